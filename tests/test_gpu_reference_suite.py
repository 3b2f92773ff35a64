"""The reference's own hot-path tests, unchanged, against the drop-in.

`__graft_entry__.build()` keeps a travelling copy of /root/reference/pkg/{src/rnscope,tests} under
baseline/_ref/ (git-ignored, shipped to the GPU box by gpurun; never part of the repo's history).
tests/refshim/refshim.py aliases `rnscope` to paper_2512_18345_b200 and pytest runs
test_{rns,transform,baseconv,keyswitch,vectors}.py from that copy in a subprocess."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
REF_TESTS = ROOT / "baseline" / "_ref" / "ref_tests"
FILES = ["test_rns.py", "test_transform.py", "test_baseconv.py", "test_keyswitch.py", "test_vectors.py"]

# Tests of the reference that cannot hold for a device engine, each with the reason.
DESELECT = {
}


@pytest.mark.parametrize("name", FILES)
def test_reference_test_file_passes_against_the_drop_in(name, tmp_path):
    if not (REF_TESTS / name).exists():
        pytest.skip("no travelling copy of the reference tests (baseline/_ref/ref_tests); "
                    "run __graft_entry__.build() where /root/reference exists")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "refshim"), str(ROOT), env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-p", "refshim", "-q", "-x", "--no-header", "-p", "no:cacheprovider",
           str(REF_TESTS / name)]
    for node, _why in DESELECT.items():
        if node.startswith(name):
            cmd += ["--deselect", str(REF_TESTS / node)]
    res = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1500)
    tail = "\n".join((res.stdout + res.stderr).splitlines()[-40:])
    assert res.returncode == 0, f"{name} against the drop-in:\n{tail}"
    print(tail.splitlines()[-1] if tail else "")
