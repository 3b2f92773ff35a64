"""Regenerate data/params/*.json with this package's own prime and root search.
tests/test_host_logic.py checks them against the reference's shipped moduli
(tests/golden/golden.json)."""
from pathlib import Path

from paper_2512_18345_b200.params import generate_parameter_set, sub_parameter_set

here = Path(__file__).resolve().parent / "params"
generate_parameter_set(4096, 12, 3, 1 << 40, 64, 32).save(here / "verify_small.json")
ks48 = generate_parameter_set(65536, 48, 4, 1 << 40, 32768, 32)
ks48.save(here / "ks48.json")
sub_parameter_set(ks48, 24).save(here / "ks24.json")
sub_parameter_set(ks48, 12).save(here / "ks12.json")
