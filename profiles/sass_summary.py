"""Per-kernel SASS opcode summary of csrc/libckks_b200.so (sm_100a cubins only):
    python profiles/sass_summary.py > profiles/r2_sass_summary.txt
For every kernel: instruction count, the integer / FP64 / tensor / memory opcode classes the hot
loops are built from, and the Blackwell-specific opcodes the profiling guide asks to look for
(UTCxMMA = tcgen05.mma, LDTM/STTM = tensor memory, UTMALDG/UTMASTG = tensor TMA, UBLKCP = bulk TMA copy,
SYNCS = mbarrier, UCGABAR = barrier.cluster, ST (generic, not STG / STS) = st.shared::cluster into another
CTA's shared memory, ACQBULK/PREEXIT = PDL,
256-bit LDG/STG).  Evidence of what the library is -- and is not -- built from."""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_2512_18345_b200" / "csrc" / "libckks_b200.so"
CLASSES = [
    ("IMAD.HI", r"^IMAD\.HI"), ("IMAD.WIDE", r"^IMAD\.WIDE"), ("IMAD", r"^IMAD(?!\.HI|\.WIDE|\.MOV|\.IADD)"),
    ("IMAD.MOV/IADD", r"^IMAD\.(MOV|IADD)"), ("VIADDMNMX", r"^VIADDMNMX"), ("IADD3", r"^IADD3"), ("LOP3/SHF", r"^(LOP3|SHF)"),
    ("DMMA", r"^DMMA"), ("DFMA/DADD", r"^(DFMA|DADD|DMUL)"), ("HMMA/IMMA", r"^(HMMA|IMMA)"),
    ("UTCxMMA", r"^UTC.*MMA"), ("LDTM/STTM", r"^(LDTM|STTM)"), ("UTMALDG/STG", r"^UTMA(LDG|STG)"), ("UBLKCP", r"^UBLKCP"), ("SYNCS(mbarrier)", r"^SYNCS"),
    ("UCGABAR(cluster barrier)", r"^UCGABAR"), ("ST(DSMEM)", r"^ST(\.|$)"),
    ("LDGSTS", r"^LDGSTS"), ("LDG", r"^LDG"), ("LDG.256", r"^LDG.*\.256"), ("STG", r"^STG"), ("STG.256", r"^STG.*\.256"),
    ("LDS", r"^LDS"), ("STS", r"^STS"), ("BAR", r"^BAR"), ("PDL", r"^(ACQBULK|PREEXIT)"), ("SHFL", r"^SHFL"),
]


def main():
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    kernels, name = collections.OrderedDict(), None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            name = re.sub(r"\(.*", "", name).replace("void ", "").replace("ckks::", "")
            kernels[name] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m and name:
            kernels[name]["_total"] += 1
            op = m.group(1)
            for label, pat in CLASSES:
                if re.match(pat, op):
                    kernels[name][label] += 1
    archs = sorted(set(re.findall(r"arch = (sm_\w+)", out)))
    print(f"# {LIB.name}: cubin architectures {archs}; {len(kernels)} kernels")
    labels = [c for c, _ in CLASSES]
    total = collections.Counter()
    for k, c in kernels.items():
        total.update(c)
        body = "  ".join(f"{lab}={c[lab]}" for lab in labels if c[lab])
        print(f"{k}\n    instructions={c['_total']}  {body}")
    print("\n# whole library")
    print("  ".join(f"{lab}={total[lab]}" for lab in labels))
    print("# Hopper/Blackwell opcodes: UTCxMMA (tcgen05.mma) = %d, LDTM/STTM (tensor memory) = %d, UTMALDG/UTMASTG (tensor TMA) = %d, "
          "UBLKCP (bulk async copy = TMA engine, cp.async.bulk) = %d with SYNCS (mbarrier) = %d; PDL (ACQBULK/PREEXIT) = %d, "
          "256-bit LDG/STG = %d" % (total["UTCxMMA"], total["LDTM/STTM"], total["UTMALDG/STG"], total["UBLKCP"],
                                    total["SYNCS(mbarrier)"], total["PDL"], total["LDG.256"] + total["STG.256"]))


if __name__ == "__main__":
    sys.exit(main())
