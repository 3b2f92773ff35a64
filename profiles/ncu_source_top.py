"""Top instructions by warp-stall samples from an ncu source page
(`ncu -i X.ncu-rep --page source --csv > src.csv`): per kernel the stall-reason totals, the
executed-opcode mix and the `top` instructions with their three main stall reasons.
Usage: ncu_source_top.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
for bi, st in enumerate(starts):
    h = rows[st + 1]
    end = starts[bi + 1] if bi + 1 < len(starts) else len(rows)
    blk = rows[st + 2:end]
    ia, isamp, iex = h.index("Source"), h.index("# Samples"), h.index("Instructions Executed")
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    num = lambda r, i: int(r[i]) if i < len(r) and r[i].isdigit() else 0
    tot = sum(num(r, isamp) for r in blk)
    print(f"== {rows[st][1][:90]}\n   samples {tot}, SASS instructions {len(blk)}")
    agg = {s_: sum(num(r, h.index(s_)) for r in blk) for s_ in stalls}
    print("   stalls:", ", ".join(f"{k[6:]}={v}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v))
    mix = {}
    for r in blk:
        parts = r[ia].split()
        if not parts:
            continue
        op = (parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]).split(".")[0]
        mix[op] = mix.get(op, 0) + num(r, iex)
    total = sum(mix.values()) or 1
    print("   executed mix:", ", ".join(f"{k} {100 * v / total:.1f}%" for k, v in sorted(mix.items(), key=lambda kv: -kv[1])[:10]))
    for r in sorted(blk, key=lambda r: -num(r, isamp))[:top_n]:
        why = {s_[6:]: num(r, h.index(s_)) for s_ in stalls if num(r, h.index(s_)) > 0}
        why = ", ".join(f"{k}={v}" for k, v in sorted(why.items(), key=lambda kv: -kv[1])[:3])
        print(f"   {num(r, isamp):5d} samples  x{num(r, iex):7d}  {r[ia][:64]:64s} {why}")
