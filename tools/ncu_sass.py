"""Per-opcode totals of an `ncu --page source --csv --print-source sass` dump (first kernel in
the dump): shared-memory wavefronts, executed warp instructions, stall samples.
usage: python tools/ncu_sass.py dump.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
hdr = rows[h[0]]
end = h[1] - 1 if len(h) > 1 else len(rows)
wi, si, ii, sa = (hdr.index(k) for k in ("L1 Wavefronts Shared", "Source", "Instructions Executed", "# Samples"))
tot = 0; by = {}; ninst = 0; nsamp = 0
def fl(x):
    try: return float(x or 0)
    except ValueError: return 0.0
for r in rows[h[0] + 1:end]:
    if len(r) < len(hdr): continue
    t = r[si].split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "")
    op = op.rstrip(";")
    b = by.setdefault(op, [0, 0, 0])
    b[0] += fl(r[wi]); b[1] += fl(r[ii]); b[2] += fl(r[sa])
    tot += fl(r[wi]); ninst += fl(r[ii]); nsamp += fl(r[sa])
print(f"shared wavefronts {tot:.0f}  warp instructions {ninst:.0f}  samples {nsamp:.0f}")
print(f"{'opcode':28s} {'wavefronts':>12s} {'warp-instr':>12s} {'samples':>8s}")
for k, v in sorted(by.items(), key=lambda kv: -kv[1][2])[:30]:
    print(f"{k:28s} {v[0]:12.0f} {v[1]:12.0f} {v[2]:8.0f}")
