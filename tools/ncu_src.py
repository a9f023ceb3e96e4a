"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump by source line:
stall samples (total and per reason), instructions and shared-memory wavefronts.
usage: python tools/ncu_src.py dump.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
# the dump holds one section per file; find header rows
agg = collections.defaultdict(lambda: collections.Counter())
cur_file = None; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path": cur_file = r[1].split("/")[-1]; hdr = None; continue
    if len(r) == 2: continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr): continue
    d = dict(zip(hdr, r))
    # SASS rows carry an Address; the CUDA-source rows repeat aggregated counts: use SASS rows only
    if not d.get("Address"): continue
    key = (cur_file, d["Line No"])
    def f(k):
        try: return float(d.get(k, 0) or 0)
        except ValueError: return 0.0
    a = agg[key]
    a["samples"] += f("# Samples"); a["inst"] += f("Instructions Executed")
    a["wf"] += f("L1 Wavefronts Shared"); a["wf_ideal"] += f("L1 Wavefronts Shared Ideal")
    for k in ("stall_long_sb", "stall_short_sb", "stall_mio", "stall_wait", "stall_selected", "stall_barrier", "stall_math", "stall_lg", "stall_not_selected"):
        a[k] += f(k)
tot = sum(a["samples"] for a in agg.values()) or 1
twf = sum(a["wf"] for a in agg.values())
print(f"total samples {tot:.0f}, shared wavefronts {twf:.0f} (ideal {sum(a['wf_ideal'] for a in agg.values()):.0f})")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    rs = " ".join(f"{k[6:]}={a[k]:.0f}" for k in a if k.startswith("stall_") and a[k] > 0.02 * a["samples"])
    print(f"{key[0]}:{key[1]:>4}  {100*a['samples']/tot:5.1f}%  inst={a['inst']:.0f} wf={a['wf']:.0f}/{a['wf_ideal']:.0f}  {rs}")
