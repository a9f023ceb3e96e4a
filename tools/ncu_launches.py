"""Aggregate an ncu launch list (--csv, metrics gpu__time_duration.sum [+ dram__bytes_*]) per
kernel name: launches, total/mean duration, DRAM bytes.  usage: python tools/ncu_launches.py x.csv [skip_first_n]"""
import csv, sys, collections, re
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ii = hdr.index("ID")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = collections.defaultdict(lambda: collections.Counter())
unit = {}
ui = hdr.index("Metric Unit")
for r in rows[1:]:
    if int(r[ii]) < skip: continue
    name = re.sub(r"\(.*", "", r[ki])
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    if r[mi] == "gpu__time_duration.sum":
        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(u, 1.0)
        agg[name]["us"] += v; agg[name]["n"] += 1
    elif r[mi].startswith("dram__bytes"):
        v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        agg[name][r[mi]] += v
tot = sum(a["us"] for a in agg.values()) or 1
tb = sum(a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"] for a in agg.values())
print(f"total {tot/1e3:.2f} ms over {sum(a['n'] for a in agg.values())} launches; DRAM {tb/1e9:.3f} GB")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    b = a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]
    print(f"{k[:70]:70s} n={a['n']:5d} total={a['us']/1e3:9.3f} ms ({100*a['us']/tot:4.1f}%) mean={a['us']/a['n']:8.1f} us  dram={b/1e9:7.3f} GB  {b/1e3/max(a['us'],1e-9):6.0f} GB/s")
