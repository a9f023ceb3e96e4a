"""One line per launch of an `ncu --page raw --csv` dump: duration, shared-memory wavefronts,
LSU data-pipe and FP64 pipe utilisation, issue slots, bank conflicts, DRAM bytes, top stalls.
usage: python tools/ncu_raw.py dump.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
names = {'us': 'gpu__time_duration.sum', 'smem_wf': 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
         'lsu%': 'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
         'fp64%': 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
         'issue%': 'smsp__issue_active.avg.pct_of_peak_sustained_active',
         'conflicts': 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
         'dram_rd_MB': 'dram__bytes_read.sum', 'dram_wr_MB': 'dram__bytes_write.sum',
         'warps': 'sm__warps_active.avg.per_cycle_active', 'regs': 'launch__registers_per_thread'}
st = [i for i, h in enumerate(hdr) if 'pcsamp_warps_issue_stalled' in h and 'not_issued' not in h]
for r in rows[2:]:
    d = {k: r[hdr.index(v)] for k, v in names.items() if v in hdr}
    top = sorted([(float(r[i]), hdr[i].split('stalled_')[1]) for i in st if r[i]], reverse=True)[:6]
    tot = sum(float(r[i]) for i in st if r[i]) or 1
    print(r[hdr.index('Kernel Name')][:36], ' '.join(f"{k}={v[:9]}" for k, v in d.items()))
    print('    stalls:', ' '.join(f"{n}={100*v/tot:.0f}%" for v, n in top))
