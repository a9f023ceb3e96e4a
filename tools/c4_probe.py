"""Config-4 Newton-PCG fine path probe: runs bench.py's config4 leg once (128 systems x 4
Newton steps at 511^2) and prints its JSON.  Under ncu (metrics gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum; see profiles/r02_c4_*), tools/ncu_launches.py
aggregates the launch list per kernel."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

print(json.dumps(bench.config4_block(bench.measured_peaks()[0]["hbm_gbs"])), flush=True)
