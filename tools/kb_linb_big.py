"""LINEAR_B kernel timing at the bench's launch shape (many slices of 1023^2 per launch)."""
import sys, json
sys.path.insert(0, '.')
from tools.kbench import linb_2d
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 256
print(json.dumps(linb_2d(1025, ns, 16)), flush=True)
