"""LINEAR_B kernel timing at the config-5 shape (64 slices x 16 steps) and config-3 shape."""
import sys, json
sys.path.insert(0, '.')
from tools.kbench import linb_2d
shapes = ((1025, 64, 16), (257, 64, 64)) if len(sys.argv) < 2 else ((1025, 64, int(sys.argv[1])),)
for nx, ns, st in shapes:
    print(json.dumps(linb_2d(nx, ns, st)), flush=True)
