import sys, json
sys.path.insert(0,'.')
from tools.kbench import linb_2d
for nx,ns,st in ((1025,1,16),(1025,4,16),(1025,16,16),(1025,64,16),(257,64,64),(257,8,64)):
    print(json.dumps(linb_2d(nx,ns,st)), flush=True)
