B=$PWD/paper_2304_14074_b200/csrc/build/cb/libchp_cb.so
for nb in 148 64 32 16; do echo blocks=$nb; CHP_LIB=$B CHP_C2_BLOCKS=$nb python tools/ttt.py 3 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['seconds'], d['k'])"; done
