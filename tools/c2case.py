import sys
sys.path.insert(0, ".")
sys.argv = ["kbench"]
import importlib.util
spec = importlib.util.spec_from_file_location("kb", "tools/kbench.py")
kb = importlib.util.module_from_spec(spec); spec.loader.exec_module(kb)
import json
print(json.dumps(kb.coarse_sweep(1025, 4)))
