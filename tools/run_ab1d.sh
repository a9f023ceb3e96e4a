# A/B of 1D library variants (CHP_LIB) on the kernel bench, then config 2 TtT
timeout 900 python -m pytest tests/test_gpu_1d.py -m gpu -x -q 2>&1 | tail -2
for L in "$@"; do
  echo "== $L"; CHP_LIB=$PWD/$L timeout 300 python tools/kbench.py 1d
done
timeout 600 python tools/ttt.py 2 > gpurun_out/ttt_c2.jsonl 2>&1; cut -c1-200 gpurun_out/ttt_c2.jsonl | tail -1
