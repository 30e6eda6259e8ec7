# DEBUG: PDL phase breaks of the grid build — the ragged/noise test sequence three times
for i in 1 2 3; do
  r=$(timeout 200 python -m pytest tests/test_gpu_ops.py -q -m gpu -x -k "ragged or splat or system_operators or backward or noise or sigma or constant" 2>&1 | tail -1)
  echo "run $i => $r"
done
