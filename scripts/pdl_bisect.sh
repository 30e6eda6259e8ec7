# DEBUG: PDL phase breaks of the grid build (FBS_PDL_BREAK mask: 1 alloc, 2 free, 4 copy/event, 8 entry, 16 named, 32 phases)
for m in 63 31; do
  r=$(FBS_PDL_BREAK=$m timeout 200 python -m pytest tests/test_gpu_ops.py -q -m gpu -x -k "ragged or splat or system_operators or backward" 2>&1 | tail -1)
  echo "mask $m => $r"
done
