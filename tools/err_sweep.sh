# Gram error vs bound E for several chunk sizes (diagnostic)
for ck in 1 2 4 8 1000; do
  echo "chunk_kb=$ck"
  CIL_TC_CHUNK_KB=$ck timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "gram_error" -s 2>&1 | grep -E "max err"
done
