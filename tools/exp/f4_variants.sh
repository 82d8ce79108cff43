for v in 0 1 2; do
  echo "== variant $v"
  GFQ_F4_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_f4.py -x -q 2>&1 | tail -1
  GFQ_F4_VARIANT=$v timeout 300 python tools/f4_bench.py 2 2>&1 | grep -E '"k": 8192' 
done
