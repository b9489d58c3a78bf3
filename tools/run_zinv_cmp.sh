timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k zinv 2>&1 | tail -1
for lib in "" paper_2508_19138_b200/variants/old.so; do
  L=${lib:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== lib ${lib:-new}"
  for nb in "640 8" "1024 1" "1024 8" "2048 1" "2048 8" "4096 1" "512 128"; do NEGF_B200_LIB=$L timeout 120 python tools/zinv_bench.py $nb 2>&1 | grep zinv; done
done
