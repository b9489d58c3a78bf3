# cluster-panel CTA size for 32-column panels: 512 threads (256 rows/CTA, default) vs 256 threads (128 rows/CTA)
# (variant: python tools/build_variant.py nt256 -DNEGF_ZINV_NT256_MAX=2048)
V=$PWD/paper_2508_19138_b200/variants/nt256.so
NEGF_B200_LIB=$V timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "zinv" 2>&1 | tail -1
for lib in "" $V; do
  L=${lib:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== lib ${lib:-default}"
  for nb in "768 1" "1024 1" "1024 2" "1024 8" "1536 2" "2048 1" "2048 2" "2048 8" "512 128"; do NEGF_B200_LIB=$L timeout 120 python tools/zinv_bench.py $nb 2>&1 | grep zinv; done
  NEGF_B200_LIB=$L timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['iteration_s'], d['stage_s_both_iterations'])"
done
