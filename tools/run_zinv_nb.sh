# cluster-panel width for the largest blocks: 16 columns x 8 CTAs (default above 2048) vs 32 columns x 16 CTAs
# (non-portable cluster; variant: python tools/build_variant.py nb32all -DNEGF_ZINV_NB32_MAX=4096)
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "zinv" 2>&1 | tail -1
NEGF_B200_LIB=$PWD/paper_2508_19138_b200/variants/nb32all.so timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "zinv_large" 2>&1 | tail -1
for lib in "" paper_2508_19138_b200/variants/nb32all.so; do
  L=${lib:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== lib ${lib:-default}"
  for nb in "4096 1" "4096 2" "3000 1" "2049 2"; do NEGF_B200_LIB=$L timeout 120 python tools/zinv_bench.py $nb 2>&1 | grep zinv; done
done
