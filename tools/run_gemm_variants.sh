# build first: python tools/build_variant.py b8s4m3 -DNEGF_BULK_BK=8 -DNEGF_BULK_STAGES=4 -DNEGF_BULK_MINB=3;
#   b16s2m3 -DNEGF_BULK_BK=16 -DNEGF_BULK_STAGES=2 -DNEGF_BULK_MINB=3; b32s2m2 -DNEGF_BULK_BK=32 -DNEGF_BULK_STAGES=2 -DNEGF_BULK_MINB=2
# DMMA GEMM variants: cp.async kernel (algo 2) vs the TMA-engine bulk-copy + mbarrier kernel (algo 3),
# bulk-kernel tile/stage variants built by tools/build_variant.py into paper_2508_19138_b200/variants/
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "zgemm" 2>&1 | tail -2
for lib in "" paper_2508_19138_b200/variants/b8s4m3.so paper_2508_19138_b200/variants/b16s2m3.so paper_2508_19138_b200/variants/b32s2m2.so; do
  L=${lib:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== lib ${lib:-default (bulk BK16 3 stages 2 CTA/SM)}"
  NEGF_B200_LIB=$L timeout 120 python tools/gemm_vs_cublas.py 128 256 2,3
  NEGF_B200_LIB=$L timeout 120 python tools/gemm_vs_cublas.py 8 1024 2,3
done
