# build first: python tools/build_variant.py t6464 -DNEGF_BULK_BN=64 -DNEGF_BULK_WN=4 -DNEGF_BULK_MINB=1;
#   t12832 -DNEGF_BULK_BM=128 -DNEGF_BULK_WM=4 -DNEGF_BULK_MINB=1; t6432s3 -DNEGF_BULK_STAGES=3 -DNEGF_BULK_MINB=1; k24 -DNEGF_BULK_BK=24
# bulk-copy GEMM tile/stage variants (algo 3 forces the bulk kernel), RGF-like shapes
for lib in "" paper_2508_19138_b200/variants/t6464.so paper_2508_19138_b200/variants/t12832.so paper_2508_19138_b200/variants/t6432s3.so paper_2508_19138_b200/variants/k24.so; do
  L=${lib:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== lib ${lib:-default (bulk 64x32 BK32 2 stages 2 CTA/SM)}"
  NEGF_B200_LIB=$L timeout 120 python tools/gemm_vs_cublas.py 4 2048 3
  NEGF_B200_LIB=$L timeout 120 python tools/gemm_vs_cublas.py 16 512 3
  NEGF_B200_LIB=$L timeout 120 python tools/gemm_vs_cublas.py 128 256 3
done
