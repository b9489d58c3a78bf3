# 3M cp.async kernel with 32x32 warp tiles (2 warps per 64x32 CTA, 8 warps/SM like cuBLAS's Z kernel) vs 32x16 (default)
for lib in "" w1m4 w1m3; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== ${lib:-default}"
  for sh in "128 256" "16 512" "8 1024"; do NEGF_B200_LIB=$L python tools/gemm_vs_cublas.py $sh 2 2>&1 | grep negf; done
done
