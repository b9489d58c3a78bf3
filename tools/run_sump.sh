# 3M operand sums once per CTA and stage into a shared-memory plane (sump) vs per warp fragment (default)
NEGF_B200_LIB=$PWD/paper_2508_19138_b200/variants/sump.so timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "zgemm or zinv" 2>&1 | grep -E "passed|failed" | head -3
for lib in "" sump "" sump; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== ${lib:-default}"
  NEGF_B200_LIB=$L python tools/gemm_vs_cublas.py 147 256 2 2>&1 | grep negf
  NEGF_B200_LIB=$L python tools/perf_carrier.py 64 256 147xm1x2x1 2>&1 | grep energies
done
