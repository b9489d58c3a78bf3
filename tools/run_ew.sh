# elementwise kernel with all plain-term loads issued up front (default) vs before (oldew)
timeout 900 python -m pytest tests/test_gpu_rgf.py tests/test_gpu_large_shapes.py tests/test_gpu_obc.py -x -q 2>&1 | grep -E "passed|failed" | head -3
for lib in "" oldew ""; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== ${lib:-default}"
  NEGF_B200_LIB=$L python tools/perf_carrier.py 64 256 147xm1x2x1 147x1x2x1 2>&1 | grep energies
done
