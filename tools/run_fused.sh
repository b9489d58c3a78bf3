# fused sweep (T = Pinv R formed in the sweep, default) vs T in the one-CTA panel kernel (nofuse)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_rgf.py -x -q -k "zinv or rgf" 2>&1 | grep -E "passed|failed|^E " | head -5
for lib in "" nofuse; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== ${lib:-default}"
  for nb in "256 128" "512 8" "512 16" "300 7"; do NEGF_B200_LIB=$L python tools/zinv_bench.py $nb 2>&1 | grep zinv; done
  NEGF_B200_LIB=$L python tools/perf_carrier.py 64 256 128xm1x2x1 2>&1 | grep energies
  NEGF_B200_LIB=$L timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['iteration_s'])"
done
