# one-CTA panel with one barrier per column (candidate rows published with the candidates; default) vs two (twobar)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_rgf.py -x -q -k "zinv or rgf" 2>&1 | grep -E "passed|failed|^E " | head -3
for lib in "" twobar "" twobar; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== ${lib:-default}"
  for nb in "256 147" "512 8"; do NEGF_B200_LIB=$L python tools/zinv_bench.py $nb 2>&1 | grep zinv; done
  NEGF_B200_LIB=$L python tools/perf_carrier.py 64 256 147xm1x2x1 2>&1 | grep energies
done
NEGF_B200_LIB= timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 default', d['iteration_s'])"
NEGF_B200_LIB=$PWD/paper_2508_19138_b200/variants/twobar.so timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 twobar', d['iteration_s'])"
