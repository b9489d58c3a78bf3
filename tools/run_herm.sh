# anti-Hermitian products on lower-triangle tiles (default) vs full products (noherm variant)
true
for lib in "" h3 noherm; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== ${lib:-default}"
  NEGF_B200_LIB=$L python tools/perf_carrier.py 64 256 128xm1x2x1 128x1x2x1 2>&1 | grep energies
  NEGF_B200_LIB=$L timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_s_both_iterations']; print('c3', round(d['iteration_s'],4), 'G', round(s['G: OBC+RGF'],4), 'wrgf', round(s['W: RGF'],4))"
done
