# real x complex kernel (V stored as doubles) for the W assembly vs the 2-product Gauss path (nodz) and tile variants
timeout 600 python -m pytest tests/test_gpu_scba.py -x -q 2>&1 | tail -1
for lib in "" m5 bk8 bk32 n64 ""; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  NEGF_B200_LIB=$L timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_s_both_iterations']; print('${lib:-default}', round(d['iteration_s'],4), 'asm', round(s['W: assembly'],4), 'wrgf', round(s['W: RGF'],4), 'G', round(s['G: OBC+RGF'],4))"
done
