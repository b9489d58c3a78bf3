# bulk-copy 3M kernel with the operand-disjoint DMMA order (default) vs before (old variant)
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k zgemm 2>&1 | tail -1
for lib in "" old; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== ${lib:-default}"
  for sh in "16 512" "8 1024" "4 2048"; do NEGF_B200_LIB=$L python tools/gemm_vs_cublas.py $sh 3 2>&1 | grep negf; done
  NEGF_B200_LIB=$L timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_s_both_iterations']; print('c3', round(d['iteration_s'],4), 'G', round(s['G: OBC+RGF'],4), 'wrgf', round(s['W: RGF'],4))"
done
