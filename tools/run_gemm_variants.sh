# DMMA GEMM variants (tools/build_variant.py into paper_2508_19138_b200/variants/) vs the default library
for lib in "" paper_2508_19138_b200/variants/pf.so; do
  L=${lib:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== lib ${lib:-default}"
  NEGF_B200_LIB=$L timeout 120 python tools/gemm_vs_cublas.py 128 256 2,0
  NEGF_B200_LIB=$L timeout 120 python tools/gemm_vs_cublas.py 8 1024 2
  NEGF_B200_LIB=$L timeout 600 python bench.py --steps 2 --warmup 2 --alt-steps 0 --scgw '' --c4 '' --no-cpu-baseline \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 value', round(d['value'],2), 'gemm TF', round(d['roofline']['achieved'],2))"
done
