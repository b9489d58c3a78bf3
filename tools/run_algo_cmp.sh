# GEMM algo 2 (cp.async 3M) vs 3 (bulk-copy/mbarrier 3M) on the bench workloads
for a in 2 3; do
  echo "== NEGF_GEMM_ALGO=$a"
  NEGF_GEMM_ALGO=$a timeout 120 python tools/gemm_vs_cublas.py 128 512 $a
  NEGF_GEMM_ALGO=$a timeout 900 python bench.py --steps 3 --warmup 2 --alt-steps 2 --scgw 64x512x16 --no-cpu-baseline \
    | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
c4=d['c4_rgf_rate']; c3=d['scgw_iteration']
print('C2 value', round(d['value'],2), 'alt', round(d['greater_alt']['value'],2), 'gemm TF', round(d['roofline']['achieved'],2))
print('C4 it', round(c4['iteration_s'],3), 'G', round(c4['rgf_tflops_model_G_incl_obc'],2), 'W', round(c4['rgf_tflops_model_W_rgf'],2), 'exec frac', round(c4['rgf_executed_frac_of_peak_W_rgf'],3), c4['stage_s_rank0'])
print('C3 it', round(c3['iteration_s'],3), 'G', round(c3['rgf_tflops_model_G_incl_obc'],2), 'W', round(c3['rgf_tflops_model_W_rgf'],2), c3['stage_s_rank0'])
"
done
