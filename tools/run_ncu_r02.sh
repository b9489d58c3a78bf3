# ncu launch list + one full capture of the top kernels for the C2 batch (round 2)
run() { python bench.py --steps 1 --warmup 1 --alt-steps 0 --scgw "" --c4 "" --no-cpu-baseline --n-e 128 --e2e-steps 0; }
run > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2600 -c 2600 --csv --log-file gpurun_out/launches_r02.csv \
  python bench.py --steps 1 --warmup 1 --alt-steps 0 --scgw "" --c4 "" --no-cpu-baseline --n-e 128 --e2e-steps 0 \
  > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"zgemm_kernel|zinv_panel" -s 400 -c 4 -o gpurun_out/prof_r02 \
  python bench.py --steps 1 --warmup 1 --alt-steps 0 --scgw "" --c4 "" --no-cpu-baseline --n-e 128 --e2e-steps 0 \
  > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
