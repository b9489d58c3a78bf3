# final 1-GPU measurements: bench (driver-like settings), then the ncu launch list of one C2 batch and a full
# capture of the top kernels (each ncu command only after the same command exited 0 without ncu)
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final_n1.json 2> gpurun_out/bench_final_n1.err; echo bench_rc=$?
run() { python bench.py --steps 1 --warmup 1 --alt-steps 0 --scgw "" --c4 "" --no-cpu-baseline --n-e 128 --e2e-steps 0; }
run > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2600 -c 2600 --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 1 --warmup 1 --alt-steps 0 --scgw "" --c4 "" --no-cpu-baseline --n-e 128 --e2e-steps 0 \
  > gpurun_out/ncu_launch.log 2>&1; echo launch_rc=$?
python tools/launch_summary.py gpurun_out/launches_final.csv > gpurun_out/launches_c2_final.csv
ncu --set full --clock-control none --import-source on -k regex:"zgemm_kernel" -s 400 -c 2 -o gpurun_out/prof_final \
  python bench.py --steps 1 --warmup 1 --alt-steps 0 --scgw "" --c4 "" --no-cpu-baseline --n-e 128 --e2e-steps 0 \
  > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
