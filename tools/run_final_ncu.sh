# launch list of one C2 batch (147 energies) with the final code + ncu --set full of the streamed sweep
run() { python bench.py --steps 1 --warmup 1 --alt-steps 0 --scgw "" --c4 "" --no-cpu-baseline --n-e 147 --e2e-steps 0; }
run > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2600 -c 2600 --csv --log-file gpurun_out/launches_final2.csv \
  python bench.py --steps 1 --warmup 1 --alt-steps 0 --scgw "" --c4 "" --no-cpu-baseline --n-e 147 --e2e-steps 0 \
  > gpurun_out/ncu_launch2.log 2>&1; echo launch_rc=$?
python tools/launch_summary.py gpurun_out/launches_final2.csv > gpurun_out/launches_c2_final2.csv
ncu --set full --clock-control none --import-source on -k regex:"zinv_sweep" -s 20 -c 1 -o gpurun_out/prof_sweep \
  python tools/zinv_bench.py 256 147 > gpurun_out/ncu_sweep.log 2>&1; echo sweep_rc=$?
head -12 gpurun_out/launches_c2_final2.csv | cut -c1-150
