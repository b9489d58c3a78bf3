# final 1-GPU check after the streamed inversion sweep: full GPU suite, smoke, bench (driver-like settings)
timeout 2300 python -m pytest tests/ -q -m gpu 2>&1 | grep -v OMP | grep -E "FAILED|passed|failed|^E  .*assert" | head -20
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final5_n1.json 2> gpurun_out/bench_final5_n1.err; echo bench_rc=$?
