# energy slices on side streams (ScbaOptions.rgf_streams / CarrierSolver(streams=)) at the C3 and C2 shapes
timeout 600 python -m pytest tests/test_gpu_scba.py -x -q 2>&1 | tail -1
for st in 1 2; do
  NEGF_RGF_STREAMS=$st timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 streams=$st', d['iteration_s'], {k: round(v, 3) for k, v in d['stage_s_both_iterations'].items()})"
done
python tools/perf_carrier.py 64 256 128xm1x2x1 128xm2x2x1 2>&1 | grep energies
