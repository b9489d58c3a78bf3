# ScbaOptions.greater="identity" in the GW loop: parity tests + C3-shape rate both ways
timeout 900 python -m pytest tests/test_gpu_scba.py -x -q 2>&1 | tail -2
for g in recursion identity; do
  NEGF_GREATER=$g timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 $g', d['iteration_s'], d['stage_s_both_iterations'], d['identity_defects'])"
done
