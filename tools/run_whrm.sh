# anti-Hermitian W diagonal sources on half the tiles (default) vs full products (nowh variant); then the GPU suite
for lib in "" nowh; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  NEGF_B200_LIB=$L timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_s_both_iterations']; print('${lib:-default}', round(d['iteration_s'],4), 'asm', round(s['W: assembly'],4), 'wrgf', round(s['W: RGF'],4))"
done
timeout 2300 python -m pytest tests/ -q -m gpu 2>&1 | grep -v OMP | grep -E "FAILED|passed|failed|^E  .*assert" | head -20
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
