# streamed sweep (32-row CTAs) above 512 too (swall) vs the default threshold 512
for lib in "" swall; do
  L=${lib:+$PWD/paper_2508_19138_b200/variants/$lib.so}; L=${L:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== ${lib:-default}"
  for nb in "768 8" "1024 8" "2048 2" "2048 8" "4096 1"; do NEGF_B200_LIB=$L python tools/zinv_bench.py $nb 2>&1 | grep zinv; done
done
