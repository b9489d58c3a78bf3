for lib in "" paper_2508_19138_b200/variants/sweep1024.so; do
  L=${lib:-$PWD/paper_2508_19138_b200/libnegf_b200.so}
  echo "== lib ${lib:-default}"
  for nb in "1024 1" "1024 8" "2048 1" "2048 2" "2048 8" "4096 1"; do NEGF_B200_LIB=$L timeout 120 python tools/zinv_bench.py $nb; done
done
