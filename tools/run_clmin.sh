# one-CTA 16-column panels (default at 512) vs 2-CTA cluster 32-column panels at 512, after the streamed sweep
for cm in "" 257; do
  echo "== NEGF_ZINV_CLUSTER_MIN=${cm:-default}"
  for nb in "512 8" "512 16"; do NEGF_ZINV_CLUSTER_MIN=$cm python tools/zinv_bench.py $nb 2>&1 | grep zinv; done
  NEGF_ZINV_CLUSTER_MIN=$cm timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['iteration_s'])"
done
