# build first: python tools/build_variant.py pack4 -DNEGF_CONV_PACK_MINB=4; pack5 -DNEGF_CONV_PACK_MINB=5
# conv roofline (bench.conv_roofline) with the default library and packed-row occupancy variants
for lib in "" paper_2508_19138_b200/variants/pack4.so paper_2508_19138_b200/variants/pack5.so; do
  echo "== lib ${lib:-default}"
  NEGF_B200_LIB=${lib:-$PWD/paper_2508_19138_b200/libnegf_b200.so} timeout 300 python -c "
import sys, json, torch; sys.argv=['x']; sys.path.insert(0,'.')
import bench
r = bench.conv_roofline(torch.device('cuda:0'), lengths=(128, 512, 1024))
print(json.dumps({k: {q: round(v[q]['achieved']) for q in v} for k, v in r['lengths'].items()}))
"
done
