# final code on 4 GPUs: every GPU test, bench at N=2 and N=4 (driver-style torchrun), the full C3 iteration
timeout 2400 python -m pytest tests/ -q -m gpu 2>&1 | grep -v OMP | grep -E "FAILED|passed|failed|^E  .*assert" | head -20
for n in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/bench_final4_n$n.json 2> gpurun_out/bench_final4_n$n.err
  echo "n=$n rc=$?"
done
timeout 1500 python -m torch.distributed.run --standalone --nproc-per-node 4 tools/c3_full.py 16 8 2048 2 > gpurun_out/c3_full_final4.json 2> gpurun_out/c3_full_final4.err
tail -c 300 gpurun_out/c3_full_final4.json
