# final code, 147-energy C2 batches: bench at N=4 (driver-style torchrun)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_final5_n4.json 2> gpurun_out/bench_final5_n4.err
echo "n=4 rc=$?"
