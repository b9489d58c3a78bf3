# final code: full C3 iteration on 4 GPUs (reference algorithm) and the C5 DD scaling (balanced plan)
timeout 1500 python -m torch.distributed.run --standalone --nproc-per-node 4 tools/c3_full.py 16 8 2048 2 > gpurun_out/c3_full_final5.json 2> gpurun_out/c3_full_final5.err
tail -c 1200 gpurun_out/c3_full_final5.json
for n in 1 2; do timeout 300 python -m torch.distributed.run --standalone --nproc-per-node $n tools/dd_bench.py 32 4096 1 2>&1 | grep DD_BENCH; done
for n in 3 4; do timeout 300 python -m torch.distributed.run --standalone --nproc-per-node $n tools/dd_bench.py 32 4096 1 balanced 2>&1 | grep DD_BENCH; done
