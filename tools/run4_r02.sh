set -x
timeout 900 python -m pytest tests/test_gpu_dd.py tests/test_gpu_kernels.py tests/test_gpu_obc.py tests/test_gpu_memo.py tests/test_gpu_rgf.py -x -q 2>&1 | tail -4
for n in 1 2 4; do timeout 300 python -m torch.distributed.run --standalone --nproc-per-node $n tools/dd_bench.py 32 4096 1 2>&1 | grep DD_BENCH; done
timeout 300 python -m torch.distributed.run --standalone --nproc-per-node 4 tools/dd_bench.py 32 4096 1 balanced 2>&1 | grep DD_BENCH
timeout 300 python -m torch.distributed.run --standalone --nproc-per-node 3 tools/dd_bench.py 32 4096 1 balanced 2>&1 | grep DD_BENCH
for n in 1 2 4; do timeout 300 python -m torch.distributed.run --standalone --nproc-per-node $n tools/dd_bench.py 32 512 8 2>&1 | grep DD_BENCH; done
for b in 8 16 128; do timeout 60 python tools/zinv_bench.py 512 $b; NEGF_ZINV_CLUSTER_MIN=257 timeout 60 python tools/zinv_bench.py 512 $b; done
timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 single', d['iteration_s'], d['stage_s_both_iterations'])"
NEGF_ZINV_CLUSTER_MIN=257 timeout 300 python tools/c3_rate.py 64 512 16 8 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 cluster', d['iteration_s'], d['stage_s_both_iterations'])"
