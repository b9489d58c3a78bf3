# GEMM / inversion / RGF GPU tests and the C2 shape GEMM after the 3M stage rewrite
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_rgf.py tests/test_gpu_obc.py -x -q 2>&1 | tail -1
for sh in "128 256" "16 512" "8 1024"; do python tools/gemm_vs_cublas.py $sh 2,0,3 2>&1 | grep -v "^\*"; done
