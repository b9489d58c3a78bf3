# ncu --set full of cuBLAS's ZGEMM (torch.bmm, 128 x 256^3 and 8 x 1024^3) for comparison with the library's 3M kernel
python tools/gemm_vs_cublas.py 128 256 2 || exit 1
ncu --metrics gpu__time_duration.sum -c 12 python tools/gemm_vs_cublas.py 128 256 2 2>&1 | grep -E "^  [a-zA-Z_].*\(|Context|void|gemm" | head -30
ncu --set full --clock-control none -k regex:'^(?!.*zgemm_kernel)(?!.*elementwise)(?!.*normal)(?!.*distribution).*' -s 0 -c 1 -o gpurun_out/ncu_cublas256 -f python tools/gemm_vs_cublas.py 128 256 2 > gpurun_out/ncu_cublas256.log 2>&1
ncu --set full --clock-control none -k regex:'^(?!.*zgemm_kernel)(?!.*elementwise)(?!.*normal)(?!.*distribution).*' -s 0 -c 1 -o gpurun_out/ncu_cublas1024 -f python tools/gemm_vs_cublas.py 8 1024 2 > gpurun_out/ncu_cublas1024.log 2>&1
tail -3 gpurun_out/ncu_cublas256.log
