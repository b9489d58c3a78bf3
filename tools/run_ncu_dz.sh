# ncu --set full of the real x complex (W assembly) kernel at the C3 shape (one launch)
python tools/c3_rate.py 64 512 8 8 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none -k regex:zgemm_dz_kernel -s 10 -c 1 -o gpurun_out/prof_dz -f python tools/c3_rate.py 64 512 8 8 > gpurun_out/ncu_dz.log 2>&1; echo rc=$?
