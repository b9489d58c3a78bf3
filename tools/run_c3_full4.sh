# full C3 SCGW iteration (2048 energies, r_cut 16) on 4 GPUs: reference algorithm and with G^> by the identity
for g in recursion identity; do
  NEGF_GREATER=$g timeout 1500 python -m torch.distributed.run --standalone --nproc-per-node 4 tools/c3_full.py 16 8 2048 2 > gpurun_out/c3_full_$g.json 2> gpurun_out/c3_full_$g.err
  tail -c 1500 gpurun_out/c3_full_$g.json
done
