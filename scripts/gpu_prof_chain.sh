set -x
mkdir -p gpurun_out
python scripts/prof_chain.py C3 64 > gpurun_out/prof_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_rk4 -s 2 -c 1 -o gpurun_out/prof_c3 python scripts/prof_chain.py C3 64 > gpurun_out/ncu_c3.log 2>&1; echo ncu3 rc=$?
python scripts/prof_chain.py C4 1024 > gpurun_out/prof_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain_rk4 -s 1 -c 1 -o gpurun_out/prof_c4 python scripts/prof_chain.py C4 1024 > gpurun_out/ncu_c4.log 2>&1; echo ncu4 rc=$?
python - <<'PY' > gpurun_out/cublas_kernels.txt 2>&1
import torch
a=torch.randn(4096,4096,dtype=torch.float64,device='cuda'); b=torch.randn(4096,2048,dtype=torch.float64,device='cuda')
for _ in range(3): a@b
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,launch__cluster_dim_x --clock-control none python -c "
import torch
a=torch.randn(4096,4096,dtype=torch.float64,device='cuda'); b=torch.randn(4096,2048,dtype=torch.float64,device='cuda')
for _ in range(3): a@b
torch.cuda.synchronize()" > gpurun_out/ncu_cublas.log 2>&1; echo ncu5 rc=$?
