import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes, torch, json
from paper_1702_02207_b200 import _native
lib=_native.lib(); sink=torch.empty(1024,dtype=torch.float64,device='cuda'); ops=ctypes.c_int64(0)
st=torch.cuda.current_stream().cuda_stream
res={}
for mode,name in ((0,'dfma_lane_inst'),(1,'dadd_lane_inst'),(2,'dmma_flops'),(3,'dmma+dfma_flops')):
    best=0
    for it in (1000,10000,10000):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        a.record(); rc=lib.osc_bench_fp64(it,mode,sink.data_ptr(),ctypes.byref(ops),st); b.record(); torch.cuda.synchronize()
        assert rc==0, _native.last_error()
        best=max(best, ops.value/(a.elapsed_time(b)*1e-3))
    res[name]=best
for n in (4096, 8192):
    A=torch.randn(n,n,dtype=torch.float64,device='cuda'); B=torch.randn(n,n,dtype=torch.float64,device='cuda')
    for _ in range(2): A@B
    torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): A@B
    b.record(); torch.cuda.synchronize()
    res[f'cublas_dgemm_{n}_flops']=5*2*n**3/(a.elapsed_time(b)*1e-3)
M,K,N=4096,4096,1024
A=torch.randn(M,K,dtype=torch.float64,device='cuda'); B=torch.randn(K,N,dtype=torch.float64,device='cuda')
for _ in range(3): A@B
torch.cuda.synchronize(); a.record()
for _ in range(20): A@B
b.record(); torch.cuda.synchronize()
res['cublas_dgemm_4096x4096x1024_flops']=20*2*M*K*N/(a.elapsed_time(b)*1e-3)
print(json.dumps(res, indent=1))
