import time, torch
N = 129**3
B = 8*N/1e9
h = torch.empty(N, dtype=torch.float64).pin_memory()
d = torch.empty(N, dtype=torch.float64, device="cuda")
def wall(fn, reps=20):
    fn(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/reps
for k in (1,2,4,8):
    ss=[torch.cuda.Stream() for _ in range(k)]
    ch=(N+k-1)//k
    def f():
        for i,s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*ch:(i+1)*ch].copy_(h[i*ch:(i+1)*ch], non_blocking=True)
    t=wall(f); print("H2D streams=%d %.1f GB/s"%(k,B/t))
# bigger buffer
N2=8*N; h2=torch.empty(N2,dtype=torch.float64).pin_memory(); d2=torch.empty(N2,dtype=torch.float64,device='cuda')
t=wall(lambda: d2.copy_(h2,non_blocking=True)); print("H2D 137MB %.1f GB/s"%(8*N2/1e9/t))
t=wall(lambda: h2.copy_(d2,non_blocking=True)); print("D2H 137MB %.1f GB/s"%(8*N2/1e9/t))
# zero-copy kernel read of host memory via UVA: torch can't directly; use cupy-free approach: torch's .to with mapped? skip
import subprocess
print(subprocess.run(['nvidia-smi','--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max','--format=csv'],capture_output=True,text=True).stdout)
