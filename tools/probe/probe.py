import torch, time, os, subprocess
print("nproc", os.cpu_count())
print(subprocess.run("lscpu | head -20", shell=True, capture_output=True, text=True).stdout)
d = torch.device("cuda")
for (m,n,k) in [(8192,8192,8192),(2000,1024,500),(500,1024,2000),(2000,64,500)]:
    a = torch.randn(m,k,dtype=torch.float64,device=d); b = torch.randn(k,n,dtype=torch.float64,device=d)
    for _ in range(3): c = a@b
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): c=a@b
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/10
    print(f"cublas dgemm {m}x{n}x{k}: {2*m*n*k/ms/1e9:.2f} TFLOP/s ({ms*1e3:.1f} us)")
