import torch, time, numpy as np
dev = torch.device("cuda", 0)
d = torch.empty(1 << 30, dtype=torch.int32, device=dev)   # 4 GB
for trial in range(4):
    h = torch.empty(1 << 30, dtype=torch.int32, pin_memory=True)
    h.numpy()[:] = 1
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        d.copy_(h, non_blocking=True); torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"trial {trial} rep {rep}: {4.295/(t1-t0):.1f} GB/s", flush=True)
    del h
