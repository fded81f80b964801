import torch, time
dev = torch.device("cuda", 0)
for mb in (4, 18, 64):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device=dev)
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    for _ in range(3): d.copy_(h, non_blocking=True); h2.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e0.record(); [d.copy_(h, non_blocking=True) for _ in range(10)]; e1.record(); [h2.copy_(d, non_blocking=True) for _ in range(10)]; e2.record()
    torch.cuda.synchronize()
    print(f"{mb} MB: H2D {10*n/e0.elapsed_time(e1)/1e6:.1f} GB/s, D2H {10*n/e1.elapsed_time(e2)/1e6:.1f} GB/s")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    e0.record()
    with torch.cuda.stream(s1):
        [d.copy_(h, non_blocking=True) for _ in range(10)]
    d2 = torch.empty_like(d)
    with torch.cuda.stream(s2):
        [h2.copy_(d2, non_blocking=True) for _ in range(10)]
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2); e1.record(); torch.cuda.synchronize()
    print(f"   concurrent H2D+D2H: {20*n/e0.elapsed_time(e1)/1e6:.1f} GB/s total")
