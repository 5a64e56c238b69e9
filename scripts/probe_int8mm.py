import torch, time
torch.cuda.set_device(0)
for (M, K, N) in ((16384, 12800, 64), (16384, 1600, 64), (1600, 16384, 64), (16384, 6400, 64), (4096, 4096, 4096)):
    a = torch.randint(-128, 127, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (K, N), dtype=torch.int8, device="cuda")
    try:
        c = torch._int_mm(a, b)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): c = torch._int_mm(a, b)
        e.record(); torch.cuda.synchronize()
        t = s.elapsed_time(e) / 10
        print(M, K, N, f"{t:.3f} ms", f"{2*M*K*N/t/1e9:.1f} TOPS")
    except Exception as ex:
        print(M, K, N, "ERR", ex)
