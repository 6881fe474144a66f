"""H2D bandwidth of one 79 MB pinned batch: one copy vs K chunks on K streams."""
import torch
nbytes = 79148544
x = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
for K in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(K)]
    chunk = (x.numel() + K - 1) // K
    def go():
        for k, s in enumerate(streams):
            with torch.cuda.stream(s):
                y[k * chunk:(k + 1) * chunk].copy_(x[k * chunk:(k + 1) * chunk], non_blocking=True)
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream()
    e0.record(main)
    for s in streams:
        s.wait_event(e0)
    for _ in range(10):
        go()
    for s in streams:
        main.wait_stream(s)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"K={K}: {ms:.3f} ms per batch = {nbytes / ms / 1e6:.1f} GB/s")
