import torch, json
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda").view(torch.int64).random_()
y = torch.empty(205 << 20, dtype=torch.bfloat16, device="cuda").uniform_()
out = {}
for name, t, f in [("sum_int64_1GB", x, lambda t: t.sum()), ("sum_bf16_215MB", y, lambda t: t.float().sum() if False else t.sum(dtype=torch.float32)),
                   ("copy_1GB", x, lambda t: t.clone())]:
    for _ in range(3): f(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f(t)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nbytes = t.numel() * t.element_size() * (2 if "copy" in name else 1)
    out[name] = round(nbytes / ms / 1e6, 1)
print(json.dumps(out))
