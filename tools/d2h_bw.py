"""Host<->device copy ceiling for the end-to-end leg: 1.6 GB (C2's output) device -> pinned host, timed
with CUDA events, one stream and two streams (halves)."""
import torch

n = 1600010896 // 4
d = torch.empty(n, dtype=torch.int32, device="cuda")
h = torch.empty(n, dtype=torch.int32).pin_memory()
s2 = [torch.cuda.Stream(), torch.cuda.Stream()]
for _ in range(2):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    h.copy_(d, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"D2H 1.6 GB pinned, one stream: {ms:.2f} ms = {1.6e9 / (ms / 1e3) / 1e9:.1f} GB/s")
torch.cuda.synchronize()
e0.record()
for _ in range(3):
    half = n // 2
    for k, st in enumerate(s2):
        st.wait_event(e0)
        with torch.cuda.stream(st):
            h[k * half:(k + 1) * half].copy_(d[k * half:(k + 1) * half], non_blocking=True)
for st in s2:
    torch.cuda.current_stream().wait_stream(st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"D2H 1.6 GB pinned, two streams: {ms:.2f} ms = {1.6e9 / (ms / 1e3) / 1e9:.1f} GB/s")
