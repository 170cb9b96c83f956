"""Pinned host -> device copy rate on this box (the floor under C3's e2e): one 11.3 GB transfer
in 64 MiB and 1 GiB pieces, timed with CUDA events."""
import torch

tot = int(11.3e9)
host = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
dev = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for piece in (64 << 20, 256 << 20, 1 << 30):
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            left = tot
            while left > 0:
                k = min(piece, left)
                dev[:k].copy_(host[:k], non_blocking=True)
                left -= k
            e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"piece {piece >> 20} MiB: {ms:.1f} ms for {tot / 1e9:.1f} GB = {tot / ms / 1e6:.1f} GB/s", flush=True)
