"""Host link bandwidth (pinned H2D / D2H, 16 MB, best of 5) next to kbg_grid_pass's phase timeline."""
import os
import subprocess
import sys
import time

import torch

a = torch.empty(2 << 20, dtype=torch.float64).pin_memory()
d = torch.empty(2 << 20, dtype=torch.float64, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(a, non_blocking=True)), ("d2h", lambda: a.copy_(d, non_blocking=True))):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {16.777 / best:.1f} GB/s", flush=True)
