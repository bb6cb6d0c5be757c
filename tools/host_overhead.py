"""Host enqueue cost vs device time per MiCRO step at c1 size (is the GPU starved?)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_00967_b200 import engine  # noqa: E402

n_g = 11_700_000
m = engine.Micro(n_g, 1, density=0.01, initial_threshold=0.0258, dense_output=False)
x = torch.zeros(n_g, device="cuda")
m.set_model(x)
G = [torch.empty(n_g, device="cuda") for _ in range(8)]
for i, g in enumerate(G):
    engine.synth_gaussian(g, 1, 0, i)
for t in range(300):
    m.step([G[t % 8]], 0.01, t)
torch.cuda.synchronize()
for timing in (False, True):
    m.kernel_timing(timing)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    h0 = time.perf_counter()
    for t in range(300, 1300):
        m.step([G[t % 8]], 0.01, t)
    h1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    print(f"kernel_timing={timing}: host enqueue {1e6 * (h1 - h0) / 1000:.1f} us/step, device {1e3 * a.elapsed_time(b) / 1000:.1f} us/step")
    m.kernel_times(1024)
