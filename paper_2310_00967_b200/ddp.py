"""PyTorch DDP communication hook: MiCRO in place of DDP's dense all-reduce
(SURVEY.md §8f-4 — the gradient producer side of the path).

    from paper_2310_00967_b200.ddp import MicroHookState, micro_hook
    model = DDP(model, device_ids=[local_rank])
    model.register_comm_hook(MicroHookState(density=0.01), micro_hook)

Each DDP bucket (a flat gradient of numel b) gets its own MiCRO context with
its own residuals and thresholds (keyed by bucket index and size; DDP
rebuilds its buckets once after the first iteration, which starts fresh
contexts).  Per bucket and iteration the hook runs the reference's MiCRO
iteration (harness.cpp:121-224) on this rank's gradient — error-feedback
accumulate, exclusive cyclic partition, threshold select, the exchange and
the worker-order sparse sum — and hands DDP back the averaged sparse
gradient g/n (the dense output), which the optimizer then applies.

``eta`` scales the gradient inside the accumulator (acc = e + eta*G).  The
reference's simulator applies the learning rate there (x -= g/n); with a
torch optimizer applying the learning rate itself, keep ``eta = 1`` so error
feedback runs in gradient units.  Gradients in bf16/fp16 are accumulated in
fp32 (the library's compute type) and cast back.  ``state_dtype=torch.float64``
keeps the residuals, thresholds' arithmetic and sums in fp64 (the reference's
own arithmetic) while the fp32 bucket gradients are read as they are
(micro_config.grad_dtype = MICRO_GRAD_F32: widened exactly on load).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .engine import Micro


class MicroHookState:
    def __init__(self, process_group=None, *, density: float = 0.01, initial_threshold: float | None = None,
                 scaling_factor: float = 0.01, eta: float = 1.0, transport: str = "peer",
                 comm_device=None, state_dtype: torch.dtype = torch.float32, **micro_kw):
        self.pg = process_group
        self.density = density
        self.initial_threshold = initial_threshold
        self.scaling_factor = scaling_factor
        self.eta = eta
        self.transport = transport
        self.comm_device = comm_device
        if state_dtype not in (torch.float32, torch.float64):
            raise ValueError(f"state_dtype must be float32 or float64, not {state_dtype}")
        self.kw = dict(micro_kw, dtype=state_dtype, grad_dtype=torch.float32)
        self.t = 0
        self.contexts: dict[tuple[int, int], object] = {}

    def _delta0(self, g: torch.Tensor) -> float:
        if self.initial_threshold is not None:
            return self.initial_threshold
        # warm start at the (1-d) quantile of |eta*G| for a Gaussian of the
        # bucket's RMS; the controller takes it from there
        import statistics
        rms = float(g.float().pow(2).mean().sqrt()) if g.numel() else 0.0
        return statistics.NormalDist().inv_cdf(1.0 - self.density / 2.0) * self.eta * rms or 0.01

    def context(self, index: int, grad: torch.Tensor):
        key = (index, grad.numel())
        m = self.contexts.get(key)
        if m is None:
            for k in [k for k in self.contexts if k[0] == index]:  # DDP rebuilt this bucket
                self.contexts.pop(k).close()
            world = dist.get_world_size(self.pg) if dist.is_initialized() else 1
            kw = dict(density=self.density, initial_threshold=self._delta0(grad),
                      scaling_factor=self.scaling_factor, dense_output=True, device=grad.device, **self.kw)
            if world == 1:
                m = Micro(grad.numel(), 1, **kw)
            else:
                from .dist import DistMicro
                m = DistMicro(grad.numel(), group=self.pg, comm_device=self.comm_device,
                              transport=self.transport, **kw)
            self.contexts[key] = m
        return m

    def close(self):
        for m in self.contexts.values():
            m.close()
        self.contexts.clear()


def micro_hook(state: MicroHookState, bucket) -> torch.futures.Future:
    """DDP comm hook: the bucket's gradient becomes MiCRO's g/n."""
    g = bucket.buffer()
    if g.numel() == 0:
        fut = torch.futures.Future()
        fut.set_result(g)
        return fut
    m = state.context(bucket.index(), g)
    g32 = g if g.dtype == torch.float32 else g.float()
    m.step([g32.contiguous()], state.eta, state.t)
    g.copy_(m.dense_device())  # g/n: sums at the union / n, zero elsewhere (cast to g's dtype)
    if bucket.is_last():
        state.t += 1
    fut = torch.futures.Future()
    fut.set_result(g)
    return fut
