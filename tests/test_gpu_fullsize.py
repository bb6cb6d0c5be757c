"""BASELINE's full size (C3: n_g = 138M fp32, d = 0.01): bit-exact against the
C restatement for a few iterations, then size-independent properties over a
longer run — no build-up, ascending union, the strict threshold predicate,
bitwise error-feedback conservation and the model update.  GPU only."""
import numpy as np
import pytest
import torch

from oracle import Oracle, OracleCluster

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2310_00967_b200 import engine, sparsim

N_G = 138_000_000


def test_c3_bit_exact_vs_restatement():
    o = Oracle()
    d, delta0, eta = 0.01, 0.025758293035489, 0.01
    m = engine.Micro(N_G, 1, density=d, initial_threshold=delta0)
    x = torch.zeros(N_G, device="cuda")
    m.set_model(x)
    ref = OracleCluster(N_G, 1, density=d, delta0=delta0, model=True)
    for t in range(3):
        G = o.gaussian(1, 0, t, N_G)[None, :]
        m.step([torch.from_numpy(G[0]).cuda()], eta, t)
        r = ref.step(G, eta, t)
        idx, sums = m.union()
        assert np.array_equal(idx.astype(np.int64), r["union_idx"]), t
        assert np.array_equal(sums, r["union_sum"]), t
        assert m.query().deltas[0] == r["delta_next"][0]
        assert np.array_equal(m.residual(0), ref.e[0]), t
        assert np.array_equal(x.cpu().numpy(), ref.x), t
    m.close()


def test_c3_properties_long_run():
    eta = 0.01
    m = engine.Micro(N_G, 1, density=0.01, initial_threshold=0.025758293035489)
    x = torch.zeros(N_G, device="cuda")
    m.set_model(x)
    g = torch.empty(N_G, device="cuda")
    for t in range(60):
        engine.synth_gaussian(g, 2, 0, t)
        e_t = m.residual_device(0).clone()
        x_t = x.clone()
        delta = float(m.query().deltas[0])
        m.step([g], eta, t)
        if t % 10 and t != 59:
            continue
        pi, ps, Kt = m.union_device()
        K = int(Kt.item())
        idx = engine.device_view(pi, K, torch.int32, m.device).long()
        sums = engine.device_view(ps, K, torch.float32, m.device)
        acc = sparsim.accumulate(e_t, eta, g)                     # e + eta*G, two roundings
        assert K == m.query().counts[0]                           # no build-up (n = 1: union = selection)
        assert bool((idx[1:] > idx[:-1]).all())                   # ascending
        sel = torch.zeros(N_G, dtype=torch.bool, device="cuda")
        sel[idx] = True
        thr = torch.tensor(delta, dtype=torch.float64, device="cuda")
        assert torch.equal(sel, acc.double().abs() > thr)         # strict |acc| > delta, exactly
        assert torch.equal(sums, acc[idx])                        # the sums are acc (n = 1)
        e_next = m.residual_device(0)
        sent = torch.zeros_like(acc)
        sent[idx] = acc[idx]
        assert torch.equal(e_next + sent, acc)                    # conservation, bitwise
        assert torch.equal(e_next[idx], torch.zeros(K, device="cuda"))
        want_x = x_t.clone()
        want_x[idx] = x_t[idx] - sums                             # x -= g/n with n = 1
        assert torch.equal(x, want_x)
    m.close()


def test_maximum_size_int32_indices():
    """The largest gradient the int32 index format admits (n_g = 2^31 - 2,
    8.6 GB per fp32 vector), two workers: the last partition ends one short
    of 2^31, so every index, unit base and partition bound sits at the edge
    of int32.  Size-independent properties against torch on the same
    inputs: the exact strict predicate count, the union = the ascending
    selected indices, the sums, and bitwise error-feedback conservation."""
    n_g, eta = 2**31 - 2, 0.01
    torch.cuda.empty_cache()
    m = engine.Micro(n_g, 2, density=0.0005, initial_threshold=3.48 * eta, dense_output=False,
                     record_error_norm=False)
    G = [torch.empty(n_g, device="cuda") for _ in range(2)]
    for t in range(2):
        for i in range(2):
            engine.synth_gaussian(G[i], 17, i, t)
        e0 = [m.residual_device(i).clone() for i in range(2)]
        delta = m.query().deltas.copy()
        m.step(G, eta, t)
        idx, sums = m.union()
        it = torch.from_numpy(idx.astype(np.int64)).cuda()
        want_i, want_s = [], []
        for i in range(2):  # partition(n_g, 2, t, i): contiguous halves, cyclic in t
            acc = e0[i] + torch.tensor(eta, dtype=torch.float32) * G[i]
            s, e = (0, n_g // 2) if (t + i) % 2 == 0 else (n_g // 2, n_g)
            sel = torch.nonzero(acc[s:e].abs().double() > delta[i]).flatten() + s
            want_i.append(sel)
            del acc
        order = sorted(range(2), key=lambda i: int(want_i[i][0]) if want_i[i].numel() else 0)
        wi = torch.cat([want_i[i] for i in order])
        assert torch.equal(it, wi), t
        assert int(idx[-1]) > 2**31 - 2**24  # the top of int32 is reached
        # sums: both workers' accumulators at the union, in worker order from +0
        acc0 = e0[0] + torch.tensor(eta, dtype=torch.float32) * G[0]
        s01 = torch.zeros(it.numel(), device="cuda") + acc0[it]
        del acc0
        acc1 = e0[1] + torch.tensor(eta, dtype=torch.float32) * G[1]
        s01 = s01 + acc1[it]
        assert torch.equal(torch.from_numpy(sums).cuda(), s01), t
        # conservation: e_{t+1} + (acc at the union) == acc, elementwise, worker 1
        e1 = m.residual_device(1)
        sent = torch.zeros_like(acc1)
        sent[it] = acc1[it]
        assert torch.equal(e1 + sent, acc1), t
        del acc1, sent, e0, s01
        torch.cuda.empty_cache()
    m.close()
    del G
    torch.cuda.empty_cache()
