"""World-size-2 gloo test (CPU) of the expert-parallel plumbing (paper_2511_15015_b200/ep.py ep_forward_dist):
counts/rows/meta all-to-alls, the owner-side forward and the return all-to-all, with a CPU stand-in pool
whose three calls follow dx.h's dx_ep_dispatch / dx_moe_forward_routed / dx_ep_combine contracts using the
oracle.  The EP result must be bitwise the oracle's single-process layer on the global batch.
"""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
E, K, H, I, G_SZ, T = 8, 2, 64, 128, 32, 6


class OraclePool:
    """CPU stand-in implementing the EP calls' contracts (tests only)."""

    def __init__(self, rank, G, weights):
        self.rank, self.G, self.e_loc, self.W = rank, G, E // G, weights
        self.last = None

    def dx_ep_dispatch(self, layer, x, T_, send_rows, send_meta, send_counts, router_w=None, router_bias=None,
                       logits=None):
        import oracle
        idx, gate = oracle.route(logits.numpy(), K)
        ents = sorted(range(T_ * K), key=lambda i: (idx.flat[i], i))      # by global expert, then (t, j)
        xs = x.view(torch.int16).numpy()
        pos_of = {}
        for p, i in enumerate(ents):
            send_rows.view(torch.int16)[p] = torch.from_numpy(xs[i // K].copy())
            send_meta[p, 0] = int(idx.flat[i]) % self.e_loc
            send_meta[p, 1] = int(np.float32(gate.flat[i]).view(np.int32))
            pos_of[i] = p
        for o in range(self.G):
            send_counts[o] = int(sum(1 for i in ents if idx.flat[i] // self.e_loc == o))
        self.last = pos_of

    def dx_moe_forward_routed(self, layer, rows, R, meta, y_rows, tokens_global):
        import oracle
        for r in range(R):
            e = self.rank * self.e_loc + int(meta[r, 0])
            g = np.array([[np.int32(int(meta[r, 1])).view(np.float32)]], np.float32)
            x = rows.view(torch.int16)[r:r + 1].numpy().view(np.uint16)
            Y, _ = oracle.moe_ffn(x, np.array([[e]], np.int32), g, {e: self.W[e]}, H, I)
            y_rows.view(torch.int16)[r] = torch.from_numpy(Y[0, 0].view(np.int16).copy())

    def dx_ep_combine(self, layer, back_rows, T_, y):
        import oracle
        b = oracle.bits_to_f32(back_rows.view(torch.int16).numpy().view(np.uint16)).astype(np.float64)
        for t in range(T_):
            acc = 0.0 * b[0]
            for j in range(K):
                acc = acc + b[self.last[t * K + j]]
            y.view(torch.int16)[t] = torch.from_numpy(
                np.array([oracle.f64_to_bf16_rn(v) for v in acc], np.uint16).view(np.int16))


def _weights():
    import oracle
    import synth
    return {e: oracle.expert_tier(synth.expert_master(2, 0, e, H, I), H, I, G_SZ, 16, 4, e % 3 == 0) for e in range(E)}


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_2511_15015_b200 import ep
    pool = OraclePool(rank, world, _weights())
    bufs = ep.EPBuffers(T, K, H, world, E // world, "cpu")
    lg = torch.from_numpy(synth.trace_logits(2, 0, rank, T, E, 1.2))
    x = torch.from_numpy(synth.normal_bf16(2, 0, rank, 0, (T, H)).view(np.int16)).view(torch.bfloat16)
    y = torch.zeros(T, H, dtype=torch.bfloat16)
    R = ep.ep_forward_dist(pool, bufs, 0, x, T, y, logits=lg)
    np.save(f"{out_path}.{rank}.npy", y.view(torch.int16).numpy())
    np.save(f"{out_path}.{rank}.R.npy", np.array([R]))
    dist.destroy_process_group()


def test_ep_plumbing_two_ranks_gloo(tmp_path):
    sys.path.insert(0, ROOT)
    import oracle
    import synth
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "y")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    ys = np.concatenate([np.load(f"{out}.{r}.npy").view(np.uint16) for r in range(2)])
    lg = np.concatenate([synth.trace_logits(2, 0, r, T, E, 1.2) for r in range(2)])
    x = np.concatenate([synth.normal_bf16(2, 0, r, 0, (T, H)) for r in range(2)])
    idx, gate = oracle.route(lg, K)
    _, y_ref = oracle.moe_ffn(x, idx, gate, _weights(), H, I)
    assert np.array_equal(ys, y_ref)
    assert sum(int(np.load(f"{out}.{r}.R.npy")[0]) for r in range(2)) == 2 * T * K
