"""Expert-parallel plumbing: GPU r owns experts [r*E/G, (r+1)*E/G); tokens are
data-parallel.  Per layer:  dx_ep_dispatch -> all-to-all(counts, rows, meta) -> dx_moe_forward_routed on the
owner -> all-to-all(results back) -> dx_ep_combine.  Every arithmetic step runs in libdx.so; this module only
moves buffers with torch.distributed (NCCL on GPUs, gloo in the CPU tests) -- the "plumbing" of the spec.

`ep_forward_dist` is the one-process-per-GPU path.  `ep_forward_local` runs G pools inside one process with the
all-to-all done by tensor copies; it exercises exactly the same calls and is how the EP kernels are checked on
a single GPU.
"""
from __future__ import annotations

import torch


class EPBuffers:
    """Send / receive buffers of one rank (rows are bf16 [n][H] viewed as bytes for the collectives)."""

    def __init__(self, max_tokens: int, k: int, H: int, G: int, e_loc: int, device):
        n_send = max_tokens * k
        n_recv = G * max_tokens * min(k, e_loc)
        self.k, self.H, self.G = k, H, G
        self.send_rows = torch.empty(n_send, H, dtype=torch.bfloat16, device=device)
        self.send_meta = torch.empty(n_send, 2, dtype=torch.int32, device=device)
        self.send_counts = torch.zeros(G, dtype=torch.int32, device=device)
        self.recv_counts = torch.zeros(G, dtype=torch.int32, device=device)
        self.recv_rows = torch.empty(n_recv, H, dtype=torch.bfloat16, device=device)
        self.recv_meta = torch.empty(n_recv, 2, dtype=torch.int32, device=device)
        self.y_rows = torch.empty(n_recv, H, dtype=torch.bfloat16, device=device)
        self.back_rows = torch.empty(n_send, H, dtype=torch.bfloat16, device=device)


def _bytes(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.uint8)


def ep_forward_dist(pool, bufs: EPBuffers, layer: int, x, T: int, y, group=None, tokens_global=None,
                    router_w=None, router_bias=None, logits=None):
    """One MoE layer under expert parallelism, one process per GPU (torch.distributed group)."""
    import torch.distributed as dist
    k = bufs.k
    pool.dx_ep_dispatch(layer, x, T, bufs.send_rows, bufs.send_meta, bufs.send_counts, router_w=router_w,
                        router_bias=router_bias, logits=logits)
    dist.all_to_all_single(bufs.recv_counts, bufs.send_counts, group=group)
    sc = bufs.send_counts.tolist()                    # v1: counts to the host (one sync per layer)
    rc = bufs.recv_counts.tolist()
    R = sum(rc)
    dist.all_to_all_single(_bytes(bufs.recv_rows[:R]), _bytes(bufs.send_rows[:T * k]), rc, sc, group=group)
    dist.all_to_all_single(bufs.recv_meta[:R], bufs.send_meta[:T * k], rc, sc, group=group)
    if tokens_global is None:
        tokens_global = T * bufs.G
    pool.dx_moe_forward_routed(layer, bufs.recv_rows, R, bufs.recv_meta, bufs.y_rows, tokens_global)
    dist.all_to_all_single(_bytes(bufs.back_rows[:T * k]), _bytes(bufs.y_rows[:R]), sc, rc, group=group)
    pool.dx_ep_combine(layer, bufs.back_rows, T, y)
    return R


def ep_forward_local(pools, bufs_list, layer: int, xs, Ts, ys, router_w=None, router_bias=None, logits_list=None):
    """The same layer for G ranks emulated in one process: pools[r] owns expert block r."""
    G = len(pools)
    k = bufs_list[0].k
    for r in range(G):
        pools[r].dx_ep_dispatch(layer, xs[r], Ts[r], bufs_list[r].send_rows, bufs_list[r].send_meta,
                                bufs_list[r].send_counts, router_w=router_w, router_bias=router_bias,
                                logits=None if logits_list is None else logits_list[r])
    counts = [b.send_counts.tolist() for b in bufs_list]           # counts[src][dst]
    send_off = [[sum(counts[s][:d]) for d in range(G)] for s in range(G)]
    tokens_global = sum(Ts)
    recv_src_off = []
    for d in range(G):
        off, offs = 0, []
        for s in range(G):
            n = counts[s][d]
            offs.append(off)
            if n:
                bufs_list[d].recv_rows[off:off + n].copy_(bufs_list[s].send_rows[send_off[s][d]:send_off[s][d] + n])
                bufs_list[d].recv_meta[off:off + n].copy_(bufs_list[s].send_meta[send_off[s][d]:send_off[s][d] + n])
            off += n
        recv_src_off.append(offs)
        pools[d].dx_moe_forward_routed(layer, bufs_list[d].recv_rows, off, bufs_list[d].recv_meta,
                                       bufs_list[d].y_rows, tokens_global)
    for s in range(G):
        for d in range(G):
            n = counts[s][d]
            if n:
                o = recv_src_off[d][s]
                bufs_list[s].back_rows[send_off[s][d]:send_off[s][d] + n].copy_(bufs_list[d].y_rows[o:o + n])
        pools[s].dx_ep_combine(layer, bufs_list[s].back_rows, Ts[s], ys[s])
    return counts
