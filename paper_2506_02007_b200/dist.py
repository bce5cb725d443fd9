"""Host-side rank exchange over torch.distributed (gloo) for es_ctx_create_exchange.

Production multi-GPU runs use NCCL inside the library (es_ctx_create_nccl); this
exchange lets several ranks share one GPU (tests) or run without NCCL.  Only exact
operations go through it: rank-ordered all-gathers, min/max, integer sums and
"one owner contributes" sums.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

_DT = {0: np.float64, 1: np.int64}


def gloo_exchange(group=None):
    """Returns (allgather, allreduce) Python callables for Context(exchange=...)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    ops = {0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MIN, 2: dist.ReduceOp.MAX}

    def allgather(user, send, recv, nbytes):
        try:
            src = np.frombuffer((C.c_ubyte * nbytes).from_address(send), dtype=np.uint8).copy()
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(outs, torch.from_numpy(src), group=group)
            flat = torch.cat(outs).numpy()
            C.memmove(recv, flat.ctypes.data, nbytes * world)
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a failed exchange
            return 1

    def allreduce(user, buf, count, dtype, op):
        try:
            dt = _DT[dtype]
            arr = np.frombuffer((C.c_ubyte * (count * 8)).from_address(buf), dtype=dt)
            t = torch.from_numpy(arr.copy())
            dist.all_reduce(t, op=ops[op], group=group)
            C.memmove(buf, t.numpy().ctypes.data, count * 8)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    return allgather, allreduce
