"""Wait-queue policies: the reference's `PolicyKind` and `select_grants`
(memshare/policy.py:23-74) with the selection computed on the GPU.

  fifo   longest prefix (in enqueue order) that fits; a misfit head blocks
  mmu    first-fit greedy in queue order, skipping misfits
  pfifo  restrict to the highest waiting priority, then fifo
  pmmu   restrict to the highest waiting priority, then mmu

`select_grants(queue, free, kind)` keeps the reference signature (entries
need .client/.nbytes/.priority; returns the granted clients in queue order)
and runs as a one-queue launch of K4 `select_grants_batch`;
`select_grants_batch` evaluates many queues in one launch (one warp each).
"""

from __future__ import annotations

import ctypes
import enum
from typing import Iterable, Sequence

import numpy as np

from . import _lib


class PolicyKind(enum.Enum):
    FIFO = "fifo"
    MMU = "mmu"
    PRIORITY_FIFO = "pfifo"
    PRIORITY_MMU = "pmmu"

    @classmethod
    def parse(cls, name: str) -> "PolicyKind":
        """Case-insensitive; ValueError otherwise (memshare/policy.py:29-36)."""
        try:
            return cls(str(name).lower())
        except ValueError:
            raise ValueError(
                f"unknown policy {name!r} (expected fifo|mmu|pfifo|pmmu)") from None

    @property
    def code(self) -> int:
        return _CODES[self]

    @classmethod
    def from_code(cls, code: int) -> "PolicyKind":
        return _FROM_CODE[code]


_CODES = {PolicyKind.FIFO: 0, PolicyKind.MMU: 1,
          PolicyKind.PRIORITY_FIFO: 2, PolicyKind.PRIORITY_MMU: 3}
_FROM_CODE = {v: k for k, v in _CODES.items()}


def as_policy(p) -> PolicyKind:
    if isinstance(p, PolicyKind):
        return p
    if isinstance(p, (int, np.integer)):
        return PolicyKind.from_code(int(p))
    return PolicyKind.parse(p)


def policy_mask(policies: Iterable) -> tuple[int, tuple[PolicyKind, ...]]:
    """Bit mask for sg_batch.policy_mask and the policies in output order
    (increasing code)."""
    kinds = {as_policy(p) for p in policies}
    if not kinds:
        raise ValueError("at least one policy is required")
    ordered = tuple(sorted(kinds, key=lambda k: k.code))
    mask = 0
    for k in ordered:
        mask |= 1 << k.code
    return mask, ordered


def _torch_cuda():
    import torch
    if not torch.cuda.is_available():
        raise _lib.SgpuUnavailable("select_grants runs on the GPU; no CUDA device is available")
    return torch


def select_grants_batch(queues: Sequence[tuple[Sequence[int], Sequence[int]]],
                        free: Sequence[int], kinds: Sequence, device=None) -> list[np.ndarray]:
    """Evaluate many queues in one launch.  queues[q] = (nbytes, priorities)
    in enqueue order; returns one boolean granted-mask per queue."""
    torch = _torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    sizes = [len(q[0]) for q in queues]
    off = np.zeros(len(queues) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    nb = np.concatenate([np.asarray(q[0], dtype=np.int64) for q in queues]) if off[-1] else \
        np.zeros(1, dtype=np.int64)
    pr_list = []
    for q in queues:
        p = np.asarray(q[1], dtype=np.int64)
        if p.size and (p.min() < -(1 << 31) or p.max() >= (1 << 31)):
            # only order and equality matter to the policies: dense ranks
            _, p = np.unique(p, return_inverse=True)
        pr_list.append(p.astype(np.int32))
    pr = np.concatenate(pr_list) if off[-1] else np.zeros(1, dtype=np.int32)
    fr = np.asarray(free, dtype=np.int64)
    kd = np.asarray([as_policy(k).code for k in kinds], dtype=np.uint32)
    t_off = torch.from_numpy(off).to(dev)
    t_nb = torch.from_numpy(nb).to(dev)
    t_pr = torch.from_numpy(pr).to(dev)
    t_fr = torch.from_numpy(fr).to(dev)
    t_kd = torch.from_numpy(kd.view(np.int32)).to(dev)
    t_g = torch.zeros(max(int(off[-1]), 1), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        rc = _lib.lib().sg_select_grants_batch(
            len(queues), ctypes.c_void_p(t_off.data_ptr()), ctypes.c_void_p(t_nb.data_ptr()),
            ctypes.c_void_p(t_pr.data_ptr()), ctypes.c_void_p(t_fr.data_ptr()),
            ctypes.c_void_p(t_kd.data_ptr()), ctypes.c_void_p(t_g.data_ptr()),
            ctypes.c_void_p(stream.cuda_stream))
    _lib.check(rc, "sg_select_grants_batch")
    g = t_g.cpu().numpy().astype(bool)
    return [g[off[i]:off[i + 1]] for i in range(len(queues))]


def select_grants(queue, free: int, kind) -> list:
    """Return the clients to grant, in queue order, with sum(nbytes) <= free
    (memshare/policy.py:52-74).  `queue` holds waiting entries for one
    device in enqueue order; entries need .client, .nbytes, .priority."""
    kind = as_policy(kind)
    if not queue:
        return []
    sizes = [int(e.nbytes) for e in queue]
    prios = [int(e.priority) for e in queue]
    mask = select_grants_batch([(sizes, prios)], [int(free)], [kind])[0]
    return [e.client for e, m in zip(queue, mask) if m]


__all__ = ["PolicyKind", "select_grants", "select_grants_batch", "policy_mask", "as_policy"]
