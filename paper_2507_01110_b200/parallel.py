"""View-sharded training across GPUs: the sparse gradient exchange.

Each rank renders its own view (one process per GPU, torch.distributed /
NCCL over NVLink).  Before ADAM the per-view gradients of the touched
Gaussians are summed over ranks on the *union* of touched nodes:

  1. all_gather of the row counts, then of the node-id lists (4 B/id)
  2. every rank forms the same sorted union U of node ids
  3. each rank scatter-adds its packed per-row gradients into a
     union-indexed buffer (f32, 92 B/node)
  4. one all_reduce(sum) of that buffer
  5. ADAM runs on U on every rank (replicated master params stay identical)

Parity contract: the reduced gradient of node i equals the sum
over ranks of the single-view gradients at identical parameters.  Only the
collectives and index plumbing live here; works with NCCL (GPU) or gloo
(CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .core import SECTIONS

COLS = [c for _, c in SECTIONS]


def _sections(buf: torch.Tensor, rows: int):
    out, off = [], 0
    for c in COLS:
        out.append(buf[off * rows:(off + c) * rows].view(rows, c))
        off += c
    return out


def union_of_rows(row_node: torch.Tensor, group=None):
    """All-gather the ranks' touched node ids; returns (sorted union U,
    position in U of each local row)."""
    world = dist.get_world_size(group)
    n = torch.tensor([row_node.numel()], dtype=torch.int64, device=row_node.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(max(counts), 1)
    padded = torch.full((cap,), -1, dtype=torch.int64, device=row_node.device)
    padded[:row_node.numel()] = row_node.to(torch.int64)
    gathered = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(gathered, padded, group=group)
    allids = torch.cat([g[:c] for g, c in zip(gathered, counts)])
    U = torch.unique(allids, sorted=True)
    pos = torch.searchsorted(U, row_node.to(torch.int64))
    return U, pos


def sparse_grad_allreduce(row_node: torch.Tensor, grads: torch.Tensor, rows: int, group=None,
                          wire_dtype=torch.float32):
    """Sum packed per-row gradients (section-major, `rows` rows) over ranks
    on the union of touched nodes.  Returns (U int64, packed f64 grads of
    |U| rows)."""
    U, pos = union_of_rows(row_node[:rows], group)
    nU = U.numel()
    buf = torch.zeros(23 * nU, dtype=wire_dtype, device=grads.device)
    for dst, src in zip(_sections(buf, nU), _sections(grads[:23 * rows], rows)):
        dst.index_add_(0, pos, src.to(wire_dtype))
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return U, buf.to(torch.float64)
