"""View-sharded training across GPUs: the sparse gradient exchange (K11-exchange).

Each rank (one process per GPU) renders its own view.  Before ADAM the
per-view gradients of the touched Gaussians are combined on the union U of
every rank's render rows, with owner-sharded ADAM (csrc/exchange.cu):

  1. all-gather of the row counts and the padded node-id lists (4 B/id);
  2. on-device union: ids OR-ed into a node bitmap; owner(id) =
     (id >> 5) mod N; U laid out owner-major (owner chunks sorted by id);
  3. each rank buckets its R gradient rows by owner and ships them point to
     point (a sparse reduce-scatter: 192 B per row, not a dense |U| buffer);
  4. the owner sums the received rows source by source (deterministic) and
     runs ADAM on its chunk only — moments and step counts live with the
     owner, so per-rank ADAM cost is O(|U|/N);
  5. the owners broadcast their updated attribute rows and every rank writes
     all of U into its replicated node records.

The node records are the authoritative state on every rank; the render rows
of SPTs are read from them (glod_gather_plan.spt_from_master), so a rank
never renders values another rank has already updated (the per-rank store
and cache keep the reference's decision counters).

Parity contract: the gradient ADAM applies to node i is the sum
over ranks of that step's single-view gradients at identical parameters.

`NcclExchange` is the product path: glod_grad_exchange /
glod_param_allgather with an NCCL communicator owned by the C library.
`GroupExchange` runs the same device phases with the collectives of a
torch.distributed process group (any backend; gloo stages through host
memory) — it is what runs two ranks on one GPU, where NCCL refuses a
duplicate device.  `exchange_with_group` is written against a phases object
so its collective sequence is testable on CPU (tests/test_parallel.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

F = 23          # attribute values per node
ROW = F + 1     # wire row: owner-local position + 23 gradients


def owner_of(ids, nranks: int):
    """owner(id) = (id >> 5) mod N: 32-node words dealt round-robin."""
    return (np.asarray(ids, dtype=np.int64) >> 5) % nranks


class _Ctx:
    """A glod_xchg context (phases; optionally an NCCL communicator)."""

    def __init__(self, nranks: int, rank: int, capacity: int, nccl_id: bytes | None = None):
        self.nranks, self.rank, self.capacity = int(nranks), int(rank), int(capacity)
        h = C.c_void_p()
        uid = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _lib.check(_lib.lib().glod_xchg_create(self.nranks, self.rank, self.capacity, uid, C.byref(h)))
        self._h = h
        self.offsets = [0] * (self.nranks + 1)

    def __del__(self):
        try:
            if self._h:
                _lib.load().glod_xchg_destroy(self._h)
        except Exception:
            pass

    def stats(self) -> dict:
        out = (C.c_int64 * 4)()
        _lib.check(_lib.lib().glod_xchg_stats(self._h, out))
        return {"union": out[0], "owned": out[1], "bytes_sent": out[2], "bytes_received": out[3]}

    def owned(self):
        """(ids int32 [n], packed section-major grads f64 [23·n], n)."""
        ids, g, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        _lib.check(_lib.lib().glod_xchg_owned(self._h, C.byref(ids), C.byref(g), C.byref(n)))
        n = int(n.value)
        return (_lib.device_view(ids.value or 0, (n,), torch.int32),
                _lib.device_view(g.value or 0, (F * n,), torch.float64), n)


class NcclExchange(_Ctx):
    """Product path: the whole exchange inside the C library over NCCL."""

    def __init__(self, capacity: int, group=None):
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = [None]
        if rank == 0:
            buf = C.create_string_buffer(128)
            _lib.check(_lib.lib().glod_nccl_unique_id(buf))
            uid = [buf.raw]
        dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        super().__init__(world, rank, capacity, uid[0])

    def reduce(self, row_node: torch.Tensor, grads: torch.Tensor, R: int) -> int:
        n = C.c_int64()
        _lib.check(_lib.lib().glod_grad_exchange(self._h, _lib.ptr(row_node), _lib.ptr(grads), int(R),
                                                 C.byref(n), _lib.stream_ptr()))
        return int(n.value)

    def allgather_params(self, records: torch.Tensor, stride: int):
        _lib.check(_lib.lib().glod_param_allgather(self._h, _lib.ptr(records), int(stride), _lib.stream_ptr()))


class DevicePhases(_Ctx):
    """The exchange's device phases without a communicator (see GroupExchange)."""

    def union(self, ids_all: torch.Tensor):
        off = (C.c_int64 * (self.nranks + 1))()
        _lib.check(_lib.lib().glod_xchg_union(self._h, _lib.ptr(ids_all), int(ids_all.numel()), off,
                                              _lib.stream_ptr()))
        self.offsets = [int(x) for x in off]
        return self.offsets

    def union_ids(self) -> torch.Tensor:
        p, n = C.c_void_p(), C.c_int64()
        _lib.check(_lib.lib().glod_xchg_union_ids(self._h, C.byref(p), C.byref(n)))
        return _lib.device_view(p.value or 0, (int(n.value),), torch.int32)

    def pack(self, row_node: torch.Tensor, grads: torch.Tensor, R: int):
        counts = (C.c_int64 * self.nranks)()
        p = C.c_void_p()
        _lib.check(_lib.lib().glod_xchg_pack(self._h, _lib.ptr(row_node), _lib.ptr(grads), int(R), counts,
                                             C.byref(p), _lib.stream_ptr()))
        counts = [int(x) for x in counts]
        return _lib.device_view(p.value or 0, (sum(counts), ROW), torch.float64), counts

    def begin_accumulate(self) -> int:
        n = C.c_int64()
        _lib.check(_lib.lib().glod_xchg_begin_accumulate(self._h, None, C.byref(n), _lib.stream_ptr()))
        return int(n.value)

    def accumulate(self, rows: torch.Tensor):
        rows = rows.contiguous()
        _lib.check(_lib.lib().glod_xchg_accumulate(self._h, _lib.ptr(rows), int(rows.shape[0]),
                                                   _lib.stream_ptr()))

    def pack_params(self, records: torch.Tensor, stride: int) -> torch.Tensor:
        p = C.c_void_p()
        _lib.check(_lib.lib().glod_xchg_pack_params(self._h, _lib.ptr(records), int(stride), C.byref(p),
                                                    _lib.stream_ptr()))
        return _lib.device_view(p.value or 0, (self.offsets[-1], F), torch.float64)

    def scatter_params(self, records: torch.Tensor, stride: int):
        _lib.check(_lib.lib().glod_xchg_scatter_params(self._h, _lib.ptr(records), int(stride),
                                                       _lib.stream_ptr()))


# ---------------------------------------------------------------------------
# The exchange over a torch.distributed process group, against a phases
# object (DevicePhases on the GPU; a numpy stand-in in the CPU tests).
# ---------------------------------------------------------------------------
def _comm_device(group):
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")


def _all_gather_var(t: torch.Tensor, n: int, group, fill=-1):
    """All-gather of a variable-length 1-D tensor (counts first, padded)."""
    world = dist.get_world_size(group)
    dev = _comm_device(group)
    cnt = torch.tensor([n], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(max(counts), 1)
    pad = torch.full((cap,), fill, dtype=t.dtype, device=dev)
    pad[:n] = t[:n].to(dev)
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat(out), counts


def exchange_with_group(ph, row_node, grads, R: int, group=None) -> int:
    """Phases 1-4 with the group's collectives; returns the owned row count."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = _comm_device(group)
    ids_all, _ = _all_gather_var(row_node, R, group)
    ph.union(ids_all.to(row_node.device))
    send, counts = ph.pack(row_node, grads, R)
    cm = torch.tensor(counts, dtype=torch.int64, device=dev)
    mat = [torch.zeros_like(cm) for _ in range(world)]
    dist.all_gather(mat, cm, group=group)
    recv_counts = [int(m[rank].item()) for m in mat]
    send_d = send.to(dev)
    starts = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    inbox = [None] * world
    ops = []
    for p in range(world):
        if p == rank:
            inbox[p] = send_d[starts[p]:starts[p + 1]]
            continue
        inbox[p] = torch.empty((recv_counts[p], ROW), dtype=torch.float64, device=dev)
        if counts[p]:
            ops.append(dist.P2POp(dist.isend, send_d[starts[p]:starts[p + 1]].contiguous(), p, group))
        if recv_counts[p]:
            ops.append(dist.P2POp(dist.irecv, inbox[p], p, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    n = ph.begin_accumulate()
    for p in range(world):                     # source by source, rank order
        if recv_counts[p]:
            ph.accumulate(inbox[p].to(send.device))
    return n


def params_with_group(ph, records, stride: int, group=None):
    """Phase 5: owners broadcast their chunk; everyone scatters all of U."""
    world = dist.get_world_size(group)
    dev = _comm_device(group)
    buf = ph.pack_params(records, stride)
    off = ph.offsets
    host = buf.to(dev)
    for o in range(world):
        if off[o + 1] > off[o]:
            chunk = host[off[o]:off[o + 1]].contiguous()
            dist.broadcast(chunk, src=dist.get_global_rank(group, o) if group is not None else o, group=group)
            host[off[o]:off[o + 1]] = chunk
    buf.copy_(host.to(buf.device))
    ph.scatter_params(records, stride)


class GroupExchange:
    """DevicePhases + a process group's collectives (NcclExchange's API)."""

    def __init__(self, capacity: int, group=None):
        self.group = group
        self.ph = DevicePhases(dist.get_world_size(group), dist.get_rank(group), capacity)

    def reduce(self, row_node, grads, R: int) -> int:
        return exchange_with_group(self.ph, row_node, grads, R, self.group)

    def allgather_params(self, records, stride: int):
        params_with_group(self.ph, records, stride, self.group)

    def owned(self):
        return self.ph.owned()

    def stats(self) -> dict:
        return self.ph.stats()


def make_exchange(capacity: int, group=None):
    """NCCL inside the library when the group runs NCCL; otherwise the
    group's own collectives around the device phases."""
    if dist.get_backend(group) == "nccl":
        return NcclExchange(capacity, group)
    return GroupExchange(capacity, group)
