"""Out-of-core scene store in pinned host DRAM.

Mirrors the reference store's data model (store.py:143-333): attributes as
six little-endian f32 sections in *slot* order — every non-SPT node first
(ascending id), then each SPT's records in record order — so an SPT cut
prefix is one contiguous range per section.  Where the reference reads
prefixes from a file/memory backing, this store keeps the sections in
page-locked host memory *interleaved* — one 92-B row per slot, the six
sections as column slices of a [nslots, 23] array — so an SPT prefix
(store.py:304-312) is ONE contiguous range and moves to HBM as one
copy-engine transfer (cudaMemcpyAsync); write-back is the reverse copy.
The .glod file keeps the reference's section-major layout (disk mode reads
it directly).  Byte counters follow the reference exactly
(`attribute_bytes_read += prefix_len · 92`, store.py:311).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .core import BYTES_PER_GAUSSIAN_F32, SECTIONS, AttributeArrays


class NotFoundError(KeyError):
    pass


class InvalidBlockError(ValueError):
    pass


@dataclass
class AttributeBlock:
    """Attributes of an SPT record prefix, in record order (store.py:130-140).
    `attrs` is an AttributeArrays (host) or a packed device tensor."""

    spt_id: int
    prefix_len: int
    attrs: object

    def __post_init__(self):
        if isinstance(self.attrs, AttributeArrays) and len(self.attrs) != self.prefix_len:
            raise InvalidBlockError("block arrays do not match prefix_len")


def slot_order(h, hspt) -> np.ndarray:
    """slot → node (store.py:143-154)."""
    flat = hspt.flat_records()
    in_spt = np.zeros(h.capacity, dtype=bool)
    in_spt[flat["nodes"]] = True
    alive = np.ones(h.capacity, dtype=bool)
    if h.free:
        alive[np.asarray(h.free, dtype=np.int64)] = False
    head = np.nonzero(alive & ~in_spt)[0]
    return np.concatenate([head, flat["nodes"]]).astype(np.int64)


def alloc_rows(nslots: int, location: str = "host", pin: bool = True, interleaved: bool = True):
    """One [nslots, 23] f32 array (page-locked host memory, or HBM for
    location="device") and the six attribute sections as column-slice views
    of it (interleaved rows: glod_store_view.row_stride = 23).  With
    interleaved=False: six separate section arrays (the file's layout;
    row_stride = 0) and rows = None."""
    def empty(shape):
        if location == "device":
            return torch.empty(shape, dtype=torch.float32, device="cuda")
        return torch.empty(shape, dtype=torch.float32, pin_memory=pin and torch.cuda.is_available())
    if not interleaved:
        return None, [empty((nslots, cols)) for _, cols in SECTIONS]
    rows = empty((nslots, 23))
    secs, off = [], 0
    for _, cols in SECTIONS:
        secs.append(rows[:, off:off + cols])
        off += cols
    return rows, secs


def fill_section(sec: torch.Tensor, values) -> None:
    """Write one section (an (nslots, cols) array) into its column slice."""
    v = torch.from_numpy(np.ascontiguousarray(np.asarray(values, dtype=np.float32)).reshape(sec.shape))
    sec.copy_(v.to(sec.device) if sec.is_cuda else v)


class HostStore:
    """Pinned host store + per-SPT directory, built from (hierarchy, hspt).

    `location="device"` keeps the same sections in HBM instead (config C2,
    a fully device-resident scene): every transfer path is unchanged, the
    copies just become device-to-device."""

    bytes_per_gaussian = BYTES_PER_GAUSSIAN_F32

    def __init__(self, h, hspt, pin: bool = True, location: str = "host", interleaved: bool = True):
        if location not in ("host", "device"):
            raise ValueError("location must be 'host' or 'device'")
        self.location = location
        flat = hspt.flat_records()
        self.slot_to_node = slot_order(h, hspt)
        self.nslots = int(self.slot_to_node.size)
        self.record_offset = flat["offset"].astype(np.int64)
        self.record_count = flat["count"].astype(np.int64)
        self.total_records = int(self.record_count.sum())
        self.rows, self.sections = alloc_rows(self.nslots, location, pin, interleaved)
        for (name, cols), sec in zip(SECTIONS, self.sections):
            fill_section(sec, np.asarray(getattr(h.attrs, name))[self.slot_to_node])
        self.attribute_bytes_read = 0

    @staticmethod
    def from_scene(scene, location: str = "host") -> "HostStore":
        """The store of an open scene: our scenefile.Scene (sections read from
        the file straight into pinned memory) or the reference's
        store.Scene (store.py:237-280; sections read through its backing)."""
        if hasattr(scene, "host_store"):
            return scene.host_store(location)
        st = HostStore.__new__(HostStore)
        st.location = location
        st.slot_to_node = np.asarray(scene.slot_to_node, dtype=np.int64).copy()
        st.nslots = int(scene.nslots)
        st.record_offset = np.asarray(scene.spt_dir["record_offset"], dtype=np.int64)
        st.record_count = np.asarray(scene.spt_dir["record_count"], dtype=np.int64)
        st.total_records = int(st.record_count.sum())
        st.attribute_bytes_read = 0
        st.rows, st.sections = alloc_rows(st.nslots, location)
        buf = getattr(scene.backing, "buf", None)
        for (name, cols), sec in zip(SECTIONS, st.sections):
            off, length = scene.sections[name]
            raw = bytes(buf[off:off + length]) if buf is not None else scene.backing.read(off, length)
            fill_section(sec, np.frombuffer(raw, dtype="<f4").reshape(st.nslots, cols))
        return st

    def to_scene(self, scene) -> None:
        """Write the sections back into an open scene (every slot, the
        reference's write_back, store.py:323-333)."""
        if hasattr(scene, "save_store"):
            scene.save_store(self)
            return
        for (name, cols), sec in zip(SECTIONS, self.sections):
            off, length = scene.sections[name]
            data = sec.cpu().numpy().astype("<f4", copy=False).tobytes()
            if len(data) != length:
                raise InvalidBlockError(f"store section {name!r} does not match the scene")
            scene.backing.write(off, data)

    # -- directory ----------------------------------------------------------
    def _check(self, spt_id: int):
        if spt_id < 0 or spt_id >= self.record_count.size:
            raise NotFoundError(f"unknown spt_id {spt_id}")

    def spt_slot_start(self, spt_id: int) -> int:
        self._check(spt_id)
        return self.nslots - self.total_records + int(self.record_offset[spt_id])

    # -- host (drop-in) API -------------------------------------------------
    def load_spt_prefix(self, spt_id: int, prefix_len: int) -> AttributeBlock:
        self._check(spt_id)
        if prefix_len > int(self.record_count[spt_id]):
            raise InvalidBlockError(f"prefix {prefix_len} exceeds record count "
                                    f"{int(self.record_count[spt_id])}")
        s = self.spt_slot_start(spt_id)
        parts = []
        for (name, cols), sec in zip(SECTIONS, self.sections):
            a = sec[s:s + prefix_len].cpu().numpy().copy()
            parts.append(a if cols > 1 else a[:, 0])
        self.attribute_bytes_read += prefix_len * self.bytes_per_gaussian
        return AttributeBlock(spt_id, int(prefix_len), AttributeArrays(*parts))

    def write_back(self, block: AttributeBlock) -> None:
        self._check(block.spt_id)
        if block.prefix_len > int(self.record_count[block.spt_id]):
            raise InvalidBlockError("block longer than the SPT")
        if not isinstance(block.attrs, AttributeArrays):
            raise InvalidBlockError("host write_back needs an AttributeArrays block")
        s = self.spt_slot_start(block.spt_id)
        for (name, cols), sec in zip(SECTIONS, self.sections):
            v = np.asarray(getattr(block.attrs, name), dtype=np.float32).reshape(block.prefix_len, cols)
            sec[s:s + block.prefix_len] = torch.from_numpy(v).to(sec.device)

    # -- device path ----------------------------------------------------------
    def prefix_to_device(self, spt_id: int, prefix_len: int, out_f32: torch.Tensor) -> None:
        """Six async H2D copies of the prefix into a packed f32 staging block
        (section-major, prefix_len rows).  Counts bytes like the reference."""
        s = self.spt_slot_start(spt_id)
        P = int(prefix_len)
        off = 0
        for (name, cols), sec in zip(SECTIONS, self.sections):
            out_f32[off:off + cols * P].view(P, cols).copy_(sec[s:s + P], non_blocking=True)
            off += cols * P
        self.attribute_bytes_read += P * self.bytes_per_gaussian

    def device_to_store(self, spt_id: int, prefix_len: int, src_f32: torch.Tensor) -> None:
        """Async D2H write-back of a packed f32 block (store.py:323-333)."""
        s = self.spt_slot_start(spt_id)
        P = int(prefix_len)
        off = 0
        for (name, cols), sec in zip(SECTIONS, self.sections):
            sec[s:s + P].copy_(src_f32[off:off + cols * P].view(P, cols), non_blocking=True)
            off += cols * P

    def device_view(self):
        """glod_store_view of the store (device-mapped addresses of the pinned
        rows; row_stride 23 for the interleaved layout)."""
        if getattr(self, "_view", None) is None:
            import ctypes as C
            from . import _lib
            v = _lib.StoreView()
            rows = getattr(self, "rows", None)
            if rows is not None:            # interleaved: sections at column offsets of one row
                base = rows.data_ptr()
                if not rows.is_cuda:
                    dp = C.c_void_p()
                    _lib.check(_lib.lib().glod_host_device_ptr(C.c_void_p(base), C.byref(dp)))
                    base = dp.value
                off = 0
                for k, (_, cols) in enumerate(SECTIONS):
                    v.section[k] = base + 4 * off
                    off += cols
                v.row_stride = 23
            else:
                for k, sec in enumerate(self.sections):
                    if sec.is_cuda:
                        v.section[k] = sec.data_ptr()
                        continue
                    dp = C.c_void_p()
                    _lib.check(_lib.lib().glod_host_device_ptr(C.c_void_p(sec.data_ptr()), C.byref(dp)))
                    v.section[k] = dp.value
            v.nslots = self.nslots
            self._view = v
        return self._view

    def memory_report(self, gaussian_count: int | None = None) -> dict:
        """store.py:395-411 accounting (92 B attrs, 184 B optimiser, 12 B SPT)."""
        n = self.nslots if gaussian_count is None else gaussian_count
        attr = self.bytes_per_gaussian
        return {"attribute_bytes_per_gaussian": attr, "optimizer_bytes_per_gaussian": 2 * attr,
                "spt_metadata_bytes_per_gaussian": 12, "topology_bytes_per_node": 12,
                "gaussian_count": int(n), "attribute_total_bytes": int(n) * attr,
                "optimizer_total_bytes": int(n) * 2 * attr, "spt_metadata_total_bytes": int(n) * 12,
                "training_bytes_per_gaussian": attr + 2 * attr + 12 + 12}


class DiskStore(HostStore):
    """Disk mode (the reference's FileBacking,
    store.py:84-112): the six attribute sections stay in the .glod file.
    The device cache pread()s missed prefixes into pinned bounce buffers and
    copies them to HBM (prefetches overlap the GPU's work on the current
    step) and pwrite()s write-backs (glod_cache_set_file); nothing of the
    store is held in host memory.  `sections` are read-only memory maps of
    the file for host-side inspection (they show the file as written so
    far; call the cache's flush_io() first)."""

    def __init__(self, scene):
        import os
        self.location = "disk"
        self.path = str(scene.path)
        self.slot_to_node = np.asarray(scene.slot_to_node, dtype=np.int64).copy()
        self.nslots = int(scene.nslots)
        self.record_offset = np.asarray(scene.spt_dir["record_offset"], dtype=np.int64)
        self.record_count = np.asarray(scene.spt_dir["record_count"], dtype=np.int64)
        self.total_records = int(self.record_count.sum())
        self.attribute_bytes_read = 0
        self.section_offsets = np.array([scene.sections[name][0] for name, _ in SECTIONS], dtype=np.int64)
        self.fd = os.open(self.path, os.O_RDWR)

    def __del__(self):
        import os
        try:
            os.close(self.fd)
        except Exception:
            pass

    @property
    def sections(self):
        out = []
        for (name, cols), off in zip(SECTIONS, self.section_offsets):
            m = np.memmap(self.path, dtype="<f4", mode="r", offset=int(off), shape=(self.nslots, cols))
            out.append(torch.from_numpy(np.array(m)))
        return out

    def load_spt_prefix(self, spt_id: int, prefix_len: int) -> AttributeBlock:
        self._check(spt_id)
        if prefix_len > int(self.record_count[spt_id]):
            raise InvalidBlockError(f"prefix {prefix_len} exceeds record count "
                                    f"{int(self.record_count[spt_id])}")
        s = self.spt_slot_start(spt_id)
        parts = []
        for (name, cols), off in zip(SECTIONS, self.section_offsets):
            a = np.fromfile(self.path, dtype="<f4", count=prefix_len * cols, offset=int(off) + 4 * cols * s)
            parts.append(a.reshape(prefix_len, cols) if cols > 1 else a)
        self.attribute_bytes_read += prefix_len * self.bytes_per_gaussian
        return AttributeBlock(spt_id, int(prefix_len), AttributeArrays(*parts))

    def write_back(self, block: AttributeBlock) -> None:
        import os
        self._check(block.spt_id)
        s = self.spt_slot_start(block.spt_id)
        for (name, cols), off in zip(SECTIONS, self.section_offsets):
            v = np.asarray(getattr(block.attrs, name), dtype="<f4").reshape(block.prefix_len, cols)
            os.pwrite(self.fd, v.tobytes(), int(off) + 4 * cols * s)

    def device_view(self):
        from . import _lib
        v = _lib.StoreView()
        v.nslots = self.nslots
        return v

    def to_scene(self, scene) -> None:
        """The file is the store: nothing to copy (flush the cache first)."""
