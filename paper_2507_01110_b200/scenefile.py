"""Scene files: the reference's bit-exact little-endian
`.glod` format (store.py:1-40, write_scene :157-234, Scene._parse :245-280),
read straight into the pinned host store.

Layout (store.py): a 40-B header (magic, version, gaussian/node counts, SH
degree, section count), a table of 32-B section entries (16-B name, offset,
length), then 64-B-aligned sections: six f32 attribute sections in *slot*
order (non-SPT nodes ascending, then each SPT's records in record order),
topology (`parents`, `children`, u32 with 0xFFFFFFFF = NONE), `slot_to_node`,
`node_to_slot`, `upper_nodes`, `pass_roots`, the SPT directory, the packed
12-B SPT records and a `meta` record.

This module mirrors the reference's API for it — `write_scene`,
`open_scene` → `Scene` with `read_hierarchy`, `read_hspt`, `read_spt`,
`load_spt_prefix`, `write_back`, `spt_slot_start`, `memory_report` — and
adds the device path's entry points:

  * `Scene.host_store(location)`: a `HostStore` whose six sections are read
    from the file directly into page-locked host memory (one sequential read
    per section, no intermediate copy), ready for the trainer's copy-engine
    prefetch;
  * `Scene.save_store(store)`: the trained store written back into the file
    in place (the reference's write_back, store.py:323-333, for every slot).

Parsing and writing are host byte formatting; nothing here is on the per-view
path.
"""
from __future__ import annotations

import struct

import numpy as np

from .core import AttributeArrays, EmptySceneError, LodConfig
from .hierarchy import NONE, Hierarchy
from .hspt import Hspt
from .spt import RECORD_DTYPE, Spt
from .store import AttributeBlock, HostStore, InvalidBlockError, NotFoundError, slot_order

MAGIC = b"GLOD"
VERSION = 1
ALIGN = 64
U32_NONE = 0xFFFFFFFF

SPT_DIR_DTYPE = np.dtype([("spt_id", "<u4"), ("root", "<u4"), ("root_center", "<f4", (3,)),
                          ("record_offset", "<u8"), ("record_count", "<u4")])
META_DTYPE = np.dtype([("root", "<u4"), ("size_threshold", "<f8"), ("min_subtree", "<u4"),
                       ("lod_threshold", "<f8"), ("lod_metric", "<u1")])
_HEADER = struct.Struct("<4sIQQB3xII4x")  # 40 bytes
_SECTION = struct.Struct("<16sQQ")        # 32 bytes


class CorruptFileError(ValueError):
    pass


def _align(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


def _attr_specs(sh_cols: int):
    return [("means", 3), ("scales", 3), ("rotations", 4), ("opacities", 1), ("base_colors", 3),
            ("sh_rest", sh_cols)]


def attribute_bytes_per_gaussian(sh_degree: int) -> int:
    return 4 * sum(c for _, c in _attr_specs(3 * ((sh_degree + 1) ** 2 - 1)))


def write_scene(h, hspt, path) -> None:
    """Serialise hierarchy + HSPT (store.py:157-234), byte for byte."""
    h, hspt = Hierarchy.from_any(h), Hspt.from_any(hspt)
    if h.node_count == 0:
        raise EmptySceneError("refusing to write an empty scene")
    slot_to_node = slot_order(h, hspt)
    nslots = slot_to_node.size
    node_to_slot = np.full(h.capacity, U32_NONE, dtype=np.uint32)
    node_to_slot[slot_to_node] = np.arange(nslots, dtype=np.uint32)
    sh_cols = h.attrs.sh_rest.shape[1]
    sections = [(name, np.asarray(getattr(h.attrs, name))[slot_to_node].astype("<f4").tobytes())
                for name, _ in _attr_specs(sh_cols)]
    parent = h.parent.astype(np.int64)
    sections.append(("parents", np.where(parent == NONE, U32_NONE, parent).astype("<u4").tobytes()))
    kids = h.children.astype(np.int64)
    sections.append(("children", np.where(kids == NONE, U32_NONE, kids).astype("<u4").tobytes()))
    sections.append(("slot_to_node", slot_to_node.astype("<u4").tobytes()))
    sections.append(("node_to_slot", node_to_slot.tobytes()))
    sections.append(("upper_nodes", np.asarray(hspt.upper_nodes).astype("<u4").tobytes()))
    sections.append(("pass_roots", np.asarray(hspt.passthrough_roots).astype("<u4").tobytes()))
    S = len(hspt.spts)
    sdir = np.zeros(S, dtype=SPT_DIR_DTYPE)
    counts = np.array([s.subtree_size for s in hspt.spts], dtype=np.int64)
    sdir["spt_id"] = np.arange(S)
    sdir["root"] = [s.root for s in hspt.spts]
    if S:
        sdir["root_center"] = np.stack([np.asarray(s.root_center) for s in hspt.spts]).astype(np.float32)
        sdir["record_offset"] = np.concatenate([[0], np.cumsum(counts)[:-1]])
    sdir["record_count"] = counts
    rec = np.empty(int(counts.sum()), dtype=RECORD_DTYPE)
    if S:
        rec["key_self"] = np.concatenate([s.key_self for s in hspt.spts]).astype(np.float32)
        rec["key_parent"] = np.concatenate([s.key_parent for s in hspt.spts]).astype(np.float32)
        rec["node"] = np.concatenate([s.nodes for s in hspt.spts]).astype(np.uint32)
    sections.append(("spt_dir", sdir.tobytes()))
    sections.append(("spt_records", rec.tobytes()))
    meta = np.zeros(1, dtype=META_DTYPE)
    meta[0]["root"] = h.root
    meta[0]["size_threshold"] = hspt.size_threshold
    meta[0]["min_subtree"] = hspt.min_subtree
    meta[0]["lod_threshold"] = hspt.lod.threshold
    meta[0]["lod_metric"] = 0 if hspt.lod.metric == "max_scale" else 1
    sections.append(("meta", meta.tobytes()))

    table_at = _HEADER.size
    cursor = _align(table_at + _SECTION.size * len(sections))
    offsets = []
    for _, data in sections:
        offsets.append(cursor)
        cursor = _align(cursor + len(data))
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MAGIC, VERSION, h.leaf_count, h.node_count, h.attrs.sh_degree, 0, len(sections)))
        for i, (name, data) in enumerate(sections):
            f.seek(table_at + i * _SECTION.size)
            f.write(_SECTION.pack(name.encode().ljust(16, b"\x00"), offsets[i], len(data)))
            f.seek(offsets[i])
            f.write(data)
        if f.tell() < cursor:
            f.seek(cursor - 1)
            f.write(b"\x00")


class Scene:
    """Open scene file (store.py:238-415): demand reads of SPT prefixes,
    write-back, and the pinned-store / device entry points."""

    def __init__(self, path, mode: str = "r+b"):
        self.path = path
        self.f = open(path, mode)
        self.attribute_bytes_read = 0
        self._parse()

    # -- parsing (store.py:245-280) ------------------------------------------
    def _read(self, off: int, n: int) -> bytes:
        self.f.seek(off)
        data = self.f.read(n)
        if len(data) != n:
            raise CorruptFileError(f"truncated read at byte {off}")
        return data

    def _parse(self):
        magic, version, gcount, ncount, sh_degree, _, nsect = _HEADER.unpack(self._read(0, _HEADER.size))
        if magic != MAGIC:
            raise CorruptFileError("bad magic at byte 0")
        if version != VERSION:
            raise CorruptFileError(f"unsupported version {version} at byte 4")
        self.gaussian_count, self.node_count, self.sh_degree = gcount, ncount, sh_degree
        self.sh_cols = 3 * ((sh_degree + 1) ** 2 - 1)
        self.sections = {}
        for i in range(nsect):
            at = _HEADER.size + i * _SECTION.size
            name, off, length = _SECTION.unpack(self._read(at, _SECTION.size))
            if off % ALIGN:
                raise CorruptFileError(f"section misaligned at byte {at}")
            self.sections[name.rstrip(b"\x00").decode()] = (off, length)
        meta = np.frombuffer(self._read(*self._section("meta")), dtype=META_DTYPE)[0]
        self.root = int(meta["root"])
        self.size_threshold = float(meta["size_threshold"])
        self.min_subtree = int(meta["min_subtree"])
        self.lod = LodConfig(threshold=float(meta["lod_threshold"]),
                             metric="max_scale" if meta["lod_metric"] == 0 else "surface_area")
        self.spt_dir = np.frombuffer(self._read(*self._section("spt_dir")), dtype=SPT_DIR_DTYPE)
        self.slot_to_node = np.frombuffer(self._read(*self._section("slot_to_node")), dtype="<u4").astype(np.int64)
        self.nslots = self.slot_to_node.size

    def _section(self, name):
        if name not in self.sections:
            raise CorruptFileError(f"missing section {name!r}")
        return self.sections[name]

    @property
    def bytes_per_gaussian(self) -> int:
        return attribute_bytes_per_gaussian(self.sh_degree)

    def _spt_entry(self, spt_id: int):
        if spt_id < 0 or spt_id >= self.spt_dir.size:
            raise NotFoundError(f"unknown spt_id {spt_id}")
        return self.spt_dir[spt_id]

    def spt_slot_start(self, spt_id: int) -> int:
        entry = self._spt_entry(spt_id)
        return self.nslots - int(self.spt_dir["record_count"].sum()) + int(entry["record_offset"])

    # -- reference API ---------------------------------------------------------
    def _read_slots(self, start: int, count: int) -> AttributeArrays:
        arrays = {}
        for name, cols in _attr_specs(self.sh_cols):
            off, _ = self._section(name)
            data = self._read(off + 4 * cols * start, 4 * cols * count)
            arr = np.frombuffer(data, dtype="<f4")
            arrays[name] = arr.reshape(count, cols) if cols > 1 else arr
            self.attribute_bytes_read += len(data)
        return AttributeArrays(**arrays)

    def load_spt_prefix(self, spt_id: int, prefix_len: int) -> AttributeBlock:
        entry = self._spt_entry(spt_id)
        if prefix_len > int(entry["record_count"]):
            raise InvalidBlockError(f"prefix {prefix_len} exceeds record count {entry['record_count']}")
        attrs = self._read_slots(self.spt_slot_start(spt_id), int(prefix_len))
        return AttributeBlock(spt_id=spt_id, prefix_len=int(prefix_len), attrs=attrs)

    def write_back(self, block: AttributeBlock) -> None:
        entry = self._spt_entry(block.spt_id)
        if block.prefix_len > int(entry["record_count"]):
            raise InvalidBlockError("block longer than the SPT")
        start = self.spt_slot_start(block.spt_id)
        for name, cols in _attr_specs(self.sh_cols):
            off, _ = self._section(name)
            data = np.asarray(getattr(block.attrs, name)).astype("<f4").tobytes()
            if len(data) != 4 * cols * block.prefix_len:
                raise InvalidBlockError(f"bad {name} array length")
            self.f.seek(off + 4 * cols * start)
            self.f.write(data)

    def read_spt(self, spt_id: int) -> Spt:
        entry = self._spt_entry(spt_id)
        off, _ = self._section("spt_records")
        rec = np.frombuffer(self._read(off + int(entry["record_offset"]) * RECORD_DTYPE.itemsize,
                                       int(entry["record_count"]) * RECORD_DTYPE.itemsize), dtype=RECORD_DTYPE)
        return Spt.from_packed(int(entry["root"]), entry["root_center"].astype(np.float64), rec)

    def read_hierarchy(self) -> Hierarchy:
        parents = np.frombuffer(self._read(*self._section("parents")), dtype="<u4")
        children = np.frombuffer(self._read(*self._section("children")), dtype="<u4").reshape(-1, 2)
        cap = parents.size
        slots = self._read_slots(0, self.nslots)
        self.attribute_bytes_read -= self.nslots * self.bytes_per_gaussian   # not a demand read
        attrs = AttributeArrays.zeros(cap, dtype=np.float64)
        if attrs.sh_rest.shape[1] != self.sh_cols:
            attrs.sh_rest = np.zeros((cap, self.sh_cols))
        attrs.put(self.slot_to_node, slots.astype(np.float64))
        alive = np.zeros(cap, dtype=bool)
        alive[self.slot_to_node] = True
        parent = np.where(parents == U32_NONE, NONE, parents.astype(np.int64))
        kids = np.where(children == U32_NONE, NONE, children.astype(np.int64))
        return Hierarchy(attrs=attrs, parent=parent.astype(np.int32), children=kids.astype(np.int32),
                         root=self.root, free=list(np.nonzero(~alive)[0]))

    def read_hspt(self) -> Hspt:
        upper = np.frombuffer(self._read(*self._section("upper_nodes")), dtype="<u4").astype(np.int64)
        pass_roots = np.frombuffer(self._read(*self._section("pass_roots")), dtype="<u4").astype(np.int64)
        spts = [self.read_spt(i) for i in range(self.spt_dir.size)]
        return Hspt(upper_nodes=upper, spts=spts, passthrough_roots=pass_roots,
                    size_threshold=self.size_threshold, min_subtree=self.min_subtree, lod=self.lod,
                    spt_id_of={s.root: i for i, s in enumerate(spts)})

    def memory_report(self, gaussian_count: int | None = None) -> dict:
        n = self.gaussian_count if gaussian_count is None else gaussian_count
        attr = self.bytes_per_gaussian
        return {"attribute_bytes_per_gaussian": attr, "optimizer_bytes_per_gaussian": 2 * attr,
                "spt_metadata_bytes_per_gaussian": RECORD_DTYPE.itemsize, "topology_bytes_per_node": 12,
                "gaussian_count": int(n), "attribute_total_bytes": int(n) * attr,
                "optimizer_total_bytes": int(n) * 2 * attr,
                "spt_metadata_total_bytes": int(n) * RECORD_DTYPE.itemsize,
                "training_bytes_per_gaussian": attr + 2 * attr + RECORD_DTYPE.itemsize + 12}

    # -- device path -------------------------------------------------------------
    def host_store(self, location: str = "host") -> HostStore:
        """HostStore over this file's slots (the SPT directory gives the
        per-SPT record offsets/counts): every attribute section read and
        interleaved into page-locked rows (or HBM for location="device")."""
        import torch
        if self.sh_cols != 9:
            raise ValueError("the device path keeps degree-1 SH (9 columns)")
        st = HostStore.__new__(HostStore)
        st.location = location
        st.slot_to_node = self.slot_to_node.copy()
        st.nslots = int(self.nslots)
        st.record_offset = self.spt_dir["record_offset"].astype(np.int64)
        st.record_count = self.spt_dir["record_count"].astype(np.int64)
        st.total_records = int(st.record_count.sum())
        st.attribute_bytes_read = 0
        from .store import alloc_rows, fill_section
        st.rows, st.sections = alloc_rows(st.nslots, location)
        tmp = np.empty(self.nslots * 9, dtype="<f4")
        for (name, cols), sec in zip(_attr_specs(self.sh_cols), st.sections):
            off, length = self._section(name)
            buf = tmp[:self.nslots * cols]
            self.f.seek(off)
            if self.f.readinto(memoryview(buf).cast("B")) != length:
                raise CorruptFileError(f"truncated section {name!r}")
            fill_section(sec, buf.reshape(self.nslots, cols))
        return st

    def disk_store(self):
        """Disk mode: a store that stays in this file (store.DiskStore)."""
        from .store import DiskStore
        if self.sh_cols != 9:
            raise ValueError("the device path keeps degree-1 SH (9 columns)")
        self.f.flush()
        return DiskStore(self)

    def save_store(self, store: HostStore) -> None:
        """Write the store's sections back into the file (store.py:323-333 for
        every slot), e.g. after training or at a flush."""
        import torch
        torch.cuda.synchronize()
        for (name, cols), sec in zip(_attr_specs(self.sh_cols), store.sections):
            off, length = self._section(name)
            data = sec.cpu().numpy().astype("<f4", copy=False).tobytes()
            if len(data) != length:
                raise InvalidBlockError(f"store section {name!r} does not match the file")
            self.f.seek(off)
            self.f.write(data)
        self.f.flush()

    def close(self):
        self.f.close()


def open_scene(path, mode: str = "r+b") -> Scene:
    return Scene(path, mode)
