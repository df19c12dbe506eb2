"""ORACLE — test infrastructure only (see oracle/glod_oracle.py header).

CPU restatement of the reference's serve path, `ServeSession.handle_pose`
(protocol.py:165-193) with its wire codecs (protocol.py:40-49, 76-96), on top
of the C oracle cut (glod_oracle.cut_hspt, hspt.py:104-158).  Produces the
reference's message bytes for a camera path; the Stats trailer's cut_ms
float is written as 0.0 (it is a wall-clock measurement).

Pinned by tests/test_serve.py against tests/golden/serve_cases.npz (the
reference's own ServeSession output, tests/golden/make_golden.py).
"""
from __future__ import annotations

import struct

import numpy as np

from . import glod_oracle as O

_COLS = (3, 3, 4, 1, 3, 9)   # means, scales, rotations, opacities, base_colors, sh_rest


def wire_attrs(sections, ids) -> bytes:
    """protocol._wire_attrs (protocol.py:40-49) of rows `ids`: each section
    as contiguous little-endian f32, row-major within the section."""
    return b"".join(np.ascontiguousarray(sec[ids], dtype="<f4").tobytes() for sec in sections)


def frame(t, payload: bytes) -> bytes:
    return struct.pack("<BI", t, len(payload)) + payload


class ServeOracle:
    """Per-client state of ServeSession (protocol.py:152-163)."""

    def __init__(self, d: dict):
        self.d = d
        sh = np.zeros((d["sh_rest"].shape[0], 9))
        c = min(d["sh_rest"].shape[1], 9)
        sh[:, :c] = d["sh_rest"][:, :c]
        self.sections = [d["means"], d["scales"], d["rotations"], d["opacities"], d["base_colors"], sh]
        cap = d["children"].shape[0]
        kind = np.full(cap, -1, np.int32)
        kind[d["spt_root"]] = np.arange(d["spt_root"].size, dtype=np.int32)
        if d["pass_roots"].size:
            kind[d["pass_roots"]] = -2
        cnt = d["spt_count"]
        self.kind = kind
        self.off = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64) if cnt.size else cnt
        self.resident_spts: dict = {}
        self.resident_upper = np.empty(0, dtype=np.int64)
        self.bytes_sent = 0

    def handle_pose(self, position, planes) -> list:
        d = self.d
        rs = O.cut_hspt(int(d["root"]), d["children"], self.kind, d["means"], d["scales"], self.off,
                        d["spt_count"], d["spt_root"], d["spt_center"], d["key_self"], d["key_parent"],
                        d["rec_node"], position, float(d["lod_threshold"]), int(d["lod_metric"]), planes)
        out, loaded = [], 0
        new = {int(s): sel for s, sel in zip(rs["spt_id"], rs["selected"]) if sel.size > 0}
        for sid in list(self.resident_spts):                      # protocol.py:176-179
            if sid not in new:
                del self.resident_spts[sid]
                out.append(frame(3, struct.pack("<I", sid)))
        for sid, nodes in new.items():                            # :180-187
            have = self.resident_spts.get(sid)
            if have is not None and np.array_equal(have, nodes):
                continue
            out.append(frame(2, struct.pack("<II", sid, nodes.size) + wire_attrs(self.sections, nodes)))
            self.resident_spts[sid] = nodes
            loaded += nodes.size
        upper = np.concatenate([rs["upper"], rs["passthrough"]])  # :188-192
        if not np.array_equal(upper, self.resident_upper):
            out.append(frame(4, struct.pack("<I", upper.size) + wire_attrs(self.sections, upper)))
            self.resident_upper = upper
            loaded += upper.size
        self.bytes_sent += sum(len(m) for m in out)
        n_rs = rs["upper"].size + rs["passthrough"].size + sum(s.size for s in rs["selected"])
        out.append(frame(5, struct.pack("<IIQf", n_rs, loaded, self.bytes_sent, 0.0)))
        return out
