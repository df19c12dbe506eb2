"""Adapters between golden-vector arrays, the product types and the oracle."""
from __future__ import annotations

import numpy as np

from paper_2507_01110_b200.core import AttributeArrays, Camera, LodConfig
from paper_2507_01110_b200.hierarchy import Hierarchy
from paper_2507_01110_b200.hspt import Hspt
from paper_2507_01110_b200.spt import Spt


def hierarchy_of(d) -> Hierarchy:
    attrs = AttributeArrays(d["means"], d["scales"], d["rotations"], d["opacities"],
                            d["base_colors"], d["sh_rest"])
    return Hierarchy(attrs=attrs, parent=d["parent"].astype(np.int32),
                     children=d["children"].astype(np.int32), root=int(d["root"]))


def hspt_of(d) -> Hspt:
    cnt = d["spt_count"]
    off = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64) if cnt.size else cnt
    spts = [Spt(root=int(r), root_center=d["spt_center"][i],
                nodes=d["rec_node"][o:o + c], key_self=d["key_self"][o:o + c],
                key_parent=d["key_parent"][o:o + c])
            for i, (r, o, c) in enumerate(zip(d["spt_root"], off, cnt))]
    lod = LodConfig(float(d["lod_threshold"]), ("max_scale", "surface_area")[int(d["lod_metric"])])
    return Hspt(upper_nodes=d["upper_nodes"], spts=spts, passthrough_roots=d["pass_roots"],
                size_threshold=float(d["size_threshold"]), min_subtree=int(d["min_subtree"]),
                lod=lod, spt_id_of={int(r): i for i, r in enumerate(d["spt_root"])})


def camera_of(d, p) -> Camera:
    return Camera(position=d[p + "position"], orientation=d[p + "orientation"],
                  focal=tuple(d[p + "focal"]), principal_point=tuple(d[p + "pp"]),
                  resolution=tuple(int(x) for x in d[p + "res"]), near=float(d[p + "near"]),
                  far=float(d[p + "far"]))


def view_cfg(d, v):
    return LodConfig(float(d[f"v{v}_T"]), ("max_scale", "surface_area")[int(d[f"v{v}_metric"])])


def oracle_cut_hspt(d, v, cull=None):
    """Run the C oracle on golden case arrays for view v."""
    from oracle import glod_oracle as O
    cap = d["children"].shape[0]
    kind = np.full(cap, -1, np.int32)
    kind[d["spt_root"]] = np.arange(d["spt_root"].size, dtype=np.int32)
    if d["pass_roots"].size:
        kind[d["pass_roots"]] = -2
    cnt = d["spt_count"]
    off = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64) if cnt.size else cnt
    c = bool(d[f"v{v}_cull"]) if cull is None else cull
    planes = d[f"v{v}_planes"] if c else None
    return O.cut_hspt(int(d["root"]), d["children"], kind, d["means"], d["scales"], off, cnt,
                      d["spt_root"], d["spt_center"], d["key_self"], d["key_parent"],
                      d["rec_node"], d[f"v{v}_position"], float(d[f"v{v}_T"]),
                      int(d[f"v{v}_metric"]), planes)


def golden_rs(d, v):
    p = f"v{v}_rs_"
    cnt = d[p + "sel_count"]
    b = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    return {"upper": d[p + "upper"], "passthrough": d[p + "pass"], "spt_id": d[p + "spt_id"],
            "d_root": d[p + "d_root"], "prefix_len": d[p + "prefix_len"],
            "selected": [d[p + "sel"][b[j]:b[j + 1]] for j in range(cnt.size)]}


def assert_rs_equal(got, want, where=""):
    """Bit-exact RenderSet comparison (order, ids, d_root bits, prefix)."""
    np.testing.assert_array_equal(got["upper"], want["upper"], err_msg=f"{where} upper")
    np.testing.assert_array_equal(got["passthrough"], want["passthrough"], err_msg=f"{where} pass")
    np.testing.assert_array_equal(got["spt_id"], want["spt_id"], err_msg=f"{where} spt ids")
    assert np.array_equal(np.asarray(got["d_root"]).view(np.uint64),
                          np.asarray(want["d_root"]).view(np.uint64)), f"{where} d_root bits"
    np.testing.assert_array_equal(got["prefix_len"], want["prefix_len"], err_msg=f"{where} prefix")
    assert len(got["selected"]) == len(want["selected"])
    for j, (a, b) in enumerate(zip(got["selected"], want["selected"])):
        np.testing.assert_array_equal(a, b, err_msg=f"{where} spt #{j} selection")


def rs_dict(rs):
    return {"upper": rs.upper, "passthrough": rs.passthrough,
            "spt_id": np.array([s.spt_id for s in rs.per_spt], dtype=np.int64),
            "d_root": np.array([s.d_root for s in rs.per_spt], dtype=np.float64),
            "prefix_len": np.array([s.prefix_len for s in rs.per_spt], dtype=np.int64),
            "selected": [s.selected for s in rs.per_spt]}
