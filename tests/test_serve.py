"""Serve path: ServeSession.handle_pose message streams.

* the oracle restatement (oracle/serve_oracle.py) is pinned to the
  reference's own ServeSession output (tests/golden/serve_cases.npz);
* the device path (paper_2507_01110_b200.protocol: K2/K1 cut + one
  glod_wire_pack launch) is byte-identical to the golden streams and to the
  oracle on a larger generated scene (the Stats trailer's cut_ms is a
  wall-clock value and is masked);
* the host codecs mirror the reference's protocol tests
  (pkg/tests/test_protocol.py).
"""
from __future__ import annotations

import struct

import numpy as np
import pytest

from oracle.serve_oracle import ServeOracle
from paper_2507_01110_b200 import protocol as P
from paper_2507_01110_b200.core import AttributeArrays

from .conftest import golden
from .helpers import camera_of, hierarchy_of, hspt_of


def case_arrays(d, c):
    p = f"c{c}_"
    return {k[len(p):]: d[k] for k in d.files if k.startswith(p)}


def golden_msgs(cd, v):
    lens = cd[f"v{v}_lens"]
    buf = cd[f"v{v}_bytes"].tobytes()
    b = np.concatenate([[0], np.cumsum(lens)])
    return [buf[b[i]:b[i + 1]] for i in range(lens.size)]


def masked(msgs):
    """Zero the Stats trailer's cut_ms (last 4 bytes of the last message)."""
    assert msgs and msgs[-1][0] == P.MSG_STATS
    return list(msgs[:-1]) + [msgs[-1][:-4] + b"\0\0\0\0"]


def test_oracle_matches_reference_streams():
    d = golden("serve_cases.npz")
    for c in range(int(d["n_cases"])):
        cd = case_arrays(d, c)
        srv = ServeOracle(cd)
        for v in range(int(cd["n_views"])):
            got = srv.handle_pose(cd[f"v{v}_position"], cd[f"v{v}_planes"])
            assert masked(got) == masked(golden_msgs(cd, v)), f"case {c} pose {v}"


def test_codecs_roundtrip():
    rng = np.random.default_rng(0)
    a = AttributeArrays.zeros(5)
    a.means = rng.normal(size=(5, 3))
    a.scales = rng.uniform(0.1, 1, (5, 3))
    a.rotations = rng.normal(size=(5, 4))
    a.opacities = rng.uniform(size=5)
    a.base_colors = rng.uniform(size=(5, 3))
    a.sh_rest = rng.normal(size=(5, 9))
    msg, end = P.decode_message(P.encode_spt_load(7, a))
    assert msg["type"] == "spt_load" and msg["spt_id"] == 7 and msg["count"] == 5
    for name in ("means", "scales", "rotations", "opacities", "base_colors", "sh_rest"):
        np.testing.assert_array_equal(getattr(msg["attrs"], name),
                                      getattr(a, name).astype(np.float32).astype(np.float64))
    stream = P.encode_spt_evict(3) + P.encode_upper_set(a) + P.encode_stats(10, 5, 1000, 1.5)
    kinds = [m["type"] for m in P.decode_stream(stream)]
    assert kinds == ["spt_evict", "upper_set", "stats"]
    with pytest.raises(P.ProtocolError):
        P.decode_message(b"\x02\x00")
    with pytest.raises(P.ProtocolError):
        P.decode_message(P.frame(2, b"\x00" * 4)[:-1])
    with pytest.raises(P.ProtocolError):
        P.decode_message(P.frame(9, b""))
    with pytest.raises(P.ProtocolError):
        P.decode_message(P.frame(2, struct.pack("<II", 1, 2) + b"\x00" * 10))


@pytest.mark.gpu
def test_device_serve_matches_reference_streams():
    d = golden("serve_cases.npz")
    for c in range(int(d["n_cases"])):
        cd = case_arrays(d, c)
        sess = P.ServeSession(hierarchy=hierarchy_of(cd), hspt=hspt_of(cd), lod=hspt_of(cd).lod)
        for v in range(int(cd["n_views"])):
            got = sess.handle_pose(camera_of(cd, f"v{v}_"))
            assert masked(got) == masked(golden_msgs(cd, v)), f"case {c} pose {v}"


@pytest.mark.gpu
def test_device_serve_vs_oracle_generated():
    """20k-leaf designed scene, 1080p orbit path with a repeated pose; the
    replayed client ends with the server's resident set."""
    from paper_2507_01110_b200.core import Frustum
    from paper_2507_01110_b200.scenegen import SceneSpec, designed_scene, orbit_views, scene_extent
    h, hs, cfg = designed_scene(SceneSpec(n_leaves=20_000, spt_leaves=256, seed=3))
    E = scene_extent(20_000)
    cams = orbit_views(10, 1.4 * E, 0.5 * E, seed=4, jitter=0.3, target_jitter=0.2 * E)
    cams.insert(4, cams[3])
    flat = hs.flat_records()
    arrays = {"means": h.attrs.means, "scales": h.attrs.scales, "rotations": h.attrs.rotations,
              "opacities": h.attrs.opacities, "base_colors": h.attrs.base_colors,
              "sh_rest": h.attrs.sh_rest, "children": h.children, "root": h.root,
              "spt_root": flat["roots"], "pass_roots": hs.passthrough_roots, "spt_count": flat["count"],
              "spt_center": flat["centers"], "key_self": flat["key_self"],
              "key_parent": flat["key_parent"], "rec_node": flat["nodes"],
              "lod_threshold": cfg.threshold, "lod_metric": cfg.metric_code}
    srv = ServeOracle(arrays)
    sess = P.ServeSession(hierarchy=h, hspt=hs, lod=cfg)
    client = P.ClientReplay()
    loads = 0
    for i, cam in enumerate(cams):
        got = sess.handle_pose(cam)
        want = srv.handle_pose(cam.position, Frustum.from_camera(cam).planes)
        assert masked(got) == masked(want), f"pose {i}"
        for m in P.decode_stream(b"".join(got)):
            client.apply(m)
            loads += m["type"] == "spt_load"
    assert loads > 10
    assert client.resident_counts() == sess.resident_counts()
    assert client.unknown_evictions == 0
