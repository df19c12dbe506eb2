"""K6 radix sort: stable (key, value) order against numpy's stable argsort,
with heavy key duplication (ties must keep input order, renderer.py:127)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2507_01110_b200 import _lib  # noqa: E402


@pytest.mark.parametrize("width,n,bits", [(64, 1, 64), (64, 1000, 64), (64, 300_000, 64),
                                          (32, 5_000_000, 13), (32, 77_777, 32), (64, 2_500_000, 40)])
def test_sort_pairs_stable(width, n, bits):
    rng = np.random.default_rng(n + bits)
    hi = min(2 ** bits, 2 ** 63)
    keys = rng.integers(0, max(hi // max(n // 8, 1), 2), n, dtype=np.uint64) if bits > 20 else \
        rng.integers(0, 2 ** bits, n, dtype=np.uint64)
    if bits == 64:   # fp64-depth-like keys: positive doubles as uint64, many exact ties
        d = rng.uniform(1.0, 300.0, n)
        d[::7] = d[0]
        keys = d.view(np.uint64).copy()
    dt = np.uint64 if width == 64 else np.uint32
    keys = keys.astype(dt)
    vals = np.arange(n, dtype=np.int32)
    tk = torch.from_numpy(keys.view(np.int64 if width == 64 else np.int32)).cuda()
    tk2 = torch.empty_like(tk)
    tv = torch.from_numpy(vals).cuda()
    tv2 = torch.empty_like(tv)
    L = _lib.lib()
    scratch = torch.empty(int(L.glod_sort_scratch_bytes(n)), dtype=torch.uint8, device="cuda")
    alt = C.c_int32(0)
    fn = L.glod_sort_pairs_u64 if width == 64 else L.glod_sort_pairs_u32
    _lib.check(fn(_lib.ptr(tk), _lib.ptr(tk2), _lib.ptr(tv), _lib.ptr(tv2), n, 0, bits,
                  _lib.ptr(scratch), scratch.numel(), C.byref(alt), _lib.stream_ptr()))
    out_v = (tv2 if alt.value else tv).cpu().numpy()
    out_k = (tk2 if alt.value else tk).cpu().numpy().view(dt)
    want = np.argsort(keys, kind="stable")
    np.testing.assert_array_equal(out_v, want.astype(np.int32))
    np.testing.assert_array_equal(out_k, keys[want])
