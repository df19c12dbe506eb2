"""Micro-benchmark: pinned-store prefix transfers (zero-copy kernel vs cudaMemcpyAsync)."""
import ctypes as C
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2507_01110_b200 import _lib
from paper_2507_01110_b200.core import SECTIONS

N = 20_000_000
secs = [torch.empty((N, c), dtype=torch.float32).pin_memory() for _, c in SECTIONS]
for s in secs:
    s.fill_(1.5)
view = _lib.StoreView()
for k, s in enumerate(secs):
    dp = C.c_void_p()
    _lib.check(_lib.lib().glod_host_device_ptr(C.c_void_p(s.data_ptr()), C.byref(dp)))
    view.section[k] = dp.value
view.nslots = N
rng = np.random.default_rng(0)
for n_items, rows_each in [(120, 8000), (600, 1600), (30, 32000)]:
    starts = np.sort(rng.choice(N // rows_each - 1, n_items, replace=False)) * rows_each
    blocks = [torch.empty(23 * rows_each, dtype=torch.float64, device="cuda") for _ in range(n_items)]
    tab = np.zeros((n_items, 7), np.int64)     # glod_prefix_item incl. overlay, overlay_rows, src
    for i in range(n_items):
        tab[i] = (starts[i], rows_each, 23 * rows_each * i, blocks[i].data_ptr(), 0, 0, 0)
    dtab = torch.from_numpy(tab).cuda()
    total = 23 * rows_each * n_items
    mb = total * 4 / 1e6
    for load, name in ((1, "load"), (0, "write")):
        fn = _lib.lib().glod_store_load_prefixes if load else _lib.lib().glod_store_write_back
        for rep in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            _lib.check(fn(C.byref(view), _lib.ptr(dtab), n_items, total, _lib.stream_ptr()))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
        print(f"zero-copy {name}: items={n_items} rows={rows_each} {mb:.0f} MB in {dt*1e3:.2f} ms = {mb/1e3/dt:.1f} GB/s")
    # memcpy path: 6 ranges per item into a staging f32 buffer
    staging = torch.empty(total, dtype=torch.float32, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        off = 0
        for i in range(n_items):
            for (nm, c), s in zip(SECTIONS, secs):
                staging[off:off + c * rows_each].view(rows_each, c).copy_(s[starts[i]:starts[i] + rows_each], non_blocking=True)
                off += c * rows_each
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"memcpy(torch) load: {mb:.0f} MB in {dt*1e3:.2f} ms = {mb/1e3/dt:.1f} GB/s")
    big = torch.empty(total, dtype=torch.float32).pin_memory()
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        staging.copy_(big, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"single memcpy H2D: {mb:.0f} MB in {dt*1e3:.2f} ms = {mb/1e3/dt:.1f} GB/s")
