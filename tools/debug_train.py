"""Debug: compare GPU vs oracle train steps row by row."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from tests.test_train_gpu import make_case, snapshot, restore, NAMES
from paper_2507_01110_b200.core import AttributeArrays
from oracle import glod_oracle as O

tr, orc, lrs = make_case()
for it in range(1, 6):
    snap = snapshot(tr)
    got = tr.train_step(it)
    restore(orc, snap)
    # replicate the oracle's gather to compare rows
    want, extra = orc.train_step(it, view=got["view"])
    R = got["gaussians_rendered"]
    rows = AttributeArrays.from_packed(tr._rows[:23 * R].cpu().numpy(), R)
    node = tr._row_node[:R].cpu().numpy()
    print(it, {k: (got[k], want[k]) for k in ("view", "loss", "gaussians_rendered", "cache_hits", "gaussians_loaded_from_store")})
    print("   row nodes equal:", np.array_equal(node, extra["row_nodes"]))
    # oracle rows: re-gather from snapshot state
    restore(orc, snap)
    cam, target = orc.views[got["view"]]
    rs = orc.cut(cam)
    print("   stats", tr.last_stats)
    img_gpu = tr.rast.forward(tr._rows[:23 * R], R, tr.views[got["view"]][0]).cpu().numpy()
    A = {k: getattr(rows, k) for k in NAMES}
    img_o, _ = O.render_forward(A, cam)
    print("   image(gpu rows) gpu vs oracle maxabs", np.abs(img_gpu - img_o).max())
    print("   oracle-image vs extra image maxabs", np.abs(img_o - extra["image"]).max())
