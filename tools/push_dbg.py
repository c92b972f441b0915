"""Debug aid: one register / register_batch call on golden meshes (run under timeout)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1411_2141_b200 as mrb  # noqa: E402
from conftest import golden  # noqa: E402

mode = sys.argv[1]
names = sys.argv[2].split(",")
gs = [golden(n) for n in names]
ims = [(mrb.ImageGrid(g["re"].shape[1], g["re"].shape[0], g["re"]),
        mrb.ImageGrid(g["te"].shape[1], g["te"].shape[0], g["te"]),
        mrb.TriMesh(g["V"], g["T_in"])) for g in gs]
cfg = mrb.SolverConfig(tau=0.001, max_iterations=int(os.environ.get("IT", "25")),
                       smoothing_passes=int(os.environ.get("PASSES", "1")), energy_tolerance=0.0)
if mode == "batch":
    out = mrb.register_batch([a for a, _, _ in ims], [b for _, b, _ in ims], [m for _, _, m in ims],
                             cfg, precision="f32")
    print("batch ok", [o[1].iterations_run for o in out])
else:
    for a, b, m in ims:
        u, rep = mrb.register(a, b, m, cfg, precision="f32")
        print("single ok", rep.iterations_run, m.n_vertices)
