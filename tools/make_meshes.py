"""Generate and cache content-adaptive meshes with the REFERENCE mesher.

Runs only in the build container (it imports the reference package from
/root/reference, which does not exist on the GPU box).  The mesh is an input
to the registration path, produced once outside the timed region and fed
identically to both sides (BASELINE.json north_star).

Output: data/meshes/<cfg>_s<seed>[_x255].npz with V float64 (n,2) and
T int32 (m,3) (the reference's TriMesh arrays after its CCW reorientation).

usage: python tools/make_meshes.py c1 0 [c2 0-63 ...] [--x255] [-j N]
"""
import argparse
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "data", "meshes")


def mesh_path(cfg, seed, x255=False):
    return os.path.join(OUT, f"{cfg}_s{seed}{'_x255' if x255 else ''}.npz")


def one(job):
    cfg, seed, x255 = job
    sys.path.insert(0, REF)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    import meshreg as mr
    from paper_1411_2141_b200.synthetic import CONFIGS, make_pair

    path = mesh_path(cfg, seed, x255)
    if os.path.exists(path):
        return path, 0.0
    spec = CONFIGS[cfg]
    re, te = make_pair(spec, seed, scale=255.0 if x255 else 1.0)
    t0 = time.time()
    img = mr.ImageGrid(spec.size, spec.size, te.astype(np.float64))
    mesh = mr.generate_mesh(img, mr.NodeBudget(spec.target_nodes), mr.MeshGenConfig(seed=0))
    dt = time.time() - t0
    tmp = path + ".tmp.npz"
    np.savez_compressed(tmp, V=mesh.vertices, T=mesh.triangles.astype(np.int32),
                        mesher_seconds=dt)
    os.replace(tmp, path)
    return path, dt


def parse_seeds(s):
    out = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("items", nargs="+", help="cfg seeds pairs, e.g. c2 0-63")
    ap.add_argument("--x255", action="store_true")
    ap.add_argument("-j", type=int, default=1)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    jobs = []
    for cfg, seeds in zip(a.items[0::2], a.items[1::2]):
        jobs += [(cfg, s, a.x255) for s in parse_seeds(seeds)]
    if a.j > 1:
        from multiprocessing import Pool
        with Pool(a.j) as p:
            for path, dt in p.imap_unordered(one, jobs):
                print(f"{path} {dt:.1f}s", flush=True)
    else:
        for j in jobs:
            path, dt = one(j)
            print(f"{path} {dt:.1f}s", flush=True)
