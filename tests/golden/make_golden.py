"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container only (imports /root/reference/pkg/src/meshreg, which
does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/<case>.npz.  Each file holds the inputs (images, mesh) and
the reference's outputs for the hot path: displacement u,
energy trace, iterations run, MSD before/after, dense field, warped image, the
CSR operators (L, grad_x_op, grad_y_op, vertex_average_op), connectivity and
the pixel->triangle map captured from the reference's own `densify`.
The reference ships no golden files; these pin both the
oracle (oracle/meshreg_oracle.py) and the B200 path.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import meshreg as mr  # noqa: E402
import meshreg.densefield as mr_df  # noqa: E402
from meshreg import synthetic  # noqa: E402
from scipy import ndimage  # noqa: E402

from paper_1411_2141_b200.synthetic import PairSpec, make_pair  # noqa: E402


class _Capture:
    """Stand-in for the numpy module inside meshreg.densefield that records
    the pixel->triangle map and weights arrays `densify` allocates and fills
    (densefield.py:148-149), so the golden map is the reference's own."""

    def __init__(self):
        self.arrays = {}

    def __getattr__(self, name):
        return getattr(np, name)

    def full(self, *a, **k):
        out = np.full(*a, **k)
        self.arrays["tri_of"] = out
        return out

    def zeros(self, shape, *a, **k):
        out = np.zeros(shape, *a, **k)
        if isinstance(shape, tuple) and len(shape) == 3 and shape[2] == 3:
            self.arrays["weights"] = out
        return out


def reference_pixel_map(mesh, w, h):
    cap = _Capture()
    mr_df.np = cap
    try:
        mr.densify(mesh, np.zeros((mesh.n_vertices, 2)), w, h)
    finally:
        mr_df.np = np
    return cap.arrays["tri_of"], cap.arrays["weights"]


def csr_parts(prefix, A):
    A = A.tocsr() if hasattr(A, "tocsr") else A
    assert A.has_canonical_format
    return {f"{prefix}_indptr": A.indptr.astype(np.int64),
            f"{prefix}_indices": A.indices.astype(np.int64),
            f"{prefix}_data": A.data.astype(np.float64)}


def mesh_parts(mesh, with_ops=True):
    out = {"V": mesh.vertices.copy(), "T_in": mesh.triangles.copy(),
           "T": mesh.triangles.copy(), "edges": mesh.edges.astype(np.int64),
           "valence": mesh.valence.astype(np.int64), "boundary": mesh.boundary.copy(),
           "ring_ptr": np.concatenate([[0], np.cumsum([len(r) for r in mesh.rings])]).astype(np.int64),
           "ring_idx": np.concatenate(mesh.rings).astype(np.int64),
           "inc_ptr": np.concatenate([[0], np.cumsum([len(r) for r in mesh.incident])]).astype(np.int64),
           "inc_idx": np.concatenate(mesh.incident).astype(np.int64)}
    if with_ops:
        g = mesh.geometry
        out.update(csr_parts("L", mr.build_laplacian(mesh)))
        out.update(csr_parts("gx", g.grad_x_op))
        out.update(csr_parts("gy", g.grad_y_op))
        out.update(csr_parts("avg", g.vertex_average_op))
        out.update(areas=g.areas, coeffs=g.coeffs, vertex_areas=g.vertex_areas)
    return out


def run_register(re, te, mesh, cfg, dense=True):
    u, rep = mr.register(re, te, mesh, cfg)
    out = {"u": u, "trace": np.array(rep.energy_trace), "iterations_run": rep.iterations_run,
           "msd_before": rep.msd_before, "msd_after": rep.msd_after,
           "cfg": np.array([cfg.tau, cfg.lam, cfg.max_iterations, cfg.smoothing_passes,
                            cfg.energy_tolerance])}
    if dense:
        d = mr.densify(mesh, u, te.width, te.height)
        out.update(ux=d.ux, uy=d.uy, warped=mr.warp_image(te, d).data)
    return out


def smooth_image(w, h, seed, amplitude=60.0):
    """Same construction as the reference conftest.random_smooth_image."""
    rng = np.random.default_rng(seed)
    data = ndimage.gaussian_filter(rng.standard_normal((h, w)), 2.0, mode="nearest")
    lo, hi = data.min(), data.max()
    return mr.ImageGrid(w, h, 120.0 + amplitude * (data - lo) / max(hi - lo, 1e-12) - amplitude / 2)


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def case_generated(name, size, blobs, peak, target, iters, scale, passes=1, tol=0.0,
                   unit=False, pixel_map=True, tau=0.005):
    spec = PairSpec(name, size, blobs, 0, peak, target, iters)
    re32, te32 = make_pair(spec, seed=3, scale=scale)
    re = mr.ImageGrid(size, size, re32.astype(np.float64))
    te = mr.ImageGrid(size, size, te32.astype(np.float64))
    mesh = mr.generate_mesh(te, mr.NodeBudget(target), mr.MeshGenConfig(seed=0))
    cfg = mr.SolverConfig(tau=tau, max_iterations=iters, smoothing_passes=passes,
                          energy_tolerance=tol)
    out = dict(re=re32, te=te32, **mesh_parts(mesh), **run_register(re, te, mesh, cfg))
    if pixel_map:
        tri_of, wts = reference_pixel_map(mesh, size, size)
        out.update(tri_of=tri_of.astype(np.int32), pm_weights=wts)
    if unit:
        rng = np.random.default_rng(11)
        u = rng.uniform(-1.5, 1.5, (mesh.n_vertices, 2))
        grad = rng.uniform(-50, 50, (mesh.n_vertices, 2))
        L = mr.build_laplacian(mesh)
        out.update(
            unit_u=u, unit_grad=grad,
            unit_warp_sample=mr.warp_sample(te, mesh.vertices, u),
            unit_energy=mr.energy(re, te, mesh, u),
            unit_energy_gradient=mr.energy_gradient(re, te, mesh, u),
            unit_vgrad=mr.vertex_gradient_all(mesh, mesh.geometry, te.sample(*mesh.vertices.T)),
            unit_smooth2=mr.smooth_displacement(L, u, 0.8, 2),
            unit_step=mr.step(u, grad, mr.SolverConfig(), L, mesh.vertices, (size, size)),
            unit_msd=mr.msd(te, re),
        )
    save(name, **out)


def main():
    # small generated pairs ([0,1] and x255 large motion), full pipeline
    case_generated("gen64", 64, 8, 2.0, 150, 40, 1.0, unit=True)
    case_generated("gen64_x255", 64, 8, 2.0, 400, 40, 255.0, unit=True, tau=0.001)
    case_generated("gen64_p0", 64, 8, 2.0, 400, 20, 25.0, passes=0, pixel_map=False,
                   tau=0.001)
    case_generated("gen64_p2", 64, 8, 2.0, 400, 30, 255.0, passes=2, pixel_map=False,
                   tau=0.001)
    case_generated("gen96_tol", 96, 10, 3.0, 400, 100, 25.0, tol=1e-6, pixel_map=False,
                   tau=0.001)

    # reference fixture (acceptance C3 pattern, test_acceptance.py:116-134),
    # float64 images that are NOT fp32-representable
    w = 256
    ref = synthetic.smooth_texture(w, w, seed=7)
    bump = synthetic.random_bump_field(w, w, seed=107, n_bumps=3, max_amplitude=4.0)
    _, te = synthetic.warped_pair(ref, bump)
    mesh = mr.generate_mesh(te, mr.NodeBudget(3000), mr.MeshGenConfig(seed=1))
    cfg = mr.SolverConfig(tau=0.005, lam=0.8, max_iterations=100)
    tri_of, _ = reference_pixel_map(mesh, w, w)
    save("accept_c3", re=ref.data, te=te.data, **mesh_parts(mesh, with_ops=False),
         **run_register(ref, te, mesh, cfg), tri_of=tri_of.astype(np.int32))

    # plateau shift (test_registration.py:334-346 pattern)
    w = 64
    ref = synthetic.smooth_texture(w, w, seed=11, low=100, high=156)
    field = synthetic.plateau_shift_field(w, w, shift=(1.5, 0.5))
    _, te = synthetic.warped_pair(ref, field)
    mesh = mr.generate_mesh(te, mr.NodeBudget(300), mr.MeshGenConfig(seed=2))
    save("plateau64", re=ref.data, te=te.data, **mesh_parts(mesh),
         **run_register(ref, te, mesh, mr.SolverConfig(max_iterations=30)))

    # identical images: tolerance exit (test_registration.py:292-300)
    img = smooth_image(48, 48, seed=9)
    mesh = mr.generate_mesh(img, mr.NodeBudget(80), mr.MeshGenConfig(seed=1))
    save("identical48", re=img.data, te=img.data, **mesh_parts(mesh, with_ops=False),
         **run_register(img, img, mesh, mr.SolverConfig()))

    # divergence guard (test_registration.py:325-331)
    ref = synthetic.smooth_texture(64, 64, seed=7, low=20, high=235)
    field = synthetic.plateau_shift_field(64, 64, shift=(2.0, 0.0))
    _, te = synthetic.warped_pair(ref, field)
    mesh = mr.generate_mesh(te, mr.NodeBudget(500), mr.MeshGenConfig(seed=1))
    try:
        mr.register(ref, te, mesh, mr.SolverConfig(tau=0.1))
        msg = ""
    except mr.DivergenceError as exc:
        msg = str(exc)
    save("diverge64", re=ref.data, te=te.data, **mesh_parts(mesh, with_ops=False),
         error=np.array(msg), cfg=np.array([0.1, 0.8, 100, 1, 1e-6]))

    # pixel-grid engine (baseline.py)
    from meshreg.baseline import register_pixelwise, grid_umbrella_smooth
    for name, w, seed, shift, kw in (("pixel64", 64, 11, (1.5, 0.5), dict(iterations=30)),
                                     ("pixel96_p1", 96, 5, (2.0, 0.0),
                                      dict(iterations=40, smoothing_passes=1, tau=0.004)),
                                     ("pixel48_lam0", 48, 9, (1.0, 0.0),
                                      dict(iterations=15, lam=0.0))):
        ref = synthetic.smooth_texture(w, w, seed=seed, low=100, high=156)
        field = synthetic.plateau_shift_field(w, w, shift=shift)
        _, te = synthetic.warped_pair(ref, field)
        out, rep = register_pixelwise(ref, te, **kw)
        kwv = dict(tau=0.005, lam=0.8, iterations=100, smoothing_passes=3)
        kwv.update(kw)
        save(name, re=ref.data, te=te.data, ux=out.ux, uy=out.uy,
             warped=mr.warp_image(te, out).data, trace=np.array(rep.energy_trace),
             iterations_run=rep.iterations_run, msd_before=rep.msd_before,
             msd_after=rep.msd_after,
             cfg=np.array([kwv["tau"], kwv["lam"], kwv["iterations"], kwv["smoothing_passes"]]))
    rng = np.random.default_rng(5)
    img = smooth_image(16, 13, seed=3)
    pts = rng.uniform([-1.0, -1.0], [17.0, 14.0], (200, 2))
    gx, gy = img.sample_gradient(pts[:, 0], pts[:, 1])
    plane = rng.uniform(-5, 5, (11, 7))
    save("pixel_units", img=img.data, pts=pts, gx=gx, gy=gy, plane=plane,
         smooth=grid_umbrella_smooth(plane, 0.6))
    ref = synthetic.smooth_texture(48, 48, seed=7, low=20, high=235)
    field = synthetic.plateau_shift_field(48, 48, shift=(2.0, 0.0))
    _, te = synthetic.warped_pair(ref, field)
    try:
        register_pixelwise(ref, te, tau=0.2)
        msg = ""
    except mr.DivergenceError as exc:
        msg = str(exc)
    save("pixel_diverge48", re=ref.data, te=te.data, error=np.array(msg))

    # output formats (densefield.py:215-251): the reference's own MRDF bytes
    # and node CSV for a small registered field
    import tempfile
    from meshreg.densefield import save_field, save_node_displacements_csv
    g64 = np.load(os.path.join(HERE, "gen64.npz"))
    fld = mr.DenseField(g64["ux"], g64["uy"])
    mesh64 = mr.TriMesh(g64["V"], g64["T_in"])
    with tempfile.TemporaryDirectory() as td:
        save_field(fld, os.path.join(td, "f.mrdf"))
        save_node_displacements_csv(mesh64, g64["u"], os.path.join(td, "u.csv"))
        mrdf = np.frombuffer(open(os.path.join(td, "f.mrdf"), "rb").read(), np.uint8)
        csv_text = open(os.path.join(td, "u.csv"), encoding="ascii").read()
    save("formats", mrdf=mrdf, csv=np.array(csv_text))

    # full BASELINE config 1 pair (seed 0) on the cached reference mesh
    mpath = os.path.join(ROOT, "data", "meshes", "c1_s0.npz")
    if os.path.exists(mpath):
        from paper_1411_2141_b200.synthetic import CONFIGS
        spec = CONFIGS["c1"]
        m = np.load(mpath)
        for scale, tag in ((1.0, "c1"), (255.0, "c1_x255")):
            re32, te32 = make_pair(spec, 0, scale=scale)
            mp = mpath if scale == 1.0 else mpath.replace(".npz", "_x255.npz")
            if not os.path.exists(mp):
                continue
            m = np.load(mp)
            mesh = mr.TriMesh(m["V"], m["T"].astype(np.int64))
            re = mr.ImageGrid(256, 256, re32.astype(np.float64))
            te = mr.ImageGrid(256, 256, te32.astype(np.float64))
            cfg = mr.SolverConfig(max_iterations=spec.iterations, energy_tolerance=0.0)
            out = run_register(re, te, mesh, cfg)
            extra = {}
            if tag == "c1":
                tri_of, _ = reference_pixel_map(mesh, 256, 256)
                extra = dict(tri_of=tri_of.astype(np.int32), **{
                    k: v for k, v in mesh_parts(mesh).items()
                    if k.startswith(("L_", "gx_", "gy_", "avg_"))})
            save(tag, re=re32, te=te32, V=m["V"], T_in=m["T"].astype(np.int64),
                 T=mesh.triangles.copy(), **out, **extra)


def _bytes(path):
    with open(path, "rb") as fh:
        return np.frombuffer(fh.read(), np.uint8)


def _text(path):
    with open(path, "r", encoding="utf-8") as fh:
        return np.array(fh.read())


def cli_goldens():
    """The reference CLI itself (cli.py) on small pairs: its input files, the
    meshes its `mesh` command makes, every file `register` / `bench` /
    `metrics` write, their exit codes and stdout; plus the reference's image
    readers on PGM/PNG variants (image.py:190-296)."""
    import contextlib
    import io
    import tempfile
    from meshreg.cli import main as ref_main

    def run(argv):
        out, err = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
            rc = ref_main([str(a) for a in argv])
        return rc, out.getvalue(), err.getvalue()

    with tempfile.TemporaryDirectory() as td:
        d = lambda *p: os.path.join(td, *p)  # noqa: E731
        # the reference's CLI test pair (test_cli.py:13-22)
        ref = synthetic.smooth_texture(96, 96, seed=5, low=100, high=156)
        field = synthetic.plateau_shift_field(96, 96, shift=(2.0, 0.0))
        _, te = synthetic.warped_pair(ref, field)
        mr.save_image(ref, d("ref.png"))
        mr.save_image(te, d("template.pgm"))
        rc_m, out_m, _ = run(["mesh", "--template", d("template.pgm"), "--nodes", 400,
                              "--seed", 3, "--out", d("m")])
        assert rc_m == 0
        rc, out, err = run(["register", "--ref", d("ref.png"), "--template", d("template.pgm"),
                            "--mesh", d("m", "mesh.json"), "--iters", 40, "--out", d("r")])
        assert rc == 0, err
        rec = dict(ref_png=_bytes(d("ref.png")), te_pgm=_bytes(d("template.pgm")),
                   mesh_json=_text(d("m", "mesh.json")), mesh_node=_text(d("m", "mesh.node")),
                   mesh_ele=_text(d("m", "mesh.ele")), stdout=np.array(out),
                   mesh_quality_json=_text(d("m", "quality.json")),
                   mesh_stdout=np.array(out_m))
        # register without --mesh: the CLI meshes the template itself
        rc, out_g, err = run(["register", "--ref", d("ref.png"), "--template", d("template.pgm"),
                              "--nodes", 300, "--seed", 2, "--iters", 30, "--out", d("g")])
        assert rc == 0, err
        rec.update(gen_stdout=np.array(out_g), gen_mesh_json=_text(d("g", "mesh.json")),
                   gen_report_json=_text(d("g", "report.json")))
        for name in ("field.bin", "warped.png", "difference.png"):
            rec[name.replace(".", "_")] = _bytes(d("r", name))
        for name in ("mesh.json", "nodes.csv", "report.json", "manifest.json"):
            rec["out_" + name.replace(".", "_")] = _text(d("r", name))
        rec["warped"] = mr.load_image(d("r", "warped.png")).data
        rec["difference"] = mr.load_image(d("r", "difference.png")).data
        rec["ref"] = mr.load_image(d("ref.png")).data
        rec["te"] = mr.load_image(d("template.pgm")).data

        # divergence exit code 4 (test_cli.py:165-180) on a reference mesh
        r2 = synthetic.smooth_texture(96, 96, seed=7, low=40, high=220)
        bump = synthetic.random_bump_field(96, 96, seed=42, n_bumps=2, max_amplitude=4.0,
                                           sigma_range=(20, 35))
        _, t2 = synthetic.warped_pair(r2, bump)
        mr.save_image(r2, d("r2.pgm"))
        mr.save_image(t2, d("t2.pgm"))
        assert run(["mesh", "--template", d("t2.pgm"), "--nodes", 500, "--out", d("m2")])[0] == 0
        rc4, _, err4 = run(["register", "--ref", d("r2.pgm"), "--template", d("t2.pgm"),
                            "--mesh", d("m2", "mesh.json"), "--tau", 0.01, "--out", d("o2")])
        assert rc4 == 4, (rc4, err4)
        rec.update(div_ref_pgm=_bytes(d("r2.pgm")), div_te_pgm=_bytes(d("t2.pgm")),
                   div_mesh_json=_text(d("m2", "mesh.json")), div_stderr=np.array(err4))

        # bench over a 3-slice stack, meshes from the reference's `mesh` with the
        # bench's own budget and seed (test_cli.py:255-268)
        os.makedirs(d("s"))
        for i, sl in enumerate(synthetic.slice_stack(48, 48, 3, seed=4, max_shift=1.0)):
            mr.save_image(sl, d("s", f"s{i}.pgm"))
            rec[f"slice{i}_pgm"] = _bytes(d("s", f"s{i}.pgm"))
        for i in range(2):
            assert run(["mesh", "--template", d("s", f"s{i}.pgm"), "--nodes", 150,
                        "--out", d("bm", f"s{i}")])[0] == 0
            rec[f"bench_mesh{i}_json"] = _text(d("bm", f"s{i}", "mesh.json"))
        rcb, outb, errb = run(["bench", "--dir", d("s"), "--nodes", 150, "--iters", 15,
                               "--out", d("b")])
        assert rcb == 0, errb
        rec["bench_json"] = _text(d("b", "bench.json"))

        rcx, outx, _ = run(["metrics", "--ref", d("ref.png"), "--template", d("template.pgm"),
                            "--out", d("x")])
        assert rcx == 0
        rec["metrics_stdout"] = np.array(outx)

        # image readers: P2 with comments, 16-bit P5, RGB / 16-bit / LA PNGs
        from PIL import Image as PILImage
        rng = np.random.default_rng(11)
        a8 = rng.integers(0, 256, (7, 9)).astype(np.uint8)
        a16 = rng.integers(0, 65536, (5, 6)).astype(np.uint16)
        rgb = rng.integers(0, 256, (4, 5, 3)).astype(np.uint8)
        with open(d("p2.pgm"), "w") as fh:
            fh.write("P2\n# a comment\n9 7\n# another\n200\n")
            fh.write(" ".join(str(int(v) * 200 // 255) for v in a8.ravel()) + "\n")
        with open(d("p5_16.pgm"), "wb") as fh:
            fh.write(b"P5 6 5 65535\n" + a16.astype(">u2").tobytes())
        PILImage.fromarray(rgb, mode="RGB").save(d("rgb.png"))
        PILImage.fromarray(a16.astype(np.int32), mode="I").save(d("i16.png"))
        PILImage.fromarray(np.dstack([a8, 255 - a8]), mode="LA").save(d("la.png"))
        for name in ("p2.pgm", "p5_16.pgm", "rgb.png", "i16.png", "la.png"):
            key = name.replace(".", "_")
            rec["io_" + key] = _bytes(d(name))
            rec["io_" + key + "_data"] = mr.load_image(d(name)).data
        mr.save_image(mr.ImageGrid(9, 7, a8.astype(np.float64) + 0.5), d("w.pgm"))
        rec["io_saved_pgm"] = _bytes(d("w.pgm"))
        rec["io_saved_src"] = a8.astype(np.float64) + 0.5
    save("cli", **rec)


if __name__ == "__main__":
    if sys.argv[1:] != ["cli"]:
        main()
    cli_goldens()
