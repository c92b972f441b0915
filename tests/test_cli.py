"""Command-line front end and file formats (reference cli.py, image.py:190-296,
meshgen.py:400-452) against the reference CLI's own
outputs (tests/golden/cli.npz, written by make_golden.py `cli`).

CPU tests: readers / writers bit-exact with the reference, config-file
precedence, and every exit code that is decided before the GPU runs.  GPU
tests: `register`, `bench`, `metrics`, `warp` end to end; fp64 state, so the
tolerances are those of the fp64 parity tests (fields within 1e-10 relative
before the fp32 file rounding, MSDs within 1e-10).
"""
import io
import json
import os

import numpy as np
import pytest

import paper_1411_2141_b200 as mrb
from conftest import golden
from paper_1411_2141_b200 import cli

G = golden("cli")


def put(path, arr):
    with open(path, "wb") as fh:
        fh.write(np.asarray(arr, np.uint8).tobytes())
    return str(path)


def text(key):
    return str(G[key])


def read_json(path):
    with open(path, "r", encoding="utf-8") as fh:
        return json.load(fh)


@pytest.fixture
def pair(tmp_path):
    d = tmp_path / "in"
    d.mkdir()
    ref = put(d / "ref.png", G["ref_png"])
    te = put(d / "template.pgm", G["te_pgm"])
    mesh = d / "mesh.json"
    mesh.write_text(text("mesh_json"), encoding="ascii")
    return ref, te, str(mesh)


# ---- formats (CPU) -------------------------------------------------------------
@pytest.mark.parametrize("name", ["p2_pgm", "p5_16_pgm", "rgb_png", "i16_png", "la_png"])
def test_image_readers_match_reference(tmp_path, name):
    path = put(tmp_path / name.replace("_pgm", ".pgm").replace("_png", ".png"), G["io_" + name])
    img = mrb.load_image(path)
    assert np.array_equal(img.data, G["io_" + name + "_data"])


def test_image_writer_and_cli_inputs_match_reference(tmp_path, pair):
    src = G["io_saved_src"]
    mrb.save_image(mrb.ImageGrid(src.shape[1], src.shape[0], src), tmp_path / "w.pgm")
    assert (tmp_path / "w.pgm").read_bytes() == G["io_saved_pgm"].tobytes()
    ref, te, _ = pair
    assert np.array_equal(mrb.load_image(ref).data, G["ref"])
    assert np.array_equal(mrb.load_image(te).data, G["te"])
    # PNG writer: decoded pixels identical (the encoder's bytes are Pillow's)
    mrb.save_image(mrb.load_image(ref), tmp_path / "again.png")
    assert np.array_equal(mrb.load_image(tmp_path / "again.png").data, G["ref"])
    with pytest.raises(ValueError, match="unsupported output extension"):
        mrb.save_image(mrb.load_image(ref), tmp_path / "x.tif")


def test_reader_errors(tmp_path):
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P5\n64 64\n255\n" + bytes(16))
    with pytest.raises(mrb.FileFormatError, match="PGM pixel data truncated"):
        mrb.load_image(bad)
    (tmp_path / "z.pgm").write_bytes(b"P5\n0 4\n255\n")
    with pytest.raises(mrb.FileFormatError, match="zero-dimension"):
        mrb.load_image(tmp_path / "z.pgm")
    (tmp_path / "m.pgm").write_bytes(b"P2\n2 2\n70000\n1 2 3 4\n")
    with pytest.raises(mrb.FileFormatError, match="maxval 70000 out of range"):
        mrb.load_image(tmp_path / "m.pgm")
    (tmp_path / "t.txt").write_bytes(b"hello")
    with pytest.raises(mrb.FileFormatError, match="unsupported image format"):
        mrb.load_image(tmp_path / "t.txt")


def test_mesh_formats_match_reference(tmp_path):
    (tmp_path / "m.json").write_text(text("mesh_json"), encoding="ascii")
    (tmp_path / "m.node").write_text(text("mesh_node"), encoding="ascii")
    (tmp_path / "m.ele").write_text(text("mesh_ele"), encoding="ascii")
    a = mrb.load_mesh_json(tmp_path / "m.json")
    b = mrb.load_mesh(str(tmp_path / "m"))
    assert np.array_equal(a.vertices, b.vertices) and np.array_equal(a.triangles, b.triangles)
    # register's mesh.json is the (CCW-oriented) mesh written back
    mrb.save_mesh_json(a, tmp_path / "out.json")
    assert (tmp_path / "out.json").read_text(encoding="ascii") == text("out_mesh_json")
    mrb.save_mesh(a, str(tmp_path / "w"))
    c = mrb.load_mesh(str(tmp_path / "w"))
    assert np.array_equal(c.vertices, a.vertices) and np.array_equal(c.triangles, a.triangles)
    (tmp_path / "bad.json").write_text('{"nodes": [[0, 0]]}', encoding="ascii")
    with pytest.raises(mrb.FileFormatError, match="malformed mesh file"):
        mrb.load_mesh_json(tmp_path / "bad.json")


def test_config_file_precedence(tmp_path):
    cfg = tmp_path / "run.cfg"
    cfg.write_text("# solver settings\ntau = 0.004\niters = 15\nnodes = 180\nlambda = 0.7\n"
                   "flag = true\nname = 'abc'\n")
    assert cli.parse_config_file(cfg) == {"tau": 0.004, "iters": 15, "nodes": 180,
                                          "lambda": 0.7, "flag": True, "name": "abc"}
    args = cli.build_parser().parse_args(["register", "--config", str(cfg), "--iters", "10"])
    p = cli.resolve(args, ["tau", "lam", "iters", "nodes", "seed"])
    assert p == {"tau": 0.004, "lam": 0.7, "iters": 10, "nodes": 180, "seed": 0}
    args = cli.build_parser().parse_args(["register"])
    assert cli.resolve(args, ["tau", "lam", "iters"]) == {"tau": 0.005, "lam": 0.8, "iters": 100}


def test_exit_codes_before_the_gpu(tmp_path, pair, capsys):
    ref, te, mesh = pair
    o = str(tmp_path / "o")
    assert cli.main(["register", "--ref", ref, "--template", te, "--mesh", mesh,
                     "--tau", "-0.1", "--out", o]) == 2
    assert cli.main(["register", "--ref", ref, "--template", te, "--mesh", mesh,
                     "--lambda", "1.0", "--out", o]) == 2
    assert cli.main(["register", "--ref", ref, "--template", te, "--nodes", "2",
                     "--out", o]) == 2
    assert cli.main(["register", "--ref", str(tmp_path / "nope.png"), "--template", te,
                     "--out", o]) == 3
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P5\n64 64\n255\n" + bytes(16))
    assert cli.main(["register", "--ref", ref, "--template", str(bad), "--out", o]) == 3
    small = tmp_path / "small.pgm"
    mrb.save_image(mrb.ImageGrid(32, 32, np.zeros((32, 32))), small)
    assert cli.main(["register", "--ref", ref, "--template", str(small), "--mesh", mesh,
                     "--out", o]) == 2
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("tau 0.004\n")
    assert cli.main(["register", "--ref", ref, "--template", te, "--config", str(cfg),
                     "--out", o]) == 2
    capsys.readouterr()
    assert cli.main(["mesh", "--template", te, "--nodes", "3", "--out", o]) == 2
    assert "nodes must be an integer >= 4" in capsys.readouterr().err
    assert cli.main(["mesh", "--out", o]) == 2
    assert cli.main(["mesh", "--template", str(tmp_path / "nope.pgm"), "--out", o]) == 3
    assert not os.path.exists(o)  # nothing written on failure
    one = tmp_path / "one"
    one.mkdir()
    mrb.save_image(mrb.ImageGrid(32, 32, np.zeros((32, 32))), one / "only.pgm")
    assert cli.main(["bench", "--dir", str(one), "--out", o]) == 2
    mixed = tmp_path / "mixed"
    mixed.mkdir()
    mrb.save_image(mrb.ImageGrid(32, 32, np.zeros((32, 32))), mixed / "a.pgm")
    mrb.save_image(mrb.ImageGrid(48, 32, np.zeros((32, 48))), mixed / "b.pgm")
    assert cli.main(["bench", "--dir", str(mixed), "--out", o]) == 2
    assert cli.main(["warp", "--template", te, "--field", str(tmp_path / "nope.bin"),
                     "--out", o]) == 3


def test_bench_table_layout():
    summary = {"pairs": [{"template": "a.pgm", "reference": "b.pgm", "msd_before": 1.0,
                          "mesh_msd": 0.5, "pixel_msd": 0.25, "mesh_total_time": 1.5,
                          "pixel_time": 2.0}],
               "mean_msd_mesh": 0.5, "mean_msd_pixel": 0.25, "total_time_mesh": 1.5,
               "total_time_pixel": 2.0}
    lines = cli.bench_table(summary).splitlines()
    assert lines[0].startswith("pair") and lines[1] == "-" * len(lines[0])
    assert lines[2] == f"{'a.pgm->b.pgm':<24}{1.0:>12.3f}{0.5:>12.3f}{0.25:>12.3f}" \
                       f"{1.5:>10.2f}{2.0:>10.2f}"
    assert lines[-1].startswith("mean / total")


# ---- end to end (GPU) ----------------------------------------------------------
def _run_register(pair, out, extra=()):
    ref, te, mesh = pair
    return cli.main(["register", "--ref", ref, "--template", te, "--mesh", mesh,
                     "--iters", "40", "--out", str(out), *extra])


def relinf(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.gpu
def test_register_outputs_match_reference_cli(tmp_path, pair, capsys):
    out = tmp_path / "r"
    assert _run_register(pair, out) == 0
    stdout = json.loads(capsys.readouterr().out)
    want = json.loads(text("stdout"))
    assert stdout["iterations_run"] == want["iterations_run"]
    assert stdout["msd_after"] == pytest.approx(want["msd_after"], rel=1e-10)
    rep, ref_rep = read_json(out / "report.json"), json.loads(text("out_report_json"))
    assert set(rep) == set(ref_rep)
    assert rep["iterations_run"] == ref_rep["iterations_run"]
    assert rep["config"] == ref_rep["config"]
    assert relinf(rep["energy_trace"], ref_rep["energy_trace"]) < 1e-12
    assert rep["msd_before"] == pytest.approx(ref_rep["msd_before"], rel=1e-12)
    assert rep["msd_after"] == pytest.approx(ref_rep["msd_after"], rel=1e-10)
    # field.bin: MRDF header identical, planes are the fp32 rounding of fields
    # that agree to 1e-10 (at most one fp32 ulp apart)
    mine = (out / "field.bin").read_bytes()
    theirs = G["field_bin"].tobytes()
    assert len(mine) == len(theirs) and mine[:16] == theirs[:16]
    a = np.frombuffer(mine[16:], "<f4")
    b = np.frombuffer(theirs[16:], "<f4")
    assert np.all(np.abs(a.astype(np.float64) - b) <= np.spacing(np.abs(b)) + 1e-30)
    for name, key in (("warped.png", "warped"), ("difference.png", "difference")):
        got = mrb.load_image(out / name).data
        assert np.abs(got - G[key]).max() <= 1.0 and np.mean(got != G[key]) < 1e-3, name
    assert (out / "mesh.json").read_text(encoding="ascii") == text("out_mesh_json")
    rows = np.loadtxt(io.StringIO((out / "nodes.csv").read_text()), delimiter=",", skiprows=1)
    want_rows = np.loadtxt(io.StringIO(text("out_nodes_csv")), delimiter=",", skiprows=1)
    assert np.array_equal(rows[:, :2], want_rows[:, :2])
    assert relinf(rows[:, 2:], want_rows[:, 2:]) < 1e-10
    assert (out / "nodes.csv").read_text().splitlines()[0] == \
        text("out_nodes_csv").splitlines()[0]
    man, ref_man = read_json(out / "manifest.json"), json.loads(text("out_manifest_json"))
    assert man["command"] == ref_man["command"] == "register"
    assert man["parameters"] == ref_man["parameters"] and man["seed"] == ref_man["seed"]
    assert man["outputs"] == ref_man["outputs"]
    by_name = lambda m: {os.path.basename(k): v for k, v in m["inputs"].items()}  # noqa: E731
    assert by_name(man) == by_name(ref_man)


@pytest.mark.gpu
def test_register_deterministic_outputs(tmp_path, pair):
    """Acceptance criterion 7 (test_acceptance.py:226-264): two runs give the
    same field bytes, the same report (timing aside) and the same manifest."""
    runs = []
    for name in ("run1", "run2"):
        assert _run_register(pair, tmp_path / name) == 0
        rep = read_json(tmp_path / name / "report.json")
        rep.pop("wall_time")
        runs.append(((tmp_path / name / "field.bin").read_bytes(), rep,
                     read_json(tmp_path / name / "manifest.json")))
    assert runs[0] == runs[1]


@pytest.mark.gpu
def test_register_divergence_exits_4(tmp_path, capsys):
    r = put(tmp_path / "r2.pgm", G["div_ref_pgm"])
    t = put(tmp_path / "t2.pgm", G["div_te_pgm"])
    (tmp_path / "m.json").write_text(text("div_mesh_json"), encoding="ascii")
    rc = cli.main(["register", "--ref", r, "--template", t, "--mesh", str(tmp_path / "m.json"),
                   "--tau", "0.01", "--out", str(tmp_path / "o")])
    assert rc == 4
    # same message; the energies in it are fp64 device sums (1e-12 relative)
    import re
    num = re.compile(r"-?\d+\.\d+(?:e[-+]?\d+)?")
    got, want = capsys.readouterr().err, text("div_stderr")
    assert num.sub("#", got) == num.sub("#", want)
    assert np.allclose([float(v) for v in num.findall(got)],
                       [float(v) for v in num.findall(want)], rtol=1e-12, atol=0)


@pytest.mark.gpu
def test_bench_matches_reference(tmp_path, capsys):
    s = tmp_path / "s"
    s.mkdir()
    for i in range(3):
        put(s / f"s{i}.pgm", G[f"slice{i}_pgm"])
    meshes = tmp_path / "meshes"
    meshes.mkdir()
    for i in range(2):
        (meshes / f"s{i}.json").write_text(text(f"bench_mesh{i}_json"), encoding="ascii")
    out = tmp_path / "b"
    assert cli.main(["bench", "--dir", str(s), "--meshes", str(meshes), "--nodes", "150",
                     "--iters", "15", "--out", str(out)]) == 0
    assert "mean / total" in capsys.readouterr().out
    got, want = read_json(out / "bench.json"), json.loads(text("bench_json"))
    assert len(got["pairs"]) == len(want["pairs"]) == 2
    for p, q in zip(got["pairs"], want["pairs"]):
        assert (p["template"], p["reference"], p["mesh_nodes"]) == \
               (q["template"], q["reference"], q["mesh_nodes"])
        for key in ("mesh_msd", "pixel_msd", "msd_before"):
            assert p[key] == pytest.approx(q[key], rel=1e-9), key
    assert got["mean_msd_mesh"] == pytest.approx(np.mean([p["mesh_msd"] for p in got["pairs"]]))
    assert got["iterations"] == want["iterations"]
    assert (out / "bench.txt").exists() and (out / "manifest.json").exists()


@pytest.mark.gpu
def test_metrics_and_warp_roundtrip(tmp_path, pair, capsys):
    ref, te, _ = pair
    assert cli.main(["metrics", "--ref", ref, "--template", te,
                     "--out", str(tmp_path / "m")]) == 0
    got, want = json.loads(capsys.readouterr().out), json.loads(text("metrics_stdout"))
    assert (got["width"], got["height"], got["max_abs_diff"]) == \
           (want["width"], want["height"], want["max_abs_diff"])
    assert got["msd"] == pytest.approx(want["msd"], rel=1e-12)
    assert read_json(tmp_path / "m" / "metrics.json") == got
    assert _run_register(pair, tmp_path / "r") == 0
    assert cli.main(["warp", "--template", te, "--field", str(tmp_path / "r" / "field.bin"),
                     "--out", str(tmp_path / "w")]) == 0
    a = mrb.load_image(tmp_path / "r" / "warped.png").data
    b = mrb.load_image(tmp_path / "w" / "warped.png").data
    assert np.abs(a - b).max() <= 1.0 and np.mean(a != b) < 1e-3


# ---- the mesher through the CLI (GPU; meshgen.py, cli.py:202-223) --------------
@pytest.mark.gpu
def test_mesh_command_matches_reference_cli(tmp_path, pair, capsys):
    """`mesh --nodes 400 --seed 3`: mesh.node / mesh.ele / mesh.json /
    quality.json byte-identical to the reference CLI's files."""
    _, te, _ = pair
    out = tmp_path / "m"
    assert cli.main(["mesh", "--template", te, "--nodes", "400", "--seed", "3",
                     "--out", str(out)]) == 0
    assert json.loads(capsys.readouterr().out) == json.loads(text("mesh_stdout"))
    for name in ("mesh.json", "mesh.node", "mesh.ele", "quality.json"):
        key = {"quality.json": "mesh_quality_json"}.get(name, name.replace(".", "_"))
        assert (out / name).read_text(encoding="ascii") == text(key), name
    man = read_json(out / "manifest.json")
    assert man["command"] == "mesh" and man["seed"] == 3
    assert man["outputs"] == sorted(["mesh.node", "mesh.ele", "mesh.json", "quality.json"])


@pytest.mark.gpu
def test_register_without_mesh_meshes_the_template(tmp_path, pair, capsys):
    """`register` with no --mesh meshes the template itself (cli.py:250-258)."""
    ref, te, _ = pair
    out = tmp_path / "g"
    assert cli.main(["register", "--ref", ref, "--template", te, "--nodes", "300", "--seed", "2",
                     "--iters", "30", "--out", str(out)]) == 0
    got, want = json.loads(capsys.readouterr().out), json.loads(text("gen_stdout"))
    assert got["iterations_run"] == want["iterations_run"]
    assert got["msd_after"] == pytest.approx(want["msd_after"], rel=1e-10)
    assert (out / "mesh.json").read_text(encoding="ascii") == text("gen_mesh_json")
    rep, ref_rep = read_json(out / "report.json"), json.loads(text("gen_report_json"))
    assert relinf(rep["energy_trace"], ref_rep["energy_trace"]) < 1e-12


@pytest.mark.gpu
def test_bench_meshes_each_template_like_the_reference(tmp_path, capsys):
    """`bench` with no mesh arguments meshes every template with the bench's
    own budget and seed (cli.py:330-336): same node counts and MSDs."""
    s = tmp_path / "s"
    s.mkdir()
    for i in range(3):
        put(s / f"s{i}.pgm", G[f"slice{i}_pgm"])
    out = tmp_path / "b"
    assert cli.main(["bench", "--dir", str(s), "--nodes", "150", "--iters", "15",
                     "--out", str(out)]) == 0
    capsys.readouterr()
    got, want = read_json(out / "bench.json"), json.loads(text("bench_json"))
    for p, q in zip(got["pairs"], want["pairs"]):
        assert p["mesh_nodes"] == q["mesh_nodes"]
        for key in ("mesh_msd", "pixel_msd", "msd_before"):
            assert p[key] == pytest.approx(q[key], rel=1e-9), key
