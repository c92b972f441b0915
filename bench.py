#!/usr/bin/env python
"""Benchmark of the B200 mesh-registration path (BASELINE.json metric).

Metric: Mpx*iter/s = sum over pairs of W*H*iterations_run / time (SURVEY.md
§8(d)), whole job over all ranks.  Default workload = BASELINE config 4 as
written: ONE job of 64 independent 512x512 pairs (config-2 pairs, seeds
0..63, reference-mesher meshes, 200 iterations, tau=0.005, lam=0.8, 1
smoothing pass, energy_tolerance=0 so every pair runs all 200 iterations)
sharded across the N GPUs: rank r registers seeds r, r+N, ... ("scaling":
"strong", no collective on the data path).  `--weak` gives every rank its
own 64 pairs instead (an extra measurement, not the headline).  Single-pair
workloads (c1, c2, c3, c5) at N > 1 run one replica per GPU ("replicas
only": one pair does not shard).

`--gpus N` without a torchrun environment re-launches this script under
`python -m torch.distributed.run --nproc-per-node N` (127.0.0.1 rendezvous);
under torchrun, WORLD_SIZE must equal N.  `--dry-run` runs only the
launcher, the sharding and the cross-rank timing reductions (gloo, no GPU).

  value   device time of K runs of the whole registration (loop + dense pass)
          with inputs resident in HBM, CUDA events on the library's stream,
          L2 flushed (256 MiB write) between steps outside the events.
  e2e     the same work through the C ABI batch call from pinned HOST
          buffers: per-pair device mesh setup (upload + pixel map), H2D of the
          images, the run, D2H of u / dense field / warped image, statuses.
  --impl reference   the reference algorithm (CPU oracle port of meshreg, one
          process per core, one pair each) on the same workload.

  --workload pixel   the reference's dense comparator engine (baseline.py,
          SURVEY.md §8(f) row 1) on the config-4 batch: 64 pairs of 512x512,
          200 iterations, 3 smoothing passes, same metric.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                       [--workload c4|c1|c2|c3|c5|pixel] [--pairs P] [--precision f32|f64]
                       [--weak] [--dry-run]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1411_2141_b200 import pairqueue  # noqa: E402
from paper_1411_2141_b200.synthetic import CONFIGS, make_pair  # noqa: E402

MESH_DIR = os.path.join(ROOT, "data", "meshes")
METRIC = "registration throughput (Mpx*iter/s)"
UNIT = "Mpx*iter/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4", "c5", "pixel"])
    ap.add_argument("--pairs", type=int, default=None)
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-pairs", type=int, default=6)
    ap.add_argument("--weak", action="store_true",
                    help="every GPU registers its own --pairs pairs (weak scaling)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher + sharding + timing reductions only (gloo, no GPU)")
    return ap.parse_args(argv)


# --------------------------------------------------------------------------- inputs
def mesh_file(cfg, seed):
    return os.path.join(MESH_DIR, f"{cfg}_s{seed}.npz")


def fallback_mesh(size, target):
    """Deterministic structured triangulation used only when the cached
    reference-mesher mesh is absent (reported in config.mesh)."""
    k = max(2, int(round(np.sqrt(target))))
    xs = np.linspace(0.0, size - 1.0, k)
    gx, gy = np.meshgrid(xs, xs)
    V = np.stack([gx.ravel(), gy.ravel()], axis=1)
    T = []
    for j in range(k - 1):
        for i in range(k - 1):
            a, b, c, d = j * k + i, j * k + i + 1, (j + 1) * k + i, (j + 1) * k + i + 1
            T += [(a, b, d), (a, d, c)]
    return V, np.array(T, np.int64)


def workload_spec(name):
    spec = CONFIGS["c2" if name in ("c4", "pixel") else name]
    mesh_cfg = spec.name
    return spec, mesh_cfg


def load_pair(name, used):
    """(re, te, V, T, mesh_kind, seed) for one pair of the workload."""
    spec, mesh_cfg = workload_spec(name)
    re, te = make_pair(spec, used)
    if os.path.exists(mesh_file(mesh_cfg, used)):
        d = np.load(mesh_file(mesh_cfg, used))
        V, T = d["V"], d["T"].astype(np.int64)
        kind = ("package-mesher (bit-identical to the reference mesher)" if "mesher" in d.files
                else "reference-mesher")
    else:
        V, T, kind = package_mesh(spec, te, mesh_cfg, used)
    return re, te, V, T, kind, used


def package_mesh(spec, te, mesh_cfg, seed):
    """The mesh the reference mesher would make (generate_mesh on the
    template, NodeBudget(target), MeshGenConfig(seed=0)), built
    by this package's mesher, whose meshes are bit-identical to the
    reference's (tests/test_mesher.py, C1-C3 at full size).  Untimed; cached
    in data/meshes.  Used when the reference-mesher cache is absent (a fresh
    checkout, or C5, where the reference mesher would need ~10 h)."""
    from paper_1411_2141_b200 import ImageGrid, MeshGenConfig, NodeBudget, generate_mesh
    try:
        m = generate_mesh(ImageGrid(spec.size, spec.size, te.astype(np.float64)),
                          NodeBudget(spec.target_nodes), MeshGenConfig(seed=0))
    except Exception as exc:  # noqa: BLE001 - no GPU: structured stand-in, reported
        print(f"bench: package mesher unavailable ({exc}); structured mesh", file=sys.stderr)
        V, T = fallback_mesh(spec.size, spec.target_nodes)
        return V, T, "fallback-structured"
    V, T = m.vertices.copy(), m.triangles.copy()
    try:
        os.makedirs(MESH_DIR, exist_ok=True)
        tmp = mesh_file(mesh_cfg, seed) + f".{os.getpid()}.tmp.npz"
        np.savez_compressed(tmp, V=V, T=T.astype(np.int32), mesher="package")
        os.replace(tmp, mesh_file(mesh_cfg, seed))
    except OSError:
        pass
    return V, T, "package-mesher (bit-identical to the reference mesher)"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()  # sampling is live before the timed region starts
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.skip = len(self.lines)  # samples taken before the timed region
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines[getattr(self, "skip", 0):] or self.lines[-1:]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- dist
def dist_setup():
    info = pairqueue.rank_info()
    return info.rank, info.world, info.local


def dist_init(backend, local):
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return dist


def reduce_max(value, world, dist, device):
    return pairqueue.max_over_ranks(value, world, device)


def barrier(world, dist):
    pairqueue.barrier(world)


def job_seeds(args, rank, world):
    """(this rank's pair seeds, pairs in the whole job, scaling)."""
    P = args.pairs or (64 if args.workload in ("c4", "pixel") else 1)
    if args.weak:
        return pairqueue.weak_seeds(rank, P), P * world, "weak"
    if P < world:  # one pair does not shard: one replica per GPU
        return list(range(P)), P * world, "weak"
    return pairqueue.shard_seeds(rank, world, P), P, "strong"


def seeds_text(seeds, rank, world, weak):
    if world == 1 or weak:
        return f"{seeds[0]}..{seeds[-1]}" if len(seeds) > 1 else str(seeds[0])
    return f"rank r of {world} owns seeds r, r+{world}, ... (rank 0: {seeds[0]}..{seeds[-1]})"


# --------------------------------------------------------------------------- ours
def mesh_handles(lib, meshes, deferred=False):
    """Mesh handles for many meshes at once: the full host build
    (mrb_mesh_build_many, the library's host worker pool) or, deferred, only
    the host checks + orientation (mrb_mesh_create_many; the connectivity,
    geometry, fused operator and topology are then built on the GPU inside
    mrb_register_many)."""
    arrs = [(np.ascontiguousarray(V, np.float64), np.ascontiguousarray(T, np.int64))
            for V, T in meshes]
    k = len(arrs)
    n = np.array([V.shape[0] for V, _ in arrs], np.int64)
    m = np.array([T.shape[0] for _, T in arrs], np.int64)
    Vp = (C.c_void_p * k)(*(V.ctypes.data for V, _ in arrs))
    Tp = (C.c_void_p * k)(*(T.ctypes.data for _, T in arrs))
    out = (C.c_void_p * k)()
    bad = C.c_int32(-1)
    err = C.create_string_buffer(512)
    fn = lib.mrb_mesh_create_many if deferred else lib.mrb_mesh_build_many
    rc = fn(k, n.ctypes.data, Vp, m.ctypes.data, Tp, out, C.byref(bad), err, 512)
    if rc != 0:
        raise RuntimeError(f"mesh {bad.value}: {err.value.decode()}")
    return list(out)


def check(lib, ctx, rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: code {rc}: {lib.mrb_last_error(ctx).decode()}")


def run_ours(args, rank, world, local):
    import torch
    from paper_1411_2141_b200 import _lib

    torch.cuda.set_device(local)
    os.environ["MESHREG_B200_DEVICE"] = str(local)  # the package's default context (mesher)
    dist = dist_init("nccl", local) if world > 1 else None
    device = torch.device("cuda", local)
    lib = _lib.load()
    ctx = _lib.context(local)
    stream = torch.cuda.ExternalStream(lib.mrb_ctx_stream(ctx), device=device)

    spec, _ = workload_spec(args.workload)
    seeds, total, scaling = job_seeds(args, rank, world)
    P = len(seeds)
    pairs = [load_pair(args.workload, s) for s in seeds]
    W = H = spec.size
    iters = spec.iterations
    npx = W * H
    cfg = _lib.mrb_config(0.005, 0.8, 0.0, iters, 1,
                          _lib.PREC_F32 if args.precision == "f32" else _lib.PREC_F64, 0)
    handles = mesh_handles(lib, [(p[2], p[3]) for p in pairs])
    arr = (C.c_void_p * P)(*handles)
    batch = C.c_void_p()
    check(lib, ctx, lib.mrb_batch_create(ctx, P, arr, W, H, _lib.F32, C.byref(cfg),
                                         C.byref(batch)), "batch_create")
    re_d = torch.from_numpy(np.stack([p[0] for p in pairs])).to(device)
    te_d = torch.from_numpy(np.stack([p[1] for p in pairs])).to(device)
    torch.cuda.synchronize()
    check(lib, ctx, lib.mrb_batch_set_images(batch, re_d.data_ptr(), te_d.data_ptr(), 1), "set")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)

    for _ in range(max(args.warmup, 3)):
        check(lib, ctx, lib.mrb_batch_run(batch), "run")
    check(lib, ctx, lib.mrb_batch_sync(batch), "warmup sync")

    # per-kernel launch times (CUDA events around each launch, separate pass)
    ktimes = np.zeros(5)
    check(lib, ctx, lib.mrb_batch_kernel_times(batch, ktimes.ctypes.data), "kernel_times")
    kbytes = np.zeros(4)
    lib.mrb_batch_kernel_bytes(batch, kbytes.ctypes.data)

    barrier(world, dist)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    evs = []
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            check(lib, ctx, lib.mrb_batch_run(batch), "run")
            e1.record(stream)
            evs.append((e0, e1))
    torch.cuda.synchronize()
    clocks = sampler.stop()
    barrier(world, dist)
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    t_ms = reduce_max(t_ms, world, dist, device)

    rc = lib.mrb_batch_sync(batch)
    check(lib, ctx, rc, "result status")
    it = C.c_int32()
    tot_iters = 0
    for p in range(P):
        lib.mrb_batch_pair_status(batch, p, C.byref(it), None, None, None, None, 0)
        tot_iters += it.value
    work = float(npx) * tot_iters  # px*iter per step on this rank
    value = pairqueue.job_throughput(work * args.steps, t_ms / 1e3, world, device)
    launches = int(lib.mrb_batch_launches_per_run(batch)) * args.steps
    path_cs = int(lib.mrb_batch_path(batch))
    loop_kernel = lib.mrb_batch_loop_kernel(batch).decode()
    alg_bytes = lib.mrb_batch_algorithmic_bytes(batch)
    lib.mrb_batch_destroy(batch)

    # ---- e2e through the C ABI from pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, lib, ctx, pairs, cfg, W, H, world, dist, device)

    # ---- roofline of the dominant kernel (largest share of the run)
    n_launch = {0: iters, 1: iters, 2: iters, 3: 1}
    share = {k: ktimes[k] * n_launch[k] for k in range(4)}
    dom = max(share, key=share.get)
    names = {0: loop_kernel, 1: "k_grad", 2: "k_smooth",
             3: "k_dense"}
    if path_cs:
        n_launch = {0: 1, 1: 0, 2: 0, 3: 1}
        share = {k: ktimes[k] * n_launch[k] for k in range(4)}
        dom = max(share, key=share.get)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = kbytes[dom] / (ktimes[dom] / 1e3) / 1e9
    ncu = ncu_record(args.workload, args.precision, names[dom])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, pairs[:args.cpu_pairs], spec,
                           iters=CPU_ITERS_CAP.get(args.workload, spec.iterations))

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(t_ms / args.steps, 4), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic (seeded BASELINE generator; content-adaptive meshes of the reference mesher algorithm, see config.mesh)",
            "config": {
                "workload": f"{args.workload}: {total} pairs of {W}x{H} in the job"
                            f"{f' over {world} GPUs' if world > 1 else ''}, {iters} iterations, "
                            f"{pairs[0][4]} meshes (~{int(np.mean([len(p[2]) for p in pairs]))} nodes)",
                "pairs_per_gpu": P, "global_pairs": total, "image": [W, H],
                "iterations": iters, "tau": 0.005, "lam": 0.8, "smoothing_passes": 1,
                "energy_tolerance": 0.0, "mesh": pairs[0][4],
                "pair_seeds": seeds_text(seeds, rank, world, args.weak),
                "l2": "flushed (256 MiB write) between timed steps, outside the events",
                "parallelism": f"pair-sharded dp{world} (no collective)",
                "precision": args.precision,
            },
            "gpu_launches": launches,
            "path": (f"persistent cluster kernel {loop_kernel} (cluster of {path_cs} CTAs per pair)"
                     if path_cs > 0
                     else f"whole-GPU persistent grid kernel {loop_kernel} ({-path_cs} CTAs, one "
                          "cooperative launch per pair)" if path_cs < 0
                     else "generic 3-kernel loop (CUDA graph)"),
            "kernel_ms": {names[k]: round(float(ktimes[k]), 5) for k in range(4)},
            # device ms per descent iteration of the whole batch (loop only)
            "loop_ms_per_iteration": round(float(ktimes[0] / iters if path_cs
                                                 else ktimes[0] + ktimes[1] + ktimes[2]), 6),
            "algorithmic_bytes_per_step": alg_bytes,
            "hbm_frac_whole_run": round(alg_bytes / (t_ms / args.steps / 1e3) / 1e9 / peak, 4),
            "roofline": roofline_block(names[dom], achieved, peak, ncu, ktimes[dom],
                                       "achieved = SURVEY 8(d) algorithmic bytes per launch / "
                                       "CUDA-event time (a MODEL rate: the persistent kernels "
                                       "serve those bytes from SMEM — topology, halo exchange — "
                                       "and L2 — image taps — so it can exceed the HBM peak); "
                                       "dram_frac = the DRAM bytes ncu measured per launch "
                                       "(`traffic`) over the same time; `limiter` = what ncu "
                                       "shows bounds the kernel"),
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, lib, ctx, pairs, cfg, W, H, world, dist, device):
    """The same work through the public C-ABI calls from host buffers, mesh
    setup included: mrb_mesh_create_many (host checks + orientation of the
    mesher's (V, T), the reference's TriMesh validation) and the pipelined
    mrb_register_many from pinned images: V / T upload, the per-mesh setup on
    the GPU (connectivity, geometry, node order, fused operator, fast-path
    topology, pixel map), H2D images, registration including the dense pass,
    and D2H of what the reference's register returns (u and the report:
    iterations, energy trace, MSD before / after, status; solver.py:148-208).
    A second figure adds the D2H of the dense field and warped image (what
    the CLI writes)."""
    import torch
    from paper_1411_2141_b200 import _lib

    P = len(pairs)
    npx = W * H
    re_h = torch.from_numpy(np.stack([p[0] for p in pairs])).pin_memory()
    te_h = torch.from_numpy(np.stack([p[1] for p in pairs])).pin_memory()
    n_tot = sum(len(p[2]) for p in pairs)
    u_h = torch.empty((n_tot, 2), dtype=torch.float64).pin_memory()
    dense_h = [torch.empty((P, H, W), dtype=torch.float32).pin_memory() for _ in range(3)]
    trace_h = torch.empty((P, cfg.max_iterations), dtype=torch.float64).pin_memory()
    msd_h = torch.empty((2, P), dtype=torch.float64).pin_memory()
    iters = np.zeros(P, np.int32)
    codes = np.zeros(P, np.int32)
    steps = max(1, min(args.steps, 5))
    cnt = np.zeros(2, np.int64)
    res = {}
    setup_times = []
    step_ms = {}
    mesh_in = [(np.ascontiguousarray(p[2], np.float64), np.ascontiguousarray(p[3], np.int64))
               for p in pairs]  # the mesher's arrays, as the caller holds them
    # Deferred handles (per-mesh setup on the GPU inside mrb_register_many)
    # wherever the device setup runs: every fp32 path (cluster and whole-GPU
    # grid) and the fp64 cluster path (<= 16 x 768 nodes).  The fp64 generic
    # loop builds its meshes on the host: outside the timed region, that
    # build reported on its own, like the reference arm's TriMesh construction.
    nmax = max(len(p[2]) for p in pairs)
    deferred = args.precision == "f32" or nmax <= 16 * 768
    built_ms = []
    for variant in ("report", "dense"):
        dense = [d.data_ptr() for d in dense_h] if variant == "dense" else [None] * 3
        times, tot_iters, h2d, d2h = [], 0, 0, 0
        nwarm = max(1, args.warmup)  # untimed warm-up steps (the pool and caches settle)
        for step in range(nwarm + steps):
            torch.cuda.synchronize()
            barrier(world, dist)
            lib.mrb_transfer_bytes(None, None, 1)
            if not deferred:  # host-built meshes, outside the timed region
                tb = time.perf_counter()
                handles = mesh_handles(lib, mesh_in)
                if step >= nwarm and variant == "report":
                    built_ms.append(time.perf_counter() - tb)
            t0 = time.perf_counter()
            if deferred:
                handles = mesh_handles(lib, mesh_in, deferred=True)
                if step >= nwarm and variant == "report":
                    setup_times.append(time.perf_counter() - t0)
            arr = (C.c_void_p * P)(*handles)
            rc = lib.mrb_register_many(ctx, P, arr, W, H, _lib.F32, re_h.data_ptr(),
                                       te_h.data_ptr(), C.byref(cfg), 0, _lib.F32, u_h.data_ptr(),
                                       *dense, iters.ctypes.data, msd_h[0].data_ptr(),
                                       msd_h[1].data_ptr(), trace_h.data_ptr(), codes.ctypes.data,
                                       None, 0)
            dt = time.perf_counter() - t0
            lib.mrb_transfer_bytes(cnt.ctypes.data, cnt[1:].ctypes.data, 1)
            check(lib, ctx, rc, "e2e register_many")
            if step >= nwarm:
                times.append(dt)
                tot_iters += int(iters.sum())
                h2d, d2h = int(cnt[0]), int(cnt[1])
            for h in handles:
                lib.mrb_mesh_destroy(h)
        t = reduce_max(sum(times), world, dist, device)
        res[variant] = (pairqueue.job_throughput(float(npx) * tot_iters, t, world, device), t,
                        h2d, d2h, tot_iters)
        step_ms[variant] = [round(1e3 * x, 3) for x in times]
    value, t, h2d, d2h, tot_iters = res["report"]
    ts = reduce_max(sum(setup_times), world, dist, device)
    dv, dt_, dh2d, dd2h, _ = res["dense"]
    if deferred:
        setup = {"mesh_setup": "included: mrb_mesh_create_many on the host + GPU build in "
                               "mrb_register_many",
                 "mesh_create_ms_per_step": round(1e3 * ts / steps, 3),
                 "value_with_mesh_setup": round(value, 3)}
    else:
        tb = reduce_max(sum(built_ms), world, dist, device)
        setup = {"mesh_setup": "excluded: grid-path meshes built on the host (mrb_mesh_build_many) "
                               "before the timed region, reported here",
                 "mesh_build_ms_per_step": round(1e3 * tb / steps, 3),
                 "value_with_mesh_setup": round(pairqueue.job_throughput(
                     float(npx) * res["report"][4], t + tb, world, device), 3)}
    return {"value": round(value, 3), "unit": UNIT, "steps": steps,
            "ms_per_step": round(1e3 * t / steps, 3),
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            # the per-mesh setup, inside the timed region where
            # the GPU builds it
            **setup,
            "step_ms": step_ms["report"],
            "with_dense_outputs": {"value": round(dv, 3), "ms_per_step": round(1e3 * dt_ / steps, 3),
                                   "h2d_bytes_per_step": dh2d, "d2h_bytes_per_step": dd2h,
                                   "adds": "D2H of the dense field ux/uy and the warped image "
                                           "(fp32), what the CLI writes"},
            "api": ("mrb_mesh_create_many + " if deferred else "") + "mrb_register_many (one chunk)",
            "includes": ("mesh handles from the mesher's (V, T) (host checks + orientation), "
                         "V/T upload and the per-mesh setup on the GPU (connectivity, geometry, "
                         "node order, fused operator, topology, pixel map), " if deferred else
                         "the meshes' device upload, topology and pixel map, ") +
                        "H2D images, full registration incl. densify + warp + MSD on the device, "
                        "D2H of register's results (u, iterations, energy trace, MSD "
                        "before/after, status)"}


def ncu_record(workload, precision, kernel):
    """The ncu capture of this kernel (profiles/ncu_traffic.json): DRAM bytes
    per launch and the limiter counters."""
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(tpath):
        return {}
    rec = json.load(open(tpath)).get(workload, {}).get(precision, {}).get(kernel)
    if rec is None:
        return {}
    return rec if isinstance(rec, dict) else {"dram_bytes": rec}


def roofline_block(kernel, achieved, peak, ncu, kernel_ms, note):
    traffic = ncu.get("dram_bytes")
    out = {"kernel": kernel, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
           "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
           "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
           "frac_of_8tbs_nominal": round(achieved / 8000.0, 4)}
    if traffic:
        dram = traffic / (kernel_ms / 1e3) / 1e9
        out["dram_gbs"] = round(dram, 1)
        out["dram_frac"] = round(dram / peak, 4)
    if ncu.get("limiter"):
        out["limiter"] = ncu["limiter"]
        out["ncu"] = {k: ncu[k] for k in ("issue_active_pct", "l1tex_pct", "lts_pct",
                                         "dram_pct", "warps_active_pct", "l2_hit_pct",
                                         "source") if k in ncu}
    out["note"] = note
    return out


# --------------------------------------------------------------------------- CPU legs
def _oracle_register(re, te, V, T, iters):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import meshreg_oracle as O
    m = O.Mesh(V, T)
    t0 = time.perf_counter()
    u, info = O.register(re.astype(np.float64), te.astype(np.float64), m, tau=0.005, lam=0.8,
                         max_iterations=iters, smoothing_passes=1, energy_tolerance=0.0)
    return time.perf_counter() - t0, info["iterations_run"]


# bounded CPU samples: the oracle needs minutes per C5 iteration batch
CPU_ITERS_CAP = {"c5": 3}


def cpu_baseline(args, pairs, spec, iters=None):
    """Oracle port timed single-threaded on this host (rank 0, N=1)."""
    iters = iters or spec.iterations
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    tot, work = 0.0, 0.0
    ctxm = threadpool_limits(1) if threadpool_limits else None
    try:
        for re, te, V, T, kind, used in pairs:
            dt, it = _oracle_register(re, te, V, T, iters)
            tot += dt
            work += float(spec.size) ** 2 * it
    finally:
        if ctxm is not None:
            ctxm.unregister() if hasattr(ctxm, "unregister") else None
    return {"value": round(work / tot / 1e6, 4), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{len(pairs)} of the workload's pairs (seeds {[p[5] for p in pairs]}), "
                      f"{spec.size}x{spec.size}, {iters} iterations each, full register "
                      f"(loop + densify + warp + MSD), {tot:.1f} s"}


def _ref_worker(conn, workload, seeds, iters):
    """One host core of the reference arm: its share of the job's pairs."""
    os.environ["OMP_NUM_THREADS"] = "1"
    jobs = []
    for seed in seeds:
        if workload == "pixel":
            jobs.append(make_pair(CONFIGS["c2"], seed))
        else:
            jobs.append(load_pair(workload, seed)[:4])
    conn.send("ready")

    def one(job, it):
        if workload == "pixel":
            return _oracle_pixelwise(job[0], job[1], it)
        return _oracle_register(*job, it)

    while True:
        msg = conn.recv()
        if msg == "stop":
            break
        if msg == "warm":  # untimed: page in numpy/scipy and this core's first pair
            conn.send([one(jobs[0], 2)])
        else:
            conn.send([one(job, iters) for job in jobs])


def run_reference(args, rank, world):
    """The reference algorithm on the host cores: the whole job (all its
    pairs — the same config as our arm), one process per core, each
    registering its share of the pairs in turn."""
    if rank != 0:
        return  # rank 0 alone runs the CPU reference arm
    import multiprocessing as mp
    spec, _ = workload_spec(args.workload)
    P = args.pairs or (64 if args.workload in ("c4", "pixel") else 1)
    if args.weak:
        P *= world
    cores = len(os.sched_getaffinity(0))
    nproc = max(1, min(P, cores))
    env_bak = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                              "MKL_NUM_THREADS")}
    for k in env_bak:
        os.environ[k] = "1"
    ctx = mp.get_context("spawn")
    it_ref = (PIXEL_REF_ITERS if args.workload == "pixel"
              else CPU_ITERS_CAP.get(args.workload, spec.iterations))
    procs, conns = [], []
    for i in range(nproc):
        a, b = ctx.Pipe()
        p = ctx.Process(target=_ref_worker,
                        args=(b, args.workload, list(range(i, P, nproc)), it_ref))
        p.start()
        procs.append(p)
        conns.append(a)
    for c in conns:
        c.recv()
    warm = max(args.warmup, 3)
    times, work = [], 0.0
    for step in range(warm + args.steps):
        t0 = time.perf_counter()
        for c in conns:
            c.send("warm" if step < warm else "go")
        res = [r for c in conns for r in c.recv()]
        dt = time.perf_counter() - t0
        if step >= warm:
            times.append(dt)
            work += sum(float(spec.size) ** 2 * it for _, it in res)
    for c in conns:
        c.send("stop")
    for p in procs:
        p.join()
    value = work / sum(times) / 1e6
    same = it_ref == (PIXEL_ITERS if args.workload == "pixel" else spec.iterations)
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": warm,
        "ms_per_step": round(1e3 * sum(times) / len(times), 2), "higher_is_better": True,
        "scaling": "strong" if P >= world and not args.weak else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator; content-adaptive meshes of the reference mesher algorithm, see config.mesh)",
        "config": {"workload": f"{args.workload}: {P} pairs of {spec.size}x{spec.size} in the job, "
                               f"{it_ref} iterations"
                               + ("" if same else " (bounded sample of the iterations)"),
                   "global_pairs": P, "image": [spec.size, spec.size],
                   "iterations": it_ref, "energy_tolerance": 0.0, "same_config": same,
                   "pair_seeds": f"0..{P - 1}"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": nproc, "kind": "port",
                         "sample": f"all {P} pairs per timed step ({it_ref} iterations each), one "
                                   f"process per host core ({nproc}), oracle port of meshreg "
                                   + ("register_pixelwise" if args.workload == "pixel"
                                      else "register") + " (numpy/scipy, float64)"
                                   + ("" if args.workload == "pixel" else
                                      "; the step's wall clock includes each pair's mesh "
                                      "construction from (V, T), like our arm's e2e")
                                   + "; warm-up steps run 2 iterations of one pair per core"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------------- pixel engine
PIXEL_ITERS, PIXEL_PASSES = 200, 3
PIXEL_REF_ITERS = 20  # bounded CPU sample per pair (numpy: ~0.1 s per 512x512 iteration)


def _oracle_pixelwise(re, te, iters):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import meshreg_oracle as O
    t0 = time.perf_counter()
    _, _, info = O.register_pixelwise(re.astype(np.float64), te.astype(np.float64), tau=0.005,
                                      lam=0.8, iterations=iters, smoothing_passes=PIXEL_PASSES)
    return time.perf_counter() - t0, info["iterations_run"]


def run_pixel(args, rank, world, local):
    """The dense per-pixel engine (reference baseline.py) on the config-4
    batch through the C ABI (mrb_pixel_batch_*)."""
    import torch
    from paper_1411_2141_b200 import _lib

    torch.cuda.set_device(local)
    os.environ["MESHREG_B200_DEVICE"] = str(local)  # the package's default context (mesher)
    dist = dist_init("nccl", local) if world > 1 else None
    device = torch.device("cuda", local)
    lib = _lib.load()
    ctx = _lib.context(local)
    stream = torch.cuda.ExternalStream(lib.mrb_ctx_stream(ctx), device=device)
    spec = CONFIGS["c2"]
    seeds, total, scaling = job_seeds(args, rank, world)
    used = seeds
    P = len(seeds)
    pairs = [make_pair(spec, s) for s in seeds]
    W = H = spec.size
    npx = W * H
    prec = _lib.PREC_F32 if args.precision == "f32" else _lib.PREC_F64
    pcfg = _lib.mrb_pixel_config(0.005, 0.8, PIXEL_ITERS, PIXEL_PASSES, prec, 0)
    batch = C.c_void_p()
    check(lib, ctx, lib.mrb_pixel_batch_create(ctx, P, W, H, _lib.F32, C.byref(pcfg),
                                               C.byref(batch)), "pixel_batch_create")
    re_d = torch.from_numpy(np.stack([p[0] for p in pairs])).to(device)
    te_d = torch.from_numpy(np.stack([p[1] for p in pairs])).to(device)
    torch.cuda.synchronize()
    check(lib, ctx, lib.mrb_pixel_batch_set_images(batch, re_d.data_ptr(), te_d.data_ptr(), 1),
          "set")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    for _ in range(max(args.warmup, 3)):
        check(lib, ctx, lib.mrb_pixel_batch_run(batch), "run")
    check(lib, ctx, lib.mrb_pixel_batch_sync(batch), "warmup sync")
    kt = np.zeros(2)
    check(lib, ctx, lib.mrb_pixel_batch_kernel_times(batch, kt.ctypes.data), "kernel_times")

    barrier(world, dist)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    evs = []
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            check(lib, ctx, lib.mrb_pixel_batch_run(batch), "run")
            e1.record(stream)
            evs.append((e0, e1))
    torch.cuda.synchronize()
    clocks = sampler.stop()
    barrier(world, dist)
    t_ms = reduce_max(sum(a.elapsed_time(b) for a, b in evs), world, dist, device)
    check(lib, ctx, lib.mrb_pixel_batch_sync(batch), "result status")
    it = C.c_int32()
    tot_iters = 0
    for p in range(P):
        lib.mrb_pixel_batch_pair_status(batch, p, C.byref(it), None, None, None, None, 0)
        tot_iters += it.value
    value = pairqueue.job_throughput(float(npx) * tot_iters * args.steps, t_ms / 1e3, world,
                                     device)
    launches = int(lib.mrb_pixel_batch_launches_per_run(batch)) * args.steps

    # e2e: pinned host stacks -> set_images (H2D) -> run -> get_results (D2H) -> sync
    e2e = None
    if not args.no_e2e:
        re_h = torch.from_numpy(np.stack([p[0] for p in pairs])).pin_memory()
        te_h = torch.from_numpy(np.stack([p[1] for p in pairs])).pin_memory()
        outs = [torch.empty((P, H, W), dtype=torch.float32).pin_memory() for _ in range(3)]
        cnt = np.zeros(2, np.int64)
        times = []
        steps = max(1, min(args.steps, 5))
        for step in range(1 + steps):
            torch.cuda.synchronize()
            barrier(world, dist)
            lib.mrb_transfer_bytes(None, None, 1)
            t0 = time.perf_counter()
            check(lib, ctx, lib.mrb_pixel_batch_set_images(batch, re_h.data_ptr(), te_h.data_ptr(),
                                                           0), "e2e set")
            check(lib, ctx, lib.mrb_pixel_batch_run(batch), "e2e run")
            check(lib, ctx, lib.mrb_pixel_batch_get_results(batch, _lib.F32,
                                                            *(o.data_ptr() for o in outs)), "get")
            check(lib, ctx, lib.mrb_pixel_batch_sync(batch), "e2e sync")
            dt = time.perf_counter() - t0
            lib.mrb_transfer_bytes(cnt.ctypes.data, cnt[1:].ctypes.data, 1)
            if step:
                times.append(dt)
        t = reduce_max(sum(times), world, dist, device)
        e2e = {"value": round(pairqueue.job_throughput(float(npx) * tot_iters * steps, t, world,
                                                       device), 3),
               "unit": UNIT, "steps": steps, "ms_per_step": round(1e3 * t / steps, 3),
               "h2d_bytes_per_step": int(cnt[0]), "d2h_bytes_per_step": int(cnt[1]),
               "api": "mrb_pixel_batch_set_images(host) + run + get_results + sync",
               "includes": "H2D images, full registration, D2H ux/uy/warped + statuses"}
    lib.mrb_pixel_batch_destroy(batch)

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    es = 4 if args.precision == "f32" else 8
    bytes_launch = float(P) * npx * 6 * es  # read u, write u, read (Te, Re): 3 pairs of Real
    achieved = bytes_launch / (kt[0] / 1e3) / 1e9
    ncu = ncu_record("pixel", args.precision, "k_pixel_step")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tot, work = 0.0, 0.0
        for re, te in pairs[:1]:
            dt, its = _oracle_pixelwise(re, te, PIXEL_REF_ITERS)
            tot += dt
            work += float(npx) * its
        cpu = {"value": round(work / tot / 1e6, 4), "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"1 pair (seed {used[0]}) 512x512, {PIXEL_REF_ITERS} iterations of the "
                         f"oracle register_pixelwise (numpy float64), {tot:.1f} s"}
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(t_ms / args.steps, 4), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic (seeded BASELINE generator, config-2 pairs)",
            "config": {"workload": f"pixel: {total} pairs of {W}x{H} in the job, {PIXEL_ITERS} "
                                   f"iterations, {PIXEL_PASSES} smoothing passes (reference "
                                   "baseline.py engine)",
                       "pairs_per_gpu": P, "global_pairs": total, "image": [W, H],
                       "iterations": PIXEL_ITERS, "tau": 0.005, "lam": 0.8,
                       "smoothing_passes": PIXEL_PASSES,
                       "pair_seeds": seeds_text(seeds, rank, world, args.weak),
                       "l2": "flushed (256 MiB write) between timed steps, outside the events",
                       "parallelism": f"pair-sharded dp{world} (no collective)",
                       "precision": args.precision},
            "gpu_launches": launches,
            "kernel_ms": {"k_pixel_step": round(float(kt[0]), 5), "run": round(float(kt[1]), 4)},
            "roofline": roofline_block("k_pixel_step", achieved, peak, ncu, kt[0],
                                       "algorithmic bytes = read u + write u + read (Te, Re) per "
                                       "pixel per iteration"),
            "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch_under_torchrun(n):
    """`--gpus N` with no torchrun environment: run this script as N ranks,
    one process per GPU, through torch.distributed.run (127.0.0.1
    rendezvous on a free port); rank 0 prints the JSON line."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args, rank, world):
    """The multi-rank plumbing without a GPU: sharding, barrier, max-over-
    ranks time and summed work over gloo."""
    dist = dist_init("gloo", rank) if world > 1 else None
    seeds, total, scaling = job_seeds(args, rank, world)
    barrier(world, dist)
    t = reduce_max(1.0 + rank, world, dist, "cpu")
    value = pairqueue.job_throughput(float(len(seeds)), t, world, "cpu")
    gathered = [seeds]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, seeds)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": scaling,
                          "global_pairs": total, "seeds_by_rank": gathered,
                          "max_time": t, "value": value}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main(argv=None):
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus))
    rank, world, local = dist_setup()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        run_dry(args, rank, world)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload == "pixel":
        run_pixel(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
