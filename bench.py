#!/usr/bin/env python
"""bench.py -- H-matvec dofs/s & ACA assembly entries/s (fp64) on B200.

One "step" = one H-matrix-vector product y = A x of the 3x3 Kelvin
collocation H-matrix (BASELINE.json configs[1] by default: unit-sphere
icosphere, 20480 triangles, 61440 dofs, b_min 32, eta 1, ACA eps 1e-6,
x uniform [-1,1] seed 1).  The H-matrix is assembled once on the GPU before
the timed region; assembly is timed separately and reported under
"assembly" (entries/s and fp64 roofline).

  value : dofs/s of the device-resident matvec (x, y already in HBM), K steps
          timed with CUDA events on the library's stream, max over ranks
  e2e   : the same metric through the public API with pinned host buffers
          (H2D of x and D2H of y inside every timed step)

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
        python bench.py --impl reference ...   (CPU oracle of the reference path)
Multi-GPU (torchrun): block rows sharded over ranks, x broadcast and y
summed (disjoint rows) with NCCL on the library's stream.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H-matvec dofs/s & ACA assembly entries/s (fp64), % of HBM/FP64 roofline"

CONFIGS = {
    # BASELINE.json configs[k]; meshes are synthetic (no dataset ships)
    "c1": dict(desc="icosphere L3, 1280 triangles, 3840 dofs", mesh=("icosphere", 3),
               b_min=32, eta=1.0, eps=1e-4, nrhs=1, seed=0, x="uniform"),
    "c2": dict(desc="icosphere L5, 20480 triangles, 61440 dofs", mesh=("icosphere", 5),
               b_min=32, eta=1.0, eps=1e-6, nrhs=1, seed=1, x="uniform"),
    "c3": dict(desc="voxel cube [0,1]^3 128^2/face, 196608 triangles, 589824 dofs",
               mesh=("cube", 128), b_min=64, eta=1.0, eps=1e-5, nrhs=1, seed=2,
               x="normal_dirichlet0"),
    "c4": dict(desc="ellipsoid (2,1,0.5) L6, 81920 triangles, 245760 dofs",
               mesh=("ellipsoid", 6), b_min=32, eta=1.0, eps=1e-2, nrhs=1, seed=3,
               x="bump"),
    "c5": dict(desc="icosphere L8, 1310720 triangles, 3932160 dofs, 16 RHS",
               mesh=("icosphere", 8), b_min=64, eta=1.0, eps=1e-5, nrhs=16, seed=4,
               x="normal"),
}

BETA_STOP = 0.8  # ACA stopping beta (partition eta = 1 is outside (0,1))


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def make_mesh(hm, cfg):
    kind, p = cfg["mesh"]
    if kind == "icosphere":
        return hm.Mesh.icosphere(p)
    if kind == "ellipsoid":
        return hm.Mesh.ellipsoid(p, 2.0, 1.0, 0.5)
    m = hm.Mesh.voxel_cube(p, 0.0, 1.0)
    m.label_dirichlet("x3<=0")
    return m


def make_x(hm, cfg, mesh, n_dofs):
    nrhs = cfg["nrhs"]
    kind = cfg["x"]
    if kind == "uniform":
        x = hm.random_vector(n_dofs * nrhs, cfg["seed"], "uniform")
    elif kind == "normal":
        x = hm.random_vector(n_dofs * nrhs, cfg["seed"], "normal")
    elif kind == "normal_dirichlet0":
        x = hm.random_vector(n_dofs * nrhs, cfg["seed"], "normal")
        d = mesh.arrays()["dirichlet"].astype(bool)
        x.reshape(nrhs, 3, -1)[:, :, d] = 0.0  # g_N extension (hmbem_cli.cpp:76-77)
    else:  # Gaussian bump at (2,0,0), sigma 0.05, + 1e-3 uniform noise
        c = mesh.arrays()["centroids"]
        bump = np.exp(-np.sum((c - np.array([2.0, 0, 0])) ** 2, axis=1) / (2 * 0.05 ** 2))
        x = np.tile(bump, 3) + 1e-3 * hm.random_vector(n_dofs, cfg["seed"], "uniform")
    return np.asfortranarray(x.reshape(nrhs, n_dofs).T) if nrhs > 1 else x


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, name in enumerate(names):
                if len(r) > 4 + k and r[4 + k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profile_traffic(config_name):
    """dram bytes per matvec of the streamed kernels from the committed ncu
    summary (profiles/ncu_<config>_matvec.json), if present."""
    p = os.path.join(ROOT, "profiles", f"ncu_{config_name}_matvec.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_matvec")
    except (OSError, ValueError):
        return None


def profile_pipes(config_name):
    """fp64-pipe utilisation of the assembly kernels from the committed ncu
    captures (the north star's counter for kernel evaluation): the ACA
    kernel and the near-field fill, per config when captured."""
    out = {}
    for key, fname in (("aca_fp64_pipe_pct", f"ncu_r01_aca_{config_name}_final.json"),
                       ("nearfield_fp64_pipe_pct", f"ncu_r01_{config_name}_assembly.json")):
        try:
            with open(os.path.join(ROOT, "profiles", fname)) as f:
                launches = json.load(f)["launches"]
        except (OSError, ValueError, KeyError):
            continue
        want = "aca_kernel" if key.startswith("aca") else "nearfield_kernel"
        for l in launches:
            if want in l.get("kernel", ""):
                out[key] = l.get("fp64_pipe_pct")
                out[key.replace("pct", "source")] = "profiles/" + fname
                break
    return out or None


# ---------------------------------------------------------------------------
def cpu_reference(args, cfg, emit_line: bool):
    """The reference path's CPU implementation (oracle port) on this config:
    assembly with all host threads (parallel_for over blocks) and the serial
    H-matvec (hmatrix.cpp:22-45), each step one matvec."""
    import paper_2205_04752_b200 as hm
    from oracle import oracle as orc
    mesh = make_mesh(hm, cfg)
    a = mesh.arrays()
    cores = os.cpu_count() or 1
    prob = orc.Problem.kelvin(a["vertices"], a["triangles"], 1.0, 0.3, cfg["b_min"], cfg["eta"])
    t0 = time.perf_counter()
    prob.assemble(eps=cfg["eps"], beta=BETA_STOP)
    t_asm = time.perf_counter() - t0
    _, entries = prob.assemble_time()
    n = 3 * mesh.num_triangles
    x = make_x(hm, cfg, mesh, n)
    xs = x if x.ndim == 1 else x[:, 0]
    times = []
    steps = args.steps if emit_line else 3
    warm = args.warmup if emit_line else 1
    for it in range(warm + steps):
        t0 = time.perf_counter()
        prob.matvec(xs)
        dt = time.perf_counter() - t0
        if it >= warm:
            times.append(dt)
    t_mv = float(np.mean(times))
    value = n / t_mv
    sample = (f"{cfg['desc']}: oracle assembly ({cores} threads, {t_asm:.1f} s) + "
              f"{steps} serial H-matvecs (1 RHS, {t_mv * 1e3:.1f} ms each)")
    out = {
        "cpu_baseline": {"value": value, "unit": "dofs/s", "cores": 1, "kind": "port",
                         "sample": sample, "ms_per_matvec": t_mv * 1e3},
        "assembly": {"value": entries / t_asm, "unit": "entries/s", "cores": cores,
                     "seconds": t_asm, "entries": entries},
    }
    return out, t_mv


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    res, t_mv = cpu_reference(args, cfg, emit_line=True)
    v = res["cpu_baseline"]["value"]
    line = {
        "metric": METRIC, "value": v, "unit": "dofs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_mv * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": args.config + ": " + cfg["desc"], "b_min": cfg["b_min"],
                   "eta": cfg["eta"], "eps_aca": cfg["eps"], "beta_stop": BETA_STOP,
                   "nrhs": 1},
        "cpu_baseline": res["cpu_baseline"],
        "assembly_cpu": res["assembly"],
        "e2e": {"value": v, "unit": "dofs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def weighted_entries(h):
    """sum_c w_c (sum_adm k_cb (m_b + n_b) + sum_dense m_b n_b), w_c = 1 on the
    diagonal components and 2 off it (each off-diagonal factor serves two x
    components): the multiply-adds of one RHS."""
    k, _, _, _ = h.ranks()
    blocks = h.partition_blocks()
    t = h.tree()
    m = (t.nodes[blocks[:, 0], 1] - t.nodes[blocks[:, 0], 0]).astype(np.float64)
    n = (t.nodes[blocks[:, 1], 1] - t.nodes[blocks[:, 1], 0]).astype(np.float64)
    adm = blocks[:, 2] == 1
    rb, re = h.row_range
    owned = (t.nodes[blocks[:, 0], 0] >= rb) & (t.nodes[blocks[:, 0], 1] <= re)
    w = np.array([1.0, 2.0, 2.0, 1.0, 2.0, 1.0])
    kk = np.where(k < 0, 0, k).astype(np.float64)
    lowrank = (kk * ((m + n) * (adm & owned))[None, :]).sum(axis=1)
    dense = float((m * n * (~adm & owned)).sum())
    return float((w * (lowrank + dense)).sum())


# ---------------------------------------------------------------------------
def galerkin_leg(hm, torch, mesh, cfg, device, reps=20):
    """SURVEY.md 8f rank 2 on the same mesh: the Galerkin V_Delta and V_kl
    H-matrices (pair quadrature with Sauter-Schwab rules for touching pairs)
    assembled by the same engine, and the Lame single-layer V_h matvec
    (compose_Vh) on device pointers.  Secondary object of the c2 line."""
    vh = hm.LameSingleLayer(mesh, 1.0, 0.3, b_min=cfg["b_min"], eta=cfg["eta"],
                            device=device)
    best = None
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sk, sd = vh.assemble(eps=cfg["eps"], beta=BETA_STOP, lookahead=2)
        wall = time.perf_counter() - t0
        if best is None or wall < best[0]:
            best = (wall, sk, sd)
    wall, sk, sd = best
    nt = vh.nt
    x = hm.random_vector(3 * nt, cfg["seed"], "uniform")
    xd = torch.tensor(x, dtype=torch.float64, device=f"cuda:{device}")
    yg = torch.zeros(3 * nt, dtype=torch.float64, device=f"cuda:{device}")
    yd = torch.zeros(3 * nt, dtype=torch.float64, device=f"cuda:{device}")
    s = 0.5 / vh.E * (1.0 + vh.nu) / (1.0 - vh.nu)
    c34 = 3.0 - 4.0 * vh.nu

    def vh_step():
        vh.vkl.matvec_ptr(xd.data_ptr(), yg.data_ptr(), 1)
        vh.vdelta.matvec_ptr(xd.data_ptr(), yd.data_ptr(), 3)  # diag3: 3 RHS
        torch.cuda.synchronize()
        return s * (c34 * yd + yg)

    y = vh_step()
    for _ in range(3):
        vh_step()
    t0 = time.perf_counter()
    for _ in range(reps):
        vh_step()
    ms = (time.perf_counter() - t0) / reps * 1e3
    y_host = vh.matvec(x)
    entries = sk.aca_entries + sk.dense_entries + sd.aca_entries + sd.dense_entries
    # the composed operators of the operator algebra
    # on device vectors: V_h, K_h (3N -> 3M), D_h (3N -> 3N)
    ops_t = None
    try:
        ops = hm.OperatorSet(mesh, 1.0, 0.3, b_min=cfg["b_min"], eta=cfg["eta"], device=device)
        so = ops.assemble(eps=cfg["eps"], beta=BETA_STOP, lookahead=2)
        xn = torch.tensor(hm.random_vector(3 * ops.n, 3, "uniform"), device=f"cuda:{device}")
        xm = torch.tensor(hm.random_vector(3 * ops.m, 4, "uniform"), device=f"cuda:{device}")
        ops_t = {"assembly_ms_device": sum(st_.ms_total for st_ in so)}
        for name, f_, v_ in (("vh", ops.vh_dev, xm), ("kh", ops.kh_dev, xn),
                             ("dh", ops.dh_dev, xn), ("kh_t", ops.kh_t_dev, xm)):
            f_(v_)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                f_(v_)
            torch.cuda.synchronize()
            ops_t[name + "_ms_wall"] = (time.perf_counter() - t0) / 5 * 1e3
        del ops
    except Exception as e:  # informational
        ops_t = {"error": str(e)}
    # CPU reference path (the oracle restatement, all host threads) beside
    # the device on a bounded sample: the icosphere L3 (1280 triangles)
    cpu = None
    try:
        import os as _os
        from oracle import oracle as orc
        m3 = hm.Mesh.icosphere(3)
        a3 = m3.arrays()
        t0 = time.perf_counter()
        for which in (0, 1):
            p = orc.Problem.galerkin(a3["vertices"], a3["triangles"], which,
                                     b_min=cfg["b_min"], eta=cfg["eta"])
            p.assemble(eps=cfg["eps"], beta=BETA_STOP, lookahead=2)
        cpu_s = time.perf_counter() - t0
        g3 = hm.LameSingleLayer(m3, 1.0, 0.3, b_min=cfg["b_min"], eta=cfg["eta"],
                                device=device)
        g3.assemble(eps=cfg["eps"], beta=BETA_STOP, lookahead=2)
        s3 = g3.assemble(eps=cfg["eps"], beta=BETA_STOP, lookahead=2)
        gpu_ms = s3[0].ms_total + s3[1].ms_total
        cpu = {"sample": "icosphere L3, 1280 triangles: V_kl grid + V_Delta assembly",
               "cpu_s": cpu_s, "cores": _os.cpu_count(), "kind": "port",
               "gpu_ms_device": gpu_ms, "speedup": cpu_s / (gpu_ms * 1e-3)}
    except Exception as e:  # the CPU leg is informational
        cpu = {"error": str(e)}

    return {"operator": "V_h = (1+nu)/(2E(1-nu)) [(3-4nu) diag3(V_Delta) + grid(V_kl)]",
            "assembly_ms_device": sk.ms_total + sd.ms_total, "assembly_ms_wall": wall * 1e3,
            "entries": entries, "entries_per_s": entries / ((sk.ms_total + sd.ms_total) * 1e-3),
            "nearfield_ms": sk.ms_nearfield + sd.ms_nearfield,
            "pivots": sk.pivots + sd.pivots,
            "storage_mb": vh.vkl.storage()["mb_current"] + vh.vdelta.storage()["mb_current"],
            "matvec_ms_wall": ms, "matvec_dofs_per_s": 3 * nt / (ms * 1e-3),
            "matvec_check_rel": float(np.linalg.norm(y.cpu().numpy() - y_host) /
                                      np.linalg.norm(y_host)),
            "cpu_baseline": cpu,
            "operators": ops_t}


def run_ours(args, cfg):
    import torch
    import paper_2205_04752_b200 as hm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    # torchrun (RANK set) or N > 1: the NCCL protocol runs even for one rank
    # (HMB_BENCH_NO_DIST=1 disables it for a single process)
    if world > 1 or ("RANK" in os.environ and not os.environ.get("HMB_BENCH_NO_DIST")):
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local
    torch.cuda.set_device(device)

    mesh = make_mesh(hm, cfg)
    nrhs = cfg["nrhs"]
    h = hm.HMatrix.kelvin(mesh, E=1.0, nu=0.3, b_min=cfg["b_min"], eta=cfg["eta"],
                          device=device, shard=(rank, world))
    n = h.cols
    # ---- assembly (timed on the device, best of 3 after one warm-up; the
    # first assemblies of a process also map the factor arenas) ----
    asm = []
    h.set_profiling(True)
    for _ in range(4):
        for k in ("aca", "nearfield", "compact", "relocate"):
            h.kernel_times(k, reset=True)
        st = h.assemble(eps=cfg["eps"], beta=BETA_STOP, lookahead=2)
        kt_asm = {k: h.kernel_times(k, reset=True)[0]
                  for k in ("aca", "nearfield", "compact", "relocate")}
        asm.append((st, kt_asm))
    h.set_profiling(False)
    best, best_kt = min(asm[1:], key=lambda p: p[0].ms_total)
    storage = h.storage()
    fp64_peak = hm.fp64_peak_tflops(device)

    x = make_x(hm, cfg, mesh, n)
    xt = torch.tensor(np.ascontiguousarray(x.T if x.ndim > 1 else x), dtype=torch.float64,
                      device=f"cuda:{device}")
    # library layout: dofs x nrhs column-major == nrhs x dofs row-major
    yt = torch.zeros((nrhs, h.rows) if nrhs > 1 else h.rows, dtype=torch.float64,
                     device=f"cuda:{device}")
    stream = torch.cuda.ExternalStream(h.stream(), device=f"cuda:{device}")

    def step():
        with torch.cuda.stream(stream):
            if dist is not None:
                dist.broadcast(xt, src=0)
            h.matvec_ptr(xt.data_ptr(), yt.data_ptr(), nrhs)
            if dist is not None:
                dist.all_reduce(yt)  # rows are disjoint across ranks: sum = gather

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # per-kernel device times from a separate profiled pass (not the timed one)
    h.set_profiling(True)
    KNAMES = ("gather", "hmv_stream", "hmv_zreduce", "hmv_ypart", "hmv_reduce", "hmv_blocks",
              "hmv16_z", "hmv16_zsum", "hmv16_leaf")
    for k in KNAMES:
        h.kernel_times(k, reset=True)
    for _ in range(max(3, min(args.steps, 10))):
        step()
    torch.cuda.synchronize()
    kt = {k: h.kernel_times(k, reset=True) for k in KNAMES}
    h.set_profiling(False)

    # ---- timed region: K device-resident matvecs ----
    clocks = ClockSampler(device)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)  # sampler warm-up
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = h.rows * nrhs / (ms_step * 1e-3)

    # ---- e2e through the public API with pinned host buffers ----
    xh = torch.tensor(np.ascontiguousarray(x.T if x.ndim > 1 else x),
                      dtype=torch.float64).pin_memory()
    yh = torch.zeros(yt.shape, dtype=torch.float64).pin_memory()
    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(2):
        h.matvec_ptr(xh.data_ptr(), yh.data_ptr(), nrhs, device=False)
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        if dist is not None:  # host-driven: x from host on every rank, y reduced
            h.matvec_ptr(xh.data_ptr(), yh.data_ptr(), nrhs, device=False)
            yd = yh.to(f"cuda:{device}", non_blocking=True)
            dist.all_reduce(yd)
            yh.copy_(yd)
        else:
            h.matvec_ptr(xh.data_ptr(), yh.data_ptr(), nrhs, device=False)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # ---- roofline of the dominant kernel ----
    peak, peak_src = measured_peaks()
    nsteps_prof = max(kt["gather"][1], 1)
    alg_bytes = storage["matvec_bytes"] + 8 * (nrhs - 1) * (h.rows + h.cols)
    traffic = profile_traffic(args.config) if nrhs == 1 else None
    if kt["hmv16_leaf"][1] > 0:
        # 16 RHS per pass on the fp64 tensor cores: flop-bound:
        # F = 2 nrhs sum_c w_c (sum_adm k (m + n) + sum_dense m n), w = 1 | 2
        ms_dom = (kt["hmv16_z"][0] + kt["hmv16_zsum"][0] + kt["hmv16_leaf"][0]) / nsteps_prof
        flops = 2.0 * nrhs * weighted_entries(h)
        dmma_peak = hm.dmma_peak_tflops(device)
        achieved = flops / (ms_dom * 1e-3) / 1e12
        roofline = {"bound": "tensor", "kernel": "hmv16_z + hmv16_zsum + hmv16_leaf (DMMA)",
                     "achieved": achieved, "peak": dmma_peak, "unit": "TFLOP/s",
                     "frac": achieved / dmma_peak, "traffic": traffic,
                     "peak_source": "measured (hmgpu_dmma_peak, fp64 m8n8k4 chains)",
                     "algorithmic_flops_per_step": flops,
                     "algorithmic_bytes_per_step": alg_bytes,
                     "hbm_frac": alg_bytes / (ms_dom * 1e-3) / 1e9 / peak,
                     "ms_kernel": ms_dom, "ms_matvec_device": ms_step}
        dom_launches = 4 * ((nrhs + 15) // 16)
    else:
        ms_stream = (kt["hmv_stream"][0] + kt["hmv_ypart"][0]) / max(kt["hmv_stream"][1], 1)
        ms_blocks = kt["hmv_blocks"][0] / max(kt["hmv_blocks"][1], 1)
        ms_dom = ms_stream if ms_stream > 0 else ms_blocks
        dom_name = "hmv_stream_kernel (pass A + pass B)" if ms_stream > 0 else "hmv_blocks_kernel"
        achieved = alg_bytes / (ms_dom * 1e-3) / 1e9 if ms_dom > 0 else None
        roofline = {"bound": "hbm", "kernel": dom_name,
                    "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak if achieved else None,
                    "traffic": traffic, "peak_source": peak_src,
                    "algorithmic_bytes_per_step": alg_bytes,
                    "ms_kernel": ms_dom,
                    "ms_matvec_device": ms_step,
                    "matvec_frac_incl_gather_reduce": alg_bytes / (ms_step * 1e-3) / 1e9 / peak}
        dom_launches = 3 + (kt["hmv_zreduce"][1] > 0) + (kt["hmv_ypart"][1] > 0)

    res = None
    if rank == 0 and world == 1 and not args.no_cpu:
        res, _ = cpu_reference(args, cfg, emit_line=False)
    # counted fp64 flops per entry: 30 n_q + 1 with n_q = 7 for
    # near-field pairs; ACA entries mostly far (n_q = 3); report entries/s
    asm_s = best.ms_total * 1e-3
    entries = best.aca_entries + best.dense_entries
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "dofs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded mesh + x; random_vector mt19937_64)",
        "config": {"workload": args.config + ": " + cfg["desc"], "b_min": cfg["b_min"],
                   "eta": cfg["eta"], "eps_aca": cfg["eps"], "beta_stop": BETA_STOP,
                   "lookahead": 2, "nrhs": nrhs,
                   "parallelism": f"block-row shards x{world}" if world > 1 else "1 GPU",
                   "l2": f"inputs larger than L2: {alg_bytes / 1e9:.2f} GB streamed per step"},
        "roofline": roofline,
        "e2e": {"value": h.rows * nrhs / e2e_s, "unit": "dofs/s",
                "h2d_bytes_per_step": int(8 * h.cols * nrhs),
                "d2h_bytes_per_step": int(8 * h.rows * nrhs)},
        "gpu_launches": int(args.steps * dom_launches),
        "clocks": ck,
        "assembly": {"value": entries / asm_s, "unit": "entries/s", "ms": best.ms_total,
                     "kernel_ms": best_kt, "aca_entries": best.aca_entries,
                     "dense_entries": best.dense_entries, "pivots": best.pivots,
                     "storage_mb": storage["mb_current"],
                     # counted flops: 30 n_q + 1 per component entry
                     "counted_tflops": best.counted_flops / asm_s / 1e12,
                     "fp64_peak_tflops_measured": fp64_peak,
                     "fp64_frac": best.counted_flops / asm_s / 1e12 / fp64_peak,
                     "fp64_frac_kernels": best.counted_flops /
                     ((best_kt["aca"] + best_kt["nearfield"]) * 1e-3) / 1e12 / fp64_peak,
                     "nearfield_entries_per_s": best.dense_entries /
                     (best_kt["nearfield"] * 1e-3) if best_kt["nearfield"] else None,
                     "ncu": profile_pipes(args.config)},
        "kernel_ms": {k: (v[0] / v[1] if v[1] else 0.0) for k, v in kt.items()},
    }
    if args.config == "c4" and world == 1:
        # the adaptive matvec of config 4 (Algorithm 2): full-mode assembly at
        # eps 1e-2, theta 0.7, eps_amvm 1e-6, look-ahead 2, 5 sweeps; the
        # estimator, marking walk and refinement run on the device.  One
        # untimed run first (like the matvec warm-up: the estimator's term
        # buffers, ~2 GB, come out of the stream-ordered pool on first use),
        # then a fresh assembly and the timed run
        h.assemble(eps=cfg["eps"], beta=BETA_STOP, lookahead=2)
        h.amvm_multiply(x, theta=0.7, eps_amvm=1e-6, lookahead_steps=2, max_iterations=5)
        st4 = h.assemble(eps=cfg["eps"], beta=BETA_STOP, lookahead=2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rep = h.amvm_multiply(x, theta=0.7, eps_amvm=1e-6, lookahead_steps=2,
                                 max_iterations=5)
        amvm_s = time.perf_counter() - t0
        line["amvm"] = {"seconds": amvm_s, "sweeps": len(rep.iterations),
                        "termination": rep.termination,
                        "gamma": [float(i.gamma) for i in rep.iterations],
                        "marked": [int(i.marked) for i in rep.iterations],
                        "ms_per_sweep": [float(i.ms) for i in rep.iterations],
                        "warmup_runs": 1,
                        "assembly_ms": st4.ms_total}
    if args.config == "c2" and world == 1 and not args.no_galerkin:
        try:  # secondary object: never costs the headline line
            line["galerkin"] = galerkin_leg(hm, torch, mesh, cfg, device)
        except Exception as e:
            line["galerkin"] = {"error": str(e)}
    if res is not None:
        line["cpu_baseline"] = res["cpu_baseline"]
        line["assembly"]["cpu_entries_per_s"] = res["assembly"]["value"]
        line["assembly"]["cpu_cores"] = res["assembly"]["cores"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-galerkin", action="store_true",
                    help="skip the Galerkin V_h object of the c2 line")
    ap.add_argument("--nrhs", type=int, default=0,
                    help="override the config's number of right-hand sides")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to 3 (timing rule)")
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.nrhs > 0:
        cfg["nrhs"] = args.nrhs
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
