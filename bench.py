#!/usr/bin/env python
"""SAND adaptive T-MLP query benchmark (BASELINE.json metric) on 1..8 B200s.

One step = one sand_query over the whole workload: K1 depth-map lookup -> K2 scan/scatter binning
-> K3 fused T-MLP (tcgen05), i.e. every row of SURVEY.md Sec. 8(a), inputs resident in HBM.
Default workload (N = 1) = BASELINE.json configs[2] ("C2"): 512^3 marching-cubes vertex grid
(134,217,728 points), 8 x 256 SIREN T-MLP (seeded SIREN init, BF16 MMA),
level-7 sphere-union octree.  N > 1 (one rank per GPU, NCCL; `--gpus N` self-launches under
torch.distributed.run): BASELINE.json configs[4] ("C4"), the fixed 1024^3 grid with the level-8 octree,
strong-scaled -- cut into work-balanced z-slabs, one per rank (`--scaling weak` refines the grid along z
instead); NCCL only all-gathers a small per-rank record after the timed region (no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sand|reference]
"""
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

METRIC = "adaptive T-MLP SDF queries/sec at 512³ grid (8×256 SIREN) and % tensor peak"
UNIT = "points/s"
R_DYN_30 = 2.39e-2   # run_dynamic's second exit threshold (see there)


def _peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return dict(bf16=float(mp["bf16_tflops"]), bf16_sus=float(mp["bf16_tflops_sustained"]),
                    hbm=float(mp["hbm_gbs"]), src="measured")
    except Exception:
        return dict(bf16=1590.0, bf16_sus=1400.0, hbm=6650.0, src="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx = float(f[2])
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if pw:
            out["power_w_median"] = float(np.median(pw))
        return out


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _arm_config(args, c, ws, wl_desc, global_points):
    """The `config` object of the bench line -- identical for this arm and the reference arm."""
    weak = args.scaling == "weak"
    if ws == 1:
        wl = wl_desc
    elif c.grid_R is not None:
        R = c.grid_R
        wl = (f"{args.config} weak-scaled: {R}x{R}x{R * ws} grid" if weak else
              f"{args.config} strong-scaled: the fixed {R}x{R}x{R} grid") + f", work-balanced z-slabs over {ws} ranks"
    else:
        wl = f"{args.config} x {ws} ranks" if weak else f"{args.config} split over {ws} ranks"
    dmap = {"C0": "32^3 voxel sphere map", "C1": "128^3 voxel 16-sphere map",
            "C2": "level-7 sphere-union octree (baked 128^3)", "C3": "level-7 sphere-union octree (baked 128^3)",
            "C4": "level-8 sphere-union octree (baked 256^3)"}[args.config]
    per_rank = 12 * global_points / (1 if weak else ws)
    return {"workload": wl,
            "model": f"{c.spec.L}x{c.spec.H} SIREN T-MLP (seeded SIREN init), linear tails",
            "depth_map": dmap, "global_points": global_points, "parallelism": f"dp{ws} (z-slab shards)",
            "l2": (f"inputs {per_rank / 1e9:.2f} GB per rank > 126 MB L2; no flush needed"
                   if per_rank >= 126e6 else
                   f"inputs {per_rank / 1e6:.0f} MB per rank < 126 MB L2: a 256 MB buffer is "
                   "written before every step (outside the per-step CUDA events)"),
            "full_depth_baseline": bool(args.full_depth)}


def _n1_workload(args, c):
    """The N = 1 workload description (rank 0 of one)."""
    if c.grid_R is not None:
        return f"{args.config}: {c.grid_R}x{c.grid_R}x{c.grid_R} grid, z-planes [0,{c.grid_R}) on rank 0"
    return f"{args.config}: points [0,{c.points_fn().shape[0]})"


def run_reference(args):
    """--impl reference: the plain FP32 C oracle (oracle/sand_oracle_fp32.c, OpenMP over the host cores), as it
    stands, on a bounded seeded sample of the same workload per step.  Rank 0 only."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import sandgen as g
    from oracle import fp32 as ofp
    c = g.make_config(args.config)
    p = c.params()
    R = c.grid_R
    n_step = args.ref_sample
    rng = np.random.default_rng(1234)
    cloud = c.points_fn() if R is None else None
    n_work = R ** 3 if R is not None else cloud.shape[0]
    times = []
    for it in range(args.warmup + args.steps):
        if R is not None:
            pts = _sample_grid_points(R, 0, R, R, n_step, rng)
        else:
            pts = cloud[np.sort(rng.choice(n_work, n_step, replace=False))]
        t0 = time.perf_counter()
        ofp.query_fp32(p, c.depthmap, pts)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    ms = 1e3 * float(np.mean(times))
    val = n_step / (ms / 1e3)
    sample = (f"{n_step} seeded random vertices of the {R}^3 grid per step" if R is not None else
              f"{n_step} seeded random points of the {n_work}-point cloud per step")
    global_points = n_work * ws if (R is not None and args.scaling == "weak") else n_work
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.scaling == "weak" else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _arm_config(args, c, ws, _n1_workload(args, c), global_points),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": ofp.threads(), "cpu": ofp.cpu_model(),
                             "kind": "oracle (plain FP32 C, OpenMP, -ffp-contract=off)", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


TRAFFIC_FILE = "r02_k3_traffic.json"
TRAFFIC_SRC = f"profiles/{TRAFFIC_FILE} (ncu --set full of this round's kernel, dram read+write per launch)"


def _traffic():
    """DRAM bytes per K3 launch from the committed ncu --set full capture (profiles/), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", TRAFFIC_FILE)))
        return t["dram_bytes_per_launch"]
    except Exception:
        return None


def _sine_roofline(per_depth, H, ms_mlp, clocks):
    """K3's second bound: sum_p d_p * H sines per launch against MUFU.SIN at 16 / clk / SM (4 per SMSP;
    scripts/micro/epi2.cu measures 15.3 elements / clk / SM for the sine + tail + BF16-pack chain)."""
    sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
    sines = float(sum(c * d * H for d, c in enumerate(per_depth)))
    ach = sines / (ms_mlp / 1e3) / 1e9
    peak = 148 * 16 * sm_mhz * 1e6 / 1e9
    return {"bound": "alu", "kernel": "K3 epilogue (MUFU.SIN)", "achieved": ach, "peak": peak, "unit": "Gsin/s",
            "frac": ach / peak, "sines_per_launch": sines,
            "peak_source": "derived: 148 SM x 16 MUFU.SIN / clk x median SM clock (DESIGN.md, K3 per-SM budget)"}


def _padding_waste(per_depth, H, fp32, even_bins=False):
    """Fraction of the H x H tensor FLOPs K3 executes that pad: ragged last tile per depth bucket (256-row
    pair tiles, 128-row otherwise), with even_bins (the slot-team kernel) every bucket rounded up to an even
    tile count, and, for H = 336, the width padded to 352 (zero weights)."""
    T = 128 if fp32 else 256
    HP = (H + 31) // 32 * 32 if H > 256 and not fp32 else H

    def tiles(c):
        t = -(-c // T)
        return t + (t & 1) if even_bins else t

    alg = sum(c * (d - 1) * 2.0 * H * H for d, c in enumerate(per_depth) if d >= 1)
    ex = sum(tiles(c) * T * (d - 1) * 2.0 * HP * HP for d, c in enumerate(per_depth) if d >= 1)
    return {"tile_rows": T, "padded_width": HP, "even_bins": bool(even_bins), "executed_flops": ex,
            "waste_frac": 1.0 - alg / ex if ex else 0.0}


def _cores():
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        if th:
            return int(max(th))
    except Exception:
        pass
    return os.cpu_count()


def cpu_baseline(p, depthmap, sampler, budget_s):
    """The plain FP32 C oracle timed on the host cores (OpenMP, all usable cores) on bounded seeded samples of
    this workload (rank 0, N = 1): chunks of 2^15 points drawn by `sampler(m)` until ~budget_s of oracle time."""
    from oracle import fp32 as ofp
    done, t_used, chunk = 0, 0.0, 1 << 15
    while t_used < budget_s and done < (1 << 22):
        s = sampler(chunk)
        t0 = time.perf_counter()
        ofp.query_fp32(p, depthmap, s)
        t_used += time.perf_counter() - t0
        done += s.shape[0]
    return {"value": done / t_used, "unit": UNIT, "cores": ofp.threads(), "cpu": ofp.cpu_model(),
            "kind": "oracle (plain FP32 C, OpenMP, -ffp-contract=off)",
            "sample": f"{done} seeded random points of the workload ({t_used:.1f} s of oracle time)"}


def run_populate(args):
    """Depth-map population (Eq. 5 + Eq. 6): every finest leaf of the config's octree, 25 samples
    each (8 corners + centre + 16 seeded interior points, R21), r = 1.5e-4.  One step =
    sand_populate_leaf_depths over all of them.  Single GPU (rank 0 of any launch)."""
    import torch
    import sandgen as g
    from paper_2604_25936_b200 import SAND_BF16, SandContext
    ws, rank, local = _dist()
    if rank != 0:
        return 0
    c = g.make_config(args.config if args.config != "C1" else "C2")
    p = c.params()
    oc = c.depthmap
    sel = np.nonzero(oc.leaf_level == oc.level)[0]
    samples = g.leaf_samples(oc.leaf_level[sel], oc.leaf_ijk[sel], 16, seed=5)
    n, spl = samples.shape[0], samples.shape[1]
    dev = torch.device("cuda", 0)
    ts = torch.from_numpy(np.ascontiguousarray(samples.reshape(-1, 3))).to(dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    r = 1.5e-4
    from paper_2604_25936_b200 import SAND_OPT_FP32_TENSOR
    H, L = c.spec.H, c.spec.L
    ns = n * spl
    with SandContext(c.spec.L, c.spec.H, c.spec.omega0, SAND_BF16, c.spec.tail, 0) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        st = torch.cuda.current_stream(dev)
        ctx.sand_set_stream(st.cuda_stream)

        def timed(tensor, steps):
            ctx.sand_set_option(SAND_OPT_FP32_TENSOR, tensor)
            for _ in range(args.warmup):
                ctx.sand_populate_leaf_depths(ts.data_ptr(), n, spl, r, out.data_ptr())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record(st)
            for _ in range(steps):
                ctx.sand_populate_leaf_depths(ts.data_ptr(), n, spl, r, out.data_ptr())
            e1.record(st)
            torch.cuda.synchronize(dev)
            return e0.elapsed_time(e1) / steps

        ms_simt = timed(0, max(1, min(args.steps, 3)))          # the FP32 SIMT kernel, for comparison
        d_simt = out.cpu().numpy().copy()
        clk = ClockSampler(0)
        clk.start()
        ms = timed(1, args.steps)                                # split-FP16 tensor cores where H allows
        clocks = clk.stop()
        tensor_used = H in (64, 128, 256)
    flops = ns * (6.0 * H + (L - 1) * 2.0 * H * H + L * 2.0 * H)
    sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
    ach = flops / (ms / 1e3) / 1e12
    if tensor_used:
        # executed tensor work: three H x H products per hidden layer (split operands) + the split-bias MMA
        pk = _peaks()
        exec_flops = ns * (L - 1) * (3.0 * 2 * H * H + 2.0 * 16 * H)
        roof = {"bound": "tensor", "kernel": "k_tmlp_x3 (split-FP16 x3, Eq. 5 mode)",
                "achieved": exec_flops / (ms / 1e3) / 1e12, "peak": pk["bf16"], "unit": "TFLOP/s",
                "frac": exec_flops / (ms / 1e3) / 1e12 / pk["bf16"],
                "peak_source": pk["src"] + " bf16_tflops (burst; FP16 kind::f16 has the BF16 rate)",
                "flops_formula": "executed: samples x (L-1) x (3 x 2H^2 + 2 x 16 H)", "traffic": None}
    else:
        peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12   # FP32 FMA lanes x 2 FLOP x clock (B200_PROFILING.md units)
        roof = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "peak_source": "derived: 148 SM x 128 FP32 FMA lanes x 2 FLOP x median SM clock", "traffic": None}
    d_tc = out.cpu().numpy()
    cpu = None
    if not args.no_cpu:
        import oracle
        k = min(n, 2000)
        t0 = time.perf_counter()
        oracle.populate_leaf_depths(p, samples[:k], r)
        dt = time.perf_counter() - t0
        cpu = {"value": k * spl / dt, "unit": "samples/s", "cores": _cores(), "kind": "oracle (numpy float64)",
               "cores_note": "BLAS pool for the matmuls; sin, lookup and the Eq. 5 decision on one core",
               "sample": f"first {k} leaves x {spl} samples"}
    line = {"task": "populate", "metric": "depth-map population samples/sec (Eq. 5 + Eq. 6)",
            "value": ns / (ms / 1e3), "unit": "samples/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{c.name} octree finest leaves: {n} leaves x {spl} samples, r = 1.5e-4",
                       "model": f"{L}x{H} SIREN T-MLP (seeded init)"},
            "roofline": roof, "algorithmic_tflops": ach,
            "fp32_simt": {"value": ns / (ms_simt / 1e3), "unit": "samples/s", "ms_per_step": ms_simt,
                          "speedup_of_tensor_path": ms_simt / ms,
                          "leaf_depth_agreement": float(np.mean(d_simt == d_tc))},
            "cpu_baseline": cpu, "clocks": clocks,
            "depth_hist": np.bincount(d_tc, minlength=L + 1).tolist()}
    print(json.dumps(line), flush=True)
    return 0


def run_sweep(args):
    """octree max level 6..10 (C2's spheres, bands and score bump; Sec. 3.2 / Tab. 8 of the
    paper sweeps the octree depth) and a paper-like far-field map (depth 0 = cached SDF, Eq. 7, for
    every leaf farther than 0.04 from the surface: most of the grid) on C2's 512^3 grid with C2's 8x256 net.
    Levels <= 8 are baked into a dense grid on load, 9-10 are descended on the device.  One JSON line with
    one entry per map: points/s, per-stage ms, K1 achieved HBM GB/s (13 B/pt algorithmic; + 4 B/pt far SDF
    for depth-0 points), depth histogram.  Single GPU."""
    import torch
    import sandgen as g
    from sandgen import configs as gc
    from paper_2604_25936_b200 import SAND_BF16, SandContext
    ws, rank, local = _dist()
    if rank != 0:
        return 0
    c = g.make_config("C2")
    p = c.params()
    sph = g.make_spheres(gc.SPHERE_SEED)
    dev = torch.device("cuda", 0)
    pts_np = g.grid_points(c.grid_R)
    n = pts_np.shape[0]
    pts = torch.from_numpy(pts_np).to(dev)
    sdf = torch.empty(n, dtype=torch.float32, device=dev)
    dep = torch.empty(n, dtype=torch.uint8, device=dev)
    maps = [(f"octree level {lev}", lev, gc.BANDS_8, False) for lev in (6, 7, 8, 9, 10)]
    maps.append(("far-field octree level 7 (|d| >= 0.04 -> depth 0)", 7, (0.005, 0.01, 0.02, 0.04), True))
    entries = []
    pk = _peaks()
    with SandContext(c.spec.L, c.spec.H, c.spec.omega0, SAND_BF16, c.spec.tail, 0) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        ctx.sand_reserve(n)
        st = torch.cuda.current_stream(dev)
        ctx.sand_set_stream(st.cuda_stream)
        for name, lev, bands, far in maps:
            oc = g.build_octree(sph, lev, bands, c.spec.L, score_seed=gc.SCORE_SEED, far_band=far)
            ctx.sand_load_depthmap(oc)
            for _ in range(args.warmup):
                ctx.sand_query(pts.data_ptr(), n, sdf.data_ptr(), dep.data_ptr())
            ctx.sand_get_stats()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record(st)
            for _ in range(args.steps):
                ctx.sand_query(pts.data_ptr(), n, sdf.data_ptr(), dep.data_ptr())
            e1.record(st)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / args.steps
            s2 = ctx.sand_get_stats()
            q = max(s2["queries"], 1)
            pd = [int(v) for v in s2["per_depth"][:c.spec.L + 1]]   # last query's histogram
            ms_lk = s2["ms_lookup_sum"] / q
            k1_bytes = 13.0 * n + 4.0 * pd[0]
            f_exec = sum(pd[d] * (d - 1) * 2.0 * c.spec.H ** 2 for d in range(1, c.spec.L + 1))
            ms_mlp = s2["ms_mlp_sum"] / q
            entries.append({"map": name, "max_level": lev, "n_nodes": int(oc.nodes.size),
                            "n_leaves": int(oc.leaf_depth.size), "baked": lev <= 8,
                            "value": n / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
                            "stage_ms": {"lookup": ms_lk, "bin": s2["ms_bin_sum"] / q, "mlp": ms_mlp},
                            "depth0_frac": pd[0] / n, "mean_depth": sum(d * pd[d] for d in range(len(pd))) / n,
                            "k1_hbm_gbs": k1_bytes / (ms_lk / 1e3) / 1e9, "k1_hbm_frac": k1_bytes / (ms_lk / 1e3) / 1e9 / pk["hbm"],
                            "k3_tensor_frac": (f_exec / (ms_mlp / 1e3) / 1e12 / pk["bf16"]) if ms_mlp > 0 else None,
                            "per_depth": pd})
            print(f"[sweep] {name}: {n / (ms / 1e3) / 1e9:.2f} G points/s, lookup {ms_lk:.3f} ms, "
                  f"depth-0 {pd[0] / n:.3f}", file=sys.stderr, flush=True)
    line = {"task": "sweep", "metric": "adaptive T-MLP SDF queries/sec vs octree max level and far-field share",
            "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"C2 512^3 grid ({n} points), 8x256 SIREN T-MLP, C2 spheres",
                       "hbm_peak_gbs": pk["hbm"], "bf16_peak_tflops": pk["bf16"]},
            "entries": entries}
    print(json.dumps(line), flush=True)
    return 0


def run_dynamic(args):
    """the paper's 'SAND w/o Octree' alternative -- dynamic exit on
    |t_i| < r without a depth map -- on C2's 512^3 grid and 8x256 net, next to the octree path on the
    same points.  Two thresholds: the paper's r = 1.5e-4 (with SIREN-init weights no residual is
    that small, so every point runs to L) and the 30% quantile of |t_i| over a sample (exits spread over
    the layers).  FP32 SIMT kernel (sand_query_dynamic), tile-level early exit.  Single GPU."""
    import torch
    import sandgen as g
    from paper_2604_25936_b200 import SAND_BF16, SAND_OPT_DYN_SCHEDULE, SandContext
    ws, rank, local = _dist()
    if rank != 0:
        return 0
    steps = min(args.steps, 3)
    c = g.make_config("C2")
    p = c.params()
    dev = torch.device("cuda", 0)
    pts_np = g.grid_points(c.grid_R)
    n = pts_np.shape[0]
    pts = torch.from_numpy(pts_np).to(dev)
    sdf = torch.empty(n, dtype=torch.float32, device=dev)
    dep = torch.empty(n, dtype=torch.uint8, device=dev)
    # second threshold: a fixed constant, the 30% quantile of |t_i| (i >= 2) of C2's seeded weights over
    # 4096 grid points (measured in round 1; nothing on the product bench path comes from the oracle)
    r30 = R_DYN_30
    entries = []
    with SandContext(c.spec.L, c.spec.H, c.spec.omega0, SAND_BF16, c.spec.tail, 0) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        ctx.sand_load_depthmap(c.depthmap)
        ctx.sand_reserve(n)
        st = torch.cuda.current_stream(dev)
        ctx.sand_set_stream(st.cuda_stream)

        def timed(fn, k):
            for _ in range(min(args.warmup, 3)):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record(st)
            for _ in range(k):
                fn()
            e1.record(st)
            torch.cuda.synchronize(dev)
            return e0.elapsed_time(e1) / k

        ms_oct = timed(lambda: ctx.sand_query(pts.data_ptr(), n, sdf.data_ptr(), dep.data_ptr()), 5)
        # the octree path in the dynamic path's own arithmetic (FP32 SIMT) and on the FP32-accurate tensor
        # path, so that the ratio below compares the methods, not SIMT against tensor cores
        oct_same = {}
        from paper_2604_25936_b200 import SAND_F16X3, SAND_FP32
        for pname, pcode in (("fp32_simt", SAND_FP32), ("f16x3_tensor", SAND_F16X3)):
            with SandContext(c.spec.L, c.spec.H, c.spec.omega0, pcode, c.spec.tail, 0) as cx:
                cx.sand_load_weights(g.pack_blob(p))
                cx.sand_load_depthmap(c.depthmap)
                cx.sand_reserve(n)
                cx.sand_set_stream(st.cuda_stream)
                ms_p = timed(lambda: cx.sand_query(pts.data_ptr(), n, sdf.data_ptr(), dep.data_ptr()), steps)
                oct_same[pname] = {"value": n / (ms_p / 1e3), "unit": UNIT, "ms_per_step": ms_p}
        # tile-level early exit / pools re-compacted after every layer (FP32 SIMT) / every layer on the split-FP16
        # tensor kernel with the exit selected afterwards
        for mode in ("tile", "pool", "tensor"):
            ctx.sand_set_option(SAND_OPT_DYN_SCHEDULE, {"tile": 0, "pool": 1, "tensor": 2}[mode])
            for name, r in (("paper r = 1.5e-4", 1.5e-4), (f"r = 30% quantile of |t_i| ({r30:.3e})", r30)):
                ms = timed(lambda: ctx.sand_query_dynamic(pts.data_ptr(), n, r, sdf.data_ptr(), dep.data_ptr()), steps)
                hist = np.bincount(dep.cpu().numpy(), minlength=c.spec.L + 1)[:c.spec.L + 1].tolist()
                entries.append({"mode": mode, "threshold": name, "r": r, "value": n / (ms / 1e3), "unit": UNIT,
                                "ms_per_step": ms, "exit_depth_hist": hist,
                                "mean_exit_depth": float(np.dot(np.arange(len(hist)), hist) / n)})
                print(f"[dynamic] {mode} {name}: {n / (ms / 1e3) / 1e9:.3f} G points/s ({ms:.1f} ms)", file=sys.stderr,
                      flush=True)
    cpu = None
    if not args.no_cpu:
        import oracle
        k = 20000
        t0 = time.perf_counter()
        oracle.query_dynamic(p, pts_np[:k], r30)
        dt = time.perf_counter() - t0
        cpu = {"value": k / dt, "unit": UNIT, "cores": _cores(), "kind": "oracle (numpy float64)",
               "cores_note": "BLAS pool for the matmuls; sin and the exit test on one core",
               "sample": f"first {k} grid points, r = {r30:.3e}"}
    line = {"task": "dynamic", "metric": "dynamic-exit (no octree) SDF queries/sec vs the octree path",
            "unit": UNIT, "n_gpus": 1, "steps": steps, "warmup": args.warmup, "higher_is_better": True,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"C2 512^3 grid ({n} points), 8x256 SIREN T-MLP (seeded init)"},
            "octree_path": {"value": n / (ms_oct / 1e3), "unit": UNIT, "ms_per_step": ms_oct,
                            "dtype": "bf16", "note": "sand_query with C2's level-7 octree, same points"},
            "octree_path_fp32": oct_same,
            "method_gap": {e["threshold"] + " / " + e["mode"]: e["ms_per_step"] / oct_same[
                "f16x3_tensor" if e["mode"] == "tensor" else "fp32_simt"]["ms_per_step"] for e in entries},
            "method_gap_note": "dynamic-exit time / octree-path time in the same arithmetic (SIMT schedules vs the FP32 "
                               "SIMT octree path, the tensor schedule vs the F16X3 octree path); the paper: 13.67 s / "
                               "0.378 s = 36x, P:761-762, on its trained nets where most of the grid is far field",
            "entries": entries, "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)
    return 0


def run_mesh(args):
    """marching cubes on C2's 512^3 grid (the paper's mesh extraction, P:415, P:423;
    triangulation rule DESIGN.md R24).  (a) fused: sand_mesh_grid -- the query path slab by slab (32
    planes of cubes) with each slab meshed as soon as its sdf exists, the 512^3 sdf never materialised;
    (b) unfused: sand_query over the whole grid, then sand_marching_cubes on the 537 MB sdf grid.  The MC
    kernel alone is timed in (b) (HBM-bound: 4 B of sdf per cube + 36 B per triangle).  Single GPU."""
    import torch
    import sandgen as g
    from paper_2604_25936_b200 import SAND_BF16, SandContext
    ws, rank, local = _dist()
    if rank != 0:
        return 0
    steps = min(args.steps, 5)
    c = g.make_config("C2")
    p = c.params()
    R = c.grid_R
    dev = torch.device("cuda", 0)
    n = R ** 3
    pk = _peaks()
    with SandContext(c.spec.L, c.spec.H, c.spec.omega0, SAND_BF16, c.spec.tail, 0) as ctx:
        ctx.sand_load_weights(g.pack_blob(p))
        ctx.sand_load_depthmap(c.depthmap)
        st = torch.cuda.current_stream(dev)
        ctx.sand_set_stream(st.cuda_stream)
        ntri = ctx.sand_mesh_grid(R, 0, 0, 0)
        tris = torch.empty(9 * ntri, dtype=torch.float32, device=dev)

        def timed(fn, k):
            for _ in range(min(args.warmup, 3)):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record(st)
            for _ in range(k):
                fn()
            e1.record(st)
            torch.cuda.synchronize(dev)
            return e0.elapsed_time(e1) / k

        ms_fused = timed(lambda: ctx.sand_mesh_grid(R, 0, tris.data_ptr(), ntri), steps)
        pts = torch.from_numpy(g.grid_points(R)).to(dev)
        sdf = torch.empty(n, dtype=torch.float32, device=dev)
        dep = torch.empty(n, dtype=torch.uint8, device=dev)
        ctx.sand_reserve(n)
        ms_query = timed(lambda: ctx.sand_query(pts.data_ptr(), n, sdf.data_ptr(), dep.data_ptr()), steps)
        ms_mc = timed(lambda: ctx.sand_marching_cubes(sdf.data_ptr(), R, tris.data_ptr(), ntri), steps)
        n2 = ctx.sand_marching_cubes(sdf.data_ptr(), R, tris.data_ptr(), ntri)
    mc_bytes = 4.0 * n + 36.0 * ntri
    line = {"task": "mesh", "metric": "marching-cubes mesh extraction of the 512^3 SDF grid (fused with the query path)",
            "value": n / (ms_fused / 1e3), "unit": UNIT, "n_gpus": 1, "steps": steps, "warmup": args.warmup,
            "ms_per_step": ms_fused, "higher_is_better": True, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"C2 {R}^3 grid, 8x256 SIREN T-MLP, level-7 octree, slabs of 64 cube planes"},
            "triangles": ntri, "triangles_unfused": n2,
            "unfused": {"ms_query": ms_query, "ms_marching_cubes": ms_mc, "ms_total": ms_query + ms_mc,
                        "sdf_grid_bytes": 4 * n},
            "roofline": {"bound": "hbm", "kernel": "k_mc_signs + k_mc_emit (unfused sand_marching_cubes call, host sync included)", "achieved": mc_bytes / (ms_mc / 1e3) / 1e9,
                         "peak": pk["hbm"], "unit": "GB/s", "frac": mc_bytes / (ms_mc / 1e3) / 1e9 / pk["hbm"],
                         "bytes_formula": "4 B sdf per grid vertex + 36 B per triangle", "traffic": None}}
    print(json.dumps(line), flush=True)
    return 0


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _relaunch(args):
    """`--gpus N` (N > 1) without a torchrun environment: re-exec this command under
    torch.distributed.run with one rank per GPU (rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] --gpus {args.gpus}: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def _grid_slab_device(R, k0, k1, Rz, dev):
    """Points of z-planes [k0, k1) of the R x R x Rz vertex grid, generated on the device from the same float32
    axis values as sandgen.grid_points_slab (x fastest): float32 [n][3]."""
    import torch
    import sandgen as g
    ax = torch.from_numpy(g.grid_axis(R)).to(dev)
    az = torch.from_numpy(g.grid_axis(Rz)[k0:k1].copy()).to(dev)
    nz = k1 - k0
    out = torch.empty((nz, R, R, 3), dtype=torch.float32, device=dev)
    out[..., 0] = ax.view(1, 1, R)
    out[..., 1] = ax.view(1, R, 1)
    out[..., 2] = az.view(nz, 1, 1)
    return out.view(-1, 3)


def _sample_grid_points(R, k0, k1, Rz, n, rng):
    """n seeded random vertices of z-planes [k0, k1) of the R x R x Rz grid (host, float32 [n][3])."""
    import sandgen as g
    tot = (k1 - k0) * R * R
    lin = np.sort(rng.choice(tot, min(n, tot), replace=False))
    ax, az = g.grid_axis(R), g.grid_axis(Rz)
    return np.stack([ax[lin % R], ax[(lin // R) % R], az[k0 + lin // (R * R)]], axis=1).astype(np.float32)


def run_query(args):
    """The BASELINE metric: sand_query over the configuration's points, one rank per GPU."""
    import torch
    import torch.distributed as dist

    import sandgen as g
    from paper_2604_25936_b200 import SAND_BF16, SAND_F16X3, SAND_FP32, SandContext, partition

    ws, rank, local = _dist()
    # one process per GPU; SAND_BENCH_SHARE_GPU=1 (test only) maps several ranks onto the visible GPUs
    # round-robin and uses gloo, to exercise the N > 1 path on a single-GPU box (the ranks' kernels are
    # independent: no kernel waits on another rank)
    share = os.environ.get("SAND_BENCH_SHARE_GPU") == "1"
    dev_index = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    comm = None
    if ws > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")            # NCCL logs its communicator (nranks) init
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                "collective": f"all_gather_into_tensor of {partition.RECORD_FIELDS} int64 per rank (after the timed region)"}
        if rank == 0:
            print(f"[bench] communicator: backend={comm['backend']} nranks={comm['nranks']}", file=sys.stderr, flush=True)

    c = g.make_config(args.config)
    p = c.params()
    dm = c.depthmap
    fp32 = args.prec == "fp32" or (args.prec is None and c.precision == SAND_FP32)
    x3 = args.prec == "f16x3"
    prec_code = SAND_F16X3 if x3 else SAND_FP32 if fp32 else SAND_BF16
    if args.full_depth:
        dm = g.VoxelMap(1, np.full(8, c.spec.L, np.uint8), None)
    weak = args.scaling == "weak"
    if c.grid_R is not None:
        k0, k1, Rz = partition.shard_planes(c.depthmap, c.grid_R, ws, rank, weak=weak)
        pts = _grid_slab_device(c.grid_R, k0, k1, Rz, dev)
        wl_desc = f"{args.config}: {c.grid_R}x{c.grid_R}x{Rz} grid, z-planes [{k0},{k1}) on rank {rank}"
        base_index = k0 * c.grid_R * c.grid_R
    else:
        pts_all = c.points_fn()
        n_all = pts_all.shape[0]
        if weak:   # every rank queries the whole cloud (global indices offset by rank)
            k0, k1, Rz = rank * n_all, (rank + 1) * n_all, None
            pts = torch.from_numpy(pts_all).to(dev)
        else:
            k0, k1, Rz = n_all * rank // ws, n_all * (rank + 1) // ws, None
            pts = torch.from_numpy(np.ascontiguousarray(pts_all[k0:k1])).to(dev)
        wl_desc = f"{args.config}: points [{k0},{k1})"
        base_index = k0
    n = pts.shape[0]
    sdf = torch.empty(n, dtype=torch.float32, device=dev)
    dep = torch.empty(n, dtype=torch.uint8, device=dev)

    ctx = SandContext(c.spec.L, c.spec.H, c.spec.omega0, prec_code, c.spec.tail, dev_index)
    if args.kprof:
        from paper_2604_25936_b200 import SAND_OPT_KPROF
        ctx.sand_set_option(SAND_OPT_KPROF, args.kprof)
    from paper_2604_25936_b200 import SAND_OPT_PAIR_KERNEL
    if args.pair_kernel is not None:
        ctx.sand_set_option(SAND_OPT_PAIR_KERNEL, args.pair_kernel)
    pair_mode = ctx.sand_get_option(SAND_OPT_PAIR_KERNEL)
    ctx.sand_load_weights(g.pack_blob(p))
    ctx.sand_load_depthmap(dm)
    ctx.sand_reserve(n)
    stream = torch.cuda.current_stream(dev)
    ctx.sand_set_stream(stream.cuda_stream)

    def query():
        ctx.sand_query(pts.data_ptr(), n, sdf.data_ptr(), dep.data_ptr())

    # inputs smaller than L2 (side configs such as C0, C3): flush L2 before every step by writing a buffer
    # larger than it, and time the steps one by one (the flush outside the events)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if 12 * n < 126e6 else None

    def timed(k):
        """k steps, CUDA events on the launching stream; returns device ms summed over the steps."""
        if flush is None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(k):
                query()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            return e0.elapsed_time(e1)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        for a_, b_ in evs:
            flush.fill_(1)
            a_.record(stream)
            query()
            b_.record(stream)
        torch.cuda.synchronize(dev)
        return sum(a_.elapsed_time(b_) for a_, b_ in evs)

    for _ in range(args.warmup):
        query()
    ctx.sand_get_stats()          # synchronises; resets the per-query event sums
    clk = ClockSampler(dev_index)
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    clk.start()
    ms_total = timed(args.steps)
    if ws > 1:
        dist.barrier()
    clocks = clk.stop()
    st = ctx.sand_get_stats()
    ms_mlp = st["ms_mlp_sum"] / max(st["queries"], 1)
    ms_lookup = st["ms_lookup_sum"] / max(st["queries"], 1)
    ms_bin = st["ms_bin_sum"] / max(st["queries"], 1)

    # order-independent per-rank checksums: fixed-point SDF sum and a position-weighted depth
    # hash over GLOBAL point indices, so the sum over ranks is identical for any N
    fin = torch.isfinite(sdf)
    sdf_fx = int(torch.round(torch.where(fin, sdf.double(), torch.zeros_like(sdf, dtype=torch.float64))
                             * float(1 << 24)).to(torch.int64).sum().item())
    gidx = torch.arange(n, device=dev, dtype=torch.int64) + int(base_index)
    dhash = int((dep.to(torch.int64) * (gidx % 8191 + 1)).sum().item())

    # the non-adaptive GPU baseline on the same points: an all-L depth map, same kernels (not in the timed region)
    ms_full = 0.0
    if not args.full_depth and not args.no_full_depth and not fp32 and not x3 and args.task == "query":
        ctx.sand_load_depthmap(g.VoxelMap(1, np.full(8, c.spec.L, np.uint8), None))
        k_fd = max(1, min(args.steps, 5))
        query()
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        ms_full = timed(k_fd) / k_fd * args.steps
        if ws > 1:
            dist.barrier()
        ctx.sand_load_depthmap(dm)
        ctx.sand_get_stats()

    rec = partition.make_record(n, st["per_depth"], ms_total, sdf_fx, dhash, k0, k1, st["queries"], ms_full)
    if ws > 1:
        cdev = torch.device("cpu") if share else dev   # gloo gathers host tensors
        t = torch.from_numpy(rec).to(cdev)
        allr = torch.empty(ws * t.numel(), dtype=t.dtype, device=cdev)
        dist.all_gather_into_tensor(allr, t)
        summ = partition.summarize(allr.cpu().numpy())
    else:
        summ = partition.summarize(rec)

    # end-to-end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        hp = pts.cpu().pin_memory()
        hs = torch.empty(n, dtype=torch.float32).pin_memory()
        hd = torch.empty(n, dtype=torch.uint8).pin_memory()
        ctx.sand_query_host(hp.data_ptr(), n, hs.data_ptr(), hd.data_ptr(), args.e2e_chunk)  # warm
        ts = []
        for _ in range(args.e2e_steps):
            if ws > 1:
                dist.barrier()
            t0 = time.perf_counter()
            ctx.sand_query_host(hp.data_ptr(), n, hs.data_ptr(), hd.data_ptr(), args.e2e_chunk)
            ts.append(time.perf_counter() - t0)
        t_e2e = float(np.mean(ts))
        if ws > 1:
            tt = torch.tensor([t_e2e], dtype=torch.float64, device="cpu" if share else dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_e2e = float(tt.item())
        e2e = {"value": summ["n_total"] / t_e2e, "unit": UNIT, "h2d_bytes_per_step": 12 * summ["n_total"],
               "d2h_bytes_per_step": 5 * summ["n_total"],
               "chunk_points": args.e2e_chunk or min(max(n // 8, 1 << 21), 1 << 23), "steps": args.e2e_steps,
               "timing": "host wall clock around the synchronous sand_query_host, max over ranks"}
        del hp, hs, hd
        ctx.sand_get_stats()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        rng = np.random.default_rng(99)
        if c.grid_R is not None:
            sampler = lambda m: _sample_grid_points(c.grid_R, k0, k1, Rz, m, rng)
        else:
            host = pts.cpu().numpy()
            sampler = lambda m: host[np.sort(rng.choice(n, min(m, n), replace=False))]
        cpu = cpu_baseline(p, c.depthmap, sampler, args.cpu_seconds)

    if rank == 0:
        pk = _peaks()
        ms_step = summ["ms_max"] / args.steps
        value = summ["n_total"] / (ms_step / 1e3)
        H = c.spec.H
        per_depth = summ["per_depth"]
        f_exec = sum(per_depth[d] * (d - 1) * 2.0 * H * H for d in range(1, c.spec.L + 1))
        f_ns = sum(per_depth[d] * d * 2.0 * H * H for d in range(1, c.spec.L + 1))
        f_exec_rank0 = st["flops_exec"]
        ach = f_exec_rank0 / (ms_mlp / 1e3) / 1e12
        if fp32:   # the FP32 path: roofline against the FP32 FMA pipe (148 SM x 128 lanes x 2 FLOP x clock)
            sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
            pk = dict(pk, bf16=148 * 128 * 2 * sm_mhz * 1e6 / 1e12, bf16_sus=148 * 128 * 2 * sm_mhz * 1e6 / 1e12,
                      src="derived FP32 ALU (148 SM x 128 lanes x 2 FLOP x median clock);")
        if x3:   # executed tensor work: 3 products of split FP16 operands per H x H layer (+ the split-bias MMA)
            f_exec_rank0 = st["flops_exec"] * 3.0 + sum(st["per_depth"][d] * (d - 1) * 2.0 * 16 * H
                                                         for d in range(2, c.spec.L + 1))
            ach = f_exec_rank0 / (ms_mlp / 1e3) / 1e12
        kname = ("k_tmlp_x3 (split-FP16 x3, CTA pair)" if x3 else
                 "k_query_simt (FP32, one thread per point)" if fp32 and H <= 64 else
                 "k_query_fp32 (FP32 register-blocked GEMM)" if fp32 else
                 "k_tmlp_wide (K3 fused T-MLP, CTA pair, N-halves)" if H == 336 else
                 "k_tmlp_tc4 (K3 fused T-MLP, CTA pair, one epilogue team per slot)" if pair_mode == 2 else
                 "k_tmlp_tc2 (K3 fused T-MLP, CTA pair, two N-half passes)" if pair_mode == 1 else
                 "k_tmlp_tc (K3 fused T-MLP, 1 CTA)")
        full = None
        if summ["ms_full_max"] > 0:
            ms_fd = summ["ms_full_max"] / args.steps
            full = {"value": summ["n_total"] / (ms_fd / 1e3), "unit": UNIT, "ms_per_step": ms_fd,
                    "speedup": ms_fd / ms_step,
                    "how": "same points and kernels, all-L depth map (every point at depth L), max over ranks"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if weak else "strong",
            "vs_baseline": None, "dtype": "f16x3" if x3 else "f32" if fp32 else "bf16", "data": "synthetic",
            "config": _arm_config(args, c, ws, wl_desc, summ["n_total"]),
            "roofline": {"bound": "alu" if fp32 else "tensor", "kernel": kname, "achieved": ach,
                         "peak": pk["bf16"], "unit": "TFLOP/s", "frac": ach / pk["bf16"],
                         "peak_source": pk["src"] + ("" if fp32 else " bf16_tflops (burst)"),
                         "frac_vs_sustained": ach / pk["bf16_sus"],
                         "traffic": _traffic() if (args.config == "C2" and not fp32) else None,
                         "algorithmic_flops_per_launch": f_exec_rank0,
                         "flops_formula": ("executed tensor FLOPs: 3 x sum_p (d_p - 1) 2 H^2 + split-bias MMAs" if x3 else
                                           "executed H x H FLOPs sum_p (d_p - 1) * 2 H^2 (Eq. 2 reading R3)"),
                         "ms_per_launch": ms_mlp,
                         "traffic_source": TRAFFIC_SRC if (args.config == "C2" and not fp32) else None},
            # the other pipe the step needs: one sine per hidden unit per evaluated layer (Eq. 2), MUFU.SIN
            "sine_roofline": None if fp32 else _sine_roofline(st["per_depth"], H, ms_mlp, clocks),
            "tensor_frac_step": f_exec / (ms_step / 1e3) / 1e12 / pk["bf16"],
            "tensor_frac_ns_formula": f_ns / (ms_step / 1e3) / 1e12 / pk["bf16"],
            "flops_exec_per_step": f_exec, "flops_ns_per_step": f_ns,
            "padding_waste": _padding_waste(st["per_depth"], H, fp32, even_bins=pair_mode == 2 and not fp32 and not x3
                                            and H in (64, 128, 256)),
            "stage_ms": {"lookup": ms_lookup, "bin": ms_bin, "mlp": ms_mlp},
            "per_depth": per_depth,
            "full_depth_speedup": full,
            "checksums": {"sdf_fixed_point_2^24": summ["sdf_fx"], "depth_hash": summ["depth_hash"],
                          "note": "int64 sums over all ranks: identical for any number of GPUs"},
            "shards": summ["ranges"], "comm": comm,
            "e2e": e2e, "cpu_baseline": cpu,
            "gpu_launches": 6 * args.steps * ws,   # lookup, scan x3, scatter, T-MLP per query
            "clocks": clocks,
            "hbm_lookup_gbs": (13.0 * n) / (ms_lookup / 1e3) / 1e9 if ms_lookup > 0 else None,
            # binning (K2a scans + K2b scatter): 1 B depth read + 4 B perm written per binned point, rank 0's shard
            "hbm_bin_gbs": (5.0 * sum(st["per_depth"][1:])) / (ms_bin / 1e3) / 1e9 if ms_bin > 0 else None,
            "hbm_peak_gbs": pk["hbm"],
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sand", choices=["sand", "reference"])
    ap.add_argument("--config", default=None, choices=["C0", "C1", "C2", "C3", "C4"],
                    help="BASELINE.json configs[i]; default C2 on 1 GPU (the metric's config), C4 on N > 1")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's fixed grid cut into work-balanced z-slabs; weak: the grid refined "
                         "along z to R x R x RN so every rank holds ~R^3 points")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunk", type=int, default=0, help="points per host-pipeline chunk (0: library default)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-full-depth", action="store_true", help="skip the all-L (non-adaptive) comparison run")
    ap.add_argument("--ref-sample", type=int, default=1 << 15)
    ap.add_argument("--full-depth", action="store_true", help="all-L depth map (non-adaptive GPU baseline)")
    ap.add_argument("--pair-kernel", type=int, default=None, choices=[0, 1, 2],
                    help="SAND_OPT_PAIR_KERNEL (default: the library's choice, 2 = slot-team CTA-pair kernel)")
    ap.add_argument("--kprof", type=int, default=0, help="diagnostic SAND_OPT_KPROF (per-role counters, stderr)")
    ap.add_argument("--prec", default=None, choices=["bf16", "fp32", "f16x3"],
                    help="default: the config's precision (C0 FP32, others BF16); fp32: the accurate FP32 path "
                         "(SIMT), reported against the FP32 ALU peak")
    ap.add_argument("--task", default="query", choices=["query", "populate", "sweep", "dynamic", "mesh"],
                    help="query: the adaptive SDF query path (BASELINE metric); populate: depth-map "
                         "population (Eq. 5/6, SURVEY 8(f) NEXT #1) on the config's finest octree leaves")
    args = ap.parse_args()
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        _relaunch(args)
    if ws_env is not None and int(ws_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env} (launch one rank per GPU)")
    if args.config is None:
        args.config = "C2" if args.gpus == 1 or args.task != "query" else "C4"
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        return run_reference(args)
    if args.task == "populate":
        return run_populate(args)
    if args.task == "sweep":
        return run_sweep(args)
    if args.task == "dynamic":
        return run_dynamic(args)
    if args.task == "mesh":
        return run_mesh(args)
    return run_query(args)


if __name__ == "__main__":
    sys.exit(main())
