"""Benchmark of the B200 BA hot path (BASELINE.json metric: LM iterations/s and
time-to-converge on BAL-shaped BA; obs/s of the fused residual+Jacobian).

Headline workload: synthetic Final-13682-shaped BA (BASELINE.json configs[4],
the north star's "Target": 13,682 cameras, 4,456,117 points, 28,987,644
observations), the largest configuration that fits one GPU. One "step" = one
complete LM solve (optimize, lm.hpp:205-255) from the same initial parameters
with the reference CLI's settings: LmConfig defaults, max_iterations = 50
(cli.hpp:25), the reference's default solver (SolverChoice::cholesky,
lm.hpp:34) -- on the GPU the tile-sparse Cholesky of the reduced camera
system (csrc/chol.cu). value = LM iterations per second over the K timed
solves (device time, CUDA events on the solver stream, max over ranks);
time_to_converge_s = mean device time per solve. The scene is the host
generator's (seed = camera count), the one the parity tests
check against the oracle (tests/test_gpu_parity_configs.py).

Secondary lines (``configs``): every other BASELINE.json config with the
same protocol, the north-star implicit-Schur PCG path (``pcg``: a full
Trafalgar solve, per-iteration time and HBM fraction at Venice / Final), and
per-kernel rooflines (``kernels``).

With --gpus N > 1 (torchrun, one process per GPU) the problem is sharded by
landmark over the N GPUs (NCCL allreduce of the camera-sized
sums): scaling is strong, value = LM iterations of the one joint solve / the
max over ranks of the device time. --emulate runs the same N-rank code path
on one GPU (an in-process rank group, one host thread per rank).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config NAME] [--emulate]

--impl reference times the reference's CPU algorithm -- the oracle port of
traceopt (oracle/; the reference needs Eigen and cannot be built here,
DESIGN.md) -- on this host's cores. It imports and loads nothing of the
product: its scene comes from the oracle's own generator restatement. Each
step is a bounded sample of the headline workload (see _cpu_slice_sample);
the BASELINE.md section 2 CPU runs (full solves at Ladybug-49 with PCG and
Cholesky, Trafalgar-257 and Dubrovnik-356 with Cholesky) are reported once
under "full_solves".
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASE_CFG = "final-13682"
CONFIGS = {  # name -> (cameras, points, observations), BASELINE.json
    "ladybug-49": (49, 7776, 31843),
    "trafalgar-257": (257, 65132, 225911),
    "dubrovnik-356": (356, 226730, 1255268),
    "venice-1778": (1778, 993923, 5001946),
    "final-13682": (13682, 4456117, 28987644),
}
# CPU sample of the large configs: a camera window of C / SLICE_DIV cameras
SLICE_DIV = 64
CPU_MODEL = None


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "10"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.005)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.03)  # the sample that covers the end of the region
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist_init():
    rank, world = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1)
    if world > 1:
        # NCCL's INIT lines (communicator size, ranks, NVLink/NVLS paths) on
        # stderr, so a multi-GPU run's log shows the ranks that took part
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        dist.init_process_group("gloo")
        return rank, world, dist
    return 0, 1, None


def _max_over_ranks(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------
# CPU side: the oracle port of the reference (test infrastructure; only this
# file's CPU legs run it, and only as the baseline).
# --------------------------------------------------------------------------
def _oracle():
    from oracle import oracle as O
    O.set_threads(os.cpu_count() or 1)
    return O


def _cpu_slice_sample(O, scene, name):
    """One bounded CPU sample of the headline workload, scaled to LM iter/s of
    the full scene. Venice / Final: the reference algorithm (LmConfig
    defaults, Cholesky) on a camera window of max(C / SLICE_DIV, 256) ring cameras and
    every point seen only by them (oracle.camera_window_slice: same density,
    track lengths and band structure); the sample is optimize() with
    max_iterations = 2 and its second iteration is the timed one (the first
    carries the one-time symbolic phase, NormalEquations::initialize +
    cholesky_symbolic, which a full solve amortises); LM iter/s of the full
    scene = (N_slice / N) / t_iteration. Smaller configs: the whole scene,
    same rule (the second iteration)."""
    C, P, N = CONFIGS[name]
    sub = scene
    cams = min(C, max(C // SLICE_DIV, 256))  # >= 256 ring cameras: edge effects of the window stay small
    if N > 2_000_000:
        sub = O.camera_window_slice(scene, cams)
    ns = len(sub["cam_idx"])
    prob = O.Problem(sub["poses"], sub["points"], sub["intrinsics"], sub["cam_idx"], sub["pt_idx"], sub["pixels"])
    rep = prob.optimize(O.LmConfig(max_iterations=2))
    ct = [r["cum_time_s"] for r in rep["trajectory"]]
    t_it = ct[2] - ct[1]
    del prob
    desc = (f"reference algorithm (oracle port, LmConfig defaults / Cholesky, {os.cpu_count()} threads) on "
            + (f"a camera-window slice of {name} ({cams} of {C} cameras, {len(sub['points'])} points, "
               f"{ns} observations = {ns / N:.4f} N)" if sub is not scene else f"the whole {name} scene")
            + f": the steady-state LM iteration ({t_it:.2f} s; the first, with the symbolic phase, "
              f"{ct[1] - ct[0]:.2f} s), scaled by N_sample / N")
    return (ns / N) / t_it, t_it, ns, desc


def _cpu_full_solve(O, scene, solver, max_iterations=50, pcg_budget=0):
    """A full reference solve (LmConfig defaults, max_iterations = 50 as the
    reference CLI, cli.hpp:25): wall clock around optimize, as SPEC.md:670."""
    prob = O.Problem(scene["poses"], scene["points"], scene["intrinsics"], scene["cam_idx"], scene["pt_idx"],
                     scene["pixels"])
    cfg = O.LmConfig(max_iterations=max_iterations, solver=solver, pcg_max_iters=pcg_budget)
    t0 = time.perf_counter()
    rep = prob.optimize(cfg)
    el = time.perf_counter() - t0
    del prob
    return dict(time_to_converge_s=el, lm_iterations=rep["iterations"], lm_iters_per_s=rep["iterations"] / el,
                termination=["plateau", "max_iters", "solver_failure"][rep["reason"]], final_mse=rep["final_mse"],
                pcg_iterations=sum(r["pcg_iters"] for r in rep["trajectory"]),
                solver="pcg" if solver == 1 else "cholesky")


def run_reference(args):
    rank, world, dist = _dist_init()
    if rank != 0:
        return
    O = _oracle()
    C, P, N = CONFIGS[args.config]
    scene = O.synth_bal_shaped(C, P, N, seed=C)
    vals, samples = [], []
    for i in range(args.warmup + args.steps):
        v, t_it, ns, desc = _cpu_slice_sample(O, scene, args.config)
        if i >= args.warmup:
            vals.append(v)
            samples.append(t_it)
    value = statistics.mean(vals)
    full = {}
    if not args.no_extra:
        # the CPU runs of the smaller configs, each once
        for name, solver in (("ladybug-49", 0), ("ladybug-49", 1), ("trafalgar-257", 0), ("dubrovnik-356", 0)):
            c2, p2, n2 = CONFIGS[name]
            sc = scene if name == args.config else O.synth_bal_shaped(c2, p2, n2, seed=c2)
            full[f"{name}/{'pcg' if solver else 'cholesky'}"] = _cpu_full_solve(O, sc, solver)
    threads = os.cpu_count() or 1
    line = {"impl": "reference", "metric": "lm_iters_per_s", "value": value, "unit": "LM iter/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic BAL-shaped (SURVEY.md 8d generator restated in the oracle, seed = camera count)",
            "config": {"workload": f"{args.config} BA (C={C}, P={P}, N={N}), LmConfig defaults (Cholesky), "
                                   f"max_iterations=50"},
            "cpu_baseline": {"value": value, "unit": "LM iter/s", "cores": threads, "kind": "port",
                             "cpu_model": _cpu_model(), "sample": desc,
                             "sample_iteration_s": {"mean": statistics.mean(samples), "min": min(samples)}},
            "full_solves": full,
            "e2e": {"value": value, "unit": "LM iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# --------------------------------------------------------------------------
# GPU side
# --------------------------------------------------------------------------
# FP64 peak measured on this pool's B200 by tools/lat/dmma.cu
# (profiles/r01b_fp64_peak.txt): 63.8 FMA/clk/SM (DMMA m8n8k4 f64) x 148 SMs x
# 1.965 GHz x 2 = 37.1 TFLOP/s; plain DFMA 58.5 FMA/clk/SM = 34.0 TFLOP/s.
# MEASURED_PEAKS.json carries no FP64 number; NVIDIA's nominal figure is 40.
FP64_DFMA_PEAK_TFLOPS = 34.0
FP64_PEAK_SOURCE = "measured DFMA issue peak (tools/lat/dmma.cu, profiles/r01b_fp64_peak.txt; DMMA 37.1, nominal 40)"


def _alg_bytes(kernel, st, ds=None):
    """Algorithmic HBM bytes per launch: every array element the kernel's
    function needs, read or written once (FP64 values, int32 indices; DESIGN.md
    section 4). N observations, P points, C cameras, E tile-camera entries, T
    tiles."""
    N, P, C, T, E = st["observations"], st["points"], st["cameras"], st["tiles"], st["entries"]
    if kernel == "linearize":  # obs idx+px 22, points 24 + H_pp/g_p 72, entry partials 216 w + 216 r, cameras
        return 22 * N + 96 * P + 432 * E + 368 * C + 16 * T
    if kernel == "schur_tiles":  # blob 6/obs, points 24 + H~pp^-1 48, camera record+direction 176 + partial 48
        return 6 * N + 72 * P + 224 * E + 32 * T
    if kernel == "prep_direct":  # obs index 6, V record [Q | y] 96 written; points + H_pp/g_p 96, H~pp^-1 48 w; entry RHS 48 w
        return 102 * N + 144 * P + 48 * E + 128 * C
    if kernel == "lin_prep":  # linearize + V record 96 w, H~pp^-1 48 w, entry RHS 48 w + 48 r, H~cc 168 + rhs 48 w
        return 118 * N + 144 * P + 528 * E + 584 * C + 16 * T
    if kernel == "schur_dense":  # every V record read once (96 B / obs), the pair list (8 B / pair), tiles written
        return 96 * N + 8 * ds["pairs"] + 48 * 48 * 8 * ds["tiles"]
    raise ValueError(kernel)


def _minimal_bytes(kernel, st):
    """SURVEY.md 8(d) minimal traffic of the function (inputs read once, the
    outputs the next phase needs written once; no design intermediates):
    linearisation + prep = observation index/pixels 24 N + points 24 P +
    cameras 80 C in, H_pp/g_p/H~pp^-1 (120 P) + camera blocks (216 C) out;
    PCG S*p = 280 N + 48 P + 800 C (the survey's K5 figure)."""
    N, P, C = st["observations"], st["points"], st["cameras"]
    if kernel in ("linearize", "lin_prep"):
        return 24 * N + 24 * P + 80 * C + 120 * P + 216 * C
    if kernel == "schur_tiles":  # the survey's K5 figure assumes a stored J (reads 144 B / obs per pass); the
        return 280 * N + 48 * P + 800 * C  # matrix-free tile pass recomputes J instead, so it can exceed 1
    return None


def _chol_flops(ds):
    """FP64 flops of one tile Cholesky factorisation (48 x 48 tiles): tile
    updates and triangular solves (2 * 48^3 each) + per column factor and
    inverse (~2 * 48^3 / 3)."""
    g = 2 * 48 ** 3
    return ds["tile_updates"] * g + (ds["tiles"] - ds["tile_columns"]) * g + ds["tile_columns"] * (g // 3)


def run_b200(args):
    import torch
    rank, world, dist = _dist_init()
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    import paper_2409_12190_b200 as bae
    from paper_2409_12190_b200.api import LmConfig, SolverChoice

    emulate = args.emulate and world == 1 and args.gpus > 1
    ranks = args.gpus if emulate else 1  # in-process ranks driven by this process
    peak_hbm, peak_src = _peaks()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def comm_kw():
        if world > 1:
            obj = [bae.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            return [dict(rank=rank, world=world, nccl_id=obj[0])]
        if emulate:
            g = bae.RankGroup(ranks)
            return [dict(rank=r, world=ranks, group=g) for r in range(ranks)]
        return [{}]

    def on_ranks(fn):
        """fn(r) for each in-process rank (threads when emulating)."""
        if ranks == 1:
            return [fn(0)]
        out, err = [None] * ranks, [None] * ranks

        def body(r):
            try:
                out[r] = fn(r)
            except BaseException as e:  # noqa: BLE001 - re-raised below
                err[r] = e
        ts = [threading.Thread(target=body, args=(r,)) for r in range(ranks)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out

    def make(scene):
        kws = comm_kw()
        return on_ranks(lambda r: bae.make_ba_problem(scene.poses, scene.points, scene.intrinsics,
                                                      scene.observations, device=local, **kws[r]))

    def one_solve(probs, scene, cfg):
        for p in probs:  # untimed: inputs resident before the timed solve
            p.set_parameters(scene.poses, scene.points)
        flush.zero_()  # L2 flush between timed steps (L2 = 126 MB; 256 MB written)
        torch.cuda.synchronize()
        return on_ranks(lambda r: bae.optimize(probs[r], None, None, cfg))

    def series(probs, scene, cfg, steps, warmup):
        for _ in range(warmup):
            one_solve(probs, scene, cfg)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = sum(p.launch_count() for p in probs)
        for p in probs:
            p.phase_times(reset=True)
        dev, its, inner, reps = 0.0, 0, 0, []
        for _ in range(steps):
            rs = one_solve(probs, scene, cfg)
            reps.append(rs[0])
            dev += max(r.device_seconds for r in rs)
            its += rs[0].iterations
            inner += rs[0].total_pcg_iters
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ph = probs[0].phase_times(reset=True)
        launches = sum(p.launch_count() for p in probs) - l0
        dev_max = _max_over_ranks(dist, dev)
        if not ph.get("factor") and not ph.get("pcg") and ranks == 1:
            # the LM iterations ran as captured graphs (no per-phase events):
            # one untimed solve with plain launches for the phase breakdown
            os.environ["BAE_LM_GRAPH"] = "0"
            try:
                one_solve(probs, scene, cfg)
                torch.cuda.synchronize()
                ph = {k: v * steps for k, v in probs[0].phase_times(reset=True).items()}
            finally:
                del os.environ["BAE_LM_GRAPH"]
        return dict(value=its / dev_max, dev_max=dev_max, iterations=its, inner=inner, reports=reps,
                    phases={k: v / steps for k, v in ph.items()}, launches=launches)

    def kernel_line(name, ms, nbytes, minimal=None, launches_per_solve=None):
        gbs = nbytes / (ms * 1e-3) / 1e9
        d = {"kernel": name, "us": 1e3 * ms, "bound": "hbm", "algorithmic_bytes": nbytes, "achieved": gbs,
             "unit": "GB/s", "peak": peak_hbm, "frac": gbs / peak_hbm}
        if minimal:
            d.update(minimal_bytes=minimal, frac_minimal=minimal / (ms * 1e-3) / 1e9 / peak_hbm)
        if launches_per_solve is not None:
            d["launches_per_solve"] = launches_per_solve
        return d

    def tk(prs, kind, reps):
        """time_kernel on every rank (the sharded kernels exchange sums), max."""
        return _max_over_ranks(dist, max(on_ranks(lambda r: prs[r].time_kernel(kind, reps))))

    def direct_kernels(prs, st, ds):
        """Per-kernel device time (CUDA events on the solver stream around
        back-to-back launches) and HBM fraction of the direct path."""
        ms_l, ms_p, ms_s = tk(prs, 0, 5), tk(prs, 5, 5), tk(prs, 6, 5)
        ms_lp = tk(prs, 7, 5) if world == 1 and ranks == 1 else None
        ms_c = tk(prs, 4, 10)
        out = [kernel_line("k_linearize + k_cam_linearize (residual + J + J^T J / J^T r blocks)", ms_l,
                           _alg_bytes("linearize", st), _minimal_bytes("linearize", st)),
               kernel_line("k_prep<direct> + k_cam_prep (damping, H~pp^-1, V = W L^-T, Schur RHS)", ms_p,
                           _alg_bytes("prep_direct", st)),
               kernel_line("k_schur_dense (reduced camera matrix S into its tiles)", ms_s,
                           _alg_bytes("schur_dense", st, ds))]
        if ms_lp:
            out.append(kernel_line("k_lin_prep + k_cam_lin_prep (fused linearise + prep, after an accepted step)",
                                   ms_lp, _alg_bytes("lin_prep", st), _minimal_bytes("lin_prep", st)))
        f = _chol_flops(ds)
        out.append({"kernel": "k_tile_chol_factor + k_tile_chol_backward (factor + both substitutions)",
                    "us": 1e3 * ms_c, "bound": "fp64 / dependency chain", "algorithmic_flops": f,
                    "achieved": f / (ms_c * 1e-3) / 1e12, "unit": "TFLOP/s", "peak": FP64_DFMA_PEAK_TFLOPS,
                    "peak_source": FP64_PEAK_SOURCE, "frac": f / (ms_c * 1e-3) / 1e12 / FP64_DFMA_PEAK_TFLOPS})
        return out, dict(linearize=ms_l, prep=ms_p, schur=ms_s, lin_prep=ms_lp, chol=ms_c)

    def pcg_kernels(prs, st):
        ms_sx, ms_it = tk(prs, 1, 30), tk(prs, 2, 30)
        return {"pcg_iteration_us": 1e3 * ms_it,
                "k_schur_tiles": kernel_line("k_schur_tiles (implicit Schur S*p tile pass)", ms_sx,
                                             _alg_bytes("schur_tiles", st), _minimal_bytes("schur_tiles", st)),
                "pcg_iteration_frac_minimal": _minimal_bytes("schur_tiles", st) / (ms_it * 1e-3) / 1e9 / peak_hbm}

    cfg = LmConfig(max_iterations=50)  # reference defaults: solver = cholesky (tile-sparse Cholesky)
    C, P, N = CONFIGS[args.config]
    tg = time.perf_counter()
    scene = bae.synthetic.bal_shaped(C, P, N, seed=C)
    t_gen = time.perf_counter() - tg
    t0 = time.perf_counter()
    probs = make(scene)
    t_create = _max_over_ranks(dist, time.perf_counter() - t0)
    pr = probs[0]
    stats = pr.stats()

    with ClockSampler(local) as clk:
        head = series(probs, scene, cfg, args.steps, args.warmup)
    clocks = clk.summary()
    last = head["reports"][-1]
    ds = pr.direct_stats()
    solve_ms = 1e3 * head["dev_max"] / args.steps

    kernels, kms = direct_kernels(probs, stats, ds)
    pcg_head = pcg_kernels(probs, stats)
    # roofline: the kernel with the largest share of the solve (phase times of
    # the plain-launch breakdown): the fused linearise + prep at Final
    ph = head["phases"]
    lp = next((k for k in kernels if k["kernel"].startswith("k_lin_prep")), kernels[0])
    roofline = {"bound": "hbm", "kernel": lp["kernel"], "achieved": lp["achieved"], "peak": peak_hbm,
                "unit": "GB/s", "frac": lp["frac"], "peak_source": peak_src,
                "algorithmic_bytes_per_launch": lp["algorithmic_bytes"],
                "frac_on_survey_minimal_bytes": lp.get("frac_minimal"),
                "traffic": None, "timing": "CUDA events on the solver stream, back-to-back launches after the "
                                           "timed region (time_kernel)",
                "phase_ms_per_solve": ph}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            roofline["traffic"] = json.load(open(tpath)).get(args.config, {}).get("k_lin_prep")
        except Exception:
            pass

    # --- end to end through the public API with host buffers: make_ba_problem
    # (planning, uploads) + optimize + read-back of the final parameters ---
    e2e_iters, e2e_s = 0, 0.0
    e2e_steps_s = []
    e2e_steps = max(1, min(args.steps, 5))  # host-side hiccups (page-fault stalls) dilute over five steps
    e2e_warm = 2  # untimed: host allocations, the chunk cache and the pinned staging settle
    for i in range(e2e_steps + e2e_warm):
        kws = comm_kw()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ts = time.perf_counter()

        def e2e(r):
            p2 = bae.make_ba_problem(scene.poses, scene.points, scene.intrinsics, scene.observations, device=local,
                                     **kws[r])
            return bae.optimize(p2, scene.poses, scene.points, cfg, final_state={})
        r2 = on_ranks(e2e)[0]
        torch.cuda.synchronize()
        el = time.perf_counter() - ts
        e2e_steps_s.append(el)
        if i >= e2e_warm:
            e2e_iters += r2.iterations
            e2e_s += el
    e2e_value = e2e_iters / _max_over_ranks(dist, e2e_s)
    w_iters, w_s = 0, 0.0  # warm: optimize(init params from host) + read-back on the existing problem
    for i in range(e2e_steps + 1):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ts = time.perf_counter()
        r3 = on_ranks(lambda r: bae.optimize(probs[r], scene.poses, scene.points, cfg, final_state={}))[0]
        torch.cuda.synchronize()
        el = time.perf_counter() - ts
        if i > 0:
            w_iters += r3.iterations
            w_s += el
    e2e_warm = w_iters / _max_over_ranks(dist, w_s)
    h2d = 56 * C + 24 * P + 24 * C + 24 * N + 56 * C + 24 * P  # create inputs + optimize's initial parameters
    d2h = 56 * C + 24 * P

    # --- the other BASELINE.json configs, the same protocol ---
    extra = {}
    if not args.no_extra:
        for name in CONFIGS:
            if name == args.config:
                continue
            c2, p2_, n2 = CONFIGS[name]
            sc = bae.synthetic.bal_shaped(c2, p2_, n2, seed=c2)
            ts = time.perf_counter()
            prs = make(sc)
            t_c = _max_over_ranks(dist, time.perf_counter() - ts)
            ser = series(prs, sc, cfg, 3, 1)
            r = ser["reports"][-1]
            st2, ds2 = prs[0].stats(), prs[0].direct_stats()
            k2, _ = direct_kernels(prs, st2, ds2)
            extra[name] = {
                "workload": f"{name} BA (C={c2}, P={p2_}, N={n2}), LmConfig defaults (direct solve)",
                "lm_iters_per_s": ser["value"], "time_to_converge_s": ser["dev_max"] / 3,
                "lm_iterations": r.iterations, "termination": r.reason.name, "final_mse": r.final_mse,
                "ms_per_lm_iteration": 1e3 * ser["dev_max"] / max(1, ser["iterations"]),
                "phase_ms_per_solve": ser["phases"], "create_s": t_c, "direct": ds2, "kernels": k2}
            if name in ("trafalgar-257",) and ranks == 1:
                # the north-star implicit-Schur PCG path: a full solve at the reference tolerance
                pser = series(prs, sc, LmConfig(max_iterations=50, solver=SolverChoice.pcg), 2, 1)
                extra[name]["pcg"] = {
                    "lm_iters_per_s": pser["value"], "time_to_converge_s": pser["dev_max"] / 2,
                    "pcg_iterations_per_solve": pser["inner"] / 2, "phase_ms_per_solve": pser["phases"],
                    "config": "solver=pcg (implicit-Schur PCG, block-Jacobi), pcg_tol=1e-8", **pcg_kernels(prs, st2)}
            if name == "venice-1778":
                extra[name]["pcg"] = pcg_kernels(prs, st2)
            del prs

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            O = _oracle()
            sc = dict(poses=scene.poses, points=scene.points, intrinsics=scene.intrinsics, cam_idx=scene.cam_idx,
                      pt_idx=scene.pt_idx, pixels=scene.pixels)
            v, t_it, ns, desc = _cpu_slice_sample(O, sc, args.config)
            cpu = {"value": v, "unit": "LM iter/s", "cores": os.cpu_count() or 1, "kind": "port",
                   "cpu_model": _cpu_model(), "sample": desc}
        line = {
            "metric": "lm_iters_per_s", "value": head["value"], "unit": "LM iter/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": solve_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic BAL-shaped (SURVEY.md 8d host generator, seed = camera count)",
            "config": {"workload": f"{args.config} BA (C={C}, P={P}, N={N}), LM with LmConfig defaults "
                                   f"(solver=cholesky: tile-sparse Cholesky of the reduced camera system, "
                                   f"max_iterations=50) from the same initial state each step",
                       "parallelism": (f"landmark-sharded over {args.gpus} ranks (camera-vector sums)"
                                       + (" emulated on one GPU (in-process rank group)" if emulate else "")
                                       if args.gpus > 1 else "single GPU"),
                       "l2": "flushed (256 MB write) between steps; inputs also exceed L2",
                       "tiles": stats["tiles"], "tile_camera_entries": stats["entries"], "direct": ds},
            "time_to_converge_s": head["dev_max"] / args.steps,
            "lm_iterations_per_solve": last.iterations, "final_mse": last.final_mse,
            "termination": last.reason.name, "ms_per_lm_iteration": 1e3 * head["dev_max"] / head["iterations"],
            "generate_s": t_gen, "create_s": t_create,
            "obs_per_s_residual_jacobian": N / (kms["linearize"] * 1e-3),
            "phase_ms_per_solve": head["phases"],
            "roofline": roofline,
            "kernels": kernels,
            "pcg": pcg_head,
            "configs": extra,
            "e2e": {"value": e2e_value, "unit": "LM iter/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "includes": "make_ba_problem (planning, uploads) + optimize + parameter read-back, every step",
                    "step_s": e2e_steps_s,
                    "warm": {"value": e2e_warm, "unit": "LM iter/s", "h2d_bytes_per_step": 56 * C + 24 * P,
                             "d2h_bytes_per_step": d2h,
                             "includes": "optimize(initial parameters from host) + read-back, existing problem"}},
            "gpu_launches": head["launches"],
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        if emulate:
            line["emulated_ranks"] = ranks
        print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=BASE_CFG, choices=sorted(CONFIGS))
    ap.add_argument("--emulate", action="store_true", help="--gpus N ranks as an in-process group on one GPU")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="headline config only")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
