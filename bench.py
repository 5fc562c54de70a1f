"""Benchmark of the B200 BA hot path (BASELINE.json metric: LM iterations/s and
time-to-converge on BAL-shaped BA; obs/s of the fused residual+Jacobian).

One "step" = one complete LM solve (optimize, lm.hpp:205-255) of the
synthetic Trafalgar-257-shaped problem (BASELINE.json configs[1]) from the
same initial parameters, with the reference CLI's settings (LmConfig
defaults, max_iterations = 50, cli.hpp:25) and the reference's default
solver (SolverChoice::cholesky, lm.hpp:34): on the GPU that is the dense
reduced-camera-system direct solve. value = LM iterations per second over
the K timed solves (device time, CUDA events on the solver stream), max over
ranks; time_to_converge_s = mean device time per solve. The direct solve is
the tile-sparse Cholesky of the reduced camera system (chol.cu). The larger
BASELINE.json configs (Venice-1778, Final-13682) are solved the same way and
reported under "configs". With --gpus N > 1
(torchrun, one process per GPU) the same problem is sharded by landmark over
the N GPUs (NCCL allreduce of the camera-sized sums), so the
scaling is strong: value = LM iterations of the one joint solve / the max over
ranks of the device time. The north-star
implicit-Schur PCG path (solver = pcg) is measured the same way and
reported under "pcg"; per-kernel rooflines under "kernels".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config NAME]

--impl reference times the reference's CPU algorithm (the oracle port of
traceopt, oracle/; the reference itself needs Eigen and cannot be built here,
DESIGN.md) on this host's cores, on a bounded sample of the same workload.
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

BASE_CFG = "trafalgar-257"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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
            t0 = time.time()  # the timed region is tens of ms: start it once the sampler is running
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


def _dist_init(n):
    rank, world = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1)
    if world > 1:
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


def _sum_over_ranks(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def _cpu_sample(scene, cfg_name, threads, lm_iters=2):
    """Reference algorithm (oracle port) on the host: `lm_iters` LM iterations
    with the reference default (Cholesky) solver; returns LM iters/s."""
    from oracle import oracle as O
    from paper_2409_12190_b200.api import LmConfig
    O.set_threads(threads)
    prob = O.Problem(scene.poses, scene.points, scene.intrinsics, scene.cam_idx, scene.pt_idx, scene.pixels)
    t0 = time.perf_counter()
    rep = prob.optimize(LmConfig(max_iterations=lm_iters))
    el = time.perf_counter() - t0
    return rep["iterations"] / el, el, rep


def run_reference(args):
    rank, world, dist = _dist_init(args.gpus)
    if rank != 0:
        return
    import paper_2409_12190_b200 as bae
    scene = bae.synthetic.config_scene(args.config)
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        v, el, rep = _cpu_sample(scene, args.config, threads)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.mean(vals)
    C, P, N = bae.synthetic.CONFIGS[args.config]
    sample = f"2 LM iterations (Cholesky, the reference default) of {args.config} per step"
    line = {"impl": "reference", "metric": "lm_iters_per_s", "value": value, "unit": "LM iter/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * 2 / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic BAL-shaped (SURVEY.md 8d generator, seed = camera count)",
            "config": {"workload": f"{args.config} BA (C={C}, P={P}, N={N}), LM + Cholesky"},
            "cpu_baseline": {"value": value, "unit": "LM iter/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "LM iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# B200 FP64 datasheet figure: MEASURED_PEAKS.json has no FP64 number, so the
# FP64 roofline of the Cholesky kernel is against this nominal peak.
# FP64 peak measured on this pool's B200 by tools/lat/dmma.cu (profiles/r01b_fp64_peak.txt):
# 63.8 FMA/clk/SM (mma.sync m8n8k4 f64; DFMA 58.5) x 148 SMs x 1.965 GHz x 2 = 37.1 TFLOP/s
# (NVIDIA's nominal figure is 40). MEASURED_PEAKS.json carries no FP64 number.
FP64_PEAK_TFLOPS = 37.1
FP64_PEAK_SOURCE = "measured FP64 peak (tools/lat/dmma.cu, profiles/r01b_fp64_peak.txt; nominal 40)"


def _alg_bytes(kernel, st):
    """Algorithmic HBM bytes per launch (each logically required array element
    once): fused linearisation (K1 + camera pass) and
    the implicit Schur tile pass (K5)."""
    N, P, C, T, E = st["observations"], st["points"], st["cameras"], st["tiles"], st["entries"]
    if kernel == "linearize":  # obs idx+px 22, points 24 + H_pp/g_p 72, entry partials 216 w + 216 r, cameras
        return 22 * N + 96 * P + 432 * E + 368 * C + 16 * T
    if kernel == "schur_tiles":  # blob 6/obs, points 24 + H~pp^-1 48, camera record+direction 176 + partial 48
        return 6 * N + 72 * P + 224 * E + 32 * T
    if kernel == "prep_direct":  # obs index 6, V 144 written; points + H_pp/g_p 96, H~pp^-1 48 w; entry RHS 48 w
        return 150 * N + 144 * P + 48 * E + 128 * C
    if kernel == "lin_prep":  # linearize + V 144 w, H~pp^-1 48 w, entry RHS 48 w + 48 r, H~cc 168 + rhs 48 w
        return 166 * N + 144 * P + 528 * E + 584 * C + 16 * T
    raise ValueError(kernel)


def _schur_bytes(st, ds):
    """Direct Schur assembly, algorithmic bytes: every V = W L^-T read once
    (144 B per observation), the pair list (8 B per pair), the 48 x 48 tiles
    written."""
    return 144 * st["observations"] + 8 * ds["pairs"] + 48 * 48 * 8 * ds["tiles"]


def _chol_flops(ds):
    """FP64 flops of one tile Cholesky factorisation (48 x 48 tiles): tile
    updates and triangular solves (2 * 48^3 each) + per column factor and
    inverse (~2 * 48^3 / 3)."""
    g = 2 * 48 ** 3
    return ds["tile_updates"] * g + (ds["tiles"] - ds["tile_columns"]) * g + ds["tile_columns"] * (g // 3)


def run_b200(args):
    import torch
    rank, world, dist = _dist_init(args.gpus)
    local = _env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    import paper_2409_12190_b200 as bae
    from paper_2409_12190_b200.api import LmConfig, SolverChoice

    peak_hbm, peak_kind = _peaks()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def fresh_id():
        # One problem for the whole job. N > 1: landmark-sharded over the ranks
        # -- each rank owns a point partition and its
        # observations, cameras are replicated, camera-sized partial sums are
        # allreduced with NCCL (per LM phase, and once per PCG iteration).
        if world == 1:
            return {}
        obj = [bae.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return dict(rank=rank, world=world, nccl_id=obj[0])

    def make(scene):
        return bae.make_ba_problem(scene.poses, scene.points, scene.intrinsics, scene.observations, device=local,
                                   **fresh_id())

    def one_solve(prob, scene, cfg):
        prob.set_parameters(scene.poses, scene.points)  # untimed: inputs resident before the timed solve
        flush.zero_()  # L2 flush between timed steps (L2 = 126 MB; 256 MB written)
        torch.cuda.synchronize()
        return bae.optimize(prob, None, None, cfg)

    def series(prob, scene, cfg, steps, warmup, clk=None):
        for _ in range(warmup):
            one_solve(prob, scene, cfg)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = prob.launch_count()
        prob.phase_times(reset=True)
        dev, its, inner, reps = 0.0, 0, 0, []
        for _ in range(steps):
            r = one_solve(prob, scene, cfg)
            reps.append(r)
            dev += r.device_seconds
            its += r.iterations
            inner += r.total_pcg_iters
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ph = prob.phase_times(reset=True)
        launches = prob.launch_count() - l0
        dev_max = _max_over_ranks(dist, dev)
        if not ph.get("factor") and not ph.get("pcg"):
            # the LM iteration ran as captured graphs (no per-phase events):
            # one untimed solve with plain launches for the phase breakdown
            os.environ["BAE_LM_GRAPH"] = "0"
            try:
                one_solve(prob, scene, cfg)
                torch.cuda.synchronize()
                ph = {k: v * steps for k, v in prob.phase_times(reset=True).items()}
            finally:
                del os.environ["BAE_LM_GRAPH"]
        return dict(value=its / dev_max, dev_max=dev_max, iterations=its, inner=inner, reports=reps,
                    phases={k: v / steps for k, v in ph.items()}, launches=launches)

    C, P, N = bae.synthetic.CONFIGS[args.config]
    scene = bae.synthetic.bal_shaped(C, P, N, seed=C)
    cfg = LmConfig(max_iterations=50)  # reference defaults: solver = cholesky (here: tile-sparse Cholesky)
    cfg_pcg = LmConfig(max_iterations=50, solver=SolverChoice.pcg)
    prob = make(scene)
    stats = prob.stats()
    shard_max_pts = int(_max_over_ranks(dist, prob.shard()[2]))

    with ClockSampler(local) as clk:
        head = series(prob, scene, cfg, args.steps, args.warmup)
    last = head["reports"][-1]
    ds = prob.direct_stats()

    # --- north-star implicit-Schur PCG path, same protocol ---
    pcg = series(prob, scene, cfg_pcg, max(1, min(args.steps, 3)), max(1, args.warmup // 2))

    # --- kernel-level device times (CUDA events on the solver stream) ---
    ms_lin = prob.time_kernel(0, 20)
    ms_sx = prob.time_kernel(1, 50)
    ms_pcg = prob.time_kernel(2, 50)
    ms_chol = prob.time_kernel(4, 20)
    lin_b, sx_b, chol_f = _alg_bytes("linearize", stats), _alg_bytes("schur_tiles", stats), _chol_flops(ds)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get("k_tile_chol_factor")
        except Exception:
            traffic = None
    solve_ms = 1e3 * head["dev_max"] / args.steps
    chol_share = head["phases"].get("factor", 0.0) / solve_ms if solve_ms else None
    kernels = [
        {"kernel": "k_tile_chol_factor + k_tile_chol_backward (direct solve, per LM iteration)", "us": 1e3 * ms_chol,
         "bound": "fp64 pipe / latency", "achieved": chol_f / (ms_chol * 1e-3) / 1e12, "unit": "TFLOP/s",
         "peak": FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE,
         "frac": chol_f / (ms_chol * 1e-3) / 1e12 / FP64_PEAK_TFLOPS},
        {"kernel": "k_linearize + k_cam_linearize + k_lin_totals (fused residual + Jacobian + J^T J / J^T r blocks)",
         "us": 1e3 * ms_lin, "bound": "hbm", "achieved": lin_b / (ms_lin * 1e-3) / 1e9, "unit": "GB/s",
         "peak": peak_hbm, "frac": lin_b / (ms_lin * 1e-3) / 1e9 / peak_hbm, "obs_per_s": N / (ms_lin * 1e-3)},
        {"kernel": "k_schur_tiles (implicit Schur S*p tile pass, per PCG iteration)", "us": 1e3 * ms_sx,
         "bound": "hbm", "achieved": sx_b / (ms_sx * 1e-3) / 1e9, "unit": "GB/s", "peak": peak_hbm,
         "frac": sx_b / (ms_sx * 1e-3) / 1e9 / peak_hbm},
        {"kernel": "one PCG iteration (tile pass + camera pass + update)", "us": 1e3 * ms_pcg},
    ]

    # --- end to end through the C ABI with host buffers (create + solve + read back) ---
    e2e_iters, e2e_s = 0, 0.0
    for i in range(max(1, min(args.steps, 3)) + 1):
        ids = fresh_id()  # a new communicator per problem (outside the timed region)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p2 = bae.make_ba_problem(scene.poses, scene.points, scene.intrinsics, scene.observations, device=local,
                                 **ids)
        r2 = bae.optimize(p2, scene.poses, scene.points, cfg, final_state={})
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        del p2
        if i > 0:  # the first one warms host allocations
            e2e_iters += r2.iterations
            e2e_s += el
    e2e_max = _max_over_ranks(dist, e2e_s)
    e2e_value = e2e_iters / e2e_max
    # warm variant: optimize on the existing problem through the public API
    # (initial parameters H2D, solve, final parameters D2H) -- what the
    # reference arm times (its problem is built outside the timed region)
    w_iters, w_s = 0, 0.0
    for i in range(max(1, min(args.steps, 3)) + 1):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r3 = bae.optimize(prob, scene.poses, scene.points, cfg, final_state={})
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if i > 0:
            w_iters += r3.iterations
            w_s += el
    e2e_warm = w_iters / _max_over_ranks(dist, w_s)
    h2d = 56 * C + 24 * P + 24 * C + 24 * N + 56 * C + 24 * P  # create inputs + optimize init params
    d2h = 56 * C + 24 * P

    # --- the larger BASELINE.json configs: time-to-converge with the reference defaults ---
    extra = {}
    if not args.no_extra:
        for name in ("venice-1778", "final-13682"):
            c2, p2_, n2 = bae.synthetic.CONFIGS[name]
            # the same scene family from the on-device generator (row f4): the
            # host generator's sequential reference-Rng stream takes seconds here
            tg = time.perf_counter()
            sc = bae.synthetic.bal_shaped_device(c2, p2_, n2, seed=c2, device=local)
            t_gen = time.perf_counter() - tg
            t0 = time.perf_counter()
            pr = make(sc)
            t_create = _max_over_ranks(dist, time.perf_counter() - t0)
            ser = series(pr, sc, cfg, 2, 1)
            r = ser["reports"][-1]
            ms_l = pr.time_kernel(0, 5)
            st2 = pr.stats()
            ds2 = pr.direct_stats()
            ms_p, ms_s = pr.time_kernel(5, 5), pr.time_kernel(6, 5)
            ms_lp = pr.time_kernel(7, 5) if world == 1 else None
            kern2 = []
            for kname, ms_k, nbytes in (("k_linearize + camera pass", ms_l, _alg_bytes("linearize", st2)),
                                        ("k_prep<direct> + camera pass", ms_p, _alg_bytes("prep_direct", st2)),
                                        ("k_lin_prep + k_cam_lin_prep (fused; after an accepted step)", ms_lp,
                                         _alg_bytes("lin_prep", st2)),
                                        ("k_schur_dense (Schur assembly)", ms_s, _schur_bytes(st2, ds2))):
                if ms_k is None:
                    continue
                gbs = nbytes / (ms_k * 1e-3) / 1e9
                kern2.append({"kernel": kname, "us": 1e3 * ms_k, "bound": "hbm", "algorithmic_bytes": nbytes,
                              "achieved": gbs, "unit": "GB/s", "peak": peak_hbm, "frac": gbs / peak_hbm})
            extra[name] = {
                "workload": f"{name} BA (C={c2}, P={p2_}, N={n2}), LmConfig defaults (direct solve)",
                "data": "synthetic BAL-shaped, on-device Philox generator (csrc/synth_device.cu), seed = C",
                "generate_s": t_gen,
                "lm_iters_per_s": ser["value"], "time_to_converge_s": ser["dev_max"] / 2,
                "lm_iterations": r.iterations, "termination": r.reason.name, "final_mse": r.final_mse,
                "ms_per_lm_iteration": 1e3 * ser["dev_max"] / max(1, ser["iterations"]),
                "phase_ms_per_solve": ser["phases"], "create_s": t_create,
                "obs_per_s_residual_jacobian": n2 / (_max_over_ranks(dist, ms_l) * 1e-3),
                "linearize_hbm_frac": _alg_bytes("linearize", st2) / (ms_l * 1e-3) / 1e9 / peak_hbm,
                "direct": ds2,
                "kernels": kern2,
            }
            del pr

    clocks = clk.summary()
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            v, el, _ = _cpu_sample(scene, args.config, os.cpu_count() or 1)
            cpu = {"value": v, "unit": "LM iter/s", "cores": os.cpu_count() or 1, "kind": "port",
                   "sample": f"2 LM iterations of the reference algorithm (oracle port, Cholesky) on "
                             f"{args.config}, {el:.1f} s"}
        chol_ach = chol_f / (ms_chol * 1e-3) / 1e12
        line = {
            "metric": "lm_iters_per_s", "value": head["value"], "unit": "LM iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": solve_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic BAL-shaped (SURVEY.md 8d generator, seed = camera count)",
            "config": {"workload": f"{args.config} BA (C={C}, P={P}, N={N}), LM with LmConfig defaults "
                                   f"(solver=cholesky: tile-sparse Cholesky of the reduced camera system, "
                                   f"max_iterations=50) from the same initial state each step",
                       "parallelism": (f"landmark-sharded over {world} GPUs (NCCL allreduce of camera vectors)"
                                       if world > 1 else "single GPU"),
                       "points_per_rank_max": shard_max_pts,
                       "l2": "flushed (256 MB write) between steps",
                       "tiles": stats["tiles"], "tile_camera_entries": stats["entries"], "direct": ds},
            "time_to_converge_s": head["dev_max"] / args.steps,
            "lm_iterations_per_solve": last.iterations, "final_mse": last.final_mse,
            "termination": last.reason.name,
            "obs_per_s_residual_jacobian": N / (ms_lin * 1e-3),
            "phase_ms_per_solve": head["phases"],
            "pcg": {"lm_iters_per_s": pcg["value"], "time_to_converge_s": pcg["dev_max"] / len(pcg["reports"]),
                    "pcg_iterations_per_solve": pcg["inner"] / len(pcg["reports"]),
                    "phase_ms_per_solve": pcg["phases"],
                    "config": "same workload, solver=pcg (implicit-Schur PCG, block-Jacobi), pcg_tol=1e-8"},
            "roofline": {"bound": "tensor", "kernel": "k_tile_chol_factor + k_tile_chol_backward",
                         "achieved": chol_ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": chol_ach / FP64_PEAK_TFLOPS, "traffic": traffic,
                         "peak_source": FP64_PEAK_SOURCE,
                         "share_of_step": chol_share,
                         "limiter": "latency: the dependent pivot chain along the nested-dissection tree",
                         "algorithmic_flops": "2*48^3 per tile update / solve + 2*48^3/3 per tile column"},
            "kernels": kernels,
            "configs": extra,
            "e2e": {"value": e2e_value, "unit": "LM iter/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "includes": "make_ba_problem (planning, upload) + optimize + parameter read-back, every step",
                    "warm": {"value": e2e_warm, "unit": "LM iter/s", "h2d_bytes_per_step": 56 * C + 24 * P,
                             "d2h_bytes_per_step": d2h,
                             "includes": "optimize(init params from host) + read-back on an existing problem"}},
            "gpu_launches": head["launches"],
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=BASE_CFG)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the Venice / Final time-to-converge lines")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
