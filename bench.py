"""Benchmark of the B200 batched micro-solve path (BASELINE.json north star).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

One step = one complete device-resident two-scale `fixed_point_solve` on the
configured workload (default: config 3, the largest 2D config — 16641 micro
problems of 4225 DoFs; the north star's >=60%-of-roofline bar is quoted on it).
`value` = micro DoF-iterations of the batched micro PCG / device time of those
launches (CUDA events on the launching stream, summed over the K timed steps).
`e2e` = the same metric through the C ABI with host buffers: context build from
host inputs (H2D) + solve + download of u, w, V (D2H), wall-clock per step.

Multi-GPU (torchrun): the north star puts nothing across GPUs, so
N>1 runs N independent replicas, one per GPU; `value` sums all ranks' DoF-its over
the max-over-ranks time ("scaling": "weak").

--impl reference: the reference's own cg_solve (oracle/_ref, the unmodified
reference library) on the same workload's micro systems, with all host threads,
on a bounded sample per step.  Those systems are assembled by the C oracle,
because the reference cannot express config 3's reaction/anisotropy/table.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2103_17040_b200 import configs  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def ncu_traffic(variant):
    """DRAM bytes (read + write) per launch of the hot kernel from the committed ncu --set full
    capture (profiles/r02/prof_pair_c3_r2_raw.csv for the column-pair kernel), or None."""
    path = os.path.join(ROOT, "profiles", "r02", {1: "prof_pair_c3_r2_raw.csv"}.get(variant, "none"))
    try:
        import csv
        with open(path) as f:
            rows = list(csv.reader(f))
        hdr, units, vals = rows[0], rows[1], rows[2]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        tot = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(key)
            tot += float(vals[i].replace(",", "")) * scale[units[i]]
        return tot, os.path.relpath(path, ROOT)
    except Exception:
        return None, None


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, 1965.0, "fallback"


# ----------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except Exception:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit()) if rows else None
        loaded = [v for v in sm if v > 0.5 * (smax or 1)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------- dist plumbing -
def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        return world, rank, local, dist, backend
    return 1, 0, local, None, None


def barrier(dist, backend):
    if dist is not None:
        import torch
        if backend == "nccl":
            dist.barrier(device_ids=[torch.cuda.current_device()])
        else:
            dist.barrier()


def reduce_max(dist, backend, value):
    if dist is None:
        return value
    import torch
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(dist, backend, value):
    if dist is None:
        return value
    import torch
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------ CPU baselines --
def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference_sample(cfg, budget_s=15.0, threads=None, seed=0):
    """Reference cg_solve (oracle/_ref) on a bounded sample of the workload's micro systems
    (assembled by the C oracle), all host threads.  Returns (DoF*it/s, info)."""
    from oracle import port, ref  # CPU checker / baseline only
    threads = threads or host_threads()
    o = port.OracleContext(cfg)
    n = o.n_micro
    # interior macro nodes (Dirichlet nodes have b = 0 and no iterations)
    m = cfg.macro_n
    interior = np.array([j * (m + 1) + i for j in range(1, m) for i in range(1, m)], np.int32)
    rng = np.random.default_rng(seed)
    rp, ci = o.micro_pattern()
    # calibrate: one system single-threaded
    def systems(nodes):
        vals = np.stack([o.micro_values(int(i)) for i in nodes])
        b = np.stack([0.05 * o.rhs_parts(int(i))[1] for i in nodes])  # micro_rhs with u_i = 0.05, w_i = 0
        return vals, b
    v1, b1 = systems(interior[:1])
    _, it1, t1 = ref.batched_cg(rp, ci, v1, b1, np.zeros_like(b1), cfg.inner_tol, 20000, 1)
    per_sys = max(t1, 1e-4)
    count = int(max(threads, min(len(interior), budget_s * threads / per_sys)))
    count = min(count, len(interior), 4096)
    # assemble up to 256 distinct sampled systems and tile them to `count` solves
    uniq = np.sort(rng.choice(interior, size=min(count, 256), replace=False))
    vu, bu = systems(uniq)
    reps = -(-count // len(uniq))
    vals = np.tile(vu, (reps, 1))[:count]
    b = np.tile(bu, (reps, 1))[:count]
    _, iters, secs = ref.batched_cg(rp, ci, vals, b, np.zeros_like(b), cfg.inner_tol, 20000, threads)
    if (iters < 0).any():
        raise RuntimeError("reference cg_solve failed on the sample")
    dof_it = float(n) * float(iters.sum())
    return dof_it / secs, dict(threads=threads, systems=int(count), distinct=len(uniq), seconds=secs,
                               dof_iters=dof_it,
                               iters_mean=float(iters.mean()), iters_max=int(iters.max()))


def two_scale_standin(cfg, threads=None):
    """Like-for-like end-to-end two-scale solve on the reference-expressible stand-in of the
    workload (k = 0, D = I, symbolic config-2-family map, same grids): the
    reference's AssemblyContext + fixed_point_solve (oracle/_ref, all host threads) against
    this library's context build + solve + download of u, w, V through the C ABI."""
    from oracle import ref  # CPU baseline only
    from paper_2103_17040_b200 import abi
    threads = threads or host_threads()
    red = cfg.reduced()
    ini = red.ini()
    ext = red.ext(reference_expressible=True)
    abi.Context(ini, ext).close()  # module load / allocator warm-up
    t0 = time.perf_counter()
    g = abi.Context(ini, ext)
    out = g.solve(outer_tol=red.outer_tol)
    t1 = time.perf_counter()
    g.close()
    t2 = time.perf_counter()
    r = ref.RefContext(ini, threads)
    s = r.solve(outer_tol=red.outer_tol, workers=threads)
    t3 = time.perf_counter()
    rel_v = float(np.linalg.norm(out["V"] - s["V"]) / np.linalg.norm(s["V"]))
    r.close()
    return {"reference_s": t3 - t2, "ours_s": t1 - t0, "speedup": (t3 - t2) / (t1 - t0), "cores": threads,
            "sweeps": [out["sweeps"], s["sweeps"]], "rel_l2_V": rel_v,
            "what": f"{red.name}: AssemblyContext + fixed_point_solve (reference, {threads} threads) vs "
                    "ts_ctx_create_ini + ts_fixed_point_solve + ts_download_state (B200), same INI"}


# ------------------------------------------------------------------- arms ----
def other_config_rates(names):
    """The other single-GPU BASELINE configs' micro PCG rates on this box (not bench lines: one
    warm-up + two timed device-resident fixed-point solves each), so the driver's record also
    carries the Q2 (c4) and 3D (c5) cluster kernels and the 33-wide pair kernel (c2)."""
    from paper_2103_17040_b200 import abi
    out = {}
    for name in names:
        try:
            c = configs.CONFIGS[name]
            g = abi.Context(c.ini(), c.ext())
            g.solve(download=False)
            reps = [g.solve(download=False) for _ in range(2)]
            dof = sum(r["micro_dof_iters"] for r in reps)
            ms = sum(r["micro_ms"] for r in reps)
            rate = dof / (ms * 1e-3)
            out[name] = {"value": rate, "unit": "DoF*it/s", "workload": c.description or name,
                         "two_scale_solve_s": sum(r["total_ms"] for r in reps) * 1e-3 / len(reps),
                         "sweeps": reps[-1]["sweeps"], "setup_ms_device_first_build": g.info["setup_ms"],
                         "micro_kernel": g.info["micro_kernel"],
                         "x_hbm_roofline_alg": rate * c.alg_bytes_per_dof / (peaks()[0] * 1e9)}
            g.close()
        except Exception as e:  # must not sink the headline number
            out[name] = {"unavailable": str(e)}
    return out


def run_ours(args, cfg):
    from paper_2103_17040_b200 import abi

    world, rank, local, dist, backend = dist_setup(args.gpus)
    abi.select_device(local if world > 1 else 0)
    if not abi.device_ok():
        raise SystemExit("no usable sm_100 device: " + abi.lib().ts_last_error().decode())
    table = cfg.table()
    ext = cfg.ext()
    ini = cfg.ini()
    ctx = abi.Context(ini, ext)
    info = ctx.info
    opts = ctx.default_opts()

    def step():
        return ctx.solve(download=False)

    for _ in range(args.warmup):
        step()
    barrier(dist, backend)
    with ClockSampler(local if world > 1 else 0) as clk:
        t0 = time.perf_counter()
        reps = [step() for _ in range(args.steps)]
        wall = time.perf_counter() - t0
    clocks = clk.summary()
    barrier(dist, backend)
    micro_s = sum(r["micro_ms"] for r in reps) * 1e-3
    total_s = sum(r["total_ms"] for r in reps) * 1e-3
    dof_it = sum(r["micro_dof_iters"] for r in reps)
    launches = sum(r["gpu_launches"] for r in reps)
    micro_launches = sum(r["sweeps"] for r in reps)
    micro_s_max = reduce_max(dist, backend, micro_s)
    total_s_max = reduce_max(dist, backend, total_s)
    dof_all = reduce_sum(dist, backend, dof_it)
    value = dof_all / micro_s_max

    # SURVEY.md 8d timed region (ii): isolated cold batched micro solve, u_i = 0.05, w_i = 0
    nM, nm = ctx.n_macro, ctx.n_micro
    cold = None
    if rank == 0:
        cu, cw = np.full(nM, 0.05), np.zeros(nM)
        ctx.micro_solve(cu, cw, tol=opts["inner_tol"])  # warm-up
        _, cit, crep = ctx.micro_solve(cu, cw, tol=opts["inner_tol"])
        cold = {"value": crep["micro_dof_iters"] / (crep["micro_ms"] * 1e-3), "unit": "DoF*it/s",
                "ms": crep["micro_ms"], "iters_mean": float(cit.mean()), "iters_max": int(cit.max()),
                "what": "one batched micro PCG launch over all problems from x0 = 0 with u_i = 0.05"}

    # e2e through the C ABI with host buffers (pinned), H2D + D2H inside the timed region
    ctx.close()
    pu = abi.PinnedArray((nM,))
    pw = abi.PinnedArray((nM,))
    pV = abi.PinnedArray((nM, nm))
    ptab = None
    if table is not None:
        ptab = abi.PinnedArray(table.shape)
        ptab.array[...] = table
        ext = abi.make_ext(D=cfg.D, reaction=cfg.reaction, table=ptab.array, amp=cfg.amp)
    e2e_times, e2e_dof = [], []
    for k in range(max(1, args.e2e_steps) + 1):
        barrier(dist, backend)
        t0 = time.perf_counter()
        c2 = abi.Context(ini, ext)
        t1 = time.perf_counter()
        r = c2.solve(download=False)
        t2 = time.perf_counter()
        c2.state(pu.array, pw.array, pV.array)
        t3 = time.perf_counter()
        c2.close()
        dt = time.perf_counter() - t0
        if k > 0:  # first pass warms allocator/module loading
            e2e_times.append(dt)
            e2e_dof.append(r["micro_dof_iters"])
        print(f"e2e pass {k}: {dt:.3f} s = create {t1 - t0:.3f} + solve {t2 - t1:.3f} (device {r['total_ms']:.1f} ms)"
              f" + download {t3 - t2:.3f} + destroy {time.perf_counter() - t3:.3f}", file=sys.stderr, flush=True)
    e2e_s = reduce_max(dist, backend, sum(e2e_times))
    e2e_value = reduce_sum(dist, backend, sum(e2e_dof)) / e2e_s
    h2d = (table.nbytes if table is not None else 0) + len(ini.encode())
    d2h = (2 * nM + nM * nm) * 8
    state_check = float(np.abs(pV.array).max())

    hbm_gbs, sm_max, peak_kind = peaks()
    b_csr = cfg.csr_bytes_per_dof    # CSR operator bytes per DoF-iteration
    b_alg = cfg.alg_bytes_per_dof    # the smaller of CSR and coefficient tensors (C4: tensors)
    per_launch_dofit = dof_it / micro_launches
    per_launch_s = micro_s / micro_launches
    hbm_ach = b_alg * per_launch_dofit / per_launch_s / 1e9
    # SMEM-resident kernels (column strips / pairs) keep the operator on chip for the whole
    # solve, so HBM does not bound them: the binding unit is SMEM bandwidth (ncu: SMEM
    # wavefronts ~62 % of peak, DRAM < 1 %).  micro_smem_bytes = their SMEM loads + stores per
    # DoF-iteration (the kernel's traffic model, ts_ctx_info).
    smem_b_per_dofit = float(info.get("micro_smem_bytes") or 0.0)
    variant = {0: "column strips", 1: "column pairs", 2: "generic streaming",
               3: "generic Q2 class-compact"}.get(info.get("micro_kernel"), "?")
    smem_resident = info.get("micro_kernel") in (0, 1)
    sm_mhz = clocks.get("sm_mhz") or sm_max
    smem_peak = 128.0 * 148 * sm_mhz * 1e6 / 1e9
    smem_ach = smem_b_per_dofit * per_launch_dofit / per_launch_s / 1e9

    traffic, traffic_src = ncu_traffic(info.get("micro_kernel"))
    if traffic is not None and cfg.name != "c3-large":
        traffic, traffic_src = None, None  # the committed capture is of config 3
    dram_gbs = traffic / per_launch_s / 1e9 if traffic is not None else None
    roof_hbm = {"bound": "hbm", "achieved": hbm_ach, "peak": hbm_gbs, "unit": "GB/s", "frac": hbm_ach / hbm_gbs,
                "traffic": traffic, "peak_kind": peak_kind,
                "basis": f"B_alg {b_alg:.2f} B per micro DoF-iteration (SURVEY.md 8d, the smaller of CSR "
                         f"{b_csr:.2f} B and coefficient tensors {cfg.tensor_bytes_per_dof:.2f} B) per batched-PCG "
                         "launch / launch time"}
    if smem_resident:
        roofline = {"bound": "smem", "achieved": smem_ach, "peak": smem_peak, "unit": "GB/s",
                    "frac": smem_ach / smem_peak, "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu)",
                    "traffic_source": traffic_src, "dram_gbs_measured": dram_gbs,
                    "basis": f"{smem_b_per_dofit:.1f} B SMEM loads+stores per micro DoF-iteration ({variant}, "
                             f"R={info.get('micro_rows')}) per launch / launch time; peak 128 B/clk/SM x 148 SMs "
                             f"at {sm_mhz:.0f} MHz; the operator is SMEM-resident for the whole solve, so DRAM "
                             "moves only the once-per-solve operator/rhs/state bytes (dram_gbs_measured)"}
        roof_hbm["note"] = ("the CSR-streaming bound this kernel removes (it reads the operator once per "
                            "solve, not once per iteration), hence > 1")
    else:
        roofline = dict(roof_hbm, traffic_unit="DRAM bytes per launch (ncu)", traffic_source=traffic_src)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v_cpu, cinfo = cpu_reference_sample(cfg, budget_s=args.cpu_budget)
            cpu = {"value": v_cpu, "unit": "DoF*it/s", "cores": cinfo["threads"], "kind": "reference",
                   "sample": (f"reference cg_solve (oracle/_ref) on {cinfo['systems']} solves of "
                              f"{cinfo['distinct']} sampled {cfg.name} micro systems "
                              f"(C-oracle assembled, u_i=0.05 cold start), {cinfo['threads']} threads, "
                              f"{cinfo['seconds']:.1f}s, mean {cinfo['iters_mean']:.0f} it"),
                   "seconds": cinfo["seconds"]}
            # SURVEY.md 8d also asks for the single-worker figure (reference at 1 worker)
            v1, c1 = cpu_reference_sample(cfg, budget_s=3.0, threads=1, seed=1)
            cpu["single_thread"] = {"value": v1, "unit": "DoF*it/s", "cores": 1,
                                    "sample": f"{c1['systems']} solves, {c1['seconds']:.1f}s"}
        except Exception as e:  # the CPU leg must not sink the GPU number
            cpu = {"value": None, "unit": "DoF*it/s", "cores": host_threads(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
        if not args.no_two_scale_cpu:
            try:
                cpu["two_scale_s"] = two_scale_standin(cfg)
            except Exception as e:
                cpu["two_scale_s"] = {"unavailable": str(e)}

    others = None
    if rank == 0 and world == 1 and not args.no_other_configs:
        others = other_config_rates([n for n in ("c2", "c4", "c5") if n != cfg.name])

    if rank == 0:
        line = {
            "metric": "batched micro-solve DoF*iters/s",
            "value": value,
            "unit": "DoF*it/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": 1e3 * total_s_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded; BASELINE.json config shapes)",
            "config": {
                "workload": cfg.description or cfg.name,
                "macro_problems": nM, "micro_dofs": nm, "micro_nnz": info["micro_nnz"],
                "step": "one device-resident fixed_point_solve (all sweeps, inner/outer tol "
                        f"{opts['inner_tol']:g}/{opts['outer_tol']:g})",
                "l2": f"inputs larger than L2 (micro operators {9 * nm * nM * 8 / 1e9:.1f} GB in HBM)",
                "parallelism": "replicas" if world > 1 else "single GPU",
            },
            "two_scale_solve_s": total_s_max / args.steps,
            "sweeps_per_step": reps[-1]["sweeps"],
            "micro_dof_iters_per_step": dof_it / args.steps,
            "pct_hbm_roofline_alg": 100.0 * value / world * b_alg / (hbm_gbs * 1e9),
            "roofline": roofline,
            "roofline_hbm_alg": roof_hbm,
            "e2e": {"value": e2e_value, "unit": "DoF*it/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "seconds_per_step": e2e_s / len(e2e_times),
                    "path": "ts_ctx_create_ini (host INI + pinned A-table) -> ts_fixed_point_solve -> "
                            "ts_download_state (pinned u,w,V)"},
            "cold_batched_solve": cold,
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "setup_ms_device": info["setup_ms"],
            "micro_iters_max": max(r["micro_iters_max"] for r in reps),
            "wall_s_timed": wall,
            "state_max_abs": state_check,
            "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_reference(args, cfg):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs the CPU reference; other ranks exit 0 without work
    try:
        from oracle import ref
        if not ref.available():
            raise FileNotFoundError("oracle/_ref/libtwoscale_ref.so not built")
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}), flush=True)
        return
    budget = max(2.0, args.cpu_budget / max(1, args.steps))
    for _ in range(args.warmup):
        cpu_reference_sample(cfg, budget_s=min(budget, 2.0))
    vals, infos = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, inf = cpu_reference_sample(cfg, budget_s=budget)
        vals.append(v)
        infos.append(inf)
    wall = time.perf_counter() - t0
    dof = sum(i["dof_iters"] for i in infos)
    secs = sum(i["seconds"] for i in infos)
    value = dof / secs
    line = {
        "metric": "batched micro-solve DoF*iters/s", "value": value, "unit": "DoF*it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; BASELINE.json config shapes)", "impl": "reference",
        "config": {"workload": cfg.description or cfg.name, "macro_problems": cfg.n_macro,
                   "micro_dofs": cfg.n_micro, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "DoF*it/s", "cores": infos[0]["threads"], "kind": "reference",
                         "sample": f"per step: reference cg_solve (unmodified, oracle/_ref) on "
                                   f"{infos[0]['systems']} sampled {cfg.name} micro systems assembled by the C "
                                   f"oracle (u_i=0.05 cold start), {infos[0]['threads']} threads"},
        "e2e": {"value": value, "unit": "DoF*it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3", choices=sorted(configs.CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU work for the baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the short c2 / c4 / c5 rate measurements appended to the line")
    ap.add_argument("--no-two-scale-cpu", action="store_true",
                    help="skip the reference two-scale solve on the stand-in (minutes on config 3)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    cfg = configs.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
