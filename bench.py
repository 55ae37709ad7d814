"""bench.py -- D3M factor+solve on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[3], the largest single-GPU configuration the
hot path runs standalone): blocked LDL^T with restricted Bunch-Kaufman
pivoting of the interface matrix K of a 4x4x4 subdomain grid (144 faces x
256 unknowns, K is 36,864^2 complex128, natural face order), followed by a
16-RHS block solve with one step of iterative refinement (block_solve(...,
refine=1): the reference's own solve leaves a relative residual of ~1e-10 on
this system, the GPU solve ~4e-10 unrefined and ~2e-13 refined; the refinement
flops are not counted).  One step = block_ldlt + block_solve.

  value : complex-FP64 TFLOP/s of the whole step with K and the RHS resident
          in HBM (algorithmic flops: SURVEY.md 8(d) counts)
  e2e   : the same through the public API with HOST numpy inputs (K blocks
          and RHS copied host->device, solution copied back inside the step)
  roofline : the trailing-update DMMA GEMM (dominant kernel) -- its
          algorithmic flops / its summed CUDA-event time in the timed region,
          against the FP64 DMMA peak measured live at start-up
  cpu_baseline : the CPU oracle port (oracle/: the C restatement of the
          reference's numba kernels + numpy/OpenBLAS block drivers) running
          the SAME full step (block LDL^T of K + the 16-RHS solve) on the
          host cores, timed once; the secondaries carry same-run CPU timings
          of the subdomain reductions (configs 1, 2 and 3, process pools;
          config 5's ~20 CPU-minutes per subdomain are out of a bench's reach)
  secondary : configs 1, 2, 3 and 5 (BASELINE configs[0], [1], [2], [4]),
          each with time, rate, roofline fraction and pivot-decision margins

`--impl reference` runs only the CPU oracle port on the same metric.
N > 1 (torchrun): independent replicas per GPU (the block LDL^T chain does
not shard in this tier), value = all ranks' flops / max time.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "D3M factor+solve time and complex FP64 TFLOP/s (% of B200 FP64 peak)"
WORKLOAD = ("cfg4: block LDL^T (restricted BK) of K, 4x4x4 subdomain grid, 144 faces x 256 unknowns "
            "(n=36864 complex128, natural face order) + 16-RHS block solve + 1 refinement step")
NRHS = 16
REFINE = 1           # refinement steps in the headline solve (0 = the reference's algorithm)
CPU_SAMPLE_COLUMNS = 10


# --------------------------------------------------------------------------
def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group("gloo" if os.environ.get("D3M_BENCH_GLOO") else "nccl")
        return dist, dist.get_rank(), ws
    return None, 0, 1


def _barrier(dist):
    if dist is not None:
        dist.barrier()


def _max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
def _cfg4_host():
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    K = wl.config4_matrix()
    plan = d.symbolic_factor(d.clique_graph(K), d.identity_ordering(K.nblocks), K.sizes)
    rhs = wl.config4_rhs(K, NRHS)
    return K, plan, rhs


def _solve_flops(sched, nrhs: int) -> int:
    # forward + backward: every stored L entry is one complex FMA per RHS
    # in each sweep (diagonal blocks: strict lower half)
    ent = int(sum(int(s) * (int(s) - 1) // 2 for s in sched.sizes) + int((sched.panel_rows * sched.sizes).sum()))
    return 2 * 8 * ent * nrhs


def _fp64_peak_probe():
    """Live FP64 DMMA peak on this GPU (tools/fp64_peak.cu kernel, burst)."""
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
    except (OSError, subprocess.TimeoutExpired):
        return None
    vals = [float(l.split(":")[1].split()[0]) for l in out.splitlines() if l.startswith("DMMA m8n8k4")]
    return max(vals) if vals else None


def run_ours(args):
    import torch
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import _lib
    from paper_2002_05018_b200.device import DeviceArray, to_device

    dist, rank, ws = _dist()
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    K, plan, rhs = _cfg4_host()
    # device-resident copies (value leg)
    from paper_2002_05018_b200.factor import to_device_blocks
    Kd = to_device_blocks(K)
    rhs_d = [DeviceArray(to_device(b)) for b in rhs]

    def step_dev():
        F = d.block_ldlt(Kd, plan)
        x = d.block_solve(F, rhs_d, refine=REFINE)
        return F, x

    for _ in range(args.warmup):
        F, x = step_dev()
    torch.cuda.synchronize()
    sched = F._sched
    flops_factor = sched.flops_update + sched.flops_trsm + sched.flops_bk
    flops_step = flops_factor + _solve_flops(sched, NRHS)

    # ---- timed region: device-resident inputs -------------------------------
    # (1) the headline: K steps without per-launch instrumentation
    _barrier(dist)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # a collection before each timed region; the collector stays on (the plan's
    # tables are numpy arrays built by the native planner, so a full collection
    # has little to walk)
    gc.collect()
    with ClockSampler(local) as clk:
        e0.record(s)
        for _ in range(args.steps):
            F, x = step_dev()
        e1.record(s)
        torch.cuda.synchronize()
    _barrier(dist)
    ms_total = _max_over_ranks(dist, e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    value = flops_step * ws / (ms_step * 1e-3) / 1e12
    # (2) the same K steps with CUDA events around every launch (on the stream
    # it is launched on): per-stage intervals and the roofline of the update
    # GEMMs; the instrumentation costs ~2-3% of the step, so it is kept out of (1)
    _barrier(dist)
    torch.cuda.synchronize()
    _lib.counters_reset(timing=True)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(s)
    for _ in range(args.steps):
        F, x = step_dev()
    f1.record(s)
    torch.cuda.synchronize()
    cnt = _lib.counters_read()
    _lib.counters_reset(timing=False)
    ms_step_instr = f0.elapsed_time(f1) / args.steps

    # residual check of the last step (untimed)
    res = _residual(K, rhs, [np.asarray(v) for v in x])
    refined = _refine_leg(d, F, K, rhs, rhs_d)
    # pivot-decision margins of the 144 diagonal blocks (one extra, untimed factorisation)
    del F, x
    Fm = d.block_ldlt(Kd, plan, margins=True)
    margins_cfg4 = {"decision_margin": Fm.stats.decision_margin, "argmax_gap": Fm.stats.argmax_gap}
    del Fm
    x = None

    # ---- e2e: public API with host buffers ------------------------------------
    # inputs in pinned host memory (K's blocks as views of one pinned
    # allocation, the RHS blocks pinned), copied to the device inside every
    # step; the solution is read back to numpy inside every step
    Kp, rhs_p = _pinned_inputs(K, rhs)
    h2d = 16 * sum(int(np.asarray(b).size) for b in K.blocks.values()) + 16 * sum(b.size for b in rhs)
    d2h = 16 * sum(b.size for b in rhs)
    Fh = d.block_ldlt(Kp, plan)                     # untimed e2e warm-up step
    xh = [np.asarray(v) for v in d.block_solve(Fh, rhs_p, refine=REFINE)]
    del Fh, xh
    _barrier(dist)
    torch.cuda.synchronize()
    e2e_steps = max(3, min(args.steps, 5))
    e2e_samples = []
    gc.collect()
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        Fh = d.block_ldlt(Kp, plan)
        xh = [np.asarray(v) for v in d.block_solve(Fh, rhs_p, refine=REFINE)]
        torch.cuda.synchronize()
        e2e_samples.append((time.perf_counter() - t0) * 1e3)
        del Fh                                       # the caller releases the factor before the next solve
    # median of the samples (all are reported): one host-side hiccup in a
    # few-sample run otherwise dominates the mean
    e2e_ms = _max_over_ranks(dist, float(np.median(e2e_samples)))
    e2e_value = flops_step * ws / (e2e_ms * 1e-3) / 1e12
    del xh
    # the same with plain numpy inputs (a ddsolve caller's K.blocks / RHS
    # arrays): pageable host memory, staged by the library
    Fh = d.block_ldlt(K, plan)
    xh = [np.asarray(v) for v in d.block_solve(Fh, rhs, refine=REFINE)]
    del Fh, xh
    torch.cuda.synchronize()
    np_samples = []
    gc.collect()
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        Fh = d.block_ldlt(K, plan)
        xh = [np.asarray(v) for v in d.block_solve(Fh, rhs, refine=REFINE)]
        torch.cuda.synchronize()
        np_samples.append((time.perf_counter() - t0) * 1e3)
        del Fh
    np_ms = _max_over_ranks(dist, float(np.median(np_samples)))
    e2e_numpy = {"value": round(flops_step * ws / (np_ms * 1e-3) / 1e12, 4), "unit": "TFLOP/s",
                 "ms_per_step": round(np_ms, 3), "samples_ms": [round(v, 1) for v in np_samples],
                 "statistic": "median", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                 "inputs": "numpy complex128 arrays (pageable host memory), as the reference API takes them"}
    del xh

    if rank != 0:
        return
    peak_live = _fp64_peak_probe()
    peak = peak_live if peak_live else 36.9
    # GEMM-active time = union of the update-GEMM launch intervals (critical
    # and bulk streams overlap; a plain sum would double-count)
    gemm_ms = cnt["union_ms"]["gemm"] / args.steps
    achieved_alg = sched.flops_update / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    # the tensor pipe executes 3 real products per complex product under 3M
    # (Gauss), 4 under 4M: the roofline fraction uses the EXECUTED DMMA flops
    from paper_2002_05018_b200 import _lib
    form = _lib.gemm_form(0)
    achieved = achieved_alg * form / 4.0 if achieved_alg else None
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded, workloads.config4_matrix)",
        "config": {"workload": WORKLOAD, "n": int(K.order), "supernodes": int(K.nblocks), "nrhs": NRHS,
                   "ordering": "natural", "l2": "working set 4.6 GB factor pool >> 126 MB L2 (no flush needed)",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "flops_per_step": flops_step, "flops_update": sched.flops_update,
                   "flops_trsm": sched.flops_trsm, "flops_bk": sched.flops_bk},
        "fraction_of_fp64_peak": round(value / ws / peak, 4),
        "fraction_note": ("value counts algorithmic flops (8 per complex FMA); with the 3M GEMM the tensor pipe "
                          "executes 6, so this is an effective fraction" if form == 3 else
                          "value counts algorithmic flops (8 per complex FMA, executed as 4 real DMMA products)"),
        "gemm_form": f"{form}m",
        "roofline": {"bound": "tensor", "kernel": ("zgemm3m_tma_kernel (3M, 64x32 half tiles, TMA-staged" if form == 3 else "zgemm_grouped_kernel (4M")
                               + "; trailing Schur updates, DMMA)",
                     "timing": "EXECUTED update DMMA flops (algorithmic x form/4) / union of the update-GEMM "
                               "CUDA-event intervals in the instrumented timed region (2)",
                     "achieved": round(achieved, 3) if achieved else None, "peak": round(peak, 2),
                     "achieved_algorithmic": round(achieved_alg, 3) if achieved_alg else None,
                     "peak_source": "live DMMA m8n8k4 probe (tools/fp64_peak.cu)" if peak_live else
                     "profiles/fp64_peak_r01.txt (measured DMMA burst)",
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4) if achieved else None,
                     "traffic": 7.633e8,
                     "traffic_note": "DRAM bytes per launch of a representative 5,460-tile rest-update launch "
                                     "(ncu --set full, profiles/ncu_gemm_tma_cfg4_r02v_summary.txt); algorithmic C "
                                     "traffic of that launch 7.157e8 B (1.07x)"},
        "instrumented_ms_per_step": round(ms_step_instr, 3),
        "stage_ms_per_step": {k: round(v / args.steps, 3) for k, v in cnt["union_ms"].items()},
        "stage_ms_summed_per_step": {k: round(v / args.steps, 3) for k, v in cnt["ms"].items()},
        "gpu_launches": cnt["launches"],
        "e2e": {"value": round(e2e_value, 4), "unit": "TFLOP/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "samples_ms": [round(v, 1) for v in e2e_samples], "statistic": "median"},
        "residual": res,
        "refined": refined,
        "margins": margins_cfg4,
        "clocks": clk.summary(),
    }
    line["e2e_numpy"] = e2e_numpy
    sec = {}
    if not args.no_cfg3:
        sec["cfg3"] = _cfg3_secondary(max(2, min(args.steps, 3)), peak)
    for which in (["cfg1", "cfg2"] if not args.no_fem else []) + (["cfg5"] if not args.no_cfg5 else []):
        sec[which] = _fem_secondary(which, 1 if which == "cfg5" else 4, peak)
    # the CPU legs run last: OpenBLAS worker threads keep spinning after a
    # call and would slow the host-side launches of the GPU legs
    if not args.no_cpu:
        del Kd, rhs_d
        line["cpu_baseline"] = _cpu_full_cfg4(plan, K, rhs, flops_step, ms_step)
        if "cfg1" in sec:
            sec["cfg1"]["cpu_reduce"] = _cpu_reduce_pool("cfg1", [0, 1], sec["cfg1"]["stage_ms"]["reduce"])
        if "cfg2" in sec:
            sec["cfg2"]["cpu_reduce"] = _cpu_reduce_pool("cfg2", list(range(8)), sec["cfg2"]["stage_ms"]["reduce"])
        if "cfg3" in sec:
            sec["cfg3"]["cpu_reduce"] = _cpu_reduce_pool("cfg3", list(range(8)), sec["cfg3"]["ms_per_step"],
                                                         total=64)
    if sec:
        line["secondary"] = sec
    print(json.dumps(line), flush=True)


def _pinned_inputs(K, rhs):
    """K with its blocks as views of ONE pinned host allocation and pinned RHS
    blocks (torch CPU tensors; the public API accepts them as host arrays)."""
    import torch
    import paper_2002_05018_b200 as d
    keys = list(K.blocks)
    tot = sum(int(np.asarray(K.blocks[k]).size) for k in keys)
    buf = torch.empty(tot, dtype=torch.complex128).pin_memory()
    Kp = d.BlockSparseSym(K.sizes)
    o = 0
    for k in keys:
        b = np.ascontiguousarray(np.asarray(K.blocks[k], dtype=np.complex128))
        v = buf[o:o + b.size].view(b.shape)
        v.copy_(torch.from_numpy(b))
        Kp.blocks[k] = v
        o += b.size
    rhs_p = [torch.from_numpy(np.ascontiguousarray(r)).pin_memory() for r in rhs]
    return Kp, rhs_p


def _fem_secondary(which: str, reps: int, peak: float) -> dict:
    """BASELINE configs[0] / [1] / [4]: the full D3M pipeline on the 3-D
    Nedelec FEM problems (fem3d.py; all RHS columns at once), from the
    host-built subdomain systems (sparse A_d / D_d) to the recovered global
    solution on the host: reduce (incl. H2D) -> assemble -> block LDL^T ->
    block solve -> recover (incl. D2H).  The mesh / element front end is
    excluded (it is not part of the path).  Best of ``reps`` timed runs after
    one warm-up run; the warm-up run tracks the pivot-decision margins of
    every subdomain and diagonal-block factorisation (the timed runs do not)."""
    import torch
    from paper_2002_05018_b200 import fem3d
    cfg = {"cfg1": fem3d.config1, "cfg2": fem3d.config2, "cfg5": fem3d.config5}[which]()
    model = fem3d.build_model(cfg)
    systems = fem3d.subdomain_systems(model, rhs=None)
    runs = reps + 1
    best, keep, margins = None, None, None
    for i in range(runs):
        for s in systems:
            s.factor, s._d3m_D, s._d3m_X = None, None, None
        timers = {}
        # a collection before each run (not a paused collector: the pipeline's
        # temporaries must be reclaimable, or the allocator grows instead of reusing)
        gc.collect()
        if os.environ.get("D3M_BENCH_DEBUG"):
            from paper_2002_05018_b200 import _lib as _dl
            _dl.counters_reset(timing=os.environ.get("D3M_BENCH_DEBUG") == "2")
        sol, _, R, plan, F = fem3d.solve_d3m(model, rhs=None, keep="auto", timers=timers, systems=systems,
                                             margins=(i == 0))
        if os.environ.get("D3M_BENCH_DEBUG"):
            _c = _dl.counters_read()
            _dl.counters_reset(False)
            print(which, i, {k: round(v * 1e3, 1) for k, v in timers.items()},
                  {k: round(v, 1) for k, v in _c["union_ms"].items()}, file=sys.stderr, flush=True)
        if i == 0:
            sub = [s.factor.margin for s in systems]
            margins = {"subdomain_decision_margin": min(m[0] for m in sub),
                       "subdomain_argmax_gap": min(m[1] for m in sub),
                       "k_decision_margin": F.stats.decision_margin, "k_argmax_gap": F.stats.argmax_gap,
                       "tracked_in": "the warm-up run"}
        if i > 0 and (best is None or timers["d3m_total"] < best["d3m_total"]):
            best = timers
        keep = "solution" if systems[0].factor.released else "factor"
        del F
        torch.cuda.synchronize()
    res = fem3d.global_residual(model, sol, rhs=None)
    r = int(model.f.shape[1])
    ms_sub = [sum(int(np.shape(c.D)[1]) for c in s.couplings) for s in systems]
    # algorithmic: complex symmetric LDL^T 4n^3/3 + the (m+r)-RHS solves 8n^2(m+r);
    # D^T X is a sparse product (D = s M_Gamma on interface rows) and not counted
    flops_sub = sum(4 * s.n_dofs ** 3 // 3 + 8 * s.n_dofs ** 2 * (m + r) for s, m in zip(systems, ms_sub))
    sub_tf = flops_sub / best["reduce"] / 1e12
    out = {"workload": f"{which}: {cfg.cells}^3 hex x6 tets Nedelec, {cfg.parts} subdomains, "
                       f"{model.mesh.n_edges} edges, lambda={int(R.interface_sizes.sum())}, {r} RHS",
           "d3m_ms": round(best["d3m_total"] * 1e3, 1),
           "stage_ms": {k: round(v * 1e3, 1) for k, v in best.items() if k not in ("front_end", "d3m_total")},
           "subdomain_tflops": round(sub_tf, 2),
           "roofline": {"bound": "tensor", "stage": "reduce (subdomain BK + solves, incl. H2D)",
                        "achieved": round(sub_tf, 2), "peak": round(peak, 2), "unit": "TFLOP/s",
                        "frac": round(sub_tf / peak, 4),
                        "note": "algorithmic flops (4n^3/3 + 8n^2(m+r)) over the reduce stage's wall time"},
           "margins": margins,
           "subdomain_flops": int(flops_sub), "n_subdomain": sorted({s.n_dofs for s in systems}),
           "keep": keep, "residual": res,
           "note": "wall clock with device syncs; reduce includes the sparse-block H2D, recover the D2H"}
    del systems
    return out


def _cfg3_secondary(steps: int, peak: float) -> dict:
    """BASELINE configs[2]: batched Schur complement of 64 subdomains
    (n = 2048, m = 384); the workload's output is K_D / g_d only, so the
    reduction runs in its Schur-only form (keep="schur": forward sweep,
    K = Z_D^T D^-1 Z).  Device-resident inputs for the timed value; the
    public API from numpy inputs for e2e."""
    import torch
    import paper_2002_05018_b200 as d
    from paper_2002_05018_b200 import workloads as wl
    from paper_2002_05018_b200.device import DeviceArray, to_device
    host = wl.config3_systems(64)
    dev = [d.SubdomainSystem(s.domain, DeviceArray(to_device(s.A)), DeviceArray(to_device(s.f)), s.dof_map,
                             [d.Coupling(c.interface, DeviceArray(to_device(c.D)), c.sign) for c in s.couplings])
           for s in host]
    n, m, B = 2048, 384, 64
    # flops of the reference's algorithm (an effective rate for the Schur-only
    # form, which runs the forward sweep plus Z_D^T D^-1 Z instead of both
    # sweeps): complex symmetric LDL^T 4n^3/3 (SURVEY 8(d)'s 8n^3/3 is the LU
    # count) + the (m+1)-RHS solves 8n^2(m+1); D^T X for +-1 selectors is a gather
    flops = B * (4 * n ** 3 // 3 + 8 * n * n * (m + 1))
    for s in dev:
        s._d3m_D = None
    d.reduce_domains(dev, keep="schur")
    torch.cuda.synchronize()
    s0 = torch.cuda.current_stream()
    gc.collect()
    # one event pair per step, median over the steps: single steps on this pool stall by 20-40 ms now
    # and then (host-side, with and without any of this round's kernels: tools/_sec2-style repeats)
    samples = []
    for _ in range(max(steps, 9)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for s in dev:
            s.factor = None
            s._d3m_D = None
        e0.record(s0)
        red = d.reduce_domains(dev, keep="schur")
        e1.record(s0)
        torch.cuda.synchronize()
        samples.append(e0.elapsed_time(e1))
    ms = float(np.median(samples))
    # e2e: pinned host inputs (A, D, f as pinned torch CPU tensors), copied
    # inside the timed region; all K_D / g_d read back to numpy
    host_p = [d.SubdomainSystem(s.domain, torch.from_numpy(s.A).pin_memory(),
                                torch.from_numpy(np.ascontiguousarray(s.f)).pin_memory(), s.dof_map,
                                [d.Coupling(c.interface, torch.from_numpy(np.ascontiguousarray(c.D)).pin_memory(),
                                            c.sign) for c in s.couplings]) for s in host]
    red_h = d.reduce_domains(host_p, keep="schur")               # warm-up: the same step, read-back included
    outs = [(np.asarray(K_), np.asarray(g_)) for K_, g_ in red_h]
    del red_h, outs
    torch.cuda.synchronize()
    gc.collect()
    t0 = time.perf_counter()
    red_h = d.reduce_domains(host_p, keep="schur")
    outs = [(np.asarray(K_), np.asarray(g_)) for K_, g_ in red_h]
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3
    h2d = 16 * sum(s.A.size + s.f.size + sum(c.D.size for c in s.couplings) for s in host)
    for s in dev:
        s.factor = None
        s._d3m_D = None
    d.reduce_domains(dev, keep="schur", margins=True)            # untimed: pivot-decision margins
    mg = [s.factor.margin for s in dev]
    value = flops / (ms * 1e-3) / 1e12
    out = {"workload": "cfg3: 64 subdomains, n=2048, m=384 (A_i=(M+M^T)/2, D_i one +-1 per column), K_D and g_d",
           "ms_per_step": round(ms, 3), "statistic": "median", "samples_ms": [round(v, 1) for v in samples],
           "value": round(value, 3), "unit": "TFLOP/s",
           "roofline": {"bound": "tensor", "achieved": round(value, 3), "peak": round(peak, 2), "unit": "TFLOP/s",
                        "frac": round(value / peak, 4),
                        "note": "effective: the reference algorithm's flops (4n^3/3 + 8n^2(m+1)) / device time"},
           "margins": {"decision_margin": min(m[0] for m in mg), "argmax_gap": min(m[1] for m in mg)},
           "flops_per_step": flops, "e2e": {"ms_per_step": round(e2e_ms, 1), "h2d_bytes_per_step": int(h2d),
                                             "d2h_bytes_per_step": int(16 * B * m * (m + 1))}}
    del red, red_h, host_p, outs
    return out


def _refine_leg(d, F, K, rhs, rhs_d) -> dict:
    """block_solve alone vs block_solve(refine=1) on the last factor (CUDA
    events, device-resident RHS), with the residual of each, next to the
    reference's own residual on the same system (tests/golden)."""
    import torch
    s = torch.cuda.current_stream()
    out = {}
    for refine in (0, 1):
        x = d.block_solve(F, rhs_d, refine=refine)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(3):
            x = d.block_solve(F, rhs_d, refine=refine)
        e1.record(s)
        torch.cuda.synchronize()
        out[f"solve_refine{refine}_ms"] = round(e0.elapsed_time(e1) / 3, 3)
        out[f"residual_refine{refine}"] = _residual(K, rhs, [np.asarray(v) for v in x])
    try:
        g = np.load(os.path.join(ROOT, "tests", "golden", "cfg4_residuals.npz"))
        out["reference_residual_max"] = float(g["residual"].max())
    except OSError:
        pass
    out["note"] = ("block_solve(F, g, refine=1): one fixed-precision refinement step, K x on the tensor pipe "
                   "from the factor's device copy of K; the headline step runs refine=1; refine=0 is the reference's algorithm")
    return out


def _residual(K, rhs, x) -> float:
    """max over RHS of ||K x - b|| / ||b|| (block matvec on the host)."""
    sizes = K.sizes
    Kx = [np.zeros_like(b) for b in rhs]
    for (i, j), blk in K.blocks.items():
        B = np.asarray(blk)
        Kx[i] += B @ x[j]
        if i != j:
            Kx[j] += B.T @ x[i]
    num = np.sqrt(sum(np.sum(np.abs(Kx[i] - rhs[i]) ** 2, axis=0) for i in range(len(sizes))))
    den = np.sqrt(sum(np.sum(np.abs(rhs[i]) ** 2, axis=0) for i in range(len(sizes))))
    return float((num / den).max())


def _column_flops(sizes, pattern, columns) -> int:
    """Algorithmic flops of the first `columns` block columns, counted as the
    GPU side counts them (factor._Schedule): BK 4n^3/3 (complex symmetric
    LDL^T), panel TRSM 4 R_j n_j^2, trailing updates 8 n_i n_k n_j (4 n_i^2 n_j
    for diagonal targets)."""
    fl = 0
    for j in range(columns):
        nj = int(sizes[j])
        rows = [int(i) for i in pattern[j]]
        fl += 4 * nj ** 3 // 3 + 4 * sum(int(sizes[i]) for i in rows) * nj * nj
        for a, i in enumerate(rows):
            for kk in rows[:a + 1]:
                fl += (8 if i != kk else 4) * int(sizes[i]) * int(sizes[kk]) * nj
    return fl


class _AllHostThreads:
    """BLAS on every host core for the CPU legs.  torchrun exports
    OMP_NUM_THREADS=1 to its workers, which OpenBLAS would obey: the reference
    arm at N > 1 would then run on one thread while reporting all cores.
    `threads` is what the BLAS pool reports inside the block."""

    def __enter__(self):
        import threadpoolctl
        self._lim = threadpoolctl.threadpool_limits(limits=os.cpu_count() or 1)
        self._lim.__enter__()
        blas = [p["num_threads"] for p in threadpoolctl.threadpool_info() if p.get("user_api") == "blas"]
        self.threads = max(blas) if blas else 1
        return self

    def __exit__(self, *exc):
        return self._lim.__exit__(*exc)


def _cpu_full_cfg4(plan, K, rhs, flops_step, gpu_ms):
    """The oracle port (C restatement of the reference's numba kernels +
    numpy/OpenBLAS ZGEMM on all host threads, the reference's own algorithm
    and drivers) running the SAME step as the GPU: the full block LDL^T of
    config 4 and the 16-RHS block solve, timed once on the host cores."""
    from oracle import d3m_oracle as O
    adj = O.clique_adjacency(K.nblocks, K.blocks.keys())
    oplan = O.symbolic_factor(adj, plan.order.perm, K.sizes)
    blocks = {k: np.asarray(v) for k, v in K.blocks.items()}
    with _AllHostThreads() as pool:
        O.block_ldlt(blocks, oplan, columns=1)          # warm (loads the C kernels)
        t0 = time.perf_counter()
        F = O.block_ldlt(blocks, oplan)
        t1 = time.perf_counter()
        O.block_solve(F, rhs)
        t2 = time.perf_counter()
    del F
    dt = t2 - t0
    return {"value": round(flops_step / dt / 1e12, 6), "unit": "TFLOP/s", "cores": pool.threads,
            "kind": "port", "seconds": round(dt, 2), "factor_s": round(t1 - t0, 2), "solve_s": round(t2 - t1, 2),
            "gpu_speedup_device_resident": round(dt / (gpu_ms * 1e-3), 1),
            "sample": "the full cfg4 step (block LDL^T of all 144 block columns + 16-RHS block solve, "
                      f"{flops_step / 1e12:.2f} TFLOP counted as the GPU counts them), oracle port with OpenBLAS "
                      "ZGEMM on all host threads, one run"}


def _cpu_reduce_worker(job):
    """One subdomain's reduce_domain (subdomain.py:166-184) by the oracle
    port, in a spawned process (OpenBLAS single-threaded)."""
    cfg, idx = job
    sys.path.insert(0, ROOT)
    from oracle import d3m_oracle as O
    if cfg == "cfg3":
        from paper_2002_05018_b200 import workloads as wl
        A, D, f = wl.config3_domain(idx)
    else:
        from paper_2002_05018_b200 import fem3d
        model = fem3d.build_model(getattr(fem3d, "config1" if cfg == "cfg1" else "config2")())
        s = fem3d.subdomain_systems(model, rhs=0, sparse=False)[idx]
        A, f = np.asarray(s.A), np.asarray(s.f)
        D = np.concatenate([np.asarray(c.D) for c in s.couplings], axis=1)
    O.dense_ldlt_bk(np.eye(2, dtype=complex))       # load the C kernels
    t0 = time.perf_counter()
    O.reduce_domain(A, D, f)
    return time.perf_counter() - t0


def _cpu_reduce_pool(cfg, indices, gpu_ms, total=None):
    """Same-run CPU timing of the subdomain reduction: the
    oracle port's reduce_domain on `indices` subdomains in a pool of
    single-threaded processes (subdomains are independent),
    extrapolated to all `total` subdomains at the same pool width."""
    import multiprocessing as mp
    procs = max(1, min(len(indices), os.cpu_count() or 1))
    old = os.environ.get("OPENBLAS_NUM_THREADS")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        with mp.get_context("spawn").Pool(procs) as pool:
            t0 = time.perf_counter()
            secs = pool.map(_cpu_reduce_worker, [(cfg, i) for i in indices])
            wall = time.perf_counter() - t0
    finally:
        if old is None:
            os.environ.pop("OPENBLAS_NUM_THREADS", None)
        else:
            os.environ["OPENBLAS_NUM_THREADS"] = old
    total = total or len(indices)
    per = float(np.mean(secs))
    waves = -(-total // procs)
    est = waves * max(secs) if total != len(indices) else max(secs)
    return {"kind": "port", "procs": procs, "cores": os.cpu_count(), "subdomains_timed": len(indices),
            "s_per_subdomain": round(per, 2), "wall_s": round(wall, 2),
            "all_subdomains_s": round(est, 1), "extrapolated": total != len(indices),
            "gpu_speedup": round(est / (gpu_ms * 1e-3), 1),
            "note": f"oracle reduce_domain per subdomain in {procs} single-threaded processes"
                    + (f"; {total} subdomains = {waves} waves of the slowest timed one" if total != len(indices)
                       else "")}


def run_reference(args):
    """CPU reference arm: the oracle port on rank 0, same metric."""
    dist, rank, ws = _dist()
    if rank != 0:
        return
    K, plan, rhs = _cfg4_host()
    from oracle import d3m_oracle as O
    adj = O.clique_adjacency(K.nblocks, K.blocks.keys())
    oplan = O.symbolic_factor(adj, plan.order.perm, K.sizes)
    blocks = {k: np.asarray(v) for k, v in K.blocks.items()}
    cols = args.cpu_sample_columns
    fl = _column_flops(oplan["sizes_perm"], oplan["pattern"], cols)
    with _AllHostThreads() as pool:
        for _ in range(args.warmup):
            O.block_ldlt(blocks, oplan, columns=cols)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            O.block_ldlt(blocks, oplan, columns=cols)
        dt = (time.perf_counter() - t0) / args.steps
    value = fl / dt / 1e12
    sample = (f"first {cols} of 144 block columns of the cfg4 block LDL^T per step ({fl / 1e9:.2f} GFLOP), "
              "oracle port (C restatement of the numba kernels + numpy/OpenBLAS ZGEMM, all host threads)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded, workloads.config4_matrix)", "config": {"workload": WORKLOAD},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": pool.threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-columns", type=int, default=CPU_SAMPLE_COLUMNS)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU legs (cpu_baseline, cfg1/cfg3 CPU reduce)")
    ap.add_argument("--no-cfg3", action="store_true", help="skip the secondary config-3 measurement")
    ap.add_argument("--no-fem", action="store_true", help="skip the FEM config-1/2 secondaries")
    ap.add_argument("--no-cfg5", action="store_true", help="skip FEM config 5 (~30 s, ~150 GB HBM)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
