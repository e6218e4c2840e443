"""Benchmark: DOF-updates/s per RK stage of the fused fp64 SSPRK3 DG
shallow-water step on B200 (BASELINE.json metric), with the roofline, the
CPU oracle baseline, an end-to-end host-buffer number and clock samples.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c4]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference ...     (CPU reference arm)

Workload (default, config C3 of BASELINE.json): Williamson TC6
Rossby-Haurwitz wave, p=3 (order 4), 720x360 elements, 12,441,600 DOF,
SSPRK3 with dt = 5e-3 s; synthetic = the analytic TC6 initial condition
projected on the mesh (no dataset).  N>1: the same grid split into
latitude bands (strong scaling), one process per GPU, NCCL halo exchange.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (case, nx, ny, p, dt, label)
    "c3": ("williamson_tc6", 720, 360, 3, 5e-3, "C3: Williamson TC6, order 4 (p=3), 720x360, SSPRK3"),
    "c2": ("williamson_tc2", 360, 180, 3, 0.05, "C2: Williamson TC2, order 4 (p=3), 360x180, SSPRK3"),
    "c4": ("williamson_tc5", 1440, 720, 4, 5e-4,
           "C4: Williamson TC5 (flow over an isolated mountain; orography is an extension of the "
           "reference), order 5 (p=4), 1440x720, SSPRK3"),
    "c4tc6": ("williamson_tc6", 1440, 720, 4, 5e-4,
              "C4 shape with the TC6 IC (no orography): order 5 (p=4), 1440x720, SSPRK3"),
}
# C5: order sweep 1..6 (p = 0..5) at ~1e9 DOF (SURVEY 8d grids, nx = 2 ny); one
# GPU holds the three ~8 GB states; the initial condition is projected on
# the device (host projection of 1e9 DOF is impractical)
for _p, (_nx, _ny) in enumerate([(25856, 12928), (12928, 6464), (8576, 4288), (6400, 3200),
                                 (5120, 2560), (4352, 2176)]):
    CONFIGS[f"c5p{_p}"] = ("williamson_tc6", _nx, _ny, _p, 1e-5,
                           f"C5 order sweep: order {_p + 1} (p={_p}), {_nx}x{_ny}, "
                           f"{_nx * _ny * (_p + 1) ** 2 * 3 / 1e9:.2f}e9 DOF, SSPRK3, TC6 IC")
METRIC = "DOF-updates/sec (fp64, per RK stage)"
UNIT = "DOF-updates/s"
B_ALG = 64.0 / 3.0          # algorithmic HBM bytes per DOF-update, SSPRK3 Shu-Osher


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region.

    Started before the warm-up, so the NVML start-up of nvidia-smi is not
    inside the timed region; every line is stamped on arrival and
    ``summary(t0, t1)`` keeps the samples taken while the timed region ran
    (20 ms period: several samples even in a 40 ms region)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        lines = self.lines
        if t0 is not None:
            # a sample is printed up to one period after it is taken
            inside = [ln for ts, ln in lines if t0 <= ts <= t1 + 0.03]
            later = [ln for ts, ln in lines if ts > t1 + 0.03][:1]
            lines = inside or later
        else:
            lines = [ln for _, ln in lines]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_oracle_rate(case, nx, ny, p, dt, budget_s=12.0, max_steps=None):
    """The CPU oracle (bit-exact C port of the reference path, OpenMP over
    all host threads) on the same workload; returns (rate, steps, seconds, threads)."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from oracle import oracle as O
    t, orc, X = O.build_case(case, nx, ny, p)
    threads = O.max_threads()
    dofs = nx * ny * (p + 1) ** 2 * 3
    orc.rk_steps(X, dt, 3, 1)                       # warm-up (page-in, threads)
    steps, t0 = 0, time.perf_counter()
    while True:
        X, st, _ = orc.rk_steps(X, dt, 3, 1)
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (max_steps and steps >= max_steps):
            break
    return dofs * 3 * steps / el, steps, el, threads


def host_cpu():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


REF_PY = r"""
import json, sys, time
from dgswe import cases, dg, timestep
case, nx, ny, p, dt, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5]), int(sys.argv[6])
setup = cases.build_case(cases.default_config(case).override(nx=nx, ny=ny, p=p))
op = dg.SpatialOperator(setup.mesh, p, setup.model)
st = op.project_state(setup.ic)
tab = timestep.tableau(3)
ws = timestep._RKWorkspace(st, tab.s)
timestep.rk_step(st, op.assemble_rhs, dt, tab, ws)          # warm-up (numba JIT)
t0 = time.perf_counter()
for _ in range(steps):
    timestep.rk_step(st, op.assemble_rhs, dt, tab, ws)
el = time.perf_counter() - t0
print(json.dumps({"seconds": el, "steps": steps}))
"""


def reference_python_rate(case, nx, ny, p, dt, steps):
    """The UNMODIFIED reference (pip-installed into baseline/_ref, pure
    Python + numba, single-threaded by construction) on one pinned core:
    rk_step(state, op.assemble_rhs, dt, tableau(3)) (timestep.py:149-167)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if case not in ("williamson_tc2", "williamson_tc6"):
        return {"unavailable": f"{case} is not a case of the reference (no orography)"}
    if not os.path.isdir(os.path.join(ref, "dgswe")):
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref)"}
    env = dict(os.environ, PYTHONPATH=ref, NUMBA_CACHE_DIR="/tmp/dgswe_numba_cache",
               OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
               NUMBA_NUM_THREADS="1")
    cmd = [sys.executable, "-c", REF_PY, case, str(nx), str(ny), str(p), repr(dt), str(steps)]
    if os.path.exists("/usr/bin/taskset"):
        cmd = ["taskset", "-c", "0"] + cmd
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
        out = json.loads(res.stdout.strip().splitlines()[-1])
    except Exception as exc:                          # noqa: BLE001
        return {"unavailable": f"reference run failed: {exc}"}
    dofs = nx * ny * (p + 1) ** 2 * 3
    return {"value": dofs * 3 * out["steps"] / out["seconds"], "unit": UNIT, "cores": 1,
            "kind": "reference",
            "sample": f"{out['steps']} rk_step(tableau(3)) steps of the same grid after 1 warm-up step, "
                      "unmodified reference package (baseline/_ref), pinned to one core",
            "host": host_cpu()}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    case, nx, ny, p, dt, label = CONFIGS[args.config]
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from oracle import oracle as O
    t, orc, X = O.build_case(case, nx, ny, p)
    threads = O.max_threads()
    dofs = nx * ny * (p + 1) ** 2 * 3
    for _ in range(args.warmup):
        X, _, _ = orc.rk_steps(X, dt, 3, 1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        X, _, _ = orc.rk_steps(X, dt, 3, 1)
    el = time.perf_counter() - t0
    value = dofs * 3 * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic Williamson initial condition projected on the mesh)",
        "config": {"workload": label, "case": case, "nx": nx, "ny": ny, "p": p, "dofs": dofs,
                   "dt": dt, "rk": "SSPRK3 (tableau(3), Butcher form)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full SSPRK3 steps of the {args.config.upper()} "
                                   f"grid after {args.warmup} warm-up steps; oracle/dgswe_oracle.c "
                                   "(bit-exact C port of the reference RHS/RK, OpenMP)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": host_cpu(),
    }
    if not args.no_ref_python:
        line["reference_python"] = reference_python_rate(case, nx, ny, p, dt, args.ref_steps)
    print(json.dumps(line), flush=True)


def load_traffic(config):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
        return d.get(config)
    except (OSError, ValueError):
        return None


def run_gpu(args):
    import torch
    import torch.distributed as dist
    import paper_2303_11767_b200 as P
    from paper_2303_11767_b200.bands import BandLayout, BandOperator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    same_gpu = os.environ.get("DGSWE_BENCH_SAME_GPU") == "1"   # test mode: all ranks on GPU 0
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    case, nx, ny, p, dt, label = CONFIGS[args.config]
    setup = P.build_case(P.default_config(case).override(nx=nx, ny=ny, p=p))
    op = P.SpatialOperator(setup.mesh, p, setup.model)
    dofs = nx * ny * (p + 1) ** 2 * 3
    big = args.config.startswith("c5")
    state = op.project_state(setup.ic, device=big)
    stream = torch.cuda.current_stream()

    if world == 1:
        def steps(k):
            op.ssprk3_steps(state, dt, k)
        counter = op.launch_count
        state_bytes = state.data.numel() * 8
    else:
        L = BandLayout(ny, world, rank)
        full = state.data.cpu().numpy()
        transport = os.environ.get("DGSWE_BAND_TRANSPORT", "fused")
        ok, bop = 1, None
        if transport == "fused":
            try:
                bop = BandOperator(op, L, transport="fused")
                u = bop.empty()
                u.copy_(torch.from_numpy(L.scatter(full)))
                w1, w2 = bop.empty(), bop.empty()
                bop.attach(u, w1, w2)
            except Exception as exc:                 # no peer mappings on this rank
                log(f"rank {rank}: fused exchange unavailable ({exc})")
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:                # every rank falls back together
                if bop is not None:
                    torch.cuda.synchronize()
                    bop.close()
                transport = "p2p"
        if transport != "fused":
            bop = BandOperator(op, L, transport="p2p")
            u = torch.from_numpy(L.scatter(full)).cuda()
            w1, w2 = bop.empty(), bop.empty()
        del state
        graphs = {}
        replayed = [0]                               # kernel launches inside graph replays

        def steps(k):
            if transport != "fused":
                return bop.ssprk3_steps(u, w1, w2, dt, k)
            # no host collective inside the fused steps: K nodal steps replay
            # as one CUDA graph between the batch's conversions
            bop.begin(u)
            if k not in graphs:
                bop.nodal_steps(u, w1, w2, dt, 1)       # eager warm-up of the launch path
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                c0 = bop.launch_count()
                with torch.cuda.graph(g):
                    bop.nodal_steps(u, w1, w2, dt, k)
                graphs[k] = (g, bop.launch_count() - c0)
                replayed[0] -= graphs[k][1]             # counted at capture, run at replay
            g, n = graphs[k]
            g.replay()
            replayed[0] += n
            bop.end(u)
        counter = lambda: bop.launch_count() + replayed[0]   # noqa: E731
        state_bytes = u.numel() * 8

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up (also builds the CUDA graph for k = steps); the clock sampler
    # starts here so its start-up is outside the timed region
    clk = ClockSampler(local).__enter__()
    steps(args.warmup)
    steps(args.steps)
    torch.cuda.synchronize()
    barrier()

    # timed region: K steps, device events, max over ranks
    n0 = counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    t_in = time.time()
    ev0.record(stream)
    steps(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    t_out = time.time()
    barrier()
    clk.__exit__(None, None, None)
    clocks = clk.summary(t_in, t_out)
    launches = counter() - n0
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    if world == 1:
        flags, _ = op.status()
    else:
        flags, _ = bop.status()
    if flags:
        raise SystemExit(f"device status flags {flags:#x} during the bench")
    value = dofs * 3 * args.steps / (ms * 1e-3)

    # per-stage launch times (event-timed, same stream, individual launches)
    per_stage = None
    if world == 1:
        w1, w2 = torch.zeros_like(state.data), torch.zeros_like(state.data)
        s1 = P.State(w1, nx, ny, 1, op.nphi)
        s2 = P.State(w2, nx, ny, 1, op.nphi)
        reps = 20
        times = {1: [], 2: [], 3: []}
        ctx = op._ctx
        ctx.convert(state.data, True, 0, ny)         # the stages alone, on nodal states
        ctx.set_basis(True)
        for _ in range(reps):
            for k, fn in ((1, lambda: op.stage(0.0, None, 1.0, state, dt, s1)),
                          (2, lambda: op.stage(0.75, state, 0.25, s1, 0.25 * dt, s2)),
                          (3, lambda: op.stage(1 / 3, state, 2 / 3, s2, 2 / 3 * dt, state))):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                times[k].append((a, b))
        ctx.set_basis(False)
        ctx.convert(state.data, False, 0, ny)
        torch.cuda.synchronize()
        per_stage = {k: statistics.median(a.elapsed_time(b) for a, b in v) for k, v in times.items()}
        flags, _ = op.status()
        assert flags == 0

    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    local_dofs = dofs // world
    stage_ms = ms / (3 * args.steps)                 # stages + the batch's two basis conversions
    achieved = local_dofs * B_ALG / (stage_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": load_traffic(args.config),
                "kernel": f"dgswe::stage_kernel<{p}>",
                "alg_bytes_per_launch": local_dofs * B_ALG,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}
    if per_stage:
        roofline["per_stage_ms"] = per_stage
        roofline["per_stage_gbs"] = {
            k: local_dofs * (16.0 if k == 1 else 24.0) / (v * 1e-3) / 1e9 for k, v in per_stage.items()}

    # the reference's own entry point on a device state: rk_step(state,
    # op.assemble_rhs, dt, tableau(3)) -- three stage kernels per step on the
    # state's nodal values (converted once, back when read) and the per-step
    # status read the reference's exceptions need (timestep.py:149-167)
    api = None
    if world == 1 and not args.no_api and not big:
        tab = P.tableau(3)
        st_api = P.State(state.data.clone(), nx, ny, 1, op.nphi)
        ws = P.stepping._RKWorkspace(st_api, tab.s)
        for _ in range(3):
            P.rk_step(st_api, op.assemble_rhs, dt, tab, ws)
        torch.cuda.synchronize()
        k3 = max(3, min(args.steps, 50))
        n_api = op.launch_count()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(k3):
            P.rk_step(st_api, op.assemble_rhs, dt, tab, ws)
        a1.record(stream)
        torch.cuda.synchronize()
        ms_api = a0.elapsed_time(a1) / k3
        ach = dofs * B_ALG / (ms_api / 3 * 1e-3) / 1e9
        api = {"path": "rk_step(state, op.assemble_rhs, dt, tableau(3)): 3 stage kernels (one CUDA graph replay) on the "
                       "lazily converted nodal state + 1 status read (host sync) per step",
               "value": dofs * 3 / (ms_api * 1e-3), "unit": UNIT,
               "ms_per_step": ms_api, "steps": k3, "gpu_launches": op.launch_count() - n_api,
               "achieved_gbs": ach, "frac": ach / measured_peaks().get("hbm_gbs", 6650.0)}
        del st_api, ws

    # end to end through the public API with host buffers: every step copies
    # the state from pinned host memory, runs one fused SSPRK3 step and reads
    # the result back (the reference's rk_step contract on a host state)
    e2e = None
    if big:
        pass                                         # 8 GB states: no host round trips
    elif world == 1:
        host = torch.empty_like(state.data, device="cpu").pin_memory()
        host.copy_(state.data)
        op.ssprk3_step_host(host, dt)                # warm-up (streams, buffers)
        torch.cuda.synchronize()
        k2 = max(3, min(args.steps, 20))
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k2):
            # the whole state host -> device, one SSPRK3 step, result device -> host,
            # row-pipelined (SpatialOperator.ssprk3_step_host)
            op.ssprk3_step_host(host, dt)            # one CUDA graph per step (captured in warm-up)
            flags, _ = op.status()                   # syncs: the step's result is on the host
            if flags:
                raise SystemExit(f"device status flags {flags:#x} in the e2e loop")
        e1.record(stream)
        torch.cuda.synchronize()
        el = e0.elapsed_time(e1) * 1e-3
        e2e = {"value": dofs * 3 * k2 / el, "unit": UNIT, "h2d_bytes_per_step": state_bytes,
               "d2h_bytes_per_step": state_bytes, "steps": k2,
               "path": "pinned host state -> SpatialOperator.ssprk3_step_host (C ABI row stages, copies overlapped in 16 latitude chunks) -> pinned host, per step",
               "wall_s": time.perf_counter() - t0}
    else:
        host = u.cpu().pin_memory()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k2 = max(3, min(args.steps, 20))
        e0.record(stream)
        for _ in range(k2):
            u.copy_(host, non_blocking=True)
            bop.ssprk3_step(u, w1, w2, dt)
            host.copy_(u, non_blocking=True)
            bop.status()
        e1.record(stream)
        torch.cuda.synchronize()
        el = max_over_ranks(e0.elapsed_time(e1)) * 1e-3
        e2e = {"value": dofs * 3 * k2 / el, "unit": UNIT, "h2d_bytes_per_step": state_bytes,
               "d2h_bytes_per_step": state_bytes, "steps": k2}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not big:
        rate, n, el, threads = cpu_oracle_rate(case, nx, ny, p, dt, budget_s=args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{n} full SSPRK3 steps of the same {args.config.upper()} grid "
                         f"({el:.1f} s) with the bit-exact C port of the reference path "
                         "(oracle/dgswe_oracle.c, OpenMP)",
               "host": host_cpu()}
        if not args.no_ref_python:
            cpu["reference_python"] = reference_python_rate(case, nx, ny, p, dt, args.ref_steps)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic Williamson initial condition projected on the mesh)",
            "config": {"workload": label, "case": case, "nx": nx, "ny": ny, "p": p, "dofs": dofs,
                       "dt": dt, "rk": "SSPRK3, Shu-Osher fused stages (== tableau(3))",
                       "parallelism": (f"latitude bands x{world}, halo exchange: {transport}"
                                       if world > 1 else "single GPU"),
                       "l2": f"no flush; per-stage working set {3 * dofs * 8 / 1e6:.0f} MB "
                             f"(3 states) > 126 MB L2" if args.config != "c2" else
                             "C2 states (25 MB each) fit in L2; roofline inflated"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "api_rk_step": api,
            "clocks": clocks, "gpu_launches": int(launches),
            "dofs_per_gpu": local_dofs, "per_gpu_value": value / world,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ref-python", action="store_true",
                    help="skip timing the unmodified Python reference (baseline/_ref)")
    ap.add_argument("--ref-steps", type=int, default=2, help="timed steps of the Python reference")
    ap.add_argument("--no-api", action="store_true", help="skip the rk_step (reference API) timing")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
