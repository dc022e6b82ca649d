"""bench.py — J.v residual evaluations per second on the 1M-cell config (BASELINE configs[1]),
achieved HBM GB/s against the measured B200 peak, the end-to-end J.v through the C-ABI
with host buffers, the device JFNK solve time at 1M cells, and the reference CPU solver
timed on this box's host cores.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2] [--no-jfnk] [--no-cpu]

One step = one J.v = (R(u + eps v) - R(u)) / eps over the whole mesh (inputs resident in
HBM).  The J.v working set (~0.45-0.65 GB at 1M cells) exceeds the 126 MB L2, so no L2
flush is needed between steps.  Multi-GPU (torchrun): the path does not shard with parity
 — N independent replicas, value = total J.v/s over ranks, max-over-ranks
device time ("replicas only").
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "J·v residual evals/s + achieved HBM GB/s; JFNK solve time at 1M cells"
UNIT = "J·v/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def max_over_ranks(x: float, device: str = "cuda") -> float:
    """Max of a per-rank scalar over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(steps_per_rank: int, ms_max: float, world: int) -> float:
    """Whole-job J.v/s of N independent replicas timed by the slowest rank."""
    return world * steps_per_rank / (ms_max / 1e3)


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_jv(case, mesh, u, r_u, v, n_jv: int, warm: int = 1):
    """The reference's own jacobian_vector_product (oracle/_ref: /root/reference/proj/src
    compiled by oracle/Makefile) on the host cores.  The reference is single-threaded
    (SPEC.md:390), so n_jv independent J.v calls on the same const evaluator run spread over
    all host threads (at most 32), each thread at least one.  ONE definition for both the
    reference arm and the GPU arm's cpu_baseline: value = J.v completed / wall seconds of the
    timed region, ms_per_step = wall ms / J.v completed (so steps * ms_per_step = the timed
    region).  Falls back to the C restatement (1 thread) when the reference build is absent."""
    from oracle.bind import OracleCase, RefCase, ref_available
    if ref_available():
        threads = min(os.cpu_count() or 1, 32)
        rc = RefCase(mesh, case.physics)
        rc.set_time(1.0)
        per_thread = max(1, -(-n_jv // threads))
        rc.time_jv(u, r_u, v, max(1, warm), threads)
        secs = rc.time_jv(u, r_u, v, per_thread, threads)
        done = per_thread * threads
        kind, what = "reference", "the reference's jacobian_vector_product (oracle/_ref)"
    else:
        threads = 1
        oc = OracleCase(mesh, case.physics)
        oc.set_time(1.0)
        oc.time_jv(u, r_u, v, 1)
        done = max(1, min(n_jv, 20))
        secs = oc.time_jv(u, r_u, v, done)
        kind, what = "port", "the C restatement (oracle/sfv_oracle.c)"
    return {"value": done / secs, "unit": UNIT, "cores": threads, "kind": kind, "jv_done": done,
            "seconds": secs, "ms_per_jv": 1e3 * secs / done, "cpu_model": _cpu_model(),
            "host_threads": os.cpu_count(),
            "sample": f"{done} J.v of {what} on the full {mesh.n_cells}-cell mesh, {threads} host threads "
                      f"running concurrent independent calls ({-(-done // threads)} each)"}


def reference_jfnk_sample(case, mesh, cycles: int = 1):
    """A bounded sample of the reference's JFNK solve at this config (nonlinear.cpp:173-266
    with the automatic preconditioner of run_steps, nonlinear.cpp:382-446): the preconditioner
    setup (J~ assembly + ILU(1) factor, timed alone) and the first `cycles` GMRES(30) restart
    cycles of the first Newton step, timed through jfnk_solve.  The full solve time is
    projected from them with the Krylov count of the full solve and, when a full reference
    run on this kind of host was recorded (profiles/r02_ref_jfnk_<cfg>.json), quoted."""
    from oracle.bind import RefCase, ref_available
    from paper_2502_17217_b200.abi import solver_cfg
    if not ref_available():
        return None
    ref = RefCase(mesh, case.physics)
    ref.set_time(1.0 / case.n_steps)
    kind = "lu" if 3 * mesh.n_cells <= 30000 else "ilu1"  # make_preconditioner's automatic rule
    t0 = time.perf_counter()
    ref.precond_create({"lu": 5, "ilu1": 3}[kind])
    setup = time.perf_counter() - t0
    kr = 30 * cycles
    cfg = solver_cfg(r_tol=case.r_tol, max_outer=1, max_krylov=kr, preconditioner=kind)
    u0 = case.initial_field(mesh)[0]
    t0 = time.perf_counter()
    _, rep = ref.jfnk_solve(u0, cfg)
    t_it = time.perf_counter() - t0
    iters = max(1, int(rep.krylov_iters))
    # jfnk_solve's other work in the sample: R(u0) and one line-search residual (~2 J.v)
    return {"precond": kind, "precond_setup_s": setup, "sample_krylov": iters, "sample_s": t_it,
            "per_krylov_s": t_it / iters, "cores": 1, "cpu_model": _cpu_model()}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from paper_2502_17217_b200 import cases
    from oracle.bind import RefCase, OracleCase, ref_available, ref_box_mesh
    case = cases.config(args.config)
    if ref_available() and case.kind == "box":  # the reference's own generate_box_hex + distort_mesh
        ma = case.mesh_args
        mesh = ref_box_mesh(ma["extents"], ma["divisions"], ma["kinds"], ma.get("distort", 0.0), ma.get("seed", 0))
    else:
        mesh = case.mesh()
    u, v = cases.jv_inputs(mesh, extent=case.mesh_args.get("extents"))
    ref = (RefCase if ref_available() else OracleCase)(mesh, case.physics)
    ref.set_time(1.0)
    r_u = ref.residual(u)
    del ref
    jv = reference_jv(case, mesh, u, r_u, v, args.steps, args.warmup)
    n_jv = jv["jv_done"]
    line = {
        "impl": "reference", "metric": METRIC, "value": jv["value"], "unit": UNIT, "n_gpus": ws, "steps": n_jv,
        "warmup": args.warmup, "ms_per_step": jv["ms_per_jv"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {case.notes}", "cells": mesh.n_cells, "parallelism": "host threads"},
        "cpu_baseline": {k: jv[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "host_threads")},
        "e2e": {"value": jv["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "steps_requested": args.steps,
    }
    if not args.no_jfnk:
        line["jfnk"] = reference_jfnk_summary(args.config, case, mesh)
    print(json.dumps(line), flush=True)


def reference_jfnk_summary(cfg_name, case, mesh):
    try:
        s = reference_jfnk_sample(case, mesh)
    except Exception as exc:  # reported, never required
        return {"error": str(exc)}
    if s is None:
        return {"unavailable": "reference build absent"}
    prof = os.path.join(ROOT, "profiles", f"r02_ref_jfnk_{cfg_name}.json")
    if os.path.exists(prof):
        with open(prof) as f:
            full = json.load(f)
        s["recorded_full_solve"] = full
        kr = full.get("krylov_total")
        if kr:
            s["projected_solve_seconds"] = s["precond_setup_s"] + kr * s["per_krylov_s"]
    return s


def run_ours(args):
    import ctypes as C

    import torch

    from paper_2502_17217_b200 import cases
    from paper_2502_17217_b200 import solver as sv

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    case = cases.config(args.config)
    t_setup = time.time()
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    ev.set_time(1.0)
    t_setup = time.time() - t_setup
    u_h, v_h = cases.jv_inputs(mesh, extent=case.mesh_args.get("extents"))
    u = sv.to_device(u_h)
    v = sv.to_device(v_h)
    r_u = ev.residual(u)
    out = ev.empty()
    L, h = ev.L, ev.h
    stream = torch.cuda.current_stream()

    def jv_step():
        rc = L.sfv_jv_async(h, u.data_ptr(), r_u.data_ptr(), v.data_ptr(), out.data_ptr())
        if rc:
            ev._check(rc)

    for _ in range(args.warmup):
        jv_step()
    ev._check(L.sfv_check_errors(h, None))
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = ev.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.05)
        e0.record(stream)
        for _ in range(args.steps):
            jv_step()
        e1.record(stream)
        torch.cuda.synchronize()
    launches = ev.launch_count - l0
    ms = e0.elapsed_time(e1)
    ev._check(L.sfv_check_errors(h, None))
    ms = max_over_ranks(ms)
    ms_per = ms / args.steps
    value = replica_throughput(args.steps, ms, ws)
    peak, peak_kind = _peaks()
    jv_bytes = ev.jv_bytes
    achieved = jv_bytes / (ms_per / 1e3) / 1e9

    # end to end through the C-ABI with pinned host buffers: H2D u, r_u, v; J.v; D2H out
    n = ev.n
    hu = torch.from_numpy(u_h).pin_memory()
    hr = r_u.cpu().pin_memory()
    hv = torch.from_numpy(v_h).pin_memory()
    ho = torch.empty(n, dtype=torch.float64).pin_memory()
    dp = C.POINTER(C.c_double)

    def e2e_step():
        rc = L.sfv_jv_host(h, C.cast(hu.data_ptr(), dp), C.cast(hr.data_ptr(), dp), C.cast(hv.data_ptr(), dp),
                           C.cast(ho.data_ptr(), dp), None)
        ev._check(rc)

    for _ in range(2):
        e2e_step()
    e2e_n = max(3, min(args.steps, 20))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_n):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_n
    e2e_s = max_over_ranks(e2e_s)

    # per-stage device times of the same J.v (CUDA events on the context stream), and the
    # algorithmic bytes of each stage: the roofline is quoted for the dominant kernel
    import ctypes as C
    names = ["norm_partials_kernel", "perturb_kernel", "grad_cell_kernel", "boundary_kernel", "flux_pair_kernel"]
    st_ms = (C.c_double * 5)()
    st_b = (C.c_double * 5)()
    L.sfv_jv_stage_bytes(h, st_b)
    ev._check(L.sfv_jv_stage_times(h, u.data_ptr(), r_u.data_ptr(), v.data_ptr(), out.data_ptr(),
                                   max(5, min(args.steps, 50)), st_ms))
    if st_b[0] == 0:  # the ε reduction is fused into the perturb pass (default)
        names[1] = "eps_perturb_kernel"
    stages = [{"kernel": names[k], "ms": st_ms[k], "bytes": st_b[k],
               "GBps": st_b[k] / (st_ms[k] / 1e3) / 1e9 if st_ms[k] > 0 else None} for k in range(5)
              if st_b[k] > 0]  # fused-away stages (eps reduction, boundary faces) move no bytes of their own
    top_st = max(stages, key=lambda d: d["ms"])
    top = names.index(top_st["kernel"])
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch", {}).get(names[top])

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {case.notes}", "cells": mesh.n_cells, "faces": mesh.n_faces,
                   "parallelism": "replicas only" if ws > 1 else "single GPU",
                   "l2": "J.v working set > 126 MB L2 (no flush needed)", "setup_s": round(t_setup, 2)},
        "roofline": {"bound": "hbm", "achieved": top_st["GBps"], "peak": peak, "unit": "GB/s",
                     "frac": top_st["GBps"] / peak, "peak_kind": peak_kind, "traffic": traffic,
                     "kernel": names[top], "algorithmic_bytes_per_launch": st_b[top],
                     "launch_ms": st_ms[top], "share_of_jv": st_ms[top] / sum(st_ms)},
        "jv_roofline": {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "algorithmic_bytes_per_jv": jv_bytes, "model": "SURVEY.md 8d: 96Nc+120Nf+60Nd+12Nt"},
        "stages": stages,
        "cell_dof_per_s": 3 * mesh.n_cells * value,
        "e2e": {"value": ws / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 3 * 8 * n, "d2h_bytes_per_step": 8 * n},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_jfnk:
        f0 = case.initial_field(mesh)
        cfg = case.solver()
        # untimed warm-up solve (one Newton step, a few Krylov iterations): module loading
        # and first-launch costs of the preconditioner / GMRES kernels stay out of the number
        sv.run_steps_host(ev, f0, case.solver(max_outer=1, max_krylov=3), 1)
        f, reps, wall = sv.run_steps_host(ev, f0, cfg, 1 if case.n_steps == 1 else min(case.n_steps, args.jfnk_steps))
        s = [r.summary() for r in reps]
        line["jfnk"] = {"solve_seconds": wall, "steps": len(s), "status": [x["status"] for x in s],
                        "newton": [x["outer_iters"] for x in s], "krylov_per_newton": [x["krylov_per_newton"] for x in s],
                        "final_rel_residual": [x["final_residual"] / x["initial_residual"] for x in s],
                        "path": "sfv_run_steps_host (host buffers; includes preconditioner setup)"}
    if rank == 0 and not args.no_cpu and ws == 1:
        try:  # the same measurement as the reference arm (reference_jv)
            jv = reference_jv(case, mesh, u_h, r_u.cpu().numpy(), v_h, args.cpu_jv, 1)
            line["cpu_baseline"] = {k: jv[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                                         "host_threads")}
        except Exception as exc:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-jfnk", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--jfnk-steps", type=int, default=1)
    ap.add_argument("--cpu-jv", type=int, default=32, help="J.v in the GPU arm's cpu_baseline sample")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
