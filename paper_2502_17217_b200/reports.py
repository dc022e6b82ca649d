"""metrics.csv / iterations.csv from the device solver's reports, in the reference's
format (write_metrics_csv / write_iterations_csv, /root/reference/proj/src/io.cpp:458-488):
ostream precision 12 (``%.12g``), the status names of to_string(SolveStatus)
(nonlinear.cpp:52-58).  ``reports`` are the SolveReport structs sfv_run_steps fills; each
carries at most 64 iteration records (the C-ABI's fixed record array)."""
from __future__ import annotations

from .abi import STATUS_NAME


def _g(x: float) -> str:
    """std::ostream << double with precision(12), default float field"""
    return "%.12g" % x


def write_metrics_csv(reports, path: str) -> None:
    lines = ["step,status,outer_iters,krylov_iters,initial_residual,final_residual,wall_seconds,detail"]
    outer = krylov = 0
    wall = 0.0
    for r in reports:
        detail = r.detail.decode(errors="replace") if isinstance(r.detail, bytes) else str(r.detail)
        lines.append(f"{r.step},{STATUS_NAME.get(r.status, '?')},{r.outer_iters},{r.krylov_iters},"
                     f"{_g(r.initial_residual)},{_g(r.final_residual)},{_g(r.wall_seconds)},{detail}")
        outer += r.outer_iters
        krylov += r.krylov_iters
        wall += r.wall_seconds
    lines.append(f"total,,{outer},{krylov},,,{_g(wall)},")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def write_iterations_csv(reports, path: str) -> None:
    lines = ["step,iter,r_norm,krylov_iters,s"]
    for r in reports:
        for i in range(min(r.n_records, 64)):
            it = r.records[i]
            lines.append(f"{it.step},{it.iter},{_g(it.r_norm)},{it.krylov_iters},{_g(it.s)}")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
