"""ORACLE (test infrastructure only) — APEX performance model, plain definitions.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import it.

* ``interp`` — the profiling-informed time prediction behind apex_predict_time.
  PAPER.md P:153 (§3.1 "Offline Profiler and Performance Model": profiled
  execution times "across different batch sizes and sequence lengths" inform a
  performance model); the interpolation scheme is unstated, so we take SPEC.md
  S:49-57 / S:91's reading (reading c16): bilinear over the
  (batch, kv_tokens) grid, clamped to the grid's edges on each axis.
* ``observe`` — online recalibration of that table from a measured time,
  PAPER.md P:503 (§6: "online profiling specifically for decode-intensive
  scenarios" to correct mispredictions of the offline profile).  The paper gives
  no update rule; reading c17 fixes one: (1) a point outside the grid
  first adds a grid line through it, valued at the current (clamped) predictions,
  so no prediction changes; (2) the four corners of the point's cell move by a
  normalised least-mean-squares step, corner c += alpha * e * w_c / sum(w^2) with
  e = measured - predicted and w_c the bilinear weights, after which the
  prediction at the point is exactly predicted + alpha * e.
* Eq1-Eq6 of §3.2 written out as printed.
"""
from __future__ import annotations

from bisect import bisect_right


def _axis(grid, x):
    """(i, f): x clamped into [grid[0], grid[-1]], cell i, fraction f in [0, 1]."""
    if len(grid) == 1 or x <= grid[0]:
        return 0, 0.0
    if x >= grid[-1]:
        return len(grid) - 2, 1.0
    i = bisect_right(grid, x) - 1
    return i, (x - grid[i]) / (grid[i + 1] - grid[i])


def interp(batch_grid, kv_grid, us, batch, kv_tokens) -> float:
    """Bilinear interpolation of us[i][j] (time at batch_grid[i], kv_grid[j]) with clamping."""
    i, fx = _axis(batch_grid, batch)
    j, fy = _axis(kv_grid, kv_tokens)
    i1 = min(i + 1, len(batch_grid) - 1)
    j1 = min(j + 1, len(kv_grid) - 1)
    return ((1 - fx) * (1 - fy) * us[i][j] + fx * (1 - fy) * us[i1][j]
            + (1 - fx) * fy * us[i][j1] + fx * fy * us[i1][j1])


def observe(batch_grid, kv_grid, us, batch, kv_tokens, measured_us, alpha):
    """One online-recalibration step (reading c17).  Returns new (batch_grid, kv_grid, us);
    the inputs are not modified."""
    if not (0.0 < alpha <= 1.0) or not (measured_us > 0.0) or measured_us == float("inf"):
        raise ValueError("alpha must be in (0, 1] and measured_us finite and > 0")
    bg, kg = list(batch_grid), list(kv_grid)
    u = [list(row) for row in us]
    # (1) grid lines through an outside point, valued at the current predictions
    if batch < bg[0] or batch > bg[-1]:
        row = [interp(bg, kg, u, batch, k) for k in kg]
        at = 0 if batch < bg[0] else len(bg)
        bg.insert(at, batch)
        u.insert(at, row)
    if kv_tokens < kg[0] or kv_tokens > kg[-1]:
        col = [interp(bg, kg, u, b, kv_tokens) for b in bg]
        at = 0 if kv_tokens < kg[0] else len(kg)
        kg.insert(at, kv_tokens)
        for i in range(len(bg)):
            u[i].insert(at, col[i])
    # (2) normalised LMS step on the corners of the point's cell
    e = measured_us - interp(bg, kg, u, batch, kv_tokens)
    i, fx = _axis(bg, batch)
    j, fy = _axis(kg, kv_tokens)
    i1, j1 = min(i + 1, len(bg) - 1), min(j + 1, len(kg) - 1)
    w = {}
    for (a, b), wt in (((i, j), (1 - fx) * (1 - fy)), ((i1, j), fx * (1 - fy)),
                       ((i, j1), (1 - fx) * fy), ((i1, j1), fx * fy)):
        w[(a, b)] = w.get((a, b), 0.0) + wt
    norm = sum(x * x for x in w.values())
    for (a, b), wt in w.items():
        u[a][b] += alpha * e * wt / norm
    return bg, kg, u


def t_gpuonly(t_glinear, t_gatt):            # Eq1
    return t_glinear + t_gatt


def t_overlap(t_glinear, t_gatt):            # Eq2
    return 2 * t_glinear + t_gatt


def n_gtotal(n_g, t_gatt):                   # Eq3
    return n_g * t_gatt


def n_ctotal(n_c, t_glinear, t_gatt):        # Eq4
    return n_c * (2 * t_glinear + t_gatt)


def eq5_holds(n_g, n_c, t_glinear, t_gatt) -> bool:   # Eq5
    lhs = (n_g * t_gatt + n_c * (2 * t_glinear + t_gatt)) / (2 * t_glinear + t_gatt)
    rhs = n_g * t_gatt / (t_glinear + t_gatt)
    return lhs > rhs


def eq6_threshold(t_glinear, t_gatt) -> float:        # Eq6
    return 2 * t_glinear / t_gatt + 3 + t_gatt / t_glinear


def algorithm1(n_prefill, n_gpu, n_cpu, n_g, n_c, t_glinear, t_gatt, t_glinear_pref=None, t_gatt_pref=None,
               min_cpu_ratio=8.0):
    """Algorithm 1 step by step, plus the P:378 request-ratio gate (§4.2).

    Returns "gpu_only" | "asym_pipeline" | "async_overlap"."""
    if n_cpu == 0:                                          # lines 4-6
        return "gpu_only"
    if min_cpu_ratio and min_cpu_ratio > 0 and n_cpu < min_cpu_ratio * n_gpu:
        return "gpu_only"
    if n_prefill == 0:                                      # lines 9-16 (decode-only, Eq5)
        return "asym_pipeline" if eq5_holds(n_g, n_c, t_glinear, t_gatt) else "async_overlap"
    t_overlap_with_prefill = t_glinear_pref + t_glinear + t_gatt_pref          # line 20
    lhs = (n_g * t_gatt + n_c * t_overlap_with_prefill) / (2 * t_glinear + t_gatt)   # line 21
    rhs = n_g * t_gatt / (t_glinear + t_gatt)
    return "asym_pipeline" if lhs > rhs else "async_overlap"
