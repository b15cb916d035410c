// APEX decision layer: Eq1-Eq6 and Algorithm 1 of PAPER.md
// §3.2/§3.4 as pure host functions, fed on B200 by apex_predict_time (T_gatt),
// measured linear-layer times (T_glinear) and the measured CPU attention rate
// (N_C).  Declared in include/apex.h.
#include <cmath>

#include "apex_internal.h"

namespace {
bool pos(double x) { return std::isfinite(x) && x > 0.0; }
}  // namespace

extern "C" {

// Eq6: N_G/N_C < 2 T_glinear/T_gatt + 3 + T_gatt/T_glinear
apex_status apex_pipelining_threshold(double t_glinear, double t_gatt, double *out) {
    if (!out) return apex::set_error(APEX_EINVAL, "apex_pipelining_threshold: out is NULL");
    if (!pos(t_glinear) || !pos(t_gatt))
        return apex::set_error(APEX_EINVAL, "apex_pipelining_threshold: T_glinear %g and T_gatt %g must be finite and > 0",
                               t_glinear, t_gatt);
    *out = 2.0 * t_glinear / t_gatt + 3.0 + t_gatt / t_glinear;
    return APEX_OK;
}

apex_status apex_decide(const apex_sched_input *in, apex_decision *out) {
    if (!in || !out) return apex::set_error(APEX_EINVAL, "apex_decide: in/out is NULL");
    if (in->n_prefill < 0 || in->n_gpu_decode < 0 || in->n_cpu_decode < 0)
        return apex::set_error(APEX_EINVAL, "apex_decide: negative request count (%d, %d, %d)", in->n_prefill,
                               in->n_gpu_decode, in->n_cpu_decode);
    *out = apex_decision{APEX_STRATEGY_GPU_ONLY, 0, 0.0, 0.0, 0.0};
    // Alg. 1 lines 4-6: no requests designated for CPU offload -> GPU-only
    if (in->n_cpu_decode == 0) return APEX_OK;
    // §4.2: CPU attention only pays once CPU requests >= ratio x GPU requests
    if (in->min_cpu_ratio > 0.0 && (double)in->n_cpu_decode < in->min_cpu_ratio * (double)in->n_gpu_decode) {
        out->gate_closed = 1;
        return APEX_OK;
    }
    if (!pos(in->n_g) || !pos(in->n_c) || !pos(in->t_glinear) || !pos(in->t_gatt))
        return apex::set_error(APEX_EINVAL, "apex_decide: N_G, N_C, T_glinear, T_gatt must be finite and > 0");
    const double ng = in->n_g, nc = in->n_c, tl = in->t_glinear, ta = in->t_gatt;
    const double rhs = ng * ta / (tl + ta);                     // GPU-only throughput (Eq5 right side)
    double lhs;
    if (in->n_prefill == 0) {
        // decode-only: Eq5, (N_G T_gatt + N_C (2 T_glinear + T_gatt)) / (2 T_glinear + T_gatt)
        lhs = (ng * ta + nc * (2.0 * tl + ta)) / (2.0 * tl + ta);
        apex_pipelining_threshold(tl, ta, &out->eq6_threshold);
    } else {
        if (!pos(in->t_glinear_pref) || !pos(in->t_gatt_pref))
            return apex::set_error(APEX_EINVAL, "apex_decide: T_glinear_pref and T_gatt_pref must be finite and > 0 "
                                                "when n_prefill > 0");
        // mixed (Alg. 1 lines 20-23): N_Ctotal = N_C (T_glinear_pref + T_glinear + T_gatt_pref),
        // compared over the same (2 T_glinear + T_gatt) window as printed
        const double t_ov = in->t_glinear_pref + tl + in->t_gatt_pref;
        lhs = (ng * ta + nc * t_ov) / (2.0 * tl + ta);
    }
    out->lhs = lhs;
    out->rhs = rhs;
    out->strategy = lhs > rhs ? APEX_STRATEGY_ASYM_PIPELINE : APEX_STRATEGY_ASYNC_OVERLAP;
    return APEX_OK;
}

}  // extern "C"
