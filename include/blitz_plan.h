/* blitz_plan.h -- host-side (CPU) decision kernels of the live-autoscaling data plane.
 *
 * C ABI, plain pointers and sizes.  Built into libblitz_host.so (g++ only, no CUDA),
 * loaded by paper_2412_17246_b200/_native.py through ctypes.
 *
 * Replaces (reference = /root/reference/pkg/src/scalesim):
 *   bz_pipeline_dp  <- livescale.configure_pipeline's dynamic program
 *                      (livescale.py:113-181); the Python shim keeps the
 *                      argument checks and exception mapping of livescale.py:125-137.
 */
#ifndef BLITZ_PLAN_H
#define BLITZ_PLAN_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BZ_PLAN_OK = 0,
  BZ_PLAN_INFEASIBLE = 1, /* -> PipelineError("no feasible pipeline configuration") */
  BZ_PLAN_DEADLINE = 2,   /* -> SolverDeadlineExceeded */
  BZ_PLAN_EINVAL = -1     /* -> PipelineError (argument checks) */
};

/* Solve the weighted ZigZag split.
 *   batches, layers      N >= 1, L >= 1
 *   time_l               layer-load time in layer-execution units (>= 0, may be +inf)
 *   weights[batches]     positive per-batch weights w_i
 *   first_layer_offset   C3 offset (reference default 1)
 *   source_prefix        1: C3 bounded by sum_{j<i} S_j; 0: by sum_{j<i} T_j
 *   deadline_s           < 0 for none; checked before each batch stage
 *   t_out[batches]       receives T_i (S_i = L - T_i)
 * Returns BZ_PLAN_*.
 */
int bz_pipeline_dp(int batches, int layers, double time_l, const double* weights,
                   int first_layer_offset, int source_prefix, double deadline_s, int* t_out);

#ifdef __cplusplus
}
#endif
#endif /* BLITZ_PLAN_H */
