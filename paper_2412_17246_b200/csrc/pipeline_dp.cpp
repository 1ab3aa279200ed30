// Exact layer-ownership solver for ZigZag cooperative execution.
//
// Restates the prefix-sum dynamic program of the reference
// configure_pipeline (pkg/src/scalesim/livescale.py:113-181) natively.  The
// float64 operations are issued in the reference's order so the resulting
// splits are bit-identical:
//   coeff_j = w_j * (n - j)                      (livescale.py:139)
//   cand    = value[a] + coeff_j * t             (ramp, livescale.py:149,159)
//   update only when cand > best[a + t]          (strict, livescale.py:162)
//   end     = first index of the maximum         (np.argmax, livescale.py:170)
// States a are visited in ascending order, as np.nonzero yields them.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "../../include/blitz_plan.h"

namespace {

// Largest T with time_l * (T - offset) <= cap (livescale.py:101-110).
int64_t c3_tmax(double time_l, int64_t offset, int64_t cap, int64_t layers) {
  if (time_l <= 0.0) return layers;
  if (std::isinf(time_l)) return offset < layers ? offset : layers;
  double f = std::floor(static_cast<double>(cap) / time_l + static_cast<double>(offset) + 1e-12);
  if (f > 1e15) return layers;  // far beyond any layer count; result saturates
  int64_t t = static_cast<int64_t>(f);
  while (t > offset && time_l * static_cast<double>(t - offset) > static_cast<double>(cap) + 1e-9) --t;
  if (t > layers) t = layers;
  return t < 0 ? 0 : t;
}

}  // namespace

extern "C" int bz_pipeline_dp(int batches, int layers, double time_l, const double* weights,
                              int first_layer_offset, int source_prefix, double deadline_s,
                              int* t_out) {
  if (batches < 1 || layers < 1 || time_l < 0.0 || weights == nullptr || t_out == nullptr)
    return BZ_PLAN_EINVAL;
  const auto started = std::chrono::steady_clock::now();
  const int64_t n = batches, L = layers, off = first_layer_offset;
  const double NEG = -std::numeric_limits<double>::infinity();

  std::vector<double> value(1, 0.0), next;
  std::vector<std::vector<int32_t>> parents(static_cast<size_t>(n));
  std::vector<double> ramp(static_cast<size_t>(L + 1));

  for (int64_t j = 0; j < n; ++j) {
    if (deadline_s >= 0.0) {
      double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - started).count();
      if (el > deadline_s) return BZ_PLAN_DEADLINE;
    }
    const double coeff = weights[j] * static_cast<double>(n - j);
    for (int64_t t = 0; t <= L; ++t) ramp[t] = coeff * static_cast<double>(t);
    const size_t width = static_cast<size_t>((j + 1) * L + 1);
    next.assign(width, NEG);
    std::vector<int32_t>& par = parents[static_cast<size_t>(j)];
    par.assign(width, -1);
    const int64_t live = static_cast<int64_t>(value.size());
    for (int64_t a = 0; a < live; ++a) {
      const double base = value[a];
      if (!(base > NEG)) continue;
      int64_t tmax = L;
      if (j >= 1 && j * L - 2 * a < tmax) tmax = j * L - 2 * a;
      if (time_l > 0.0) {
        const int64_t cap = source_prefix ? (j * L - a) : a;
        const int64_t c3 = c3_tmax(time_l, off, cap, L);
        if (c3 < tmax) tmax = c3;
      }
      if (tmax < 0) continue;
      double* dst = next.data() + a;
      int32_t* pdst = par.data() + a;
      for (int64_t t = 0; t <= tmax; ++t) {
        const double cand = base + ramp[t];
        if (cand > dst[t]) {
          dst[t] = cand;
          pdst[t] = static_cast<int32_t>(a);
        }
      }
    }
    value.swap(next);
  }

  size_t end = 0;
  for (size_t i = 1; i < value.size(); ++i)
    if (value[i] > value[end]) end = i;
  if (!std::isfinite(value[end])) return BZ_PLAN_INFEASIBLE;
  int64_t a = static_cast<int64_t>(end);
  for (int64_t j = n - 1; j >= 0; --j) {
    const int64_t prev = parents[static_cast<size_t>(j)][static_cast<size_t>(a)];
    t_out[j] = static_cast<int>(a - prev);
    a = prev;
  }
  return BZ_PLAN_OK;
}
