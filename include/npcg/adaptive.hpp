// reference: adaptive.hpp:11-85 — adaptive rank selection (Alg. 5) and the
// randomized power-method error estimate (Alg. 4). Draws follow the
// reference's Rng stream order exactly (Omega blocks and power vectors
// interleaved, adaptive.cpp:90,116-117,69).
#pragma once

#include <optional>

#include "nystrom.hpp"

namespace npcg {

enum class TolMode { error, ratio, fixed };
enum class SketchKind { gaussian, column_sampling };

struct AdaptiveConfig {  // adaptive.hpp:26-37
  Index ell0 = 10;
  Index ell_max = 0;
  double mu = 0.0;
  TolMode tol_mode = TolMode::error;
  std::optional<double> tau;
  Index q = 5;
  bool secondary_criterion = true;
  SketchKind sketch = SketchKind::gaussian;
  double resolved_tau() const {
    if (tau.has_value()) {
      if (!(*tau > 0.0)) throw std::invalid_argument("AdaptiveConfig: tau must be > 0");
      return *tau;
    }
    return tol_mode == TolMode::ratio ? 10.0 : 30.0;
  }
};

struct AdaptiveOutcome {  // adaptive.hpp:40-47
  NystromApproximation approximation;
  std::optional<double> error_estimate;
  Index doublings = 0;
  bool hit_cap = false;
  double posterior_condition_estimate = 0.0;
  Index ell_final = 0;
};

/// estimate_error_power (adaptive.cpp:83-109).
inline double estimate_error_power(const LinearOperator& op, const NystromApproximation& approx, Index q, Rng& rng) {
  double est = 0.0;
  const OpRef ref = device_handle(op);
  ref.check(npcg_power_estimate_rng(ref, approx.device.get(), q, rng.handle(), &est));
  return est;
}

namespace detail {
inline AdaptiveOutcome adaptive_call(const LinearOperator& op, const AdaptiveConfig& c, Rng& rng, int mode) {
  npcg_adaptive_cfg cfg{static_cast<std::int64_t>(c.ell0), static_cast<std::int64_t>(c.ell_max), c.mu, mode,
                        c.tau.has_value() ? 1 : 0, c.tau.value_or(0.0), static_cast<std::int64_t>(c.q),
                        c.secondary_criterion ? 1 : 0, c.sketch == SketchKind::gaussian ? 0 : 1};
  npcg_nys* h = nullptr;
  npcg_adaptive_outcome o{};
  const OpRef ref = device_handle(op);
  ref.check(npcg_adaptive(ref, &cfg, rng.handle(), &h, &o));
  AdaptiveOutcome out;
  out.approximation = fetch(own(h));
  if (o.has_error_estimate) out.error_estimate = o.error_estimate;
  out.doublings = o.doublings;
  out.hit_cap = o.hit_cap != 0;
  out.posterior_condition_estimate = o.posterior_condition;
  out.ell_final = o.ell_final;
  return out;
}
}  // namespace detail

/// adaptive_nystrom, strategy 1 (adaptive.cpp:111-123).
inline AdaptiveOutcome adaptive_nystrom(const LinearOperator& op, const AdaptiveConfig& c, Rng& rng) {
  if (c.tol_mode != TolMode::error) throw std::invalid_argument("adaptive_nystrom: config.tol_mode must be error");
  return detail::adaptive_call(op, c, rng, 0);
}
/// adaptive_nystrom_ratio, strategy 2 (adaptive.cpp:125-133).
inline AdaptiveOutcome adaptive_nystrom_ratio(const LinearOperator& op, const AdaptiveConfig& c, Rng& rng) {
  if (c.tol_mode != TolMode::ratio) throw std::invalid_argument("adaptive_nystrom_ratio: config.tol_mode must be ratio");
  return detail::adaptive_call(op, c, rng, 1);
}
/// fixed_rank_nystrom, strategy 3 (adaptive.cpp:135-148).
inline AdaptiveOutcome fixed_rank_nystrom(const LinearOperator& op, const AdaptiveConfig& c, Rng& rng) {
  if (c.tol_mode != TolMode::fixed) throw std::invalid_argument("fixed_rank_nystrom: config.tol_mode must be fixed");
  return detail::adaptive_call(op, c, rng, 2);
}

/// posterior_condition_estimate (adaptive.cpp:150-156).
inline double posterior_condition_estimate(double lambda_ell, double mu, double err) {
  double out = 0.0;
  check_status(npcg_posterior_condition(lambda_ell, mu, err, &out));
  return out;
}

}  // namespace npcg
