// Statistics (stats.hpp), behaviour of /root/reference/proj/src/stats.cpp:11-46.
// The 0.975 Student-t quantile solves I_x(df/2, 1/2) = 0.05 for
// x = df / (df + t^2) by bisection on x, with the regularised incomplete
// beta function evaluated by a modified-Lentz continued fraction.
#include "imbalance/stats.hpp"

#include <cmath>

#include "imbalance/errors.hpp"

namespace imb {

namespace {

// Continued fraction for I_x(a, b) (valid for x < (a+1)/(a+b+2)).
double beta_cf(double a, double b, double x) {
  const double tiny = 1e-300;
  double c = 1.0, d = 1.0 - (a + b) * x / (a + 1.0);
  if (std::fabs(d) < tiny) d = tiny;
  d = 1.0 / d;
  double h = d;
  for (int k = 1; k < 10000; ++k) {
    const double kk = static_cast<double>(k);
    double num = kk * (b - kk) * x / ((a + 2.0 * kk - 1.0) * (a + 2.0 * kk));
    for (int half = 0; half < 2; ++half) {
      d = 1.0 + num * d;
      if (std::fabs(d) < tiny) d = tiny;
      c = 1.0 + num / c;
      if (std::fabs(c) < tiny) c = tiny;
      d = 1.0 / d;
      const double step = d * c;
      h *= step;
      if (half == 1 && std::fabs(step - 1.0) < 1e-16) return h;
      num = -(a + kk) * (a + b + kk) * x / ((a + 2.0 * kk) * (a + 2.0 * kk + 1.0));
    }
  }
  return h;
}

double reg_inc_beta(double a, double b, double x) {
  if (x <= 0.0) return 0.0;
  if (x >= 1.0) return 1.0;
  const double lead = std::exp(std::lgamma(a + b) - std::lgamma(a) - std::lgamma(b) +
                               a * std::log(x) + b * std::log1p(-x));
  if (x < (a + 1.0) / (a + b + 2.0)) return lead * beta_cf(a, b, x) / a;
  return 1.0 - lead * beta_cf(b, a, 1.0 - x) / b;
}

}  // namespace

double mean(std::span<const double> xs) {
  if (xs.empty()) throw InsufficientDataError("mean of an empty sample");
  double s = 0.0;
  for (double v : xs) s += v;
  return s / static_cast<double>(xs.size());
}

double sample_stddev(std::span<const double> xs) {
  if (xs.size() < 2) throw InsufficientDataError("stddev needs at least 2 observations");
  const double mu = mean(xs);
  double ss = 0.0;
  for (double v : xs) ss += (v - mu) * (v - mu);
  return std::sqrt(ss / static_cast<double>(xs.size() - 1));
}

double t_quantile_975(int df) {
  if (df < 1) throw InsufficientDataError("t quantile needs df >= 1");
  const double a = 0.5 * static_cast<double>(df);
  // Two-sided tail 0.05: find x in (0,1) with I_x(a, 1/2) = 0.05; I is increasing in x.
  double lo = 0.0, hi = 1.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (reg_inc_beta(a, 0.5, mid) < 0.05)
      lo = mid;
    else
      hi = mid;
  }
  const double x = 0.5 * (lo + hi);
  return std::sqrt(static_cast<double>(df) * (1.0 - x) / x);
}

double ci_halfwidth95(std::span<const double> xs) {
  if (xs.size() < 2) throw InsufficientDataError("confidence interval needs >= 2 observations");
  const double n = static_cast<double>(xs.size());
  return t_quantile_975(static_cast<int>(xs.size()) - 1) * sample_stddev(xs) / std::sqrt(n);
}

Summary summarize(std::span<const double> xs) {
  Summary s;
  s.count = static_cast<int>(xs.size());
  s.mean = mean(xs);
  s.stddev = sample_stddev(xs);
  s.ci_halfwidth = ci_halfwidth95(xs);
  return s;
}

}  // namespace imb
