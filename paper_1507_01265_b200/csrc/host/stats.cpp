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

// Sum and sum of squared deviations in two passes (no cancellation).
struct Moments {
  double mean = 0.0;
  double ssd = 0.0;
  std::size_t n = 0;
};

Moments moments(std::span<const double> xs, bool need_spread) {
  Moments m;
  m.n = xs.size();
  if (m.n == 0) throw InsufficientDataError("no observations");
  if (need_spread && m.n < 2) throw InsufficientDataError("a spread needs two or more observations");
  double total = 0.0;
  for (double v : xs) total += v;
  m.mean = total / static_cast<double>(m.n);
  if (need_spread)
    for (double v : xs) m.ssd += (v - m.mean) * (v - m.mean);
  return m;
}

double stddev_of(const Moments& m) { return std::sqrt(m.ssd / static_cast<double>(m.n - 1)); }

}  // namespace

double mean(std::span<const double> xs) { return moments(xs, false).mean; }

double sample_stddev(std::span<const double> xs) { return stddev_of(moments(xs, true)); }

// 0.975 quantile of Student's t with df degrees of freedom (Boost-free):
// the two-sided 5 % tail solves I_x(df/2, 1/2) = 0.05 at x = df/(df + t^2),
// and I is increasing in x, so x is bisected to the last representable step.
double t_quantile_975(int df) {
  if (df < 1) throw InsufficientDataError("the t quantile needs one or more degrees of freedom");
  const double a = 0.5 * static_cast<double>(df);
  double lo = 0.0, hi = 1.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    (reg_inc_beta(a, 0.5, mid) < 0.05 ? lo : hi) = mid;
  }
  const double x = 0.5 * (lo + hi);
  return std::sqrt(static_cast<double>(df) * (1.0 - x) / x);
}

double ci_halfwidth95(std::span<const double> xs) {
  const Moments m = moments(xs, true);
  return t_quantile_975(static_cast<int>(m.n) - 1) * stddev_of(m) / std::sqrt(static_cast<double>(m.n));
}

Summary summarize(std::span<const double> xs) {
  const Moments m = moments(xs, true);
  const double sd = stddev_of(m);
  return Summary{static_cast<int>(m.n), m.mean, sd,
                 t_quantile_975(static_cast<int>(m.n) - 1) * sd / std::sqrt(static_cast<double>(m.n))};
}

}  // namespace imb
