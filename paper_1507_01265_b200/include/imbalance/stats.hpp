// Repeated-timing statistics for speed-function measurement. Same API as
// /root/reference/proj/include/imbalance/stats.hpp:8-33; the Student-t
// quantile is computed in-house (the reference needs Boost.Math,
// stats.cpp:5, which is absent here).
#pragma once

#include <span>

namespace imb {

struct Summary {
  int count = 0;
  double mean = 0.0;
  double stddev = 0.0;        // n-1 denominator
  double ci_halfwidth = 0.0;  // 95% two-sided Student-t
};

double mean(std::span<const double> xs);
double sample_stddev(std::span<const double> xs);
double t_quantile_975(int df);  // 0.975 point, df >= 1, strictly decreasing in df
double ci_halfwidth95(std::span<const double> xs);
Summary summarize(std::span<const double> xs);

}  // namespace imb
