// Functional performance model: the empirical speed function s(x) the FPM
// partitioner consumes. Public names and semantics follow the reference
// header /root/reference/proj/include/imbalance/fpm.hpp:13-127; the
// implementation (csrc/host/fpm.cpp) is written fresh.
//
// Unit convention on the GPU: x counts i-planes ("frames") of a slab and
// unit_cells = m*l cells per plane, so t(x) = x * unit_cells / s(x).
#pragma once

#include <cstdint>
#include <iosfwd>
#include <optional>
#include <string>
#include <utility>
#include <vector>

namespace imb {

// fpm.hpp:13-18
struct SpeedSample {
  std::int64_t x = 0;
  double speed = 0.0;
  double ci_halfwidth = 0.0;
  std::int64_t repetitions = 1;
};

// fpm.hpp:28-49 — piecewise-linear between samples, undefined outside.
class SpeedFunction {
 public:
  SpeedFunction(std::int64_t unit_cells, std::int64_t granularity,
                std::vector<SpeedSample> samples, std::string label);

  std::int64_t unit_cells() const { return unit_cells_; }
  std::int64_t granularity() const { return granularity_; }
  const std::vector<SpeedSample>& samples() const { return samples_; }
  const std::string& label() const { return label_; }
  std::int64_t min_x() const { return samples_.front().x; }
  std::int64_t max_x() const { return samples_.back().x; }
  bool in_range(double x) const;

 private:
  std::int64_t unit_cells_;
  std::int64_t granularity_;
  std::vector<SpeedSample> samples_;
  std::string label_;
};

// fpm.hpp:51-63
struct ConditionReport {
  bool satisfied = true;
  std::vector<std::pair<std::int64_t, std::int64_t>> violations;
  std::optional<std::pair<std::int64_t, std::int64_t>> max_gain_pair;
};

// fpm.hpp:65-79
enum class ShapeClass { MonotonicallyDecreasing, IncreasingConcaveThenDecreasing, Other };
const char* to_string(ShapeClass c);
struct ShapeReport {
  ShapeClass classification = ShapeClass::Other;
  std::optional<std::int64_t> peak_x;
};

// fpm.hpp:81-98 — rectangular (n, m) grid, row-major in n.
struct SpeedSurface {
  std::int64_t unit_cells = 1;
  std::int64_t granularity = 1;
  std::string label;
  std::vector<std::int64_t> n_values;
  std::vector<std::int64_t> m_values;
  std::vector<SpeedSample> samples;
  const SpeedSample& at(std::size_t ni, std::size_t mi) const {
    return samples[ni * m_values.size() + mi];
  }
  void validate() const;
};

double eval_speed(const SpeedFunction& f, double x);  // fpm.hpp:93-96
double eval_time(const SpeedFunction& f, double x);   // fpm.hpp:98-101
ConditionReport check_condition(const SpeedFunction& f);  // fpm.hpp:103
ShapeReport classify_shape(const SpeedFunction& f);       // fpm.hpp:107
SpeedFunction average(const std::vector<SpeedFunction>& fs);  // fpm.hpp:113
SpeedFunction scaled(const SpeedFunction& f, double factor);  // fpm.hpp:118
SpeedFunction slice_surface(const SpeedSurface& g, std::int64_t fixed_n);  // fpm.hpp:123

// Speed-function CSV: "# unit_cells=U granularity=G label=S",
// then "x,speed,ci_halfwidth,repetitions"; doubles written with %.17g so a
// table round-trips bit-identically. ParseError carries the 1-based line.
void write_speed_function_csv(std::ostream& os, const SpeedFunction& f);
SpeedFunction read_speed_function_csv(std::istream& is);

}  // namespace imb
