// TEST INFRASTRUCTURE ONLY — a C-ABI shim over the UNMODIFIED reference
// partitioner (/root/reference/proj/src/{fpm,partition}.cpp), compiled from
// the sources where they lie by oracle/Makefile into oracle/_ref/. Tests load
// it with ctypes as the integer-identical oracle for the product partitioner
// (SURVEY.md §8c). Nothing here is shipped; the product never links it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "imbalance/errors.hpp"
#include "imbalance/fpm.hpp"
#include "imbalance/partition.hpp"

namespace {

struct RefSample {  // same layout as imb_speed_sample in include/imb_mpdata.h
  std::int64_t x;
  double speed;
  double ci_halfwidth;
  std::int64_t repetitions;
};

thread_local std::string g_err;

imb::SpeedFunction make(std::int64_t unit, std::int64_t g, const RefSample* s, int ns) {
  std::vector<imb::SpeedSample> v;
  for (int i = 0; i < ns; ++i) v.push_back({s[i].x, s[i].speed, s[i].ci_halfwidth, s[i].repetitions});
  return imb::SpeedFunction(unit, g, std::move(v), "ref");
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const imb::RangeError& e) { g_err = e.what(); return 1; }
  catch (const imb::DomainError& e) { g_err = e.what(); return 2; }
  catch (const imb::AlignmentError& e) { g_err = e.what(); return 3; }
  catch (const imb::IncompatibleModelError& e) { g_err = e.what(); return 4; }
  catch (const imb::InsufficientDataError& e) { g_err = e.what(); return 5; }
  catch (const imb::InfeasibleError& e) { g_err = e.what(); return 6; }
  catch (const imb::TooLargeError& e) { g_err = e.what(); return 7; }
  catch (const imb::ConfigError& e) { g_err = e.what(); return 8; }
  catch (const imb::ContractError& e) { g_err = e.what(); return 9; }
  catch (const imb::ParseError& e) { g_err = e.what(); return 10; }
  catch (const std::exception& e) { g_err = e.what(); return 99; }
}

void emit(const imb::Partition& p, std::int64_t* shares, double* per_time, double* makespan,
          std::int64_t* offset) {
  for (std::size_t i = 0; i < p.shares.size(); ++i) {
    shares[i] = p.shares[i];
    per_time[i] = p.per_time[i];
  }
  *makespan = p.makespan;
  *offset = p.offset ? *p.offset : -1;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_eval_speed(std::int64_t unit, std::int64_t g, const RefSample* s, int ns, double x,
                   double* out) {
  return guard([&] { *out = imb::eval_speed(make(unit, g, s, ns), x); });
}

int ref_eval_time(std::int64_t unit, std::int64_t g, const RefSample* s, int ns, double x,
                  double* out) {
  return guard([&] { *out = imb::eval_time(make(unit, g, s, ns), x); });
}

// kind: 0 = partition_paired, 1 = partition_general, 2 = brute_force_oracle
int ref_partition(int kind, std::int64_t unit, std::int64_t g, const RefSample* s, int ns,
                  std::int64_t total, int p, int allow_idle, std::int64_t cap,
                  std::int64_t* shares, double* per_time, double* makespan,
                  std::int64_t* offset) {
  return guard([&] {
    imb::PartitionProblem pr{total, p, make(unit, g, s, ns), allow_idle != 0};
    imb::Partition r = kind == 0   ? imb::partition_paired(pr)
                       : kind == 1 ? imb::partition_general(pr)
                                   : imb::brute_force_oracle(pr, cap);
    emit(r, shares, per_time, makespan, offset);
  });
}

int ref_predict_makespan(std::int64_t unit, std::int64_t g, const RefSample* s, int ns,
                         const std::int64_t* in_shares, int p, double* per_time,
                         double* makespan) {
  return guard([&] {
    imb::Partition r =
        imb::predict_makespan(make(unit, g, s, ns), std::span<const std::int64_t>(in_shares, p));
    for (int i = 0; i < p; ++i) per_time[i] = r.per_time[static_cast<std::size_t>(i)];
    *makespan = r.makespan;
  });
}

// violations: up to cap pairs written as (x, x') into viol[2*i]; *nviol = total count.
int ref_check_condition(std::int64_t unit, std::int64_t g, const RefSample* s, int ns,
                        int* satisfied, std::int64_t* viol, int cap, int* nviol,
                        std::int64_t* max_gain_pair) {
  return guard([&] {
    imb::ConditionReport r = imb::check_condition(make(unit, g, s, ns));
    *satisfied = r.satisfied ? 1 : 0;
    *nviol = static_cast<int>(r.violations.size());
    for (int i = 0; i < *nviol && i < cap; ++i) {
      viol[2 * i] = r.violations[static_cast<std::size_t>(i)].first;
      viol[2 * i + 1] = r.violations[static_cast<std::size_t>(i)].second;
    }
    max_gain_pair[0] = r.max_gain_pair ? r.max_gain_pair->first : -1;
    max_gain_pair[1] = r.max_gain_pair ? r.max_gain_pair->second : -1;
  });
}

// classification: 0 decreasing, 1 increasing-concave-then-decreasing, 2 other
int ref_classify_shape(std::int64_t unit, std::int64_t g, const RefSample* s, int ns, int* cls,
                       std::int64_t* peak_x) {
  return guard([&] {
    imb::ShapeReport r = imb::classify_shape(make(unit, g, s, ns));
    *cls = static_cast<int>(r.classification);
    *peak_x = r.peak_x ? *r.peak_x : -1;
  });
}

int ref_improvement_search(std::int64_t unit, std::int64_t g, const RefSample* s, int ns,
                           std::int64_t balanced, int* found, std::int64_t* delta,
                           double* gain, std::int64_t* pair) {
  return guard([&] {
    auto r = imb::improvement_search(make(unit, g, s, ns), balanced);
    *found = r ? 1 : 0;
    *delta = r ? r->delta : 0;
    *gain = r ? r->gain_s : 0.0;
    pair[0] = r ? r->violating_pair.first : -1;
    pair[1] = r ? r->violating_pair.second : -1;
  });
}

// Average of nf functions sharing unit/g and ns samples each: samples[f*ns + i].
int ref_average(std::int64_t unit, std::int64_t g, const RefSample* s, int nf, int ns,
                RefSample* out) {
  return guard([&] {
    std::vector<imb::SpeedFunction> fs;
    for (int f = 0; f < nf; ++f) fs.push_back(make(unit, g, s + static_cast<std::ptrdiff_t>(f) * ns, ns));
    imb::SpeedFunction a = imb::average(fs);
    for (int i = 0; i < ns; ++i) {
      const imb::SpeedSample& q = a.samples()[static_cast<std::size_t>(i)];
      out[i] = {q.x, q.speed, q.ci_halfwidth, q.repetitions};
    }
  });
}

int ref_slice_surface(std::int64_t unit, std::int64_t g, const std::int64_t* nv, int nn,
                      const std::int64_t* mv, int nm, const RefSample* s, std::int64_t fixed_n,
                      RefSample* out, std::int64_t* out_unit) {
  return guard([&] {
    imb::SpeedSurface srf;
    srf.unit_cells = unit;
    srf.granularity = g;
    srf.label = "ref";
    srf.n_values.assign(nv, nv + nn);
    srf.m_values.assign(mv, mv + nm);
    for (int q = 0; q < nn * nm; ++q)
      srf.samples.push_back({s[q].x, s[q].speed, s[q].ci_halfwidth, s[q].repetitions});
    imb::SpeedFunction f = imb::slice_surface(srf, fixed_n);
    for (std::size_t q = 0; q < f.samples().size(); ++q) {
      const imb::SpeedSample& v = f.samples()[q];
      out[q] = {v.x, v.speed, v.ci_halfwidth, v.repetitions};
    }
    *out_unit = f.unit_cells();
  });
}

}  // extern "C"
