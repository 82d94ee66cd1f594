// imb:: workload API (workload.hpp) over the GPU team runtime. Compiled with
// -ffp-contract=off: init_fields shares recipe.cuh with the device init
// kernel and must round identically.
#include "imbalance/workload.hpp"

#include <cuda_runtime.h>

#include <cinttypes>
#include <cstdio>
#include <cstdlib>

#include "../recipe.cuh"
#include "../team.hpp"
#include "imb_mpdata.h"
#include "imbalance/errors.hpp"

namespace imb {

void StencilDomain::validate() const {
  if (n < 3 || m < 3 || l < 3) throw ContractError("domain extents must be >= 3");
  if (halo < 1) throw ContractError("halo must be >= 1");
}

GridField::GridField(const StencilDomain& d) : domain_(d) {
  d.validate();
  data_.assign(static_cast<std::size_t>(d.storage()), 0.0);
}

std::vector<double> GridField::interior() const {
  const StencilDomain& d = domain_;
  std::vector<double> out(static_cast<std::size_t>(d.cells()));
  std::size_t q = 0;
  for (std::int64_t i = 0; i < d.n; ++i)
    for (std::int64_t j = 0; j < d.m; ++j)
      for (std::int64_t k = 0; k < d.l; ++k) out[q++] = at(i, j, k);
  return out;
}

void GridField::set_interior(const std::vector<double>& v) {
  const StencilDomain& d = domain_;
  if (v.size() != static_cast<std::size_t>(d.cells())) throw ContractError("interior size mismatch");
  std::size_t q = 0;
  for (std::int64_t i = 0; i < d.n; ++i)
    for (std::int64_t j = 0; j < d.m; ++j)
      for (std::int64_t k = 0; k < d.l; ++k) at(i, j, k) = v[q++];
  halo_valid = false;
}

namespace {

std::int64_t wrap(std::int64_t a, std::int64_t n) {
  a %= n;
  return a < 0 ? a + n : a;
}
std::int64_t clampi(std::int64_t a, std::int64_t n) { return a < 0 ? 0 : (a >= n ? n - 1 : a); }

template <class Map>
void fill_halo(GridField& f, Map map) {
  const StencilDomain& d = f.domain();
  const std::int64_t h = d.halo;
  for (std::int64_t i = -h; i < d.n + h; ++i)
    for (std::int64_t j = -h; j < d.m + h; ++j)
      for (std::int64_t k = -h; k < d.l + h; ++k) {
        if (i >= 0 && i < d.n && j >= 0 && j < d.m && k >= 0 && k < d.l) continue;
        f.at(i, j, k) = f.at(map(i, d.n), map(j, d.m), map(k, d.l));
      }
  f.halo_valid = true;
}

}  // namespace

void fill_halo_clamped(GridField& f) { fill_halo(f, clampi); }
void fill_halo_periodic(GridField& f) { fill_halo(f, wrap); }

InputFields init_fields(const StencilDomain& domain, std::uint64_t seed, Recipe recipe) {
  domain.validate();
  InputFields fs{GridField(domain), GridField(domain), GridField(domain), GridField(domain),
                 GridField(domain)};
  const recipe::Params prm =
      recipe::make_params(static_cast<int>(recipe), domain.n, domain.m, domain.l, seed);
  const std::int64_t h = domain.halo;
  for (std::int64_t i = -h; i < domain.n + h; ++i)
    for (std::int64_t j = -h; j < domain.m + h; ++j)
      for (std::int64_t k = -h; k < domain.l + h; ++k) {
        double v[5];
        recipe::cell(prm, wrap(i, domain.n), wrap(j, domain.m), wrap(k, domain.l), v);
        const std::size_t o = fs.x.index(i, j, k);
        fs.x.data()[o] = v[0];
        fs.u.data()[o] = v[1];
        fs.v.data()[o] = v[2];
        fs.w.data()[o] = v[3];
        fs.rho.data()[o] = v[4];
      }
  for (GridField* g : {&fs.x, &fs.u, &fs.v, &fs.w, &fs.rho}) g->halo_valid = true;
  return fs;
}

namespace {

void stage7(const GridField& in, GridField& out, bool is_max) {
  const StencilDomain& d = in.domain();
  if (!in.halo_valid) throw ContractError("stage input halo is not filled");
  if (out.domain().storage() != d.storage()) throw ContractError("stage output domain mismatch");
  const std::size_t bytes = static_cast<std::size_t>(d.storage()) * sizeof(double);
  double *din = nullptr, *dout = nullptr;
  auto check = [](cudaError_t e) {
    if (e != cudaSuccess) throw CudaError(cudaGetErrorString(e));
  };
  check(cudaSetDevice(0));
  check(cudaMalloc(&din, 2 * bytes));
  dout = din + d.storage();
  try {
    check(cudaMemcpy(din, in.data(), bytes, cudaMemcpyHostToDevice));
    check(cudaMemcpy(dout, out.data(), bytes, cudaMemcpyHostToDevice));
    dev::launch_stage7(din, dout, d.n, d.m, d.l, d.halo, is_max, nullptr);
    check(cudaGetLastError());
    check(cudaMemcpy(out.data(), dout, bytes, cudaMemcpyDeviceToHost));
  } catch (...) {
    cudaFree(din);
    throw;
  }
  cudaFree(din);
  out.halo_valid = false;
}

}  // namespace

void stage_max7(const GridField& in, GridField& out) { stage7(in, out, true); }
void stage_min7(const GridField& in, GridField& out) { stage7(in, out, false); }

namespace {

rt::Options to_rt(const MpdataOptions& o) { return rt::Options{o.iord, o.nonos ? 1 : 0, o.fp64}; }

void upload_field(rt::Team& t, int id, const GridField& f, bool fp64) {
  const std::vector<double> v = f.interior();
  if (fp64) {
    t.upload(id, v.data(), v.size() * sizeof(double));
  } else {
    std::vector<float> s(v.begin(), v.end());
    t.upload(id, s.data(), s.size() * sizeof(float));
  }
}

// A reference caller loops over run_step, so the device team (padded-slab
// buffers, streams, events) is cached per host thread and reused while the
// domain and options stay the same; only the five fields move per call.
rt::Team& step_team(const StencilDomain& d, const MpdataOptions& o) {
  struct Cached {
    std::int64_t n = 0, m = 0, l = 0;
    int iord = 0;
    bool nonos = false, fp64 = false;
    std::unique_ptr<rt::Team> team;
  };
  thread_local Cached c;
  if (!c.team || c.n != d.n || c.m != d.m || c.l != d.l || c.iord != o.iord || c.nonos != o.nonos ||
      c.fp64 != o.fp64) {
    c.team.reset();  // free the old buffers before allocating the new ones
    c.team = std::make_unique<rt::Team>(d.n, d.m, d.l, to_rt(o), 0, 0, d.n);
    c.n = d.n;
    c.m = d.m;
    c.l = d.l;
    c.iord = o.iord;
    c.nonos = o.nonos;
    c.fp64 = o.fp64;
  }
  return *c.team;
}

}  // namespace

GridField run_step(const InputFields& fields, const StencilDomain& domain,
                   const MpdataOptions& opts) {
  domain.validate();
  for (const GridField* g : {&fields.x, &fields.u, &fields.v, &fields.w, &fields.rho})
    if (!g->halo_valid) throw ContractError("run_step input halo is not filled");
  rt::Team& team = step_team(domain, opts);
  upload_field(team, 0, fields.x, opts.fp64);
  upload_field(team, 1, fields.u, opts.fp64);
  upload_field(team, 2, fields.v, opts.fp64);
  upload_field(team, 3, fields.w, opts.fp64);
  upload_field(team, 4, fields.rho, opts.fp64);
  team.run(1, nullptr, nullptr);
  std::vector<double> out(static_cast<std::size_t>(domain.cells()));
  if (opts.fp64) {
    team.download(0, out.data(), out.size() * sizeof(double));
  } else {
    std::vector<float> s(out.size());
    team.download(0, s.data(), s.size() * sizeof(float));
    out.assign(s.begin(), s.end());
  }
  GridField g(domain);
  g.set_interior(out);
  fill_halo_periodic(g);
  return g;
}

std::uint64_t checksum(const GridField& f) {
  std::uint64_t hsh = 0xcbf29ce484222325ull;
  const StencilDomain& d = f.domain();
  for (std::int64_t i = 0; i < d.n; ++i)
    for (std::int64_t j = 0; j < d.m; ++j)
      for (std::int64_t k = 0; k < d.l; ++k) {
        const double v = f.at(i, j, k);
        const unsigned char* b = reinterpret_cast<const unsigned char*>(&v);
        for (int q = 0; q < 8; ++q) {
          hsh ^= b[q];
          hsh *= 0x100000001b3ull;
        }
      }
  return hsh;
}

std::string checksum_hex(std::uint64_t sum) {
  char buf[19];
  std::snprintf(buf, sizeof buf, "%016" PRIx64, sum);
  return buf;
}

int thread_cap() {
  if (const char* env = std::getenv("IMBALANCE_THREAD_CAP")) {
    const long v = std::strtol(env, nullptr, 10);
    if (v >= 1) return static_cast<int>(v);
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
  return count > 0 ? count : 1;
}

TeamRunner::TeamRunner(const StencilDomain& domain, int device, std::uint64_t seed, int,
                       const MpdataOptions& opts, Recipe recipe)
    : domain_(domain), device_(device) {
  domain.validate();
  if (device < 0) throw ConfigError("device index must be >= 0");
  team_ = std::make_unique<rt::Team>(domain.n, domain.m, domain.l, to_rt(opts), device, 0, domain.n);
  team_->init_recipe(static_cast<int>(recipe), seed);
}

TeamRunner::~TeamRunner() = default;

void TeamRunner::reset() { team_->reset(); }

double TeamRunner::run(int steps, const std::function<void()>& start_sync,
                       const std::function<void()>& step_sync,
                       const std::function<void()>& end_sync) {
  if (steps < 0) throw ContractError("steps must be >= 0");
  if (start_sync) start_sync();
  double total = 0.0;
  if (!step_sync) {
    team_->run(steps, &total, nullptr);
  } else {
    for (int s = 0; s < steps; ++s) {
      double c = 0.0;
      team_->run(1, &c, nullptr);
      total += c;
      step_sync();
    }
  }
  if (end_sync) end_sync();
  return total;
}

std::uint64_t TeamRunner::current_checksum() const { return team_->checksum(); }

namespace {
// C-ABI status -> the matching imb:: exception (the inverse of c_api.cpp's guard)
void check_status(int rc) {
  if (rc == 0) return;
  const std::string msg = imb_last_error();
  switch (rc) {
    case IMB_E_RANGE: throw RangeError(msg);
    case IMB_E_DOMAIN: throw DomainError(msg);
    case IMB_E_ALIGNMENT: throw AlignmentError(msg);
    case IMB_E_INCOMPATIBLE: throw IncompatibleModelError(msg);
    case IMB_E_INSUFFICIENT: throw InsufficientDataError(msg);
    case IMB_E_INFEASIBLE: throw InfeasibleError(msg);
    case IMB_E_TOOLARGE: throw TooLargeError(msg);
    case IMB_E_CONFIG: throw ConfigError(msg);
    case IMB_E_CONTRACT: throw ContractError(msg);
    case IMB_E_PARSE: throw ParseError(msg, 0);
    case IMB_E_CUDA: throw CudaError(msg);
    case IMB_E_NCCL: throw NcclError(msg);
    default: throw Error(msg);
  }
}
}  // namespace

GroupRunner::GroupRunner(const StencilDomain& domain, const std::vector<int>& devices,
                         const std::vector<std::int64_t>& shares, std::uint64_t seed,
                         const MpdataOptions& opts, Recipe recipe, bool flag_sync)
    : domain_(domain), shares_(shares), fp64_(opts.fp64) {
  domain.validate();
  if (devices.size() != shares.size() || shares.empty())
    throw ContractError("GroupRunner needs one device per share");
  const imb_domain dom{domain.n, domain.m, domain.l, domain.halo};
  const imb_opts o{opts.iord, opts.nonos ? 1 : 0, opts.fp64 ? IMB_FP64 : IMB_FP32};
  imb_group* g = nullptr;
  check_status(imb_group_create(&dom, &o, static_cast<int>(shares.size()), devices.data(),
                                shares.data(), &g));
  group_ = g;
  try {
    check_status(imb_group_set_sync(g, flag_sync ? IMB_GROUP_SYNC_FLAGS : IMB_GROUP_SYNC_EVENTS));
    check_status(imb_group_init_recipe(g, static_cast<int>(recipe), seed));
  } catch (...) {
    imb_group_destroy(g);
    group_ = nullptr;
    throw;
  }
}

GroupRunner::~GroupRunner() {
  if (group_) imb_group_destroy(static_cast<imb_group*>(group_));
}

double GroupRunner::run(int steps) {
  team_seconds_.assign(shares_.size(), 0.0);
  double wall = 0.0;
  check_status(imb_group_run(static_cast<imb_group*>(group_), steps, team_seconds_.data(), &wall));
  return wall;
}

std::uint64_t GroupRunner::current_checksum() const {
  std::uint64_t hsh = 0xcbf29ce484222325ull;
  const std::size_t elem = fp64_ ? 8 : 4;
  std::vector<unsigned char> host;
  for (std::size_t q = 0; q < shares_.size(); ++q) {
    imb_team* t = nullptr;
    check_status(imb_group_team(static_cast<imb_group*>(group_), static_cast<int>(q), &t));
    host.resize(static_cast<std::size_t>(shares_[q] * domain_.m * domain_.l) * elem);
    check_status(imb_team_download(t, 0, host.data(), host.size()));
    for (unsigned char b : host) {
      hsh ^= b;
      hsh *= 0x100000001b3ull;
    }
  }
  return hsh;
}

TeamResult run_team_workload(const StencilDomain& domain, int threads, int steps,
                             std::uint64_t seed) {
  if (threads < 1) throw ConfigError("threads must be >= 1");
  if (threads > thread_cap()) throw ConfigError("threads above the cap");
  if (steps < 1) throw ContractError("steps must be >= 1");
  TeamRunner team(domain, 0, seed);
  TeamResult r;
  r.seconds = team.run(steps);
  r.checksum = team.current_checksum();
  return r;
}

}  // namespace imb
