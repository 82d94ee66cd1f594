// The MPDATA workload API, B200-native. Type and function names, argument
// meaning and error behaviour follow the reference declaration
// /root/reference/proj/include/imbalance/workload.hpp:14-133 (which ships no
// implementation); the step itself is the real MPDATA scheme rather than the
// reference's 5-stage surrogate, run on the GPU through the
// C-ABI runtime. Additive extensions: MpdataOptions, the recipe argument of
// init_fields, fill_halo_periodic, and GroupRunner (several GPUs / slabs).
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

namespace imb {

namespace rt {
class Team;
}

// workload.hpp:14-26
struct StencilDomain {
  std::int64_t n = 3;
  std::int64_t m = 3;
  std::int64_t l = 3;
  std::int64_t halo = 1;

  std::int64_t cells() const { return n * m * l; }
  std::int64_t sn() const { return n + 2 * halo; }
  std::int64_t sm() const { return m + 2 * halo; }
  std::int64_t sl() const { return l + 2 * halo; }
  std::int64_t storage() const { return sn() * sm() * sl(); }
  void validate() const;  // ContractError unless extents >= 3 and halo >= 1
};

// workload.hpp:31-53 — dense double field with a ghost zone on every face.
class GridField {
 public:
  explicit GridField(const StencilDomain& d);
  const StencilDomain& domain() const { return domain_; }
  double& at(std::int64_t i, std::int64_t j, std::int64_t k) { return data_[index(i, j, k)]; }
  double at(std::int64_t i, std::int64_t j, std::int64_t k) const { return data_[index(i, j, k)]; }
  std::size_t index(std::int64_t i, std::int64_t j, std::int64_t k) const {
    const std::int64_t h = domain_.halo;
    return static_cast<std::size_t>(((i + h) * domain_.sm() + (j + h)) * domain_.sl() + (k + h));
  }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  // Interior copy in (i, j, k) order, and its inverse.
  std::vector<double> interior() const;
  void set_interior(const std::vector<double>& v);
  bool halo_valid = false;

 private:
  StencilDomain domain_;
  std::vector<double> data_;
};

// workload.hpp:57-59: psi (x), the staggered Courant numbers (u, v, w) and
// the density (rho = h) of one MPDATA step.
struct InputFields {
  GridField x, u, v, w, rho;
};

// Field recipes of BASELINE.json configs (default: config 2-5 recipe).
enum class Recipe : int { Uniform = 0, Gauss = 1, RotCube = 2 };

// MPDATA step options (no reference analogue).
struct MpdataOptions {
  int iord = 2;       // 1 = donor cell; each extra pass adds one corrective iteration
  bool nonos = true;  // nonoscillatory limiter
  bool fp64 = true;   // fp32 runs the same scheme in single precision
};

// workload.hpp:61-64 — every value a pure function of (seed, field, i, j, k);
// halos are filled periodically (the BASELINE boundary condition).
InputFields init_fields(const StencilDomain& domain, std::uint64_t seed,
                        Recipe recipe = Recipe::RotCube);

void fill_halo_clamped(GridField& f);   // workload.hpp:66-67
void fill_halo_periodic(GridField& f);  // periodic counterpart (BASELINE configs)

// workload.hpp:69-74 — 7-point max/min on the GPU (Listing 1, stage 8).
void stage_max7(const GridField& in, GridField& out);
void stage_min7(const GridField& in, GridField& out);

// workload.hpp:76-80 — one MPDATA step on device 0; periodic boundaries.
// Throws ContractError when any input halo is unfilled.
GridField run_step(const InputFields& fields, const StencilDomain& domain,
                   const MpdataOptions& opts = {});

std::uint64_t checksum(const GridField& f);  // workload.hpp:82-83 (FNV-1a 64, bytes)
std::string checksum_hex(std::uint64_t sum);
int thread_cap();  // workload.hpp:87-89; on the GPU build: the device count cap

// workload.hpp:94-122 — a team is one GPU advancing one sub-domain. The
// second constructor argument selects the device (the reference's `threads`).
class TeamRunner {
 public:
  TeamRunner(const StencilDomain& domain, int device, std::uint64_t seed,
             int pin_base_core = -1, const MpdataOptions& opts = {},
             Recipe recipe = Recipe::RotCube);
  ~TeamRunner();
  void reset();
  // Hooks run on the calling host thread: before timing, after every step,
  // after the last step; the returned time excludes them (workload.hpp:101-106).
  double run(int steps, const std::function<void()>& start_sync = {},
             const std::function<void()>& step_sync = {},
             const std::function<void()>& end_sync = {});
  std::uint64_t current_checksum() const;
  const StencilDomain& domain() const { return domain_; }
  int threads() const { return 1; }
  int device() const { return device_; }

 private:
  StencilDomain domain_;
  int device_;
  std::unique_ptr<rt::Team> team_;
};

// Additive extension: P teams = P slabs of one periodic grid,
// slab q = [sum(shares[:q]), +shares[q]) on devices[q] (several slabs may share
// a device). The fused step kernel pushes each slab's edge planes into its
// neighbours' halos (over NVLink between GPUs), so the result — and
// current_checksum() — is bit-identical to one TeamRunner on the whole grid.
class GroupRunner {
 public:
  GroupRunner(const StencilDomain& domain, const std::vector<int>& devices,
              const std::vector<std::int64_t>& shares, std::uint64_t seed = 42,
              const MpdataOptions& opts = {}, Recipe recipe = Recipe::RotCube,
              bool flag_sync = true);
  ~GroupRunner();
  GroupRunner(const GroupRunner&) = delete;
  GroupRunner& operator=(const GroupRunner&) = delete;
  // Advance all slabs `steps` steps in lockstep; returns the wall seconds
  // (max over teams), per-team compute seconds in last_team_seconds().
  double run(int steps);
  const std::vector<double>& last_team_seconds() const { return team_seconds_; }
  std::uint64_t current_checksum() const;  // FNV-1a over the whole grid, slabs in order
  int teams() const { return static_cast<int>(shares_.size()); }

 private:
  StencilDomain domain_;
  std::vector<std::int64_t> shares_;
  bool fp64_;
  void* group_ = nullptr;  // imb_group*
  std::vector<double> team_seconds_;
};

struct TeamResult {
  double seconds = 0.0;
  std::uint64_t checksum = 0;
};

// workload.hpp:129-133; the checksum depends only on (domain, seed, steps).
TeamResult run_team_workload(const StencilDomain& domain, int threads, int steps,
                             std::uint64_t seed = 42);

}  // namespace imb
