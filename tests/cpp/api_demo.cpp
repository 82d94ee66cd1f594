// A C++ caller of the reference-named API (include/imbalance/*.hpp) linked
// against libimb_b200.so — what a reference user recompiles. `cpu` mode
// exercises the FPM partitioner (no GPU); `gpu` mode runs the workload API.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "imbalance/errors.hpp"
#include "imbalance/fpm.hpp"
#include "imbalance/partition.hpp"
#include "imbalance/stats.hpp"
#include "imbalance/workload.hpp"

static int fails = 0;
#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                \
    }                                                         \
  } while (0)

static void cpu_part() {
  // PAPER.md:336-344 / SPEC.md:61-73 worked example.
  imb::SpeedFunction f(15360, 8, {{112, 1436742.0}, {120, 1240377.0}, {128, 1418579.0}}, "paper");
  imb::Partition p = imb::partition_paired({480, 4, f});
  CHECK((p.shares == std::vector<std::int64_t>{112, 128, 112, 128}));
  CHECK(p.offset && *p.offset == 8);
  CHECK(std::fabs(p.makespan - 1.385950) < 1e-6);
  imb::Partition g = imb::partition_general({480, 4, f});
  CHECK((g.shares == std::vector<std::int64_t>{112, 112, 128, 128}));
  bool threw = false;
  try {
    imb::partition_paired({480, 3, f});
  } catch (const imb::ContractError&) {
    threw = true;
  }
  CHECK(threw);
  CHECK(std::fabs(imb::t_quantile_975(1) - 12.706204736174705) < 1e-9);
  std::printf("cpu part: %s\n", fails ? "FAILED" : "ok");
}

static void gpu_part() {
  imb::StencilDomain d{32, 24, 64, 1};
  imb::InputFields in = imb::init_fields(d, 42);
  imb::GridField out = imb::run_step(in, d);  // one MPDATA step on device 0
  CHECK(out.halo_valid);
  double m0 = 0, m1 = 0;
  for (std::int64_t i = 0; i < d.n; ++i)
    for (std::int64_t j = 0; j < d.m; ++j)
      for (std::int64_t k = 0; k < d.l; ++k) {
        m0 += in.x.at(i, j, k) * in.rho.at(i, j, k);
        m1 += out.at(i, j, k) * in.rho.at(i, j, k);
      }
  CHECK(std::fabs(m1 - m0) <= 1e-12 * m0);  // mass conservation
  imb::TeamRunner team(d, 0, 42);
  const double secs = team.run(5);
  CHECK(secs > 0);
  const std::uint64_t c1 = team.current_checksum();
  team.reset();
  team.run(5);
  CHECK(team.current_checksum() == c1);  // deterministic
  imb::TeamResult r = imb::run_team_workload(d, 1, 5, 42);
  CHECK(r.checksum == c1);
  // Three slabs (uneven) on device 0: bit-identical to the single team.
  for (bool flags : {false, true}) {
    imb::GroupRunner grp(d, {0, 0, 0}, {10, 7, 15}, 42, {}, imb::Recipe::RotCube, flags);
    CHECK(grp.run(2) > 0);
    CHECK(grp.run(3) > 0);
    CHECK(grp.last_team_seconds().size() == 3);
    CHECK(grp.current_checksum() == c1);
  }
  bool threw = false;
  try {
    imb::GroupRunner bad(d, {0, 0}, {16, 15});  // shares must cover n
  } catch (const imb::ContractError&) {
    threw = true;
  }
  CHECK(threw);
  std::printf("gpu part: %s (checksum %s)\n", fails ? "FAILED" : "ok",
              imb::checksum_hex(c1).c_str());
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  cpu_part();
  if (gpu) gpu_part();
  return fails ? 1 : 0;
}
