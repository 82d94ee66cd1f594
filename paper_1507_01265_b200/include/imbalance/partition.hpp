// FPM partitioner: distributes the slab axis of the MPDATA grid over p
// homogeneous GPUs that share one speed function. Names and contracts are
// those of /root/reference/proj/include/imbalance/partition.hpp:17-72;
// csrc/host/partition.cpp is a fresh implementation whose outputs are
// integer-identical (shares, offset) and bit-identical (times) to it.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "imbalance/fpm.hpp"

namespace imb {

// partition.hpp:17-22
struct PartitionProblem {
  std::int64_t total = 0;
  int processors = 2;
  SpeedFunction model;
  bool allow_idle = false;
};

// partition.hpp:27-32
struct Partition {
  std::vector<std::int64_t> shares;
  std::vector<double> per_time;
  double makespan = 0.0;
  std::optional<std::int64_t> offset;
};

inline constexpr std::int64_t kDefaultOracleCap = 10'000'000;

Partition predict_makespan(const SpeedFunction& model, std::span<const std::int64_t> shares);

// Algorithm 1: symmetric offsets around n/p; even
// indices get the smaller share. Requires even p >= 2.
Partition partition_paired(const PartitionProblem& problem);

// Exact min-makespan split for any p >= 1. Among optima, the
// lexicographically smallest non-increasing share vector is chosen and
// returned in ASCENDING order — the order the reference implementation
// emits (partition.cpp:213-214), despite its header comment.
Partition partition_general(const PartitionProblem& problem);

// Exhaustive search; shares returned non-increasing (partition.cpp:238-282).
Partition brute_force_oracle(const PartitionProblem& problem,
                             std::int64_t max_compositions = kDefaultOracleCap);

// partition.hpp:60-72
struct Improvement {
  std::pair<std::int64_t, std::int64_t> violating_pair;
  std::int64_t delta = 0;
  double gain_s = 0.0;
};
std::optional<Improvement> improvement_search(const SpeedFunction& model,
                                              std::int64_t balanced_share);

// Slab offsets (prefix sums in processor order) for a share vector: the
// decomposition the GPU group uses.
std::vector<std::int64_t> slab_offsets(std::span<const std::int64_t> shares);

}  // namespace imb
