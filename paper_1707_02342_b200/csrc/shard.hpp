// shard.hpp — the partition of one controller's samples into chunks and
// fixed groups of chunks (group.cuh), shared by the device code and the
// host-only C ABI (mppi_gpu_shard_plan).
#pragma once

#ifdef __CUDACC__
#define MPPI_HD __host__ __device__
#else
#define MPPI_HD
#endif

namespace mppi_dev {

constexpr int kGroupRowsMax = 128;  // chunks per group, at most (sets the group count)

// first chunk of group g: groups are the contiguous ranges [floor(g n / G), floor((g+1) n / G))
MPPI_HD inline int group_first_chunk(int g, int n_chunks, int n_groups) {
  return static_cast<int>((static_cast<long long>(g) * n_chunks) / n_groups);
}
// G = 8 * 2^j, the smallest with ceil(n_chunks / G) <= kGroupRowsMax: a
// function of the chunk count alone, so every rank count dividing G (1, 2, 4,
// 8, ...) sees the same groups.
MPPI_HD inline int group_count(int n_chunks) {
  int g = 8;
  while (static_cast<long long>(g) * kGroupRowsMax < n_chunks) g *= 2;
  return g;
}

}  // namespace mppi_dev
