// Persistent TMA-fed grouped GEMM (big-tile class), tk_gemm_tma.cu.
#pragma once
#include <cuda.h>

#include <vector>

#include "tk_kernels.hpp"

namespace tk {

constexpr int kTmaBK = 16;        // k per stage
constexpr int kTmaStages = 6;     // ring depth (6 x 37376 B of the 227 KB of shared memory)
constexpr int kTmaAPitch = 132;   // A box / smem pitch along m (= 4 mod 16 doubles: conflict-free fragments)
constexpr int kTmaBPitch = 20;    // B box / smem pitch along k (= 4 mod 16)
constexpr int kTmaMaxGroups = 96; // tensor-map pairs in the kernel parameters (24 KB of the 32 KB limit)

// Kernel parameters: per GEMM group (indexed by GemmTile::tmap) the tensor maps of its A~ and B~ blocks,
// plus the output, the tile list and the scalars.
struct alignas(64) GemmTmaParams {
  CUtensorMap amap[kTmaMaxGroups];
  CUtensorMap bmap[kTmaMaxGroups];
  double* C;
  const GemmTile* tiles;
  int* counter;  // dynamic tile scheduler: zeroed (cudaMemsetAsync) before every launch
  int ntiles, pad_;
  double alpha, beta;
};
static_assert(sizeof(GemmTmaParams) <= 32764, "kernel parameter limit");

size_t gemm_tma_smem_bytes();
bool gemm_tma_available();  // the driver's tensor-map encoder is reachable
// Encode the maps of groups[map_groups[i]] into p.amap[i] / p.bmap[i] for the A~ / B~ base pointers;
// false if the layout does not meet TMA's alignment rules (then the cp.async kernel runs instead).
bool gemm_tma_encode(GemmTmaParams& p, const std::vector<GemmGroup>& groups, const std::vector<int>& map_groups,
                     const double* A, const double* B);
cudaError_t launch_gemm_tma(const GemmTmaParams& p, int grid, cudaStream_t st);

}  // namespace tk
