// Grouped FP64 GEMM over the coupled sectors (Alg. 8; composition = matmul P:591-609),
// the big-tile class: persistent and TMA-fed.
//
//  * One CTA per SM (grid = min(#SMs, tiles)); CTA b takes tiles b, b + grid, ... of the planner's
//    list (long K first, L2-banded raster order within a sector), so the pipeline runs across tile
//    boundaries: while the warps write one tile's C, the next tile's first k-slices are already
//    streaming in.
//  * Producer: one thread (lane 0 of warp 0) issues cp.async.bulk.tensor (TMA) loads of a 132 x 16 slice of
//    A~ (m x k) and a 20 x 128 slice of B~ (k x n) per stage into a 6-stage ring, completion counted
//    in bytes on the stage's "full" mbarrier. The boxes are 4 elements wider than the tile on their
//    contiguous axis so that shared memory holds the A stage with pitch 132 and the B stage with
//    pitch 20 doubles (both = 4 mod 16): the m8n8k4 fragment loads below are then free of bank
//    conflicts, which TMA's swizzle modes cannot give for this fragment shape. Rows / columns past
//    the block edge are zero-filled by TMA (out-of-bounds fill), so there is no predication.
//  * Consumers: all 16 warps, each a 32 x 32 sub-tile = 4 x 4 DMMA m8n8k4 fragments (mma.sync .f64,
//    SASS DMMA.8x8x4 -- tcgen05 has no f64 kind); 8-row / 8-column fragments that lie entirely past
//    the block edge are skipped (warp-uniform), so partial edge tiles cost only their real work.
//    A warp releases a stage with one arrive on its "empty" mbarrier.
// Tensor maps (one pair per GEMM group) are kernel parameters (__grid_constant__), encoded on the
// host for the workspace pointer of the call (A~ / B~ are in the library's padded workspace layout:
// leading dimensions a multiple of 4 doubles, blocks 32-byte aligned -- TMA's 16-byte rules hold).
#include <cuda.h>

#include <cstdint>

#include "tk_device.cuh"
#include "tk_gemm_tma.hpp"
#include "tk_internal.hpp"

namespace tk {

namespace {
constexpr int BM = 128, BN = 128, BK = kTmaBK, STAGES = kTmaStages;
constexpr int APITCH = kTmaAPitch, BPITCH = kTmaBPitch;
constexpr int A_STAGE = BK * APITCH, B_STAGE = BN * BPITCH;  // doubles
constexpr uint32_t STAGE_BYTES = (uint32_t)(A_STAGE + B_STAGE) * 8u;
constexpr int NCONS = 16;  // warps (4 x 4 grid of 32 x 32 sub-tiles), all consumers
constexpr int THREADS = 32 * NCONS;
constexpr int PD = STAGES - 2;  // prefetch distance: the producer waits only for a slice released 2 steps ago
}  // namespace

#ifndef TK_WARP_LATIN
#define TK_WARP_LATIN 1
#endif

size_t gemm_tma_smem_bytes() { return (size_t)STAGES * STAGE_BYTES + 2 * STAGES * sizeof(uint64_t); }

// The TMA producer is lane 0 of warp 0 (a separate producer warp would be a 17th warp: 5 warps on one
// SM sub-partition caps registers at 96 and spills the accumulators). It keeps its own cursor over the
// CTA's (tile, k-slice) sequence, PD slices ahead of the consumers, continuing into the next tile.
// Tiles are handed out dynamically (one atomicAdd per tile on a counter the host zeroes before the
// launch), in the planner's order (long K first, L2-banded raster order): the tiles in flight on the
// 148 SMs stay a contiguous window of that order, which keeps the A / B panels of a band in L2. The
// producer posts each fetched tile index into a small shared-memory ring (read by the consumers once
// the tile's first slice has landed); past the last tile it posts -1 and completes one extra "full"
// phase without data, which ends the consumers' loop.
constexpr int kRing = 8;  // > STAGES: a ring entry is overwritten only after every warp has read it
struct TmaCursor {
  int t, kt, nk, m0, n0, mi, j;  // t < 0: no tiles left (end posted)
};

__device__ __forceinline__ void tma_next_tile(const GemmTmaParams& p, TmaCursor& c, int* ring) {
  c.t = atomicAdd(p.counter, 1);
  if (c.t >= p.ntiles) c.t = -1;
  ring[c.j++ % kRing] = c.t;
  if (c.t >= 0) {
    const GemmTile& T = p.tiles[c.t];
    c.kt = 0;
    c.nk = (T.g.K + BK - 1) / BK;
    c.m0 = T.m0;
    c.n0 = T.n0;
    c.mi = T.tmap;
    tma_prefetch_desc(&p.amap[c.mi]);
    tma_prefetch_desc(&p.bmap[c.mi]);
  }
}

// issue the loads of load iteration `it` and advance the cursor; after the last tile, one data-less
// phase of the next slot carries the end marker; afterwards nothing
__device__ __forceinline__ void tma_produce(const GemmTmaParams& p, TmaCursor& c, uint32_t& it, double* As,
                                            double* Bs, uint64_t* full, uint64_t* empty, int* ring) {
  if (c.t == -2) return;
  const int s = (int)(it % STAGES);
  if (it >= (uint32_t)STAGES) mbar_wait(&empty[s], ((it / STAGES) & 1u) ^ 1u);
  ++it;
  if (c.t < 0) {  // end marker (already in the ring): release the waiting consumers
    mbar_arrive(&full[s]);
    c.t = -2;
    return;
  }
  mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
  tma_load_2d(As + s * A_STAGE, &p.amap[c.mi], c.m0, c.kt * BK, &full[s]);
  tma_load_2d(Bs + s * B_STAGE, &p.bmap[c.mi], c.kt * BK, c.n0, &full[s]);
  if (++c.kt == c.nk) tma_next_tile(p, c, ring);
}

__global__ void __launch_bounds__(THREADS, 1) gemm_tma_kernel(const __grid_constant__ GemmTmaParams p) {
  extern __shared__ __align__(1024) double tma_smem[];
  __shared__ int ring[kRing];
  double* As = tma_smem;
  double* Bs = tma_smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = threadIdx.x == 0;
  if (producer) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();  // A~ / B~ are written by the preceding permute kernels (and the counter is zeroed)
  TmaCursor cur{0, 0, 0, 0, 0, 0, 0};
  uint32_t load_it = 0;
  if (producer) {
    tma_next_tile(p, cur, ring);
    for (int d = 0; d < PD; ++d) tma_produce(p, cur, load_it, As, Bs, full, empty, ring);
  }

  // ---------------- consumers
  // Warp -> 32 x 32 sub-tile as a Latin square over the 4 SM sub-partitions (a warp runs on sub-partition
  // warp & 3, each with its own DMMA pipe): every sub-partition holds one warp of each tile-row band wm
  // and one of each column band wn, so the fragments an edge tile skips (mf / nf below) come off all four
  // pipes evenly. With wm = warp & 3 an M-edge tile idled whole sub-partitions while the others ran the
  // full k-loop, and the skipped padding (1.5 % of cfg4's tile flops) saved no time.
#if TK_WARP_LATIN
  const int wm = warp >> 2, wn = ((warp & 3) + wm) & 3;
#else
  const int wm = warp & 3, wn = warp >> 2;
#endif
  const int gq = lane >> 2, tq = lane & 3;
  uint32_t it = 0;
  for (int j = 0;; ++j) {
    // the next tile's first slice (or the end marker): its landing publishes the ring entry
    if (producer) tma_produce(p, cur, load_it, As, Bs, full, empty, ring);
    mbar_wait(&full[it % STAGES], (it / STAGES) & 1u);
    const int t = ring[j % kRing];
    if (t < 0) break;
    const int m0 = p.tiles[t].m0, n0 = p.tiles[t].n0;
    const GemmGroup g = p.tiles[t].g;
    const int nk = (g.K + BK - 1) / BK;
    // fragments past the block edge (warp-uniform): rows m0 + wm*32 + i*8, columns n0 + wn*32 + j*8
    const int mf = min(4, max(0, (g.M - m0 - wm * 32 + 7) / 8));
    const int nf = min(4, max(0, (g.N - n0 - wn * 32 + 7) / 8));
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
    for (int kt = 0; kt < nk; ++kt, ++it) {
      const int s = (int)(it % STAGES);
      if (kt > 0) {
        if (producer) tma_produce(p, cur, load_it, As, Bs, full, empty, ring);  // slice it + PD
        mbar_wait(&full[s], (it / STAGES) & 1u);
      }
      const double* as = As + s * A_STAGE + wm * 32 + gq;
      const double* bs = Bs + s * B_STAGE + (wn * 32 + gq) * BPITCH + tq;
      if (mf == 4 && nf == 4) {  // interior warps: the full 4 x 4 fragment grid, no guards
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
          double af[4], bf[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) af[i] = as[(kk + tq) * APITCH + i * 8];
#pragma unroll
          for (int j = 0; j < 4; ++j) bf[j] = bs[j * 8 * BPITCH + kk];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma884(acc[i][j], af[i], bf[j]);
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
          double af[4], bf[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) af[i] = as[(kk + tq) * APITCH + i * 8];
#pragma unroll
          for (int j = 0; j < 4; ++j) bf[j] = bs[j * 8 * BPITCH + kk];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (i >= mf) break;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (j >= nf) break;
              dmma884(acc[i][j], af[i], bf[j]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // epilogue: C = alpha * acc + beta * C (column-major, ldc); the next tile's first PD slices are in flight
    double* Cg = p.C + g.c_off;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + wm * 32 + i * 8 + gq;
      if (m >= g.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int n = n0 + wn * 32 + j * 8 + 2 * tq + c;
          if (n < g.N) {
            double* q = Cg + (int64_t)m + (int64_t)n * g.ldc;
            double v = p.alpha * acc[i][j][c];
            if (p.beta != 0.0) v = fma(p.beta, *q, v);
            *q = v;
          }
        }
    }
  }
}

// ------------------------------------------------------------------ host side
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      (void)cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<EncodeFn>(f);
  }();
  return fn;
}

bool encode_2d(CUtensorMap* m, const double* base, uint64_t d0, uint64_t d1, uint64_t ld, uint32_t b0, uint32_t b1) {
  EncodeFn f = encode_fn();
  if (!f) return false;
  const cuuint64_t dims[2] = {d0, d1};
  const cuuint64_t strides[1] = {ld * 8};
  const cuuint32_t box[2] = {b0, b1};
  const cuuint32_t es[2] = {1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

bool gemm_tma_available() { return encode_fn() != nullptr; }

bool gemm_tma_encode(GemmTmaParams& p, const std::vector<GemmGroup>& groups, const std::vector<int>& map_groups,
                     const double* A, const double* B) {
  if ((int)map_groups.size() > kTmaMaxGroups) return false;
  for (size_t i = 0; i < map_groups.size(); ++i) {
    const GemmGroup& g = groups[map_groups[i]];
    const double* a = A + g.a_off;
    const double* b = B + g.b_off;
    // TMA: global address 16-byte aligned, strides a multiple of 16 bytes (the padded workspace layout)
    if ((((uintptr_t)a) | ((uintptr_t)b)) & 15 || (g.lda & 1) || (g.ldb & 1)) return false;
    if (!encode_2d(&p.amap[i], a, (uint64_t)g.M, (uint64_t)g.K, (uint64_t)g.lda, APITCH, BK)) return false;
    if (!encode_2d(&p.bmap[i], b, (uint64_t)g.K, (uint64_t)g.N, (uint64_t)g.ldb, BPITCH, BN)) return false;
  }
  return true;
}

static PerDeviceOnce g_tma_attr;
cudaError_t launch_gemm_tma(const GemmTmaParams& p, int grid, cudaStream_t st) {
  cudaError_t e = g_tma_attr.run([] {
    return cudaFuncSetAttribute(gemm_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)gemm_tma_smem_bytes());
  });
  if (e != cudaSuccess) return e;
  static const bool pdl = knob("TK_NO_PDL", 0) == 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)THREADS);
  cfg.dynamicSmemBytes = gemm_tma_smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, gemm_tma_kernel, p);
}

}  // namespace tk
