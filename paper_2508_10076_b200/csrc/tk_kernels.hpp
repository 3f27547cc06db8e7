// Device-side descriptor tables shared by the host planner and the sm_100a kernels.
#pragma once
#include <cstdint>
#include <mutex>

#include <cuda_runtime.h>

namespace tk {

constexpr int kMaxLegs = 8;
constexpr int kMaxGroupMembers = 32;  // k_src, k_dst of one recoupling group (cfg5: <= 3; fSU2xSU2 rank 4: > 8)
#ifndef TK_MAX_ROWS
#define TK_MAX_ROWS 512  // cfg4 permutes: 512 -> 5.24 TB/s, 256 -> 4.98, 1024 -> 4.0 (tools/gpu_ab21.sh)
#endif
constexpr int kMaxRows = TK_MAX_ROWS;    // rows per rows / recoupling job (row tables in shared memory)
constexpr int kRegMembers = 8;        // destinations accumulated in registers per pass

// One uncoupled-charge group of a permute (Alg. 10): y_j = alpha * sum_i M[i][j] perm(x_i) + beta * y_j.
// Legs are listed in DESTINATION order after dropping extent-1 legs and merging legs that are
// adjacent and contiguous on both sides. A leg's stride in member m is  a[l] + b[l] * ld(m):
// codomain legs have b = 0, domain legs a = 0 (column-major blocks, reading C5).
struct PermGroup {
  int32_t ndim;
  int32_t ksrc, kdst;
  int32_t coef_off;     // into coefs: ksrc * kdst, row-major [i][j]
  int32_t src_mem;      // into members: ksrc source members
  int32_t dst_mem;      // into members: kdst destination members
  int32_t mode;         // 0 = rows (dst leg 0 is also unit-stride in src), 1 = smem-tiled transpose,
                        // 2 = box: leg 0 unit-stride on both sides, legs 1 (dst-next) and 2 (src-next)
                        //     swapped through a shared-memory box n0 x c1 x c2 (c0 = n0, ct = c1 chunk
                        //     of leg 1, R = c2 chunk of leg 2, T0 / Tt chunk counts, nrest = legs 3..)
  int32_t tleg;         // mode 1: index (dst order) of the src-fastest leg
  int32_t c0, ct;       // mode 1: chunk of leg 0 / leg tleg held in one smem tile
  int32_t R;            // mode 1: rest indices (all other legs) packed into one tile
  int32_t T0, Tt;       // mode 1: number of chunks of leg 0 / leg tleg
  int32_t lorder;       // mode 1: load-phase walk order, 3 base-3 digits (fastest first) over
                        //         {0: leg 0 chunk, 1: leg tleg chunk, 2: rest block}
  int32_t pad0_;
  int64_t nrest;        // mode 1: product of the other legs' extents
  int32_t ext[kMaxLegs];
  int64_t sa[kMaxLegs], sb[kMaxLegs];
  int64_t da[kMaxLegs], db[kMaxLegs];
  int64_t nelem;
};

struct PermMember {
  int64_t off;  // element offset of the subblock's element (0,...,0)
  int64_t ld;   // rows of its block
  int64_t d1;   // planar complex: offset of the imaginary part relative to the real part (doubles)
  int64_t d2;   // real representation of B~: offset of the [-im, re] row half (doubles)
};

// Complex modes of a permute launch. ComplexF64 contractions run as ONE real GEMM over the real
// representation of the complex blocks (north_star: "ComplexF64 via real GEMMs"; reading C21: 4 real
// products, no 3M): A~ is planar [Ar | Ai] (M x 2K), B~ is [[Br, Bi], [-Bi, Br]] (2K x 2N), so that
// A~ B~ = [Ar Br - Ai Bi | Ar Bi + Ai Br] = [Cr | Ci] = C~ (M x 2N). The permute kernels do the
// (de)interleaving in flight while they permute.
enum PermCM : int {
  kPermReal = 0,         // Float64 -> Float64
  kPermCToC = 1,         // interleaved ComplexF64 -> interleaved (tk_permute)
  kPermCToPlanar = 2,    // interleaved -> planar re | im (+d1)          (A~)
  kPermCToRealRep = 3,   // interleaved -> [[re, im], [-im, re]]          (B~)
  kPermPlanarToC = 4     // planar (+d1) -> interleaved                   (C~ -> C)
};

// A CTA work item: `count` work units of group `group` starting at unit `first`.
// mode 0 unit = one row (dst leg 0); mode 1 unit = one smem tile of c0 x ct x R elements.
#ifndef TK_PERM_THREADS
#define TK_PERM_THREADS 256  // threads per permute CTA
#endif
constexpr int kPermThreads = TK_PERM_THREADS;
constexpr int kTileElems = 4608;  // smem capacity of the two tile buffers (elements, incl. padding)
// packed jobs: `count` consecutive small single-member rows groups starting at `group` (first unused),
// so that tiny subblocks (cfg3: 9756 subblocks of ~700 elements) do not cost one CTA each
constexpr int kPackGroups = 32;
constexpr int kPackRows = 1024;
constexpr int kPackElems = 8192;
enum PermJobType : int8_t { kJobRows = 0, kJobTiled = 1, kJobPacked = 2, kJobMulti = 3, kJobSeg = 5 };
// Latency-regime jobs (kJobSeg, permutes below 2^24 elements): the planner precomputes everything a
// CTA needs into one contiguous blob -- SegHeader, `ng` SegGroup chunks (a row range of one
// single-member group each), then the source / destination offsets of every row start as int32
// (rs[nrows], rd[nrows]; offsets of permutes this small fit) -- so a CTA's prologue is one coalesced
// copy of plan data into shared memory (issued before griddepcontrol.wait, overlapping the previous
// kernel) instead of a dependent chain of job -> group -> member loads and per-row index divisions.
// Job: first = 8-byte word offset of the blob, group = its length in words (even), count = ng.
struct SegHeader {
  int32_t ng, nrows, total, pad;
};
struct SegGroup {
  int32_t estart, rstart;    // first element / first row of this chunk within the job
  uint32_t n0, fm, fs;       // row length and its division magic (FastDiv)
  uint32_t q, rem, pad;      // kPermThreads = q * n0 + rem (per-thread walk: stride kPermThreads)
  int64_t s0, d0;            // element strides along the row (source, destination)
  double c;                  // coefficient (+-1 fermionic sign)
  int64_t sd1, dd1, dd2;     // complex-mode offsets of the source / destination member (PermCM)
};
static_assert(sizeof(SegHeader) == 16 && sizeof(SegGroup) == 80, "seg blob layout");
constexpr int kSegWords = 2 + 10 * kPackGroups + kPackRows;  // rs + rd: 2 x kPackRows int32
constexpr int kRecoupleStage = 4096;  // doubles of staged recoupling sources per CTA (32 KB)
constexpr int kRecoupleDirect = 4;    // recoupling groups with <= 4 sources run beside the other jobs
struct PermJob {
  int32_t group;
  int16_t count;  // rows / tiles / packed groups of this job
  int8_t type;    // PermJobType
  int8_t op;      // which permute of a launch (0: A~ or the only one, 1: B~)
  int64_t first;
};

// One permute of a launch: data pointers, the plan's device tables, scalars.
struct PermOp {
  const void* src;
  void* dst;
  const PermGroup* groups;
  const PermMember* members;
  const double* coefs;
  const int64_t* blob;      // kJobSeg job blobs
  double alpha, beta, ims;  // ims = -1 conjugates the source (tk_contract conjA / conjB; modes 2 and 3)
};

// Grouped GEMM: C^c = alpha * A^c B^c + beta * C^c, all column-major.
struct GemmGroup {
  int64_t a_off, b_off, c_off;  // element offsets into the A~, B~, C base pointers
  int32_t M, N, K;
  int32_t lda, ldb, ldc;
  int32_t vec;                  // 1: A/B offsets and leading dims even -> 16-byte cp.async
  int32_t pad_;
};

struct GemmTile {
  int32_t group;
  int32_t m0, n0;
  int32_t pad;         // sort key (K) / skinny: rows of the tile
  int32_t k0, k1;      // k range of this tile (split-K: a slice of [0, K))
  int32_t slot;        // split-K: partial-tile slot (-1: write C directly); reduction heads: first slot
  int32_t nsplit;      // reduction heads: number of partial slots
  int32_t tmap;        // big tiles of the TMA GEMM: index of the group's tensor-map pair
  int32_t pad2_;
  GemmGroup g;         // copy of groups[group]: a CTA's descriptors arrive in one round trip
};

// One-time per-device initialisation (kernel attributes are per device; std::call_once per ordinal).
struct PerDeviceOnce {
  static constexpr int kMaxDevices = 64;
  std::once_flag flag[kMaxDevices];
  cudaError_t err[kMaxDevices] = {};
  template <class F>
  cudaError_t run(F f) {
    int d = 0;
    cudaError_t e = cudaGetDevice(&d);
    if (e != cudaSuccess) return e;
    if (d < 0 || d >= kMaxDevices) return cudaErrorInvalidDevice;
    std::call_once(flag[d], [&] { err[d] = f(); });
    return err[d];
  }
};
// every kernel attribute of tk_kernels.cu on the current device (idempotent, thread-safe)
cudaError_t ensure_kernel_attrs();

// launchers (tk_kernels.cu); each returns the status of its own launches
// ims = -1 conjugates the source (tk_contract conjA / conjB; modes 2 and 3 only). Modes 2 and 3
// write workspace only and require beta == 0.
// job table layout: [rows / tiled / packed jobs (njobs, one launch) | recoupling jobs (njobs_multi)];
// `tiled`: some job is smem-tiled (dynamic shared memory needed). Modes 2 and 3 require beta == 0.
// variant: kLaunchRowsOnly -- every job of the first launch is a rows job (leaner kernel instance)
enum PermLaunch : int { kLaunchGeneral = 0, kLaunchRowsOnly = 1 };
cudaError_t launch_permute(const PermOp& op0, const PermOp& op1, const PermJob* jobs, int njobs, int njobs_multi,
                           bool tiled, int variant, int cm, cudaStream_t st);
// tile table layout: [big (128x128 DMMA) | small (64x64 DMMA) | skinny (streaming, GemmTile.pad = rows)]
constexpr int kSkinnyMax = 16;   // skinny groups: 0 < K <= 16 and N <= 16
constexpr int kSkinnyRows = 2048;

// Gathered skinny GEMM (abelian kinds, every GEMM block with K, N <= kSkinnyMax): C~^c = A~^c B~^c
// with the rows of A~^c read straight from A -- the operand permute A -> A~ is not a separate pass.
// A GatherSeg is one A~ subblock: rows [r0, r0 + nrows) x columns [k0, k0 + nk) of its block; element
// (r0 + i, k0 + kk) is A[src + sum_l digit_l(i) * str[l] + colsrc[kk]] (digits of i over the row legs,
// fastest first) times the coefficient (neg: -1, the fermionic sign of reading C13).
constexpr int kGatherRows = 256;   // rows per tile (one per thread)
constexpr int kGatherSegs = 128;   // subblocks per tile (64 when K > 8: shared memory)
__host__ __device__ constexpr int gather_seg_cap(int kmax) { return kmax > 8 ? 64 : kmax > 4 ? 96 : kGatherSegs; }
// rows per tile by K class: 2 rows per thread while the A~ staging (K x rows doubles) stays <= 16 KB... 32 KB
#ifndef TK_GATHER_RPT
#define TK_GATHER_RPT 2  // rows per thread for K <= 8 (the A~ stage is dynamic shared memory)
#endif
__host__ __device__ constexpr int gather_rows(int kmax) { return kmax > 8 ? kGatherRows : TK_GATHER_RPT * kGatherRows; }
struct GatherSeg {
  int32_t r0, nrows, k0, nk;
  int64_t src;
  int32_t nrl, neg;
  int32_t ext[4];
  int32_t str[4];
  int32_t colsrc[kSkinnyMax];
};
static_assert(sizeof(GatherSeg) == 128, "GatherSeg layout");
struct GatherTile {
  int32_t m0, nrows;   // rows [m0, m0 + nrows) of the group's block
  int32_t seg0, nseg;  // its subblocks (row trees of those rows, every column tree), sorted by (r0, k0)
  int32_t bt;          // the group's K x N gather table for B~ (btab[bt + k * N + n]: 2 * offset into B
                       // + (coefficient < 0), or -1 for a structural zero): B needs no permute pass either
  int32_t gout0;       // -1: C~ is the output; else the output permute is folded in: the row tree starting
                       // at the tile's segment s writes column n through gouts[gout0 + s * N + n]
  GemmGroup g;
};
// Per-tile slot (kGatherSlotWords 8-byte words): the GatherTile, its first kGatherSlotSegs segments and
// the first kGatherSlotB entries of its B~ table, so a tile's descriptors arrive in one coalesced copy;
// tiles with more segments / entries read the rest from `segs` / `btab`.
constexpr int kGatherSlotSegs = 8, kGatherSlotB = 64;
constexpr int kGatherSlotWords = 10 + 16 * kGatherSlotSegs + kGatherSlotB / 2;
static_assert(sizeof(GatherTile) == 80 && kGatherSlotWords % 2 == 0, "gather slot layout");
// Output permute folded into a GEMM's stores (abelian: each C~ subblock lands in one C subblock with a
// sign): row r of a C~ row tree, column n, goes to C[base + d0 str[0] + d1 str[1] + d2 str[2]] (negated if
// neg) with (d0, d1, d2) the mixed-radix digits of r over (ext0, ext1, rest) -- the permute's row legs of
// extent > 1 in C~ order, first fastest. All columns of a row tree share the radix (host-checked).
struct GatherOut {
  int64_t base;
  int32_t str[3], neg;
  int32_t ext0, ext1;
};
static_assert(sizeof(GatherOut) == 32, "GatherOut layout");
cudaError_t launch_gather_gemm(const double* A, const double* B, double* C, const int64_t* slots, int ntiles,
                               const GatherSeg* segs, const int32_t* btab, const GatherOut* gouts, int kmax, int nmax,
                               double alpha, double oalpha, double beta, cudaStream_t st);

// split-K (small tiles of under-filled launches): partial 64x64 tiles in `parts`, then one reduction
// CTA per head tile (deterministic order)
cudaError_t launch_gemm(const double* A, const double* B, double* C, const GemmGroup* groups, const GemmTile* tiles,
                        int ntiles_big, int ntiles_small, int ntiles_skinny, const GemmTile* split_heads,
                        int nsplit_heads, double* parts, double alpha, double beta, cudaStream_t st);

// FP64 tensor-pipe probe: blocks x 8 warps, each iters x 8 DMMA m8n8k4 (2 * 8 * 8 * 4 flops each)
cudaError_t launch_dmma_probe(int blocks, long long iters, cudaStream_t st);

}  // namespace tk
