// Blockwise (truncated) singular value decomposition of a tensor map.
//
// The paper's definition (eq. svd; "extend the SVD to tensor maps by directly acting on the
// matrix representation"; Alg. 9 "Abelian tensor decomposition" P:1317-1332): permute A to
// A~ = permute(A, (p, q)), then for every coupled sector c factor the block a_c = u_c s_c vh_c; U inherits
// A~'s codomain trees, Vh its domain trees, and the new bond space W carries one sector c with
// degeneracy k_c (the number of kept singular values of block c). Truncation is global over all blocks
// (SPEC TruncationScheme): values sorted descending, a value of block c weighs d_c (quantum dimension,
// P:1536-1540), MaxTotalDim keeps greedily while sum_kept d_c <= D, RelError drops the smallest set with
// sqrt(sum_dropped d_c s^2) <= eps ||A||, ||A||^2 = sum_c d_c sum s_c^2.
//
// B200 design: the permute is the library's permute kernel (into a padded workspace); every block is
// factored by ONE CTA with a one-sided (Hestenes) Jacobi SVD -- column pairs of the tall orientation are
// orthogonalised by plane rotations in a round-robin (circle) order, N/2 disjoint pairs per round, one
// warp per pair, until no rotation is needed; the working matrix and the accumulated right rotations sit
// in shared memory when they fit (else in the L2-resident workspace). One-sided Jacobi gives singular
// values to high relative accuracy, so no Gram matrix is ever formed. A second kernel writes the kept
// columns/rows into U, S, Vh in their canonical block layouts.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>

#include "tk_plan.hpp"

namespace tk {

// ---------------------------------------------------------------- device side
struct SvdBlock {
  int64_t a_off;   // A~ block (column-major, lda)
  int64_t g_off;   // tall working matrix G (R x K, ldg): A~ in place, or its transpose
  int64_t v_off;   // K x K right rotations (ldv)
  int64_t s_off;   // K sorted singular values (doubles)
  int64_t p_off;   // K column indices in sorted order (int32, in the index region)
  int32_t M, N, lda;
  int32_t R, K, ldg, ldv;
  int32_t trans;   // 1: M < N, G = A~^T
  int32_t smem;    // 1: G and V fit in shared memory
  int32_t pad_;
};

struct SvdOut {     // extraction target of one block (canonical layouts of U, S, Vh)
  int64_t u_off, s_off, vh_off;
  int32_t k;        // kept singular values (0: block dropped)
  int32_t blk;      // SvdBlock index
};

constexpr int kSvdThreads = 1024;
constexpr int kSvdWarps = kSvdThreads / 32;
constexpr int kSvdLanes = 8;                                  // lanes per column pair
constexpr int kSvdGroups = kSvdThreads / kSvdLanes;           // pairs rotated concurrently
constexpr int kSvdMaxK = 2048;         // per-block limit on min(M, N) (shared scratch below)
constexpr int kSvdSmemBytes = 206 * 1024;
constexpr int kSvdMaxSweeps = 60;

// SvdBlock.smem: 2 = G and V in shared memory, 1 = G only (V recovered as X^T G S^-2 afterwards),
// 0 = both in the (L2-resident) workspace.

template <int L = kSvdLanes>
__device__ __forceinline__ double group_sum(double x) {  // sum over the L lanes of a pair group
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// MODE is a template parameter so that shared-memory operands compile to LDS/STS (a runtime choice
// of pointer would leave generic LD/ST on the critical path of every rotation)
template <int MODE, int L>
__device__ __forceinline__ void svd_block(const SvdBlock& b, double* __restrict__ ws, int32_t* __restrict__ idx,
                                          double* sm, double* sig, int& rotated, int debug) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = tid / L, gl = tid % L;
  const int R = b.R, K = b.K;
  // working copies: G (R x K, ld ldG) and V (K x K, ld ldV)
  constexpr bool gs = MODE >= 1, vs = MODE == 2, accv = MODE != 1;
  const int ldG = gs ? R : b.ldg, ldV = vs ? K : b.ldv;
  double* G = gs ? sm : ws + b.g_off;
  double* V = vs ? sm + (size_t)R * K : ws + b.v_off;
  const double* A = ws + b.a_off;
  for (int64_t e = tid; e < (int64_t)R * K; e += kSvdThreads) {
    const int i = (int)(e % R), j = (int)(e / R);
    const double x = b.trans ? A[j + (int64_t)i * b.lda] : A[i + (int64_t)j * b.lda];
    if (gs || b.trans) G[i + (int64_t)j * ldG] = x;
  }
  if (accv)
    for (int64_t e = tid; e < (int64_t)K * K; e += kSvdThreads) {
      const int i = (int)(e % K), j = (int)(e / K);
      V[i + (int64_t)j * ldV] = (i == j) ? 1.0 : 0.0;
    }
  __syncthreads();
  const int n = K + (K & 1);  // circle method over n players; player K (if K odd) is a bye
  // stop rotating a pair once its cosine is at the rounding level of a length-R dot product
  const double tol = 2.3e-16 * sqrt((double)R);
  int sweep = 0;
  const long long t_start = clock64();
  for (; sweep < kSvdMaxSweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    int any = 0;
    for (int r = 0; r < n - 1; ++r) {
      // groups of 8 lanes each own one disjoint column pair of round r (all lanes of a warp stay
      // converged for the group shuffles; idle groups run empty loops)
      for (int base = 0; base < n / 2; base += (kSvdThreads / L)) {
        if (base + warp * (32 / L) >= n / 2) continue;  // warp-uniform: no pair for this warp
        const int pr = base + grp;
        int p = 0, q = 0;
        bool act = pr < n / 2;
        if (act) {
          if (pr == 0) {
            p = n - 1;
            q = r;
          } else {
            p = (r + pr) % (n - 1);
            q = (r - pr + n - 1) % (n - 1);
          }
          if (p > q) {
            const int t = p;
            p = q;
            q = t;
          }
          act = q < K;
        }
        const int len = act ? R : 0;
        double* gp = G + (int64_t)p * ldG;
        double* gq = G + (int64_t)q * ldG;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = gl; i < len; i += L) {
          const double x = gp[i], y = gq[i];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = group_sum<L>(al);
        be = group_sum<L>(be);
        ga = group_sum<L>(ga);
        if (act && ga != 0.0 && fabs(ga) > tol * sqrt(al * be)) {
          // 2x2 symmetric Schur rotation of [[al, ga], [ga, be]] (Hestenes one-sided Jacobi)
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = gl; i < R; i += L) {
            const double x = gp[i], y = gq[i];
            gp[i] = c * x - s * y;
            gq[i] = s * x + c * y;
          }
          if (accv) {
            double* vp = V + (int64_t)p * ldV;
            double* vq = V + (int64_t)q * ldV;
            for (int i = gl; i < K; i += L) {
              const double x = vp[i], y = vq[i];
              vp[i] = c * x - s * y;
              vq[i] = s * x + c * y;
            }
          }
          any = 1;
        }
      }
      __syncthreads();
    }
    if (any) rotated = 1;
    __syncthreads();
    if (!rotated) break;
    __syncthreads();
  }
  if (debug && tid == 0)
    printf("[tk svd] block %d: %d x %d, mode %d, %d sweeps, %lld cycles/round\n", blockIdx.x, R, K, MODE, sweep + 1,
           (clock64() - t_start) / ((long long)(sweep + 1) * (n - 1)));
  // singular values = column norms; rank by value (descending, ties by column index)
  for (int j = warp; j < K; j += kSvdWarps) {
    const double* g = G + (int64_t)j * ldG;
    double x = 0.0;
    for (int i = lane; i < R; i += 32) x = fma(g[i], g[i], x);
    x = warp_sum(x);
    if (lane == 0) sig[j] = sqrt(x);
  }
  __syncthreads();
  double* sv = ws + b.s_off;
  int32_t* pv = idx + b.p_off;
  for (int j = tid; j < K; j += kSvdThreads) {
    const double sj = sig[j];
    int rank = 0;
    for (int i = 0; i < K; ++i) rank += (sig[i] > sj) || (sig[i] == sj && i < j);
    sv[rank] = sj;
    pv[rank] = j;
  }
  if (!accv) {
    // G = X V with X the tall input (A~ or A~^T, untouched in the workspace): V = X^T G S^-2. A warp
    // takes one row i of V: column i of X is staged in the warp's smem slot (coalesced load), then its
    // lanes sweep 32 consecutive columns j of G with 4 independent accumulators each.
    double* Vw = ws + b.v_off;
    double* xs = sm + (size_t)R * K + (size_t)warp * R;
    for (int i = warp; i < K; i += kSvdWarps) {
      for (int r = lane; r < R; r += 32) xs[r] = b.trans ? A[i + (int64_t)r * b.lda] : A[r + (int64_t)i * b.lda];
      __syncwarp();
      for (int j0 = 0; j0 < K; j0 += 32) {
        const int j = j0 + lane;
        const int jj = j < K ? j : K - 1;
        const double* g = G + (int64_t)jj * ldG;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int r = 0;
        for (; r + 3 < R; r += 4) {
          a0 = fma(xs[r], g[r], a0);
          a1 = fma(xs[r + 1], g[r + 1], a1);
          a2 = fma(xs[r + 2], g[r + 2], a2);
          a3 = fma(xs[r + 3], g[r + 3], a3);
        }
        for (; r < R; ++r) a0 = fma(xs[r], g[r], a0);
        if (j < K) {
          const double s2 = sig[j] * sig[j];
          Vw[i + (int64_t)j * b.ldv] = s2 > 0.0 ? ((a0 + a1) + (a2 + a3)) / s2 : 0.0;
        }
      }
      __syncwarp();
    }
  }
  // write the converged G (and V) back to the workspace (the extraction kernel reads them there); for
  // a non-transposed block G's home is A~ itself, which the V recovery above still reads
  __syncthreads();
  if (gs) {
    double* Gw = ws + b.g_off;
    for (int64_t e = tid; e < (int64_t)R * K; e += kSvdThreads) {
      const int i = (int)(e % R), j = (int)(e / R);
      Gw[i + (int64_t)j * b.ldg] = G[i + (int64_t)j * ldG];
    }
  }
  if (vs) {
    double* Vw = ws + b.v_off;
    for (int64_t e = tid; e < (int64_t)K * K; e += kSvdThreads) {
      const int i = (int)(e % K), j = (int)(e / K);
      Vw[i + (int64_t)j * b.ldv] = V[i + (int64_t)j * ldV];
    }
  }
}

__global__ void __launch_bounds__(kSvdThreads, 1)
    svd_jacobi_kernel(double* __restrict__ ws, int32_t* __restrict__ idx, const SvdBlock* __restrict__ blocks,
                      const int32_t* __restrict__ list, int debug) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int rotated;
  __shared__ double sig[kSvdMaxK];
  const SvdBlock b = blocks[list[blockIdx.x]];
  if (b.K == 0) return;
  if (b.smem == 2)
    svd_block<2, kSvdLanes>(b, ws, idx, sm, sig, rotated, debug);
  else if (b.smem == 1)
    svd_block<1, kSvdLanes>(b, ws, idx, sm, sig, rotated, debug);
  else
    svd_block<0, kSvdLanes>(b, ws, idx, sm, sig, rotated, debug);
}

// ---- cluster variant: the rows of G (and of V) are split over the CTAs of a thread-block cluster
// (CS = 1, 2, 4 or 8 CTAs on as many SMs); every column pair's (alpha, beta, gamma) is the sum of the
// CTAs' partial dot products, exchanged through distributed shared memory with ONE cluster barrier
// per Jacobi round (partials double-buffered by round parity). All CTAs then take the identical
// rotation and update their own rows. A round's critical path shrinks with R / CS, and blocks whose
// G + V exceed one SM's shared memory still run on-chip.
constexpr int kClusterMaxK = 512;
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ const double* map_rank(const double* p, uint32_t rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;\n" : "=l"(out) : "l"((uint64_t)p), "r"(rank));
  return (const double*)out;
}

template <int CS>
__global__ void __launch_bounds__(kSvdThreads, 1)
    svd_cluster_kernel(double* __restrict__ ws, int32_t* __restrict__ idx, const SvdBlock* __restrict__ blocks,
                       const int32_t* __restrict__ list, int debug) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double part[2][kClusterMaxK / 2][3];
  __shared__ double sig[kClusterMaxK];
  __shared__ int rotated;
  const SvdBlock b = blocks[list[blockIdx.x / CS]];
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = tid / kSvdLanes, gl = tid % kSvdLanes;
  const int R = b.R, K = b.K;
  const int Rl = (R + CS - 1) / CS, Kl = (K + CS - 1) / CS;
  const int r0 = min(R, (int)rank * Rl), r1 = min(R, r0 + Rl), nr = r1 - r0;
  const int v0 = min(K, (int)rank * Kl), v1 = min(K, v0 + Kl), nv = v1 - v0;
  double* G = sm;                      // nr x K (ld Rl), local rows r0..r1
  double* V = sm + (size_t)Rl * K;     // nv x K (ld Kl), local rows v0..v1
  const double* A = ws + b.a_off;
  for (int64_t e = tid; e < (int64_t)nr * K; e += kSvdThreads) {
    const int i = (int)(e % nr), j = (int)(e / nr);
    const int gi = r0 + i;
    G[i + (int64_t)j * Rl] = b.trans ? A[j + (int64_t)gi * b.lda] : A[gi + (int64_t)j * b.lda];
  }
  for (int64_t e = tid; e < (int64_t)nv * K; e += kSvdThreads) {
    const int i = (int)(e % nv), j = (int)(e / nv);
    V[i + (int64_t)j * Kl] = (v0 + i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int n = K + (K & 1);
  const double tol = 2.3e-16 * sqrt((double)R);
  int sweep = 0, par = 0;
  for (; sweep < kSvdMaxSweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < n - 1; ++r) {
      // (1) local partial dot products of every pair of round r
      for (int base = 0; base < n / 2; base += kSvdGroups) {
        if (base + warp * (32 / kSvdLanes) >= n / 2) continue;  // warp-uniform: no pair for this warp
        const int pr = base + grp;
        int p = 0, q = 0;
        bool act = pr < n / 2;
        if (act) {
          if (pr == 0) { p = n - 1; q = r; } else { p = (r + pr) % (n - 1); q = (r - pr + n - 1) % (n - 1); }
          if (p > q) { const int t = p; p = q; q = t; }
          act = q < K;
        }
        const int len = act ? nr : 0;
        const double* gp = G + (int64_t)p * Rl;
        const double* gq = G + (int64_t)q * Rl;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = gl; i < len; i += kSvdLanes) {
          const double x = gp[i], y = gq[i];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = group_sum(al);
        be = group_sum(be);
        ga = group_sum(ga);
        if (act && gl == 0) {
          part[par][pr][0] = al;
          part[par][pr][1] = be;
          part[par][pr][2] = ga;
        }
      }
      if (CS > 1) cluster_sync_all(); else __syncthreads();
      // (2) identical sums in every CTA (rank order), rotation, update of the local rows
      int any = 0;
      for (int base = 0; base < n / 2; base += kSvdGroups) {
        if (base + warp * (32 / kSvdLanes) >= n / 2) continue;  // warp-uniform: no pair for this warp
        const int pr = base + grp;
        int p = 0, q = 0;
        bool act = pr < n / 2;
        if (act) {
          if (pr == 0) { p = n - 1; q = r; } else { p = (r + pr) % (n - 1); q = (r - pr + n - 1) % (n - 1); }
          if (p > q) { const int t = p; p = q; q = t; }
          act = q < K;
        }
        if (!act) continue;
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int c = 0; c < CS; ++c) {
          const double* pp = CS > 1 ? map_rank(&part[par][pr][0], (uint32_t)c) : &part[par][pr][0];
          al += pp[0];
          be += pp[1];
          ga += pp[2];
        }
        if (ga == 0.0 || fabs(ga) <= tol * sqrt(al * be)) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        double* gp = G + (int64_t)p * Rl;
        double* gq = G + (int64_t)q * Rl;
        for (int i = gl; i < nr; i += kSvdLanes) {
          const double x = gp[i], y = gq[i];
          gp[i] = c * x - s * y;
          gq[i] = s * x + c * y;
        }
        double* vp = V + (int64_t)p * Kl;
        double* vq = V + (int64_t)q * Kl;
        for (int i = gl; i < nv; i += kSvdLanes) {
          const double x = vp[i], y = vq[i];
          vp[i] = c * x - s * y;
          vq[i] = s * x + c * y;
        }
        any = 1;
      }
      if (any) rotated = 1;
      par ^= 1;
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  if (debug && tid == 0 && rank == 0)
    printf("[tk svd] block %d: %d x %d, cluster %d, %d sweeps\n", list[blockIdx.x / CS], R, K, CS, sweep + 1);
  // singular values: column norms summed over the cluster (rank order)
  double* nrm = &part[par][0][0];  // reuse: K <= kClusterMaxK partial norms (3 * K / 2 >= K slots)
  for (int j = warp; j < K; j += kSvdWarps) {
    const double* g = G + (int64_t)j * Rl;
    double x = 0.0;
    for (int i = lane; i < nr; i += 32) x = fma(g[i], g[i], x);
    x = warp_sum(x);
    if (lane == 0) nrm[j] = x;
  }
  if (CS > 1) cluster_sync_all(); else __syncthreads();
  for (int j = tid; j < K; j += kSvdThreads) {
    double x = 0.0;
#pragma unroll
    for (int c = 0; c < CS; ++c) x += (CS > 1 ? map_rank(nrm, (uint32_t)c) : nrm)[j];
    sig[j] = sqrt(x);
  }
  __syncthreads();
  if (rank == 0) {
    double* sv = ws + b.s_off;
    int32_t* pv = idx + b.p_off;
    for (int j = tid; j < K; j += kSvdThreads) {
      const double sj = sig[j];
      int rk = 0;
      for (int i = 0; i < K; ++i) rk += (sig[i] > sj) || (sig[i] == sj && i < j);
      sv[rk] = sj;
      pv[rk] = j;
    }
  }
  // local rows of G and V back to the workspace (the extraction kernel reads them there)
  double* Gw = ws + b.g_off;
  double* Vw = ws + b.v_off;
  for (int64_t e = tid; e < (int64_t)nr * K; e += kSvdThreads) {
    const int i = (int)(e % nr), j = (int)(e / nr);
    Gw[r0 + i + (int64_t)j * b.ldg] = G[i + (int64_t)j * Rl];
  }
  for (int64_t e = tid; e < (int64_t)nv * K; e += kSvdThreads) {
    const int i = (int)(e % nv), j = (int)(e / nv);
    Vw[v0 + i + (int64_t)j * b.ldv] = V[i + (int64_t)j * Kl];
  }
  if (CS > 1) cluster_sync_all();  // no CTA may exit while others still read its shared memory
}

// U[:, r] = G[:, perm r] / s_r (or V[:, perm r] when transposed); Vh[r, :] = V[:, perm r]^T (or G / s);
// S = diag(s). One CTA per (block, part), part 0 = U, 1 = Vh, 2 = S.
__global__ void __launch_bounds__(256)
    svd_extract_kernel(const double* __restrict__ ws, const int32_t* __restrict__ idx,
                       const SvdBlock* __restrict__ blocks, const SvdOut* __restrict__ outs, double* __restrict__ U,
                       double* __restrict__ S, double* __restrict__ Vh) {
  const SvdOut o = outs[blockIdx.x];
  const SvdBlock b = blocks[o.blk];
  const int part = blockIdx.y;
  const int k = o.k, M = b.M, N = b.N;
  const double* sv = ws + b.s_off;
  const int32_t* pv = idx + b.p_off;
  const double* G = ws + b.g_off;
  const double* V = ws + b.v_off;
  if (part == 0) {  // U: M x k column-major
    for (int64_t e = threadIdx.x; e < (int64_t)M * k; e += blockDim.x) {
      const int i = (int)(e % M), r = (int)(e / M);
      const int j = pv[r];
      double x;
      if (!b.trans) {
        const double s = sv[r];
        x = s > 0.0 ? G[i + (int64_t)j * b.ldg] / s : 0.0;
      } else {
        x = V[i + (int64_t)j * b.ldv];
      }
      U[o.u_off + e] = x;
    }
  } else if (part == 1) {  // Vh: k x N column-major
    for (int64_t e = threadIdx.x; e < (int64_t)k * N; e += blockDim.x) {
      const int r = (int)(e % k), c = (int)(e / k);
      const int j = pv[r];
      double x;
      if (!b.trans) {
        x = V[c + (int64_t)j * b.ldv];
      } else {
        const double s = sv[r];
        x = s > 0.0 ? G[c + (int64_t)j * b.ldg] / s : 0.0;
      }
      Vh[o.vh_off + e] = x;
    }
  } else {  // S: k x k diagonal
    for (int64_t e = threadIdx.x; e < (int64_t)k * k; e += blockDim.x) {
      const int r = (int)(e % k), c = (int)(e / k);
      S[o.s_off + e] = (r == c) ? sv[r] : 0.0;
    }
  }
}

// ---------------------------------------------------------------- host side
static PerDeviceOnce g_svd_attrs;
static cudaError_t ensure_svd_attrs() {
  return g_svd_attrs.run([] {
    cudaError_t e = cudaFuncSetAttribute(svd_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSvdSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(svd_cluster_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSvdSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(svd_cluster_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSvdSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(svd_cluster_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSvdSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(svd_cluster_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSvdSmemBytes);
    return e;
  });
}

struct SvdPlan {
  Tensor* At = nullptr;
  PermPlan pa;
  PadLayout la;
  std::vector<SvdBlock> blocks;
  DevBuf d_blocks;
  // launch classes: 0 = single-CTA kernel (modes 0/1/2), 1..4 = cluster kernel with 1, 2, 4, 8 CTAs
  std::vector<int32_t> lists[5];
  int class_smem[5] = {0, 0, 0, 0, 0};
  DevBuf d_lists[5];
  size_t ws_bytes = 0, idx_off = 0;  // byte offset of the int32 index region
  int64_t n_sigma = 0;
  int smem_bytes = 0;
  std::mutex outs_mu;
  std::once_flag up_once;
  void ensure_uploaded() {
    std::call_once(up_once, [&] {
      check_cuda(ensure_svd_attrs(), "svd kernel attributes");
      pa.ensure_uploaded();
      d_blocks.upload(blocks);
      for (int c = 0; c < 5; ++c) d_lists[c].upload(lists[c]);
    });
  }
  std::map<std::string, std::unique_ptr<DevBuf>> outs;  // extraction tables per kept-count pattern
  ~SvdPlan() {
    if (At) tk_tensor_release((tk_tensor*)At);
  }
};

static PlanCache<SvdPlan> g_svd_cache;

void svd_cache_clear() { g_svd_cache.clear(); }
size_t svd_cache_size() { return g_svd_cache.size(); }

static std::shared_ptr<SvdPlan> build_svd_plan(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q);

static std::shared_ptr<SvdPlan> get_svd_plan(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q) {
  if (A.dtype != TK_F64) TK_THROW(TK_ERR_UNSUPPORTED, "tk_svd: Float64 only in this build");
  std::ostringstream os;
  os << A.sig << "#";
  for (int x : p) os << x << ",";
  os << "#";
  for (int x : q) os << x << ",";
  return g_svd_cache.get(os.str(), [&] { return build_svd_plan(A, p, q); });
}

static std::shared_ptr<SvdPlan> build_svd_plan(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q) {
  validate_perm(A, p, q);
  auto P = std::make_shared<SvdPlan>();
  P->At = permuted_tensor(A, p, q, TK_F64);
  P->la = pad_layout(*P->At);
  build_perm_plan(A, p, q, *P->At, P->pa, 8, nullptr, &P->la);
  P->pa.identity = false;  // always copy: the Jacobi sweeps work in place on A~
  // workspace: A~ | transposed G blocks | V blocks | sigma | (int32) sorted column indices
  int64_t off = P->la.total;
  int64_t nsig = 0, nidx = 0;
  for (size_t c = 0; c < P->At->blocks.size(); ++c) {
    const Block& bl = P->At->blocks[c];
    SvdBlock b{};
    b.M = (int32_t)bl.rows;
    b.N = (int32_t)bl.cols;
    b.lda = (int32_t)P->la.ld[c];
    b.a_off = P->la.off[c];
    b.trans = bl.rows < bl.cols;
    b.R = (int32_t)std::max(bl.rows, bl.cols);
    b.K = (int32_t)std::min(bl.rows, bl.cols);
    if (b.K > kSvdMaxK) TK_THROW(TK_ERR_UNSUPPORTED, "tk_svd: a block with min(rows, cols) > 2048");
    if (b.trans) {
      b.ldg = (b.R + 3) & ~3;
      b.g_off = off;
      off += (int64_t)b.ldg * b.K;
    } else {
      b.ldg = b.lda;
      b.g_off = b.a_off;
    }
    b.ldv = (b.K + 3) & ~3;
    b.v_off = off;
    off += (int64_t)b.ldv * b.K;
    b.s_off = nsig;  // relative; rebased below
    nsig += b.K;
    b.p_off = nidx;
    nidx += b.K;
    const int64_t need2 = ((int64_t)b.R * b.K + (int64_t)b.K * b.K) * 8;
    const int64_t need1 = ((int64_t)b.R * b.K + (int64_t)kSvdWarps * b.R) * 8;  // + per-warp X column slots
    b.smem = need2 <= kSvdSmemBytes ? 2 : (need1 <= kSvdSmemBytes ? 1 : 0);
    // cluster kernel: rows split over CS CTAs so that a round's critical path is <= ~48 rows per CTA
    int cls = 0;
    static const bool no_cluster = knob("TK_SVD_NO_CLUSTER", 0) != 0;
    // blocks that fit one SM's shared memory stay on the single-CTA kernel (one barrier per round, measured
    // faster there); larger ones go to the cluster kernel with ~24 rows per CTA (cfg3: 32.8 -> 15.0 ms)
    if (!no_cluster && b.K <= kClusterMaxK && b.smem == 0) {
      static const int rows_target = (int)knob("TK_SVD_ROWS", 24);
      const int want = b.R <= rows_target ? 1 : (b.R <= 2 * rows_target ? 2 : (b.R <= 4 * rows_target ? 4 : 8));
      for (int ci = 0, cs = 1; ci < 4; ++ci, cs *= 2) {
        const int64_t Rl = (b.R + cs - 1) / cs, Kl = (b.K + cs - 1) / cs;
        const int64_t need = (Rl + Kl) * b.K * 8;
        if (cs >= want && need <= kSvdSmemBytes) {
          cls = 1 + ci;
          P->class_smem[cls] = std::max<int>(P->class_smem[cls], (int)need);
          break;
        }
      }
    }
    if (cls == 0 && b.smem) P->smem_bytes = std::max<int>(P->smem_bytes, (int)(b.smem == 2 ? need2 : need1));
    P->lists[cls].push_back((int32_t)P->blocks.size());
    P->blocks.push_back(b);
  }
  const int64_t sig_base = off;
  for (auto& b : P->blocks) b.s_off += sig_base;
  off += nsig;
  P->n_sigma = nsig;
  P->idx_off = align256((size_t)off * 8);
  P->ws_bytes = align256(P->idx_off + (size_t)nidx * 4);
  return P;
}

static std::vector<int> ivec(const int32_t* v, int n) { return std::vector<int>(v, v + n); }

// Global truncation (SPEC TruncationScheme): returns kept counts per A~ block.
static std::vector<int64_t> truncation(const Tensor& At, const std::vector<SvdBlock>& blocks,
                                       const std::vector<double>& sig, int64_t max_dim, double rel_tol, double* err,
                                       double* norm) {
  struct Item {
    double s;
    int c, r;
  };
  std::vector<Item> all;
  double n2 = 0.0;
  for (size_t c = 0; c < blocks.size(); ++c) {
    const double dc = sector_dim(At.kind, At.blocks[c].coupled);
    const int64_t base = blocks[c].s_off - blocks[0].s_off;
    for (int r = 0; r < blocks[c].K; ++r) {
      const double s = sig[base + r];
      all.push_back(Item{s, (int)c, r});
      n2 += dc * s * s;
    }
  }
  // descending value; ties by canonical charge order (block index), then block-local index
  std::stable_sort(all.begin(), all.end(), [](const Item& x, const Item& y) {
    if (x.s != y.s) return x.s > y.s;
    if (x.c != y.c) return x.c < y.c;
    return x.r < y.r;
  });
  size_t nkeep = all.size();
  if (max_dim > 0) {
    double tot = 0.0;
    size_t i = 0;
    for (; i < all.size(); ++i) {
      const double dc = sector_dim(At.kind, At.blocks[all[i].c].coupled);
      if (tot + dc > (double)max_dim) break;
      tot += dc;
    }
    nkeep = std::min(nkeep, i);
  }
  if (rel_tol > 0.0) {
    // drop from the smallest while the dropped weight stays within eps^2 ||A||^2
    double dropped = 0.0;
    size_t i = all.size();
    while (i > 0) {
      const Item& it = all[i - 1];
      const double dc = sector_dim(At.kind, At.blocks[it.c].coupled);
      if (dropped + dc * it.s * it.s > rel_tol * rel_tol * n2) break;
      dropped += dc * it.s * it.s;
      --i;
    }
    nkeep = std::min(nkeep, i);
  }
  std::vector<int64_t> keep(blocks.size(), 0);
  double d2 = 0.0;
  for (size_t i = 0; i < all.size(); ++i) {
    if (i < nkeep) {
      keep[all[i].c] += 1;
    } else {
      d2 += sector_dim(At.kind, At.blocks[all[i].c].coupled) * all[i].s * all[i].s;
    }
  }
  // a kept value must have every larger value of its block kept too (sorted per block): holds because
  // the global order is descending and per-block values are sorted descending.
  if (err) *err = std::sqrt(d2);
  if (norm) *norm = std::sqrt(n2);
  return keep;
}

}  // namespace tk

using namespace tk;

#define TK_API_BEGIN try {
#define TK_API_END                  \
  return TK_OK;                     \
  }                                 \
  catch (const tk::Error& e) {      \
    tk::set_last_error(e.what());   \
    return e.code;                  \
  }                                 \
  catch (const std::exception& e) { \
    tk::set_last_error(e.what());   \
    return TK_ERR_INVALID_ARGUMENT; \
  }

extern "C" {

tk_status tk_svd_workspace(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                           size_t* bytes) {
  TK_API_BEGIN
  if (!A || !bytes || np < 0 || nq < 0) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  *bytes = get_svd_plan(*(const Tensor*)A, ivec(p, np), ivec(q, nq))->ws_bytes;
  TK_API_END
}

tk_status tk_svd(const tk_tensor* A_, const void* a, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                 void* ws, size_t ws_bytes, tk_stream stream) {
  TK_API_BEGIN
  if (!A_ || np < 0 || nq < 0) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  if (!a && A.nelems) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null data pointer");
  auto P = get_svd_plan(A, ivec(p, np), ivec(q, nq));
  if (ws_bytes < P->ws_bytes || !ws) TK_THROW(TK_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
  if (((uintptr_t)ws & 255) != 0) TK_THROW(TK_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  P->ensure_uploaded();
  cudaStream_t st = (cudaStream_t)stream;
  free_deferred(st);
  reset_launches();
  run_permute(P->pa, a, ws, 1.0, 0.0, kPermReal, 1.0, st);
  static const bool dbg = knob("TK_SVD_DEBUG", 0) != 0;
  double* wsd = (double*)ws;
  int32_t* idx = (int32_t*)((char*)ws + P->idx_off);
  if (!P->lists[0].empty()) {
    svd_jacobi_kernel<<<(unsigned)P->lists[0].size(), kSvdThreads, P->smem_bytes, st>>>(
        wsd, idx, (const SvdBlock*)P->d_blocks.p, (const int32_t*)P->d_lists[0].p, dbg ? 1 : 0);
    check_cuda(cudaPeekAtLastError(), "svd launch");
    add_launches(1);
  }
  for (int c = 1; c < 5; ++c) {
    if (P->lists[c].empty()) continue;
    const int cs = 1 << (c - 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(P->lists[c].size() * cs));
    cfg.blockDim = dim3(kSvdThreads);
    cfg.dynamicSmemBytes = (size_t)P->class_smem[c];
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const SvdBlock* bp = (const SvdBlock*)P->d_blocks.p;
    const int32_t* lp = (const int32_t*)P->d_lists[c].p;
    const int dg = dbg ? 1 : 0;
    cudaError_t err;
    switch (cs) {
      case 1: err = cudaLaunchKernelEx(&cfg, svd_cluster_kernel<1>, wsd, idx, bp, lp, dg); break;
      case 2: err = cudaLaunchKernelEx(&cfg, svd_cluster_kernel<2>, wsd, idx, bp, lp, dg); break;
      case 4: err = cudaLaunchKernelEx(&cfg, svd_cluster_kernel<4>, wsd, idx, bp, lp, dg); break;
      default: err = cudaLaunchKernelEx(&cfg, svd_cluster_kernel<8>, wsd, idx, bp, lp, dg); break;
    }
    check_cuda(err, "svd cluster launch");
    add_launches(1);
  }
  TK_API_END
}

tk_status tk_svd_spectrum(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                          const void* ws, tk_stream stream, int32_t* n_blocks, int64_t* counts, double* sigma) {
  TK_API_BEGIN
  if (!A || !ws) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  auto P = get_svd_plan(*(const Tensor*)A, ivec(p, np), ivec(q, nq));
  if (n_blocks) *n_blocks = (int32_t)P->blocks.size();
  if (counts)
    for (size_t c = 0; c < P->blocks.size(); ++c) counts[c] = P->blocks[c].K;
  if (sigma && P->n_sigma) {
    cudaStream_t st = (cudaStream_t)stream;
    check_cuda(cudaMemcpyAsync(sigma, (const double*)ws + P->blocks[0].s_off, P->n_sigma * 8, cudaMemcpyDeviceToHost, st),
               "spectrum copy");
    check_cuda(cudaStreamSynchronize(st), "spectrum sync");
  }
  TK_API_END
}

tk_status tk_svd_truncate(const tk_tensor* A_, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                          const void* ws, int64_t max_dim, double rel_tol, tk_stream stream, tk_space** W,
                          tk_tensor** U, tk_tensor** S, tk_tensor** Vh, double* trunc_err, double* norm) {
  TK_API_BEGIN
  if (!A_ || !ws || !W || !U || !S || !Vh) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  auto P = get_svd_plan(A, ivec(p, np), ivec(q, nq));
  std::vector<double> sig(P->n_sigma);
  if (P->n_sigma) {
    cudaStream_t st = (cudaStream_t)stream;
    check_cuda(cudaMemcpyAsync(sig.data(), (const double*)ws + P->blocks[0].s_off, P->n_sigma * 8,
                               cudaMemcpyDeviceToHost, st),
               "spectrum copy");
    check_cuda(cudaStreamSynchronize(st), "spectrum sync");
  }
  std::vector<int64_t> keep = truncation(*P->At, P->blocks, sig, max_dim, rel_tol, trunc_err, norm);
  // W: one sector per kept coupled block (the coupled label c, degeneracy k_c)
  std::vector<Sector> secs;
  std::vector<int64_t> degs;
  for (size_t c = 0; c < keep.size(); ++c)
    if (keep[c] > 0) {
      secs.push_back(P->At->blocks[c].coupled);
      degs.push_back(keep[c]);
    }
  Space* w = make_space(A.kind, secs, degs, false);
  std::vector<Space*> wv{w};
  std::vector<Space*> cod(P->At->cod), dom(P->At->dom);
  *U = (tk_tensor*)make_tensor(TK_F64, cod, wv);
  *S = (tk_tensor*)make_tensor(TK_F64, wv, wv);
  *Vh = (tk_tensor*)make_tensor(TK_F64, wv, dom);
  *W = (tk_space*)w;
  TK_API_END
}

tk_status tk_svd_extract(const tk_tensor* A_, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                         const void* ws, const tk_tensor* U_, void* u, const tk_tensor* S_, void* s,
                         const tk_tensor* Vh_, void* vh, tk_stream stream) {
  TK_API_BEGIN
  if (!A_ || !ws || !U_ || !S_ || !Vh_) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  const Tensor& U = *(const Tensor*)U_;
  const Tensor& S = *(const Tensor*)S_;
  const Tensor& Vh = *(const Tensor*)Vh_;
  auto P = get_svd_plan(A, ivec(p, np), ivec(q, nq));
  const Tensor& At = *P->At;
  if (U.n_dom() != 1 || S.n_cod() != 1 || S.n_dom() != 1 || Vh.n_cod() != 1 || U.n_cod() != At.n_cod() ||
      Vh.n_dom() != At.n_dom())
    TK_THROW(TK_ERR_SPACE_MISMATCH, "tk_svd_extract: U, S, Vh do not have the shapes tk_svd_truncate returns");
  for (int i = 0; i < At.n_cod(); ++i)
    if (!same_space(U.cod[i], At.cod[i])) TK_THROW(TK_ERR_SPACE_MISMATCH, "U codomain != permuted codomain of A");
  for (int i = 0; i < At.n_dom(); ++i)
    if (!same_space(Vh.dom[i], At.dom[i])) TK_THROW(TK_ERR_SPACE_MISMATCH, "Vh domain != permuted domain of A");
  const Space* w = U.dom[0];
  if (!same_space(w, S.cod[0]) || !same_space(w, S.dom[0]) || !same_space(w, Vh.cod[0]))
    TK_THROW(TK_ERR_SPACE_MISMATCH, "U, S, Vh disagree on the bond space");
  std::map<Sector, int> ublk, sblk, vblk;
  for (int i = 0; i < (int)U.blocks.size(); ++i) ublk[U.blocks[i].coupled] = i;
  for (int i = 0; i < (int)S.blocks.size(); ++i) sblk[S.blocks[i].coupled] = i;
  for (int i = 0; i < (int)Vh.blocks.size(); ++i) vblk[Vh.blocks[i].coupled] = i;
  std::vector<SvdOut> outs;
  for (size_t c = 0; c < At.blocks.size(); ++c) {
    const Sector& cs = At.blocks[c].coupled;
    const int64_t k = w->deg_of_tree_label(cs);
    if (k == 0) continue;
    if (k > P->blocks[c].K) TK_THROW(TK_ERR_SPACE_MISMATCH, "bond degeneracy exceeds the block's singular values");
    const Block& ub = U.blocks[ublk.at(cs)];
    const Block& vb = Vh.blocks[vblk.at(cs)];
    if (ub.rows != At.blocks[c].rows || vb.cols != At.blocks[c].cols || ub.cols != k || vb.rows != k)
      TK_THROW(TK_ERR_SPACE_MISMATCH, "internal: U / Vh block shapes");
    outs.push_back(SvdOut{ub.off, S.blocks[sblk.at(cs)].off, vb.off, (int32_t)k, (int32_t)c});
  }
  if (outs.empty()) return TK_OK;
  if ((U.nelems && !u) || (S.nelems && !s) || (Vh.nelems && !vh)) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null data pointer");
  // extraction table: cached in the plan per kept-count pattern (uploaded once, graph-capture safe after)
  const void* d_outs = nullptr;
  {
    std::string key((const char*)outs.data(), outs.size() * sizeof(SvdOut));
    std::lock_guard<std::mutex> g(P->outs_mu);
    auto& slot = P->outs[key];
    if (!slot) {
      slot = std::make_unique<DevBuf>();
      slot->upload(outs);
    }
    d_outs = slot->p;
  }
  cudaStream_t st = (cudaStream_t)stream;
  P->ensure_uploaded();
  reset_launches();
  svd_extract_kernel<<<dim3((unsigned)outs.size(), 3), 256, 0, st>>>(
      (const double*)ws, (const int32_t*)((const char*)ws + P->idx_off), (const SvdBlock*)P->d_blocks.p,
      (const SvdOut*)d_outs, (double*)u, (double*)s, (double*)vh);
  check_cuda(cudaPeekAtLastError(), "svd extract launch");
  add_launches(1);
  TK_API_END
}

}  // extern "C"
