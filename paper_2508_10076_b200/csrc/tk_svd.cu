// Blockwise (truncated) singular value decomposition of a tensor map, Float64 and
// ComplexF64.
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
// B200 design (round 2). The permute is the library's permute kernel (into a padded workspace). Every
// block runs a one-sided (Hestenes) Jacobi SVD on its tall orientation G = A~ (or A~^H), column pairs
// orthogonalised by plane rotations in round-robin (circle) order, until no pair needs a rotation; the
// accumulated right rotations V give A~ V = G = U S. One-sided Jacobi never forms a Gram matrix, so
// the spectrum is accurate to eps ||A|| (like LAPACK) and U / V are orthonormal to working precision.
// The block is spread over a thread-block CLUSTER of CS CTAs (CS in {1, 2, 4, 8}): every CTA owns a
// slice of the rows of G and of V (all columns), in shared memory when the slice fits (else in the
// L2-resident workspace), so a Jacobi round is
//   (A) every warp takes pairs of the round and reduces (|g_p|^2, |g_q|^2, g_p^H g_q) over the CTA's
//       rows with its 32 lanes (butterfly shuffles) -> the CTA's partial sums;
//   (B) ONE cluster barrier; every CTA reads all CS partials of each pair (distributed shared memory)
//       and sums them in rank order -- bitwise identical in every CTA, so all CTAs take the same
//       rotation and the same convergence decision -- then rotates its own rows of G and V.
// CS is chosen per block so that a CTA holds at most 64 rows of G (two per lane): the critical path
// of a round is a few shuffles, one cluster barrier and one rotation, not a length-R reduction.
// ComplexF64: gamma = |gamma| e^{i phi}; column q is rephased by e^{-i phi} and then rotated by the real
// Jacobi rotation of (alpha, beta, |gamma|) -- a unitary column operation.
// A second kernel writes the kept columns / rows into U, S, Vh in their canonical block layouts.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>

#include "tk_device.cuh"
#include "tk_plan.hpp"

namespace tk {

// ---------------------------------------------------------------- device side
struct SvdBlock {
  int64_t a_off;    // A~ block (column-major, lda), in elements of T
  int64_t g_off;    // G (R x K, ldg): A~ in place (trans = 0) or A~^H in its own region, elements of T
  int64_t v_off;    // V (K x K, ldv), elements of T
  int64_t s_off;    // K sorted singular values (doubles, from the workspace base)
  int64_t p_off;    // K column indices in sorted order (int32, in the index region)
  int64_t x_off;    // global-mode partial sums: 2 x CS x npairs x 4 doubles (from the workspace base)
  int32_t M, N, lda;
  int32_t R, K, ldg, ldv;
  int32_t trans;    // 1: M < N, G = A~^H
  int32_t cs;       // CTAs per cluster
  int32_t smem;     // 1: the CTA's rows of G and V live in shared memory; 0: in the workspace
  int32_t Rl, Kl;   // rows of G / of V per CTA
};

struct SvdOut {     // extraction target of one block (canonical layouts of U, S, Vh)
  int64_t u_off, s_off, vh_off;
  int32_t k;        // kept singular values (0: block dropped)
  int32_t blk;      // SvdBlock index
};

#ifndef TK_SVD_THREADS
#define TK_SVD_THREADS 1024
#endif
constexpr int kSvdThreads = TK_SVD_THREADS;
#ifndef TK_SVD_LANES
#define TK_SVD_LANES 8  // lanes per column pair when the rows are in shared memory (<= 64 rows per CTA)
#endif
constexpr int kSvdWarps = kSvdThreads / 32;
constexpr int kSvdRowsTarget = 64;         // rows of G per CTA (two per lane) when choosing CS
constexpr int kSvdSmemMax = 200 * 1024;    // shared-memory budget of a CTA's rows
constexpr int kSvdMaxK = 8192;             // per-block min(rows, cols) (partial-sum buffers)
constexpr int kSvdMaxSweeps = 60;

template <typename T>
struct SvNum;
template <>
struct SvNum<double> {
  static __device__ __forceinline__ double zero() { return 0.0; }
  static __device__ __forceinline__ double one() { return 1.0; }
  static __device__ __forceinline__ double abs2(double x) { return x * x; }
  static __device__ __forceinline__ double conj(double x) { return x; }
  // alpha/beta/gamma accumulation: g[0] += x y (real), g[1] unused
  static __device__ __forceinline__ void dot(double x, double y, double& gr, double&) { gr = fma(x, y, gr); }
  // y * sign(gamma): the rotation below is computed from |gamma|
  static __device__ __forceinline__ double rephase(double y, double ur, double) { return y * ur; }
  static __device__ __forceinline__ double lin(double a, double x, double b, double y) { return fma(a, x, b * y); }
  static __device__ __forceinline__ double scale(double a, double x) { return a * x; }
};
template <>
struct SvNum<double2> {
  static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ double2 one() { return make_double2(1.0, 0.0); }
  static __device__ __forceinline__ double abs2(double2 x) { return fma(x.x, x.x, x.y * x.y); }
  static __device__ __forceinline__ double2 conj(double2 x) { return make_double2(x.x, -x.y); }
  // gamma += conj(x) y
  static __device__ __forceinline__ void dot(double2 x, double2 y, double& gr, double& gi) {
    gr = fma(x.x, y.x, fma(x.y, y.y, gr));
    gi = fma(x.x, y.y, fma(-x.y, y.x, gi));
  }
  // y * conj(u), u = (ur, ui) the unit phase of gamma
  static __device__ __forceinline__ double2 rephase(double2 y, double ur, double ui) {
    return make_double2(fma(y.x, ur, y.y * ui), fma(y.y, ur, -y.x * ui));
  }
  static __device__ __forceinline__ double2 lin(double a, double2 x, double b, double2 y) {
    return make_double2(fma(a, x.x, b * y.x), fma(a, x.y, b * y.y));
  }
  static __device__ __forceinline__ double2 scale(double a, double2 x) { return make_double2(a * x.x, a * x.y); }
};

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
// (a, b, c, d) summed over the 32 lanes by a reduce-scatter butterfly (6 shuffles instead of 20): after
// it, lane l holds the total of component (l >> 3) & 3... every lane gets all four via 4 shuffles.
__device__ __forceinline__ void warp_sum4(double& a, double& b, double& c, double& d) {
  const int lane = threadIdx.x & 31;
  const bool hi16 = lane & 16;
  // level 16: keep (a, b) in the low half, (c, d) in the high half
  {
    const double s0 = hi16 ? a : c, s1 = hi16 ? b : d;  // what the partner keeps
    const double r0 = __shfl_xor_sync(0xffffffffu, s0, 16), r1 = __shfl_xor_sync(0xffffffffu, s1, 16);
    if (hi16) { c += r0; d += r1; a = c; b = d; } else { a += r0; b += r1; }
  }
  // level 8: keep the first of the pair in lanes with bit 3 clear, the second otherwise
  const bool hi8 = lane & 8;
  {
    const double sx = hi8 ? a : b;
    const double r = __shfl_xor_sync(0xffffffffu, sx, 8);
    a = (hi8 ? b : a) + r;
  }
  // levels 4, 2, 1: plain sums of the one value per lane
  a += __shfl_xor_sync(0xffffffffu, a, 4);
  a += __shfl_xor_sync(0xffffffffu, a, 2);
  a += __shfl_xor_sync(0xffffffffu, a, 1);
  // lane with bits (4, 3) = (h, e) holds component 2h + e: broadcast all four
  const double t0 = __shfl_sync(0xffffffffu, a, 0), t1 = __shfl_sync(0xffffffffu, a, 8);
  const double t2 = __shfl_sync(0xffffffffu, a, 16), t3 = __shfl_sync(0xffffffffu, a, 24);
  a = t0;
  b = t1;
  c = t2;
  d = t3;
}
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

// DSMEM messaging without a cluster-wide barrier: st.async writes into another CTA's shared memory and
// completes transaction bytes on that CTA's mbarrier; the receiver waits on its own mbarrier with
// cluster-scope acquire (no MEMBAR.GPU, which a barrier.cluster.arrive.release costs every round)
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TK_CW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TK_CW_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// pair pr of round r of the circle method over n players (player K, if K is odd, sits out); the two
// columns in either order (the rotation is symmetric under swapping them)
__device__ __forceinline__ bool round_pair_fast(int r, int pr, int n, int K, int& p, int& q) {
  const int m = n - 1;
  if (pr == 0) {
    p = m;
    q = r;
  } else {
    p = r + pr;
    if (p >= m) p -= m;
    q = r - pr;
    if (q < 0) q += m;
  }
  return p < K && q < K;
}

// pair pr of round r of the circle method over n players (player K, if K is odd, sits out)
__device__ __forceinline__ bool round_pair(int r, int pr, int n, int K, int& p, int& q) {
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
  return q < K;
}

// CS CTAs (a cluster) per block; SM: the CTA's rows of G and V in shared memory (else in the workspace).
template <int CS, typename T, bool SM, int L>
__global__ void __launch_bounds__(kSvdThreads, 1)
    svd_jacobi_kernel(void* __restrict__ wsv, int32_t* __restrict__ idx, const SvdBlock* __restrict__ blocks,
                      const int32_t* __restrict__ list, int debug) {
  const long long t_start = clock64();
  using N = SvNum<T>;
  extern __shared__ __align__(16) double svd_dyn[];
  const SvdBlock b = blocks[list[blockIdx.x / CS]];
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NG = kSvdThreads / L;  // lane groups: one column pair each per pass
  const int grp = tid / L, gl = tid % L;
  const int R = b.R, K = b.K, Rl = b.Rl, Kl = b.Kl;
  const int n = K + (K & 1), npairs = n / 2;
  const int r0 = min(R, (int)rank * Rl), nr = min(R, r0 + Rl) - r0;
  const int v0 = min(K, (int)rank * Kl), nv = min(K, v0 + Kl) - v0;
  T* base = reinterpret_cast<T*>(wsv);
  double* wsd = reinterpret_cast<double*>(wsv);
  // the CTA's rows of G (ld ldG) and V (ld ldV); partial sums [2][npairs][4] (this CTA's copy)
  T* G;
  T* V;
  int ldG, ldV;
  double* part;
  if (SM) {
    G = reinterpret_cast<T*>(svd_dyn);
    V = G + (size_t)Rl * K;
    ldG = Rl;
    ldV = Kl;
    // partial sums of every rank, [2][CS][npairs][4] (16-byte aligned: read as double2), then 2 mbarriers
    part = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(V + (size_t)Kl * K) + 15) & ~uintptr_t(15));
  } else {
    G = base + b.g_off + r0;
    V = base + b.v_off + v0;
    ldG = b.ldg;
    ldV = b.ldv;
    part = wsd + b.x_off + (size_t)rank * 2 * npairs * 4;
  }
  const T* A = base + b.a_off;
  pdl_wait();
  // G rows: A~ (in place when not transposed and not in shared memory) or A~^H; V = I
  if (SM || b.trans) {
    for (int64_t e = tid; e < (int64_t)nr * K; e += kSvdThreads) {
      const int i = (int)(e % nr), j = (int)(e / nr), gi = r0 + i;
      G[i + (int64_t)j * ldG] = b.trans ? N::conj(A[j + (int64_t)gi * b.lda]) : A[gi + (int64_t)j * b.lda];
    }
  }
  for (int64_t e = tid; e < (int64_t)nv * K; e += kSvdThreads) {
    const int i = (int)(e % nv), j = (int)(e / nv);
    V[i + (int64_t)j * ldV] = (v0 + i == j) ? N::one() : N::zero();
  }
  // SM && CS > 1: partials are pushed to every CTA (st.async), so phase B reads local shared memory only
  constexpr bool PUSH = SM && CS > 1;
  uint64_t* xbar = reinterpret_cast<uint64_t*>(part + (PUSH ? 2 * CS * npairs * 4 : 0));
  if (PUSH && tid == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_barrier_init();
  }
  if (PUSH) cluster_sync_all(); else __syncthreads();  // remote mbarriers initialised before any push
  long long tA = 0, tX = 0, tB = 0, tS = 0;  // debug: cycles in phase A, exchange, phase B, round barrier
  uint32_t xph = 0;  // phase parity of xbar[0] (bit 0) and xbar[1] (bit 1)
  const double tol = 2.3e-16 * sqrt((double)R);
  int par = 0, sweep = 0;
  for (; sweep < kSvdMaxSweeps; ++sweep) {
    int any = 0;
    for (int r = 0; r < n - 1; ++r) {
      // (A) partial (alpha, beta, gamma) of every pair of round r over this CTA's rows; a warp takes the
      // pairs warp, warp + 32, ... in batches of kPA whose reductions interleave (independent shuffles).
      // PUSH: this CTA's sums go to slot [par][rank] of every CTA (local store + st.async to the others).
      long long tq0 = debug ? clock64() : 0;
      // (A) a group of L lanes owns pairs grp, grp + NG, ... of round r: partial (alpha, beta, gamma)
      // over this CTA's rows, reduced over the group's lanes (log2 L shuffle levels). PUSH: the CTA's
      // sums go to slot [par][rank] of every CTA of the cluster (local store + st.async to the others).
      double* pp = part + par * (PUSH ? CS : 1) * npairs * 4;
      if (PUSH && tid == 0) mbar_arrive_expect_tx(&xbar[par], (uint32_t)((CS - 1) * npairs * 32));
      for (int pb = 0; pb < npairs; pb += NG) {  // group-uniform trip count: all lanes shuffle together
        const int pr = pb + grp;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        int p, q;
        if (pr < npairs && round_pair_fast(r, pr, n, K, p, q)) {
          const T* gp = G + (int64_t)p * ldG;
          const T* gq = G + (int64_t)q * ldG;
#pragma unroll 4
          for (int i = gl; i < nr; i += L) {
            const T x = gp[i], y = gq[i];
            al += N::abs2(x);
            be += N::abs2(y);
            N::dot(x, y, gr, gi);
          }
        }
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          gr += __shfl_xor_sync(0xffffffffu, gr, o);
          gi += __shfl_xor_sync(0xffffffffu, gi, o);
        }
        if (pr < npairs && gl < 2) {  // lane 0: (alpha, beta), lane 1: (gamma re, gamma im)
          double* dst = pp + ((PUSH ? rank * npairs : 0) + pr) * 4 + 2 * gl;
          const double v0 = gl ? gr : al, v1 = gl ? gi : be;
          *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
          if (PUSH) {
            const uint32_t la = smem_u32(dst), lb = smem_u32(&xbar[par]);
#pragma unroll
            for (int c = 1; c < CS; ++c) {
              const uint32_t rk = (rank + c) % CS;
              st_async_v2(mapa_u32(la, rk), v0, v1, mapa_u32(lb, rk));
            }
          }
        }
      }
      long long tq1 = debug ? clock64() : 0;
      if (PUSH) {
        __syncthreads();                                     // the local slot is complete
        mbar_wait_cluster(&xbar[par], (xph >> par) & 1u);    // every remote slot has landed
        xph ^= 1u << par;
      } else if (CS > 1) {
        cluster_sync_all();
      } else {
        __syncthreads();
      }
      long long tq2 = debug ? clock64() : 0;
      // (B) the same group sums its pair's four components over the CS ranks in rank order (identical in
      // every CTA), computes the rotation (reciprocal square roots, no divisions) and rotates the CTA's
      // rows of columns p, q of G and V
      for (int pr = grp; pr < npairs; pr += NG) {
        int p, q;
        if (!round_pair_fast(r, pr, n, K, p, q)) continue;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
#pragma unroll
        for (int cc = 0; cc < CS; ++cc) {
          const double* src;
          if (SM) src = PUSH ? pp + cc * npairs * 4 : pp;
          else src = wsd + b.x_off + (size_t)cc * 2 * npairs * 4 + par * npairs * 4;
          const double2 v01 = *reinterpret_cast<const double2*>(src + pr * 4);
          const double2 v23 = *reinterpret_cast<const double2*>(src + pr * 4 + 2);
          al += v01.x;
          be += v01.y;
          gr += v23.x;
          gi += v23.y;
        }
        const double ga2 = fma(gr, gr, gi * gi);
        if (!(ga2 > tol * tol * al * be && ga2 > 0.0)) continue;
        // Schur rotation of [[al, |ga|], [|ga|, be]] (Hestenes); column q rephased by conj(ga / |ga|)
        const double rga = rsqrt(ga2);
        const double zeta = 0.5 * (be - al) * rga;
        const double t = copysign(1.0, zeta) * __drcp_rn(fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
        const double ur = gr * rga, ui = gi * rga;
        T* gp = G + (int64_t)p * ldG;
        T* gq = G + (int64_t)q * ldG;
#pragma unroll 4
        for (int i = gl; i < nr; i += L) {
          const T x = gp[i], y = N::rephase(gq[i], ur, ui);
          gp[i] = N::lin(c, x, -sn, y);
          gq[i] = N::lin(sn, x, c, y);
        }
        T* vp = V + (int64_t)p * ldV;
        T* vq = V + (int64_t)q * ldV;
#pragma unroll 4
        for (int i = gl; i < nv; i += L) {
          const T x = vp[i], y = N::rephase(vq[i], ur, ui);
          vp[i] = N::lin(c, x, -sn, y);
          vq[i] = N::lin(sn, x, c, y);
        }
        any = 1;
      }
      long long tq3 = debug ? clock64() : 0;
      par ^= 1;
      __syncthreads();
      if (debug) {
        long long tq4 = clock64();
        tA += tq1 - tq0;
        tX += tq2 - tq1;
        tB += tq3 - tq2;
        tS += tq4 - tq3;
      }
    }
    // every CTA took the same decisions (identical sums), so the cluster agrees on convergence
    if (!__syncthreads_or(any)) break;
  }
  if (debug && tid == 0 && rank == 0)
    printf("[tk svd] block %d: %d x %d, cluster %d, %s, %d sweeps, %lld cycles/round (A %lld X %lld B %lld S %lld)\n",
           list[blockIdx.x / CS], R, K, CS, SM ? "smem" : "ws", sweep + 1,
           (clock64() - t_start) / ((long long)(sweep + 1) * (n - 1)), tA / ((long long)(sweep + 1) * (n - 1)),
           tX / ((long long)(sweep + 1) * (n - 1)), tB / ((long long)(sweep + 1) * (n - 1)),
           tS / ((long long)(sweep + 1) * (n - 1)));
  // singular values: column norms over the cluster (rank order); partial sums in this CTA's `part`
  // half `par` (its last use was round n-2 of the final sweep, read by all CTAs before they passed
  // that round's barrier... it is rewritten only after the barrier below)
  double* nrm = part + par * npairs * 4;  // >= K slots (4 * npairs >= K)
  if (CS > 1) cluster_sync_all();         // every CTA has finished reading the last round's partials
  for (int j = warp; j < K; j += kSvdWarps) {
    const T* g = G + (int64_t)j * ldG;
    double x = 0.0;
    for (int i = lane; i < nr; i += 32) x += N::abs2(g[i]);
    x = warp_sum(x);
    if (lane == 0) nrm[j] = x;
  }
  if (CS > 1) cluster_sync_all(); else __syncthreads();
  // rank 0: sigma_j = sqrt(sum_c partial_c) in rank order into its free partial-sum half, then ranked
  // descending (ties by column index)
  if (rank == 0) {
    double* sig = part + (par ^ 1) * npairs * 4;  // no CTA reads it any more (after the barrier above)
    for (int j = tid; j < K; j += kSvdThreads) {
      double x = 0.0;
#pragma unroll
      for (int c = 0; c < CS; ++c) {
        const double* src = SM ? (CS > 1 ? map_rank(nrm, (uint32_t)c) : nrm)
                               : wsd + b.x_off + (size_t)c * 2 * npairs * 4 + par * npairs * 4;
        x += src[j];
      }
      sig[j] = sqrt(x);
    }
    __syncthreads();
    double* sv = wsd + b.s_off;
    int32_t* pv = idx + b.p_off;
    for (int j = tid; j < K; j += kSvdThreads) {
      const double sj = sig[j];
      int rk = 0;
      for (int i = 0; i < K; ++i) rk += (sig[i] > sj) || (sig[i] == sj && i < j);
      sv[rk] = sj;
      pv[rk] = j;
    }
  }
  // this CTA's rows of G and V back to the workspace (the extraction kernel reads them there)
  if (SM) {
    T* Gw = base + b.g_off;
    T* Vw = base + b.v_off;
    for (int64_t e = tid; e < (int64_t)nr * K; e += kSvdThreads) {
      const int i = (int)(e % nr), j = (int)(e / nr);
      Gw[r0 + i + (int64_t)j * b.ldg] = G[i + (int64_t)j * ldG];
    }
    for (int64_t e = tid; e < (int64_t)nv * K; e += kSvdThreads) {
      const int i = (int)(e % nv), j = (int)(e / nv);
      Vw[v0 + i + (int64_t)j * b.ldv] = V[i + (int64_t)j * ldV];
    }
  }
  if (CS > 1) cluster_sync_all();  // no CTA may exit while others still read its shared memory
}

// Non-transposed block (A~ V = G = U S): U[:, r] = G[:, perm r] / s_r, Vh[r, :] = V[:, perm r]^H.
// Transposed (A~^H W = G): U[:, r] = W[:, perm r], Vh[r, :] = (G[:, perm r] / s_r)^H. S = diag(s).
// One CTA per (block, part), part 0 = U, 1 = Vh, 2 = S.
template <typename T>
__global__ void __launch_bounds__(256)
    svd_extract_kernel(const void* __restrict__ wsv, const int32_t* __restrict__ idx,
                       const SvdBlock* __restrict__ blocks, const SvdOut* __restrict__ outs, T* __restrict__ U,
                       T* __restrict__ S, T* __restrict__ Vh) {
  using N = SvNum<T>;
  const SvdOut o = outs[blockIdx.x];
  const SvdBlock b = blocks[o.blk];
  const int part = blockIdx.y;
  const int k = o.k, M = b.M, Nc = b.N;
  const T* base = reinterpret_cast<const T*>(wsv);
  const double* sv = reinterpret_cast<const double*>(wsv) + b.s_off;
  const int32_t* pv = idx + b.p_off;
  const T* G = base + b.g_off;
  const T* V = base + b.v_off;
  if (part == 0) {  // U: M x k column-major
    for (int64_t e = threadIdx.x; e < (int64_t)M * k; e += blockDim.x) {
      const int i = (int)(e % M), r = (int)(e / M);
      const int j = pv[r];
      T x;
      if (!b.trans) {
        const double s = sv[r];
        x = s > 0.0 ? N::scale(1.0 / s, G[i + (int64_t)j * b.ldg]) : N::zero();
      } else {
        x = V[i + (int64_t)j * b.ldv];
      }
      U[o.u_off + e] = x;
    }
  } else if (part == 1) {  // Vh: k x N column-major
    for (int64_t e = threadIdx.x; e < (int64_t)k * Nc; e += blockDim.x) {
      const int r = (int)(e % k), c = (int)(e / k);
      const int j = pv[r];
      T x;
      if (!b.trans) {
        x = N::conj(V[c + (int64_t)j * b.ldv]);
      } else {
        const double s = sv[r];
        x = s > 0.0 ? N::scale(1.0 / s, N::conj(G[c + (int64_t)j * b.ldg])) : N::zero();
      }
      Vh[o.vh_off + e] = x;
    }
  } else {  // S: k x k diagonal
    for (int64_t e = threadIdx.x; e < (int64_t)k * k; e += blockDim.x) {
      const int r = (int)(e % k), c = (int)(e / k);
      S[o.s_off + e] = (r == c) ? N::scale(sv[r], N::one()) : N::zero();
    }
  }
}

// ---------------------------------------------------------------- host side
template <int CS, typename T, bool SM>
static cudaError_t set_svd_attr() {
  cudaError_t e = cudaFuncSetAttribute(svd_jacobi_kernel<CS, T, SM, SM ? TK_SVD_LANES : 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SM ? 227 * 1024 : 0);
  return e;
}
template <typename T>
static cudaError_t set_svd_attrs_t() {
  cudaError_t e = set_svd_attr<1, T, true>();
  if (e == cudaSuccess) e = set_svd_attr<2, T, true>();
  if (e == cudaSuccess) e = set_svd_attr<4, T, true>();
  if (e == cudaSuccess) e = set_svd_attr<8, T, true>();
  return e;
}
static PerDeviceOnce g_svd_attrs;
static cudaError_t ensure_svd_attrs() {
  return g_svd_attrs.run([] {
    cudaError_t e = set_svd_attrs_t<double>();
    if (e == cudaSuccess) e = set_svd_attrs_t<double2>();
    return e;
  });
}

// launch classes: (log2 CS) x (shared memory, workspace)
constexpr int kSvdClasses = 8;
struct SvdPlan {
  Tensor* At = nullptr;
  bool cplx = false;
  PermPlan pa;
  PadLayout la;
  std::vector<SvdBlock> blocks;
  DevBuf d_blocks;
  std::vector<int32_t> lists[kSvdClasses];
  int class_smem[kSvdClasses] = {};
  DevBuf d_lists[kSvdClasses];
  size_t ws_bytes = 0, idx_off = 0;  // byte offset of the int32 index region
  int64_t n_sigma = 0, sig_base = 0;  // sigma region (doubles from the workspace base)
  std::mutex outs_mu;
  std::once_flag up_once;
  void ensure_uploaded() {
    std::call_once(up_once, [&] {
      check_cuda(ensure_svd_attrs(), "svd kernel attributes");
      pa.ensure_uploaded();
      d_blocks.upload(blocks);
      for (int c = 0; c < kSvdClasses; ++c) d_lists[c].upload(lists[c]);
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
  P->cplx = A.dtype == TK_C64;
  const int es = P->cplx ? 16 : 8;   // bytes per element
  const int dpe = P->cplx ? 2 : 1;   // doubles per element
  P->At = permuted_tensor(A, p, q, A.dtype);
  P->la = pad_layout(*P->At);        // offsets in elements of A's type (interleaved complex)
  build_perm_plan(A, p, q, *P->At, P->pa, es, nullptr, &P->la);
  P->pa.identity = false;  // always copy: the Jacobi sweeps work in place on A~
  // workspace (elements of T): A~ | transposed G blocks | V blocks ; then (doubles) sigma | global-mode
  // partial sums ; then (int32) sorted column indices
  static const int rows_target = (int)knob("TK_SVD_ROWS", kSvdRowsTarget);
  int64_t off = P->la.total;
  int64_t nsig = 0, nidx = 0, npart = 0;
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
    if (b.K > kSvdMaxK) TK_THROW(TK_ERR_UNSUPPORTED, "tk_svd: a block with min(rows, cols) > 8192");
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
    // cluster size: the smallest CS with <= rows_target rows of G per CTA whose rows of G and V fit the
    // shared-memory budget; else CS = 8 with the rows in the (L2-resident) workspace
    const int64_t npairs = (b.K + 1) / 2;
    b.cs = 8;
    b.smem = 0;
    for (int cs = 1; cs <= 8; cs *= 2) {
      const int64_t Rl = (b.R + cs - 1) / cs, Kl = (b.K + cs - 1) / cs;
      const int64_t bytes = (Rl + Kl) * b.K * es + 2 * cs * npairs * 32 + 32;
      if (Rl <= rows_target && bytes <= kSvdSmemMax) {
        b.cs = cs;
        b.smem = 1;
        break;
      }
    }
    if (!b.smem) {  // smallest CS whose rows fit, if any, even with more rows per lane
      for (int cs = 1; cs <= 8; cs *= 2) {
        const int64_t Rl = (b.R + cs - 1) / cs, Kl = (b.K + cs - 1) / cs;
        if ((Rl + Kl) * b.K * es + 2 * cs * npairs * 32 + 32 <= kSvdSmemMax) {
          b.cs = cs;
          b.smem = 1;
          break;
        }
      }
    }
    b.Rl = (b.R + b.cs - 1) / b.cs;
    b.Kl = (b.K + b.cs - 1) / b.cs;
    b.x_off = npart;  // relative; rebased below
    if (!b.smem) npart += (int64_t)b.cs * 2 * npairs * 4;
    int cls = 0;
    while ((1 << cls) < b.cs) ++cls;
    cls = 2 * cls + (b.smem ? 0 : 1);
    if (b.smem)
      P->class_smem[cls] =
          std::max<int>(P->class_smem[cls], (int)(((int64_t)b.Rl + b.Kl) * b.K * es + 2 * b.cs * npairs * 32 + 32));
    P->lists[cls].push_back((int32_t)P->blocks.size());
    P->blocks.push_back(b);
  }
  // doubles from the workspace base: sigma, then the global-mode partial sums
  P->sig_base = (off * dpe + 31) & ~int64_t(31);
  const int64_t x_base = (P->sig_base + nsig + 1) & ~int64_t(1);  // 16-byte aligned partial sums
  for (auto& b : P->blocks) {
    b.s_off += P->sig_base;
    b.x_off += x_base;
  }
  P->n_sigma = nsig;
  P->idx_off = align256((size_t)(x_base + npart) * 8);
  if (plan_debug()) {
    fprintf(stderr, "[tk svd] %zu blocks:", P->blocks.size());
    for (int c = 0; c < kSvdClasses; ++c)
      if (!P->lists[c].empty())
        fprintf(stderr, " cs%d/%s x%zu (smem %d B)", 1 << (c / 2), (c & 1) ? "ws" : "smem", P->lists[c].size(),
                P->class_smem[c]);
    fprintf(stderr, "\n");
  }
  P->ws_bytes = align256(P->idx_off + (size_t)nidx * 4);
  return P;
}

static std::vector<int> ivec(const int32_t* v, int n) { return std::vector<int>(v, v + n); }

template <int CS, typename T, bool SM>
static cudaError_t launch_svd_class(const SvdPlan& P, int cls, void* ws, int32_t* idx, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P.lists[cls].size() * CS));
  cfg.blockDim = dim3(kSvdThreads);
  cfg.dynamicSmemBytes = SM ? (size_t)P.class_smem[cls] : 0;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  static const int debug = std::getenv("TK_SVD_DEBUG") ? 1 : 0;  // diagnostic print only
  return cudaLaunchKernelEx(&cfg, svd_jacobi_kernel<CS, T, SM, SM ? TK_SVD_LANES : 32>, ws, idx, (const SvdBlock*)P.d_blocks.p,
                            (const int32_t*)P.d_lists[cls].p, debug);
}

// Launch classes run concurrently: class 0 on the caller's stream, the others on library-private
// streams forked from / joined to it with events (capturable: a CUDA graph gets the same fork-join).
static cudaStream_t svd_aux_stream(int i) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, cudaStream_t> st;
  const int d = current_device();
  std::lock_guard<std::mutex> g(mu);
  auto& s = st[{d, i}];
  if (!s) check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "svd stream");
  return s;
}

template <typename T>
static cudaError_t launch_svd_cls(const SvdPlan& P, int cls, void* ws, int32_t* idx, cudaStream_t st) {
  const int cs = 1 << (cls / 2);
  const bool sm = (cls & 1) == 0;
  switch (cs * 2 + (sm ? 0 : 1)) {
    case 2: return launch_svd_class<1, T, true>(P, cls, ws, idx, st);
    case 3: return launch_svd_class<1, T, false>(P, cls, ws, idx, st);
    case 4: return launch_svd_class<2, T, true>(P, cls, ws, idx, st);
    case 5: return launch_svd_class<2, T, false>(P, cls, ws, idx, st);
    case 8: return launch_svd_class<4, T, true>(P, cls, ws, idx, st);
    case 9: return launch_svd_class<4, T, false>(P, cls, ws, idx, st);
    case 16: return launch_svd_class<8, T, true>(P, cls, ws, idx, st);
    default: return launch_svd_class<8, T, false>(P, cls, ws, idx, st);
  }
}

template <typename T>
static void launch_svd_all(const SvdPlan& P, void* ws, int32_t* idx, cudaStream_t st) {
  std::vector<int> cl;
  for (int c = kSvdClasses - 1; c >= 0; --c)  // largest clusters first (the longest blocks)
    if (!P.lists[c].empty()) cl.push_back(c);
  if (cl.empty()) return;
  if (cl.size() == 1) {
    check_cuda(launch_svd_cls<T>(P, cl[0], ws, idx, st), "svd launch");
    add_launches(1);
    return;
  }
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> joins(cl.size() - 1, nullptr);
  check_cuda(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "svd event");
  for (auto& e : joins) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "svd event");
  cudaError_t err = cudaEventRecord(fork, st);
  for (size_t i = 1; i < cl.size() && err == cudaSuccess; ++i) {
    cudaStream_t a = svd_aux_stream((int)i - 1);
    err = cudaStreamWaitEvent(a, fork, 0);
    if (err == cudaSuccess) err = launch_svd_cls<T>(P, cl[i], ws, idx, a);
    if (err == cudaSuccess) err = cudaEventRecord(joins[i - 1], a);
  }
  if (err == cudaSuccess) err = launch_svd_cls<T>(P, cl[0], ws, idx, st);
  for (auto& e : joins)
    if (err == cudaSuccess) err = cudaStreamWaitEvent(st, e, 0);
  cudaEventDestroy(fork);
  for (auto& e : joins) cudaEventDestroy(e);
  check_cuda(err, "svd launch");
  add_launches((int)cl.size());
}

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
  run_permute(P->pa, a, ws, 1.0, 0.0, P->cplx ? kPermCToC : kPermReal, 1.0, st);
  int32_t* idx = (int32_t*)((char*)ws + P->idx_off);
  if (P->cplx) launch_svd_all<double2>(*P, ws, idx, st);
  else launch_svd_all<double>(*P, ws, idx, st);
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
    check_cuda(cudaMemcpyAsync(sigma, (const double*)ws + P->sig_base, P->n_sigma * 8, cudaMemcpyDeviceToHost, st),
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
    check_cuda(cudaMemcpyAsync(sig.data(), (const double*)ws + P->sig_base, P->n_sigma * 8,
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
  *U = (tk_tensor*)make_tensor(A.dtype, cod, wv);
  *S = (tk_tensor*)make_tensor(A.dtype, wv, wv);
  *Vh = (tk_tensor*)make_tensor(A.dtype, wv, dom);
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
  const dim3 grid((unsigned)outs.size(), 3);
  const int32_t* ix = (const int32_t*)((const char*)ws + P->idx_off);
  const SvdBlock* bp = (const SvdBlock*)P->d_blocks.p;
  cudaError_t e;
  if (P->cplx) {
    cudaLaunchConfig_t cfg = {grid, dim3(256), 0, st, nullptr, 0};
    e = cudaLaunchKernelEx(&cfg, svd_extract_kernel<double2>, ws, ix, bp, (const SvdOut*)d_outs, (double2*)u,
                           (double2*)s, (double2*)vh);
  } else {
    cudaLaunchConfig_t cfg = {grid, dim3(256), 0, st, nullptr, 0};
    e = cudaLaunchKernelEx(&cfg, svd_extract_kernel<double>, ws, ix, bp, (const SvdOut*)d_outs, (double*)u,
                           (double*)s, (double*)vh);
  }
  check_cuda(e, "svd extract launch");
  add_launches(1);
  TK_API_END
}

}  // extern "C"
