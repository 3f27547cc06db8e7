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
#include <tuple>

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
  int32_t tile;     // 2: svd_jacobi_panel_kernel, 1: svd_jacobi_tile_kernel, 0: svd_jacobi_kernel
  int32_t rg;       // registers per lane (tile: rows of G; panel: rows per half of a column)
  int32_t lp;       // panel: lanes per pair slot (32 or 16)
  int32_t pad_;
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

// mbarrier wait (CTA scope) that turns a lost arrival into a kernel error instead of a hung GPU: after
// ~2^34 cycles (~9 s) of waiting it traps. A Jacobi round waits a few microseconds at most.
__device__ __forceinline__ void mbar_wait_guarded(uint64_t* bar, uint32_t parity) {
  const long long t0 = clock64();
  while (true) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (clock64() - t0 > (1LL << 34)) __trap();
  }
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

// st.async of one double (the real gamma partial)
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double a, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(raddr), "d"(a),
               "r"(rbar)
               : "memory");
}

// Jacobi for the blocks of a DMRG bond (K <= 256 columns; round 2b). The kernel above is bound by
// shared-memory traffic: per round it reads G twice and reads + writes G and V once more, and its
// column-major slices put the four pairs of a warp on conflicting banks. Here one group of 8 lanes owns
// one pair for the whole round: it loads the pair's rows of G ONCE into registers (RG rows per lane
// per column), reduces (alpha, beta, gamma) over its lanes with three shuffle levels, sends the
// partial to the other CTAs of the cluster (st.async, 24 B real / 32 B complex per pair and peer),
// waits on its own mbarrier, adds the CS partials in rank order (bitwise identical in every CTA: same
// rotations, same convergence decision), rotates the registers and stores them, then streams the
// pair's rows of V (load, rotate, store). Per round the slices are read and written once: the floor is
// 2 (rows of G + rows of V) K 8 B / 128 B per cycle per SM, so the planner picks CS per block to
// balance that against the exchange (DSMEM ~20 B per cycle per SM) and the cluster-wide latency.
// Shared memory holds the slices in 8-row tiles ([row / 8][column][row % 8]): a group's 8 lanes read
// 64 contiguous bytes of a column, and the two groups of a half-warp (consecutive pairs) sit on
// different 64-byte halves of the banks.
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ int named_bar_or(int id, int nthreads, int pred) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\tselp.s32 %0, 1, 0, q;\n\t}\n"
      : "=r"(r)
      : "r"(pred), "r"(id), "r"(nthreads)
      : "memory");
  return r;
}
// tan of the Jacobi angle, t = sign(z) / (|z| + sqrt(1 + z^2)) with z = (beta - alpha) / (2 |gamma|), to
// single precision: the rotation stays orthogonal to working precision because c = rsqrt(1 + t^2) and
// s = c t are formed in double from this t; an angle off by ~1e-7 only leaves a residual ~1e-7 gamma
// that the next sweep removes. alpha, beta, |gamma| are scaled by a power of two (exponent of |gamma|)
// so that the float arithmetic neither overflows nor underflows; |z| > 2^59 takes t = 1 / (2 z) in double.
__device__ __forceinline__ double jacobi_tan(double al, double be, double ag) {
  const double d = be - al;
  if (fabs(d) > 1.152921504606847e18 * ag) return ag / d;          // |z| > 2^59: t = 1 / (2 z)
  const long long eb = (__double_as_longlong(ag) >> 52) & 0x7ff;  // biased exponent of |gamma|
  const double sc = __longlong_as_double((2046LL - eb) << 52);      // 2^(1023 - e): ag * sc in [1, 2)
  const double num = d * (0.5 * sc), den = ag * sc;
  const float z = __double2float_rn(num) / __double2float_rn(den);
  const float tf = copysignf(1.0f, z) / (fabsf(z) + sqrtf(fmaf(z, z, 1.0f)));
  return (double)tf;
}
// (c, s) of the Jacobi rotation from the single-precision tangent, made orthogonal to working precision in
// double: with d = c^2 + s^2 - 1 (|d| ~ 1e-7), scaling both by 1 - d/2 + 3d^2/8 leaves c^2 + s^2 = 1 + O(d^3).
// The angle is accurate to ~1e-7, which only leaves a residual the next sweep removes (the first sweeps).
__device__ __forceinline__ void jacobi_cs_fast(double al, double be, double ag, double& c, double& s) {
  const double t = jacobi_tan(al, be, ag);
  const float tf = (float)t;
  const float cf = rsqrtf(fmaf(tf, tf, 1.0f));
  const double cd = (double)cf, sd = cd * t;
  const double d = fma(cd, cd, fma(sd, sd, -1.0));
  const double sc = fma(d, fma(0.375, d, -0.5), 1.0);
  c = cd * sc;
  s = sd * sc;
}
constexpr int kTileL = 8;                            // lanes per pair
constexpr int kTileThreads = 768;                    // 85 registers per thread: no spills up to RG 8
constexpr int kTileMaxPairs = kTileThreads / kTileL;  // 96: K <= 192
constexpr int kTileExactSweep = 5;                   // sweeps before this one use the single-precision tangent

// DSMEM bulk copy (cp.async.bulk shared::cta -> shared::cluster), completion counted in bytes on the
// receiving CTA's mbarrier
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Shared memory of the tile kernel: G in RG 8-row tiles and V in TV tiles, each tile [K + 1][8] (column
// K is all zeros: the partner of the player sitting out when K is odd and of groups without a pair);
// the partial sums [2][CS][npairs][4]; two mbarriers.
__host__ __device__ inline int64_t tile_smem_bytes(int K, int rg, int tv, int cs, int es) {
  const int64_t npairs = (K + 1) / 2;
  return (int64_t)(rg + tv) * 8 * (K + 1) * es + 2 * cs * npairs * 32 + 16;
}

// Jacobi for the blocks of a DMRG bond (K <= 192 columns; round 2). One group of 8 lanes owns one column
// pair for the whole round: it loads the pair's rows of G once into registers (RG rows per lane and
// column), reduces (alpha, beta, gamma) over its lanes with three shuffle levels, and -- in a cluster --
// the CTA's partials go to the other CTAs as ONE bulk copy per peer (cp.async.bulk into the peer's slot
// [rank], completion on its mbarrier; st.async per pair costs ~1.6 cycles per message). Every CTA adds the
// CS partials in rank order (bitwise identical everywhere: same rotations, same convergence decision),
// rotates the registers, stores them, and streams the pair's rows of V. Only the warps that own pairs run
// the rounds (named barrier 1). Shared memory holds the slices in 8-row tiles ([row / 8][column][row % 8]):
// a group's 8 lanes read 64 contiguous bytes of a column.
template <int CS, typename T, int RG>
__global__ void __launch_bounds__(kTileThreads, 1)
    svd_jacobi_tile_kernel(void* __restrict__ wsv, int32_t* __restrict__ idx, const SvdBlock* __restrict__ blocks,
                           const int32_t* __restrict__ list, int debug) {
  using N = SvNum<T>;
  constexpr int L = kTileL;
  constexpr bool CPLX = sizeof(T) == 16;
  extern __shared__ __align__(16) double svd_dyn[];
  const SvdBlock b = blocks[list[blockIdx.x / CS]];
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  const int tid = threadIdx.x, grp = tid / L, gl = tid % L;
  const int R = b.R, K = b.K, Rl = b.Rl, Kl = b.Kl;
  const int n = K + (K & 1), npairs = n / 2, KP = K + 1;
  const int r0 = min(R, (int)rank * Rl), nr = min(R, r0 + Rl) - r0;
  const int v0 = min(K, (int)rank * Kl), nv = min(K, v0 + Kl) - v0;
  const int tv = (Kl + 7) >> 3;               // 8-row tiles of V (G has RG tiles)
  const int TS = KP * 8;                      // tile stride (elements)
  T* G = reinterpret_cast<T*>(svd_dyn);       // [RG][K + 1][8]
  T* V = G + (size_t)RG * TS;                 // [tv][K + 1][8]
  double* part = reinterpret_cast<double*>(V + (size_t)tv * TS);  // [2][CS][npairs][4]
  uint64_t* xbar = reinterpret_cast<uint64_t*>(part + 2 * CS * npairs * 4);
  const T* A = reinterpret_cast<const T*>(wsv) + b.a_off;
  if (CS > 1 && tid == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_barrier_init();
  }
  pdl_wait();
  // G: the CTA's rows of A~ (or A~^H), zero past the last row and in column K; V: rows of the identity
  for (int64_t e = tid; e < (int64_t)RG * 8 * KP; e += kTileThreads) {
    const int i = (int)(e % (RG * 8)), j = (int)(e / (RG * 8)), gi = r0 + i;
    T x = N::zero();
    if (i < nr && j < K) x = b.trans ? N::conj(A[j + (int64_t)gi * b.lda]) : A[gi + (int64_t)j * b.lda];
    G[(i >> 3) * TS + j * 8 + (i & 7)] = x;
  }
  for (int64_t e = tid; e < (int64_t)tv * 8 * KP; e += kTileThreads) {
    const int i = (int)(e % (tv * 8)), j = (int)(e / (tv * 8));
    V[(i >> 3) * TS + j * 8 + (i & 7)] = (i < nv && v0 + i == j) ? N::one() : N::zero();
  }
  if (CS > 1) cluster_sync_all(); else __syncthreads();  // remote mbarriers initialised before any copy
  const double tol = 2.3e-16 * sqrt((double)R);
  const double tol2 = tol * tol;
  uint32_t xph = 0;
  int par = 0, sweep = 0;
  const int pr = grp;
#ifdef TK_SVD_TIMERS  // per-phase cycle counters (diagnostic builds: they cost registers)
  long long tA = 0, tX = 0, tB = 0, tX0 = 0, tX1 = 0, t_start = clock64();
#endif
  // only the warps that own pairs run the rounds (named barrier 1 over them); the others wait at the
  // block barrier after the loop
  const int nact = min(kTileThreads, ((npairs * L + 31) / 32) * 32);
  if (tid < nact) {
    for (; sweep < kSvdMaxSweeps; ++sweep) {
      const bool exact = sweep >= kTileExactSweep;
      int any = 0;
      for (int r = 0; r < n - 1; ++r) {
#ifdef TK_SVD_TIMERS
        const long long tq0 = clock64();
#endif
        double* pp = part + par * CS * npairs * 4;
        int p = K, q = K;  // K: the zero column
        if (pr < npairs) {
          round_pair_fast(r, pr, n, K, p, q);
          p = p < K ? p : K;
          q = q < K ? q : K;
        }
        T* gp = G + p * 8 + gl;
        T* gq = G + q * 8 + gl;
        T xp[RG], xq[RG];
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
#pragma unroll
        for (int t = 0; t < RG; ++t) {
          xp[t] = gp[t * TS];
          xq[t] = gq[t * TS];
        }
#pragma unroll
        for (int t = 0; t < RG; ++t) {
          al += N::abs2(xp[t]);
          be += N::abs2(xq[t]);
          N::dot(xp[t], xq[t], gr, gi);
        }
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          gr += __shfl_xor_sync(0xffffffffu, gr, o);
          if (CPLX) gi += __shfl_xor_sync(0xffffffffu, gi, o);
        }
#ifdef TK_SVD_TIMERS
        const long long tq1 = clock64();
#endif
        if (CS > 1) {
          // the CTA's partials into its own slot [rank]; one bulk copy of the slot to every peer
          double* mine = pp + (size_t)rank * npairs * 4;
          if (pr < npairs && gl == 0) {
            *reinterpret_cast<double2*>(mine + pr * 4) = make_double2(al, be);
            *reinterpret_cast<double2*>(mine + pr * 4 + 2) = make_double2(gr, gi);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, nact);
#ifdef TK_SVD_TIMERS
          const long long tx0 = clock64();
#endif
          // thread 0 expects the bytes; lane 0 of warp w copies the slot to peers rank + c, c = 1 + w (mod the
          // active warps): one copy per warp, so the copies issue in parallel (lanes of one warp serialise)
          {
            const uint32_t bytes = (uint32_t)npairs * 32;
            if (tid == 0) mbar_arrive_expect_tx(&xbar[par], (uint32_t)(CS - 1) * bytes);
            if ((tid & 31) == 0) {
              const int w = tid >> 5, nw = nact >> 5;
              const uint32_t la = smem_u32(mine), lb = smem_u32(&xbar[par]);
              for (int c = 1 + w; c < CS; c += nw) {
                const uint32_t rk = (rank + c) % CS;
                bulk_s2cluster(mapa_u32(la, rk), la, bytes, mapa_u32(lb, rk));
              }
            }
          }
#ifdef TK_SVD_TIMERS
          const long long tx1 = clock64();
          tX0 += tx0 - tq1;
          tX1 += tx1 - tx0;
#endif
          mbar_wait_guarded(&xbar[par], (xph >> par) & 1u);  // CTA scope: the copies landed here
          xph ^= 1u << par;
          double a2 = 0.0, b2 = 0.0, g2 = 0.0, h2 = 0.0;
          if (pr < npairs) {
#pragma unroll
            for (int c = 0; c < CS; ++c) {
              const double* src = pp + ((size_t)c * npairs + pr) * 4;
              const double2 v01 = *reinterpret_cast<const double2*>(src);
              const double2 v23 = *reinterpret_cast<const double2*>(src + 2);
              a2 += v01.x;
              b2 += v01.y;
              g2 += v23.x;
              h2 += v23.y;
            }
          }
          al = a2;
          be = b2;
          gr = g2;
          gi = h2;
        }
#ifdef TK_SVD_TIMERS
        const long long tq2 = clock64();
#endif
        const double ga2 = fma(gr, gr, gi * gi);
        if (ga2 > tol2 * al * be && ga2 > 0.0) {
          double ur, ui, ag;
          if (CPLX) {  // the phase of gamma must be unit to working precision: double rsqrt
            const double rga = rsqrt(ga2);
            ur = gr * rga;
            ui = gi * rga;
            ag = ga2 * rga;
          } else {
            ur = gr < 0.0 ? -1.0 : 1.0;
            ui = 0.0;
            ag = fabs(gr);
          }
          double c, sn;
          if (exact) {
            const double zeta = 0.5 * (be - al) / ag;
            const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
            c = rsqrt(fma(t, t, 1.0));
            sn = c * t;
          } else {
            jacobi_cs_fast(al, be, ag, c, sn);
          }
#pragma unroll
          for (int t2 = 0; t2 < RG; ++t2) {
            const T x = xp[t2], y = N::rephase(xq[t2], ur, ui);
            gp[t2 * TS] = N::lin(c, x, -sn, y);
            gq[t2 * TS] = N::lin(sn, x, c, y);
          }
          T* vp = V + p * 8 + gl;
          T* vq = V + q * 8 + gl;
#pragma unroll 2
          for (int t2 = 0; t2 < tv; ++t2) {
            const T x = vp[t2 * TS], y = N::rephase(vq[t2 * TS], ur, ui);
            vp[t2 * TS] = N::lin(c, x, -sn, y);
            vq[t2 * TS] = N::lin(sn, x, c, y);
          }
          any = 1;
        }
        par ^= 1;
        named_bar_sync(1, nact);
#ifdef TK_SVD_TIMERS
        tA += tq1 - tq0;
        tX += tq2 - tq1;
        tB += clock64() - tq2;
#endif
      }
      if (!named_bar_or(1, nact, any)) break;
    }
  }
  __syncthreads();
  if (debug && tid == 0 && rank == 0) {
#ifdef TK_SVD_TIMERS
    const long long nrd = (long long)(sweep + 1) * max(n - 1, 1);
    printf("[tk svd tile] block %d: %d x %d, cluster %d, RG %d, %d sweeps, %lld cycles/round (A %lld X %lld [bar %lld issue %lld] B+S %lld)\n",
           list[blockIdx.x / CS], R, K, CS, RG, sweep + 1, (clock64() - t_start) / nrd, tA / nrd, tX / nrd, tX0 / nrd,
           tX1 / nrd, tB / nrd);
#else
    printf("[tk svd tile] block %d: %d x %d, cluster %d, RG %d, %d sweeps\n", list[blockIdx.x / CS], R, K, CS, RG,
           sweep + 1);
#endif
  }
  // column norms of the CTA's rows (no copy is in flight: every CTA left the loop after the same round)
  double* nrm = part;  // >= K doubles
  for (int j = tid >> 5; j < K; j += (kTileThreads / 32)) {
    double x = 0.0;
    for (int i = tid & 31; i < RG * 8; i += 32) x += N::abs2(G[(i >> 3) * TS + j * 8 + (i & 7)]);
    x = warp_sum(x);
    if ((tid & 31) == 0) nrm[j] = x;
  }
  if (CS > 1) cluster_sync_all(); else __syncthreads();
  if (rank == 0) {
    double* sig = part + 2 * CS * npairs * 4 - ((K + 1) & ~1);  // the top of the partial-sum region
    for (int j = tid; j < K; j += kTileThreads) {
      double x = 0.0;
#pragma unroll
      for (int c = 0; c < CS; ++c) x += (CS > 1 ? map_rank(nrm, (uint32_t)c) : nrm)[j];
      sig[j] = sqrt(x);
    }
    __syncthreads();
    double* sv = reinterpret_cast<double*>(wsv) + b.s_off;
    int32_t* pv = idx + b.p_off;
    for (int j = tid; j < K; j += kTileThreads) {
      const double sj = sig[j];
      int rk = 0;
      for (int i = 0; i < K; ++i) rk += (sig[i] > sj) || (sig[i] == sj && i < j);
      sv[rk] = sj;
      pv[rk] = j;
    }
  }
  // the CTA's rows of G and V back to the workspace (column-major, ld ldg / ldv)
  T* Gw = reinterpret_cast<T*>(wsv) + b.g_off;
  T* Vw = reinterpret_cast<T*>(wsv) + b.v_off;
  for (int64_t e = tid; e < (int64_t)nr * K; e += kTileThreads) {
    const int i = (int)(e % nr), j = (int)(e / nr);
    Gw[r0 + i + (int64_t)j * b.ldg] = G[(i >> 3) * TS + j * 8 + (i & 7)];
  }
  for (int64_t e = tid; e < (int64_t)nv * K; e += kTileThreads) {
    const int i = (int)(e % nv), j = (int)(e / nv);
    Vw[v0 + i + (int64_t)j * b.ldv] = V[(i >> 3) * TS + j * 8 + (i & 7)];
  }
  if (CS > 1) cluster_sync_all();  // rank 0's reads of the other CTAs' norms are done before they exit
}

// ---------------------------------------------------------------- panel kernel (round 2)
// One-sided Jacobi with the columns split over the cluster instead of the rows: the tile kernel above
// pays a cluster-wide exchange of partial sums in EVERY round (measured ~1000-2700 cycles at 8 CTAs: the
// slowest CTA's phase plus the DSMEM latency), which no amount of per-round tuning removed. Here a column
// [G rows | V rows] lives entirely in one CTA, so a rotation needs no other CTA. The K columns form
// P = 2 CS half-panels of m columns; CTA c holds two of them, T_c and B_c, and the half-panels meet in the
// round-robin (circle) order with T_0 fixed:
//   stage 0 (per sweep): all pairs among the CTA's own 2m columns (a circle tournament, 2m - 1 rounds);
//   outer round o = 1 .. P-2: after a move, all m^2 pairs (T_c[i], B_c[(i + s) mod m]), s = 0 .. m-1;
//   move: T_c -> T_{c+1} (1 <= c < CS-1), T_{CS-1} -> B_{CS-1}, B_0 -> T_1, B_c -> B_{c-1}: two DSMEM bulk
//   copies per CTA (cp.async.bulk shared::cta -> shared::cluster), P - 1 moves per sweep (the last one
//   restores the initial placement).
// Per sweep that is (P m - 1) rounds, the same count as the scalar circle order, but only P - 1 of them
// touch the cluster. Warp i owns T_c[i] in registers during an outer round; B columns stream through
// shared memory (one load + one store per warp and round). A lane holds rows lane + 32 t of a column
// (RPL per lane): G rows first (padded to a multiple of 32), then V rows.
constexpr int kPanelThreadsReal = 768, kPanelThreadsCplx = 768;
constexpr int kPanelThreads16 = 384;  // two pair slots per warp: <= 12 slots, 168 registers per thread
template <typename T>
struct PanelCfg {
  static constexpr int threads = sizeof(T) == 8 ? kPanelThreadsReal : kPanelThreadsCplx;
};
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
// bytes of shared memory: T_in, T_out, B_cur, B_in ([m][Lc] each), rotations [2][m][4] + flags [2][m],
// 2m norms, convergence flags, one mbarrier
__host__ __device__ inline int64_t panel_smem_bytes(int m, int Lc, int cs, int es) {
  return 4LL * m * Lc * es + 64LL * m + 8LL * m + 16 + 16LL * m + 16 + 16;
}

// Jacobi rotation of [[alpha, |gamma|], [|gamma|, beta]] without a division: with rho = beta - alpha,
// h = sqrt(rho^2 + 4 |gamma|^2) and d = |rho| + h, the tangent is t = sign(rho) 2|gamma| / d, so
// c = d / sqrt(d^2 + 4|gamma|^2) and s = sign(rho) 2|gamma| / sqrt(d^2 + 4|gamma|^2) -- one sqrt and one
// rsqrt (~250 cycles of dependent latency on B200 against ~450 for the textbook zeta/t/c chain), c and s
// both to working precision (c^2 + s^2 = 1 + O(eps)). rho and |gamma| are first scaled by a power of two
// (|gamma| into [1, 2)) so the squares neither overflow nor underflow; |rho| > 2^500 |gamma| gives
// c = 1, s = |gamma| / rho.
__device__ __forceinline__ void jacobi_rot(double al, double be, double ag, double& c, double& s) {
  const long long eb = (__double_as_longlong(ag) >> 52) & 0x7ff;
  const double sc = __longlong_as_double((2046LL - eb) << 52);
  const double rho = (be - al) * sc, g = ag * sc;
  if (fabs(rho) > 3.273390607896142e150) {  // 2^500
    c = 1.0;
    s = g / rho;
    return;
  }
  const double g2 = 4.0 * g * g;
  const double h = sqrt(fma(rho, rho, g2));
  const double d = fabs(rho) + h;
  const double r = rsqrt(fma(d, d, g2));
  c = d * r;
  s = copysign(2.0 * g * r, rho);
}

// (a, b, c, d) summed over each group of LP lanes (LP = 32: the reduce-scatter butterfly; LP = 16: a
// plain butterfly inside each half-warp, the fourth value only for ComplexF64)
template <int LP, bool CPLX>
__device__ __forceinline__ void group_sum4(double& a, double& b, double& c, double& d) {
  if constexpr (LP == 32) {
    warp_sum4(a, b, c, d);
  } else {
#pragma unroll
    for (int o = LP / 2; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
      if (CPLX) d += __shfl_xor_sync(0xffffffffu, d, o);
    }
  }
}

template <typename T, int RH, int LP>
__global__ void __launch_bounds__(LP == 16 ? kPanelThreads16 : PanelCfg<T>::threads, 1)
    svd_jacobi_panel_kernel(void* __restrict__ wsv, int32_t* __restrict__ idx, const SvdBlock* __restrict__ blocks,
                            const int32_t* __restrict__ list, int debug) {
  using N = SvNum<T>;
  constexpr bool CPLX = sizeof(T) == 16;
  extern __shared__ __align__(16) double svd_dyn[];
  const SvdBlock b = blocks[list[cluster_id_x()]];
  const int CS = b.cs;
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  const int R = b.R, K = b.K;
  const int m = b.Kl;  // columns per half-panel
  const int P = 2 * CS;
  const int Rp = (R + 31) & ~31, Kv = (K + 31) & ~31, Lc = Rp + Kv;
  // LP lanes per pair slot (32 or 16: two slots per warp). Warps 0 .. GW-1 (G-warps) rotate the G rows of
  // slot `pi` and decide the rotations; warps GW .. 2GW-1 (V-warps) apply each slot's rotation to its V
  // rows one round later, off the critical path
  constexpr int PPW = 32 / LP;
  const int sub = lane / LP, ll = lane % LP;
  const int GW = (m + PPW - 1) / PPW;
  const bool gw = warp < GW, vw = warp >= GW && warp < 2 * GW;
  const int pi = (gw ? warp : warp - GW) * PPW + sub;
  const bool pact = pi < m;                        // the last warp's second slot may be empty
  const int rb = gw ? 0 : Rp;                      // first row of this warp's part of a column
  const int nrow = gw ? (Rp / LP) : (Kv / LP);     // rows per lane (<= RH)
  T* Tin = reinterpret_cast<T*>(svd_dyn);
  T* Tout = Tin + (size_t)m * Lc;
  T* Bcur = Tout + (size_t)m * Lc;
  T* Bin = Bcur + (size_t)m * Lc;
  double* rot = reinterpret_cast<double*>(Bin + (size_t)m * Lc);  // [2][m][4]: c, s, (ur, ui) or (s ur, c ur)
  int* rflag = reinterpret_cast<int*>(rot + 8 * m);                  // [2][m]: rotation applied
  double* nrm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(rflag + 2 * m) + 15) & ~uintptr_t(15));  // 2m
  int* flag = reinterpret_cast<int*>(nrm + 2 * m);
  uint64_t* mbar = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(flag + 2) + 7) & ~uintptr_t(7));
  const T* A = reinterpret_cast<const T*>(wsv) + b.a_off;
  if (tid == 0) {
    mbar_init(mbar, 1);
    fence_barrier_init();
  }
  pdl_wait();
  // initial placement: CTA c holds columns 2cm .. 2cm + 2m - 1 (T: the first m, B: the next m)
  for (int64_t e = tid; e < (int64_t)2 * m * Lc; e += nthr) {
    const int k = (int)(e / Lc), i = (int)(e % Lc);
    const int j = (int)rank * 2 * m + k;
    T x = N::zero();
    if (j < K) {
      if (i < R) x = b.trans ? N::conj(A[j + (int64_t)i * b.lda]) : A[i + (int64_t)j * b.lda];
      else if (i >= Rp && i - Rp == j) x = N::one();
    }
    (k < m ? Tin + (size_t)k * Lc : Bcur + (size_t)(k - m) * Lc)[i] = x;
  }
  if (CS > 1) cluster_sync_all(); else __syncthreads();
  const double tol = 2.3e-16 * sqrt((double)R);
  const double tol2 = tol * tol;
  uint32_t mph = 0;
  int sweep = 0;
  T t[RH], u[RH];
  int big = 0;  // a rotation of this sweep had a cosine above sqrt(tol)
#ifdef TK_SVD_TIMERS
  long long pt[6] = {0, 0, 0, 0, 0, 0}, pts = 0, ptn = 0, pmv = 0;  // load, dots, reduce, rotation, update, barrier
#define TK_PT(i) do { const long long _c = clock64(); pt[i] += _c - pts; pts = _c; } while (0)
#else
#define TK_PT(i) do { } while (0)
#endif
  // G-warp: dots of (x, y) over the G rows, the rotation (slot `pi`, parity `sl`), applied to x, y
  auto g_rotate = [&](int sl) -> int {
    double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
#pragma unroll
    for (int r = 0; r < RH; ++r)
      if (r < nrow) {
        al += N::abs2(t[r]);
        be += N::abs2(u[r]);
        N::dot(t[r], u[r], gr, gi);
      }
    TK_PT(1);
    group_sum4<LP, CPLX>(al, be, gr, gi);
    TK_PT(2);
    const double ga2 = fma(gr, gr, gi * gi);
    const int doit = ga2 > tol2 * al * be && ga2 > 0.0;
    if (doit && ga2 > tol * al * be) big = 1;  // cosine above sqrt(tol)
    if (!doit) {
      if (ll == 0 && pact) rflag[sl * m + pi] = 0;
      return 0;
    }
    double c, sn, q0, q1;
    if (CPLX) {
      const double rga = rsqrt(ga2);
      q0 = gr * rga;  // the unit phase of gamma
      q1 = gi * rga;
      jacobi_rot(al, be, ga2 * rga, c, sn);
#pragma unroll
      for (int r = 0; r < RH; ++r)
        if (r < nrow) {
          const T x = t[r], y = N::rephase(u[r], q0, q1);
          t[r] = N::lin(c, x, -sn, y);
          u[r] = N::lin(sn, x, c, y);
        }
    } else {
      jacobi_rot(al, be, fabs(gr), c, sn);
      TK_PT(3);
      const double ur = gr < 0.0 ? -1.0 : 1.0;
      q0 = sn * ur;  // x' = c x - (s ur) y, y' = s x + (c ur) y
      q1 = c * ur;
#pragma unroll
      for (int r = 0; r < RH; ++r)
        if (r < nrow) {
          const T x = t[r], y = u[r];
          t[r] = N::lin(c, x, -q0, y);
          u[r] = N::lin(sn, x, q1, y);
        }
    }
    if (ll == 0 && pact) {
      double* rr = rot + (sl * m + pi) * 4;
      rr[0] = c;
      rr[1] = sn;
      rr[2] = q0;
      rr[3] = q1;
      rflag[sl * m + pi] = 1;
    }
    return 1;
  };
  // V-warp: the rotation of slot `pi`, parity `sl`, applied to x, y (V rows); returns whether one was applied
  auto v_rotate = [&](int sl) -> int {
    if (!rflag[sl * m + pi]) return 0;
    const double* rr = rot + (sl * m + pi) * 4;
    const double c = rr[0], sn = rr[1], q0 = rr[2], q1 = rr[3];
#pragma unroll
    for (int r = 0; r < RH; ++r)
      if (r < nrow) {
        if (CPLX) {
          const T x = t[r], y = N::rephase(u[r], q0, q1);
          t[r] = N::lin(c, x, -sn, y);
          u[r] = N::lin(sn, x, c, y);
        } else {
          const T x = t[r], y = u[r];
          t[r] = N::lin(c, x, -q0, y);
          u[r] = N::lin(sn, x, q1, y);
        }
      }
    return 1;
  };
  auto col = [&](int k) -> T* { return k < m ? Tin + (size_t)k * Lc : Bcur + (size_t)(k - m) * Lc; };
  for (; sweep < kSvdMaxSweeps; ++sweep) {
    int any = 0;
    big = 0;
    // ---- stage 0: circle tournament over the CTA's 2m columns (players k < m: T_in[k], else B_cur[k - m]);
    // the V-warps run one round behind (round 2m - 1 is theirs alone)
    {
      const int n2 = 2 * m;
      for (int r = 0; r < n2; ++r) {
        if (gw && r < n2 - 1) {
          int p = 0, q = 0;
          if (pact) round_pair_fast(r, pi, n2, n2, p, q);
          T* cp = col(p) + rb + ll;
          T* cq = col(q) + rb + ll;
#pragma unroll
          for (int k = 0; k < RH; ++k)
            if (k < nrow) {
              t[k] = pact ? cp[LP * k] : N::zero();
              u[k] = pact ? cq[LP * k] : N::zero();
            }
          if (g_rotate(r & 1)) {  // (an empty slot never rotates: its data are zero)
            any = 1;
#pragma unroll
            for (int k = 0; k < RH; ++k)
              if (k < nrow) {
                cp[LP * k] = t[k];
                cq[LP * k] = u[k];
              }
          }
        } else if (vw && r >= 1 && pact) {
          int p, q;
          round_pair_fast(r - 1, pi, n2, n2, p, q);
          T* cp = col(p) + rb + ll;
          T* cq = col(q) + rb + ll;
          if (rflag[((r - 1) & 1) * m + pi]) {
#pragma unroll
            for (int k = 0; k < RH; ++k)
              if (k < nrow) {
                t[k] = cp[LP * k];
                u[k] = cq[LP * k];
              }
            v_rotate((r - 1) & 1);
#pragma unroll
            for (int k = 0; k < RH; ++k)
              if (k < nrow) {
                cp[LP * k] = t[k];
                cq[LP * k] = u[k];
              }
          }
        }
        __syncthreads();
      }
    }
    // ---- outer rounds: move, then all m^2 pairs (T_c[i], B_c[(i + s) mod m]); the V-warps one round behind
    if (CS > 1) {
      if ((gw || vw) && pact) {
#pragma unroll
        for (int k = 0; k < RH; ++k)
          if (k < nrow) t[k] = Tin[(size_t)pi * Lc + rb + ll + LP * k];
      }
      for (int o = 1; o < P; ++o) {
#ifdef TK_SVD_TIMERS
        long long tmv = clock64();
#endif
        if ((gw || vw) && pact) {
#pragma unroll
          for (int k = 0; k < RH; ++k)
            if (k < nrow) Tout[(size_t)pi * Lc + rb + ll + LP * k] = t[k];
        }
        fence_proxy_async_smem();
        __syncthreads();
        cluster_sync_all();  // every CTA is done with its landing buffers (T_in, B_in)
        const uint32_t bytes = (uint32_t)((size_t)m * Lc * sizeof(T));
        if (tid == 0) mbar_arrive_expect_tx(mbar, 2 * bytes);
        if (tid == 0 || tid == 32) {  // two warps (blockDim >= 64): the copies issue in parallel
          const bool isT = tid == 0;
          const int c = (int)rank;
          uint32_t dst_rank;
          bool dst_T;
          if (isT) {
            if (c == 0) dst_rank = 0, dst_T = true;
            else if (c == CS - 1) dst_rank = (uint32_t)c, dst_T = false;
            else dst_rank = (uint32_t)(c + 1), dst_T = true;
          } else {
            if (c == 0) dst_rank = 1, dst_T = true;
            else dst_rank = (uint32_t)(c - 1), dst_T = false;
          }
          const uint32_t src = smem_u32(isT ? Tout : Bcur);
          const uint32_t dst = mapa_u32(smem_u32(dst_T ? Tin : Bin), dst_rank);
          bulk_s2cluster(dst, src, bytes, mapa_u32(smem_u32(mbar), dst_rank));
          bulk_commit_wait_read();
        }
        mbar_wait_guarded(mbar, mph & 1u);
        mph ^= 1u;
        {
          T* x = Bcur;
          Bcur = Bin;
          Bin = x;
        }
        if ((gw || vw) && pact) {
#pragma unroll
          for (int k = 0; k < RH; ++k)
            if (k < nrow) t[k] = Tin[(size_t)pi * Lc + rb + ll + LP * k];
        }
#ifdef TK_SVD_TIMERS
        pt[0] += clock64() - tmv;
        ++pmv;
#endif
        if (o == P - 1) break;  // the last move restores the initial placement
        for (int s2 = 0; s2 <= m; ++s2) {
          if (gw && s2 < m) {
#ifdef TK_SVD_TIMERS
            pts = clock64();
            ++ptn;
#endif
            T* cq = Bcur + (size_t)((pi + s2) % m) * Lc + ll;
#pragma unroll
            for (int k = 0; k < RH; ++k)
              if (k < nrow) {
                u[k] = pact ? cq[LP * k] : N::zero();
                if (!pact) t[k] = N::zero();
              }
            if (g_rotate(s2 & 1)) {
              any = 1;
#pragma unroll
              for (int k = 0; k < RH; ++k)
                if (k < nrow) cq[LP * k] = u[k];
            }
            TK_PT(4);
          } else if (vw && s2 >= 1 && pact) {
            if (rflag[((s2 - 1) & 1) * m + pi]) {
              T* cq = Bcur + (size_t)((pi + s2 - 1) % m) * Lc + Rp + ll;
#pragma unroll
              for (int k = 0; k < RH; ++k)
                if (k < nrow) u[k] = cq[LP * k];
              v_rotate((s2 - 1) & 1);
#pragma unroll
              for (int k = 0; k < RH; ++k)
                if (k < nrow) cq[LP * k] = u[k];
            }
          }
          __syncthreads();
#ifdef TK_SVD_TIMERS
          if (gw && s2 < m) TK_PT(5);
#endif
        }
      }
    }
    // ---- convergence: OR over the cluster
    // Stop after a sweep without rotations, or after a sweep whose rotations all had cosines below
    // sqrt(tol): each such rotation leaves its pair exactly orthogonal and perturbs the others by
    // O(cosine^2) < tol, so the verification sweep the first rule needs (1 of ~12) is skipped.
    const int cta_flag = (__syncthreads_or(any) ? 1 : 0) | (__syncthreads_or(big) ? 2 : 0);
    int all = cta_flag;
    if (CS > 1) {
      if (tid == 0) flag[0] = cta_flag;
      cluster_sync_all();
      all = 0;
      for (int c = 0; c < CS; ++c)
        all |= *reinterpret_cast<const int*>(map_rank(reinterpret_cast<const double*>(flag), (uint32_t)c));
      cluster_sync_all();  // flags read before anyone rewrites them
    }
    if (all != 3) break;
  }
  if (debug && tid == 0 && rank == 0) {
    printf("[tk svd panel] block %d: %d x %d, cluster %d, m %d, RH %d, LP %d, %d sweeps\n", list[cluster_id_x()], R, K,
           CS, m, RH, LP, sweep + 1);
#ifdef TK_SVD_TIMERS
    if (ptn)
      printf("[tk svd panel] outer-round cycles per round: load+dots %lld reduce %lld rotation %lld update %lld barrier %lld\n",
             pt[1] / ptn, pt[2] / ptn, pt[3] / ptn, pt[4] / ptn, pt[5] / ptn);
    if (pmv) printf("[tk svd panel] cycles per move: %lld (%lld moves)\n", pt[0] / pmv, pmv);
#endif
  }
  // column norms of the CTA's 2m columns (G rows), ranked against every column of the block
  for (int k = warp; k < 2 * m; k += nthr >> 5) {
    const T* cc = col(k);
    double x = 0.0;
    for (int i = lane; i < Rp; i += 32) x += N::abs2(cc[i]);
    x = warp_sum(x);
    if (lane == 0) nrm[k] = sqrt(x);
  }
  if (CS > 1) cluster_sync_all(); else __syncthreads();
  {
    double* sv = reinterpret_cast<double*>(wsv) + b.s_off;
    int32_t* pv = idx + b.p_off;
    for (int k = tid; k < 2 * m; k += nthr) {
      const int j = (int)rank * 2 * m + k;
      if (j >= K) continue;
      const double sj = nrm[k];
      int rk = 0;
      for (int i = 0; i < K; ++i) {
        const int c = i / (2 * m), kk = i % (2 * m);
        const double si = CS > 1 ? map_rank(nrm, (uint32_t)c)[kk] : nrm[kk];
        rk += (si > sj) || (si == sj && i < j);
      }
      sv[rk] = sj;
      pv[rk] = j;
    }
  }
  // columns back to the workspace: G rows to G (ld ldg), V rows to V (ld ldv)
  T* Gw = reinterpret_cast<T*>(wsv) + b.g_off;
  T* Vw = reinterpret_cast<T*>(wsv) + b.v_off;
  for (int64_t e = tid; e < (int64_t)2 * m * Lc; e += nthr) {
    const int k = (int)(e / Lc), i = (int)(e % Lc);
    const int j = (int)rank * 2 * m + k;
    if (j >= K) continue;
    const T x = col(k)[i];
    if (i < R) Gw[i + (int64_t)j * b.ldg] = x;
    else if (i >= Rp && i - Rp < K) Vw[i - Rp + (int64_t)j * b.ldv] = x;
  }
  if (CS > 1) cluster_sync_all();  // the other CTAs' norm reads are done before anyone exits
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
template <int CS, typename T, int RG>
static cudaError_t set_tile_attr() {
  return cudaFuncSetAttribute(svd_jacobi_tile_kernel<CS, T, RG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              227 * 1024);
}
template <int CS, typename T>
static cudaError_t set_tile_attrs_cs() {
  cudaError_t e = set_tile_attr<CS, T, 1>();
  if (e == cudaSuccess) e = set_tile_attr<CS, T, 2>();
  if (e == cudaSuccess) e = set_tile_attr<CS, T, 3>();
  if (e == cudaSuccess) e = set_tile_attr<CS, T, 4>();
  if constexpr (sizeof(T) == 8) {
    if (e == cudaSuccess) e = set_tile_attr<CS, T, 6>();
    if (e == cudaSuccess) e = set_tile_attr<CS, T, 8>();
  }
  return e;
}
template <typename T>
static cudaError_t set_tile_attrs_t() {
  cudaError_t e = set_tile_attrs_cs<1, T>();
  if (e == cudaSuccess) e = set_tile_attrs_cs<2, T>();
  if (e == cudaSuccess) e = set_tile_attrs_cs<4, T>();
  if (e == cudaSuccess) e = set_tile_attrs_cs<8, T>();
  return e;
}
template <typename T, int RH, int LP>
static cudaError_t set_panel_attr() {
  cudaError_t e = cudaFuncSetAttribute(svd_jacobi_panel_kernel<T, RH, LP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024);
  // clusters of 16 CTAs (non-portable; B200 allows them) for the largest blocks
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(svd_jacobi_panel_kernel<T, RH, LP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}
template <typename T>
static cudaError_t set_panel_attrs_t() {
  cudaError_t e = set_panel_attr<T, 1, 32>();
  if (e == cudaSuccess) e = set_panel_attr<T, 2, 32>();
  if (e == cudaSuccess) e = set_panel_attr<T, 3, 32>();
  if (e == cudaSuccess) e = set_panel_attr<T, 4, 32>();
  if (e == cudaSuccess) e = set_panel_attr<T, 5, 32>();
  if (e == cudaSuccess) e = set_panel_attr<T, 6, 32>();
  if (e == cudaSuccess) e = set_panel_attr<T, 7, 32>();
  if constexpr (sizeof(T) == 8) {
    if (e == cudaSuccess) e = set_panel_attr<T, 2, 16>();
    if (e == cudaSuccess) e = set_panel_attr<T, 4, 16>();
    if (e == cudaSuccess) e = set_panel_attr<T, 6, 16>();
    if (e == cudaSuccess) e = set_panel_attr<T, 8, 16>();
    if (e == cudaSuccess) e = set_panel_attr<T, 10, 16>();
    if (e == cudaSuccess) e = set_panel_attr<T, 12, 16>();
    if (e == cudaSuccess) e = set_panel_attr<T, 14, 16>();
  }
  return e;
}
static PerDeviceOnce g_svd_attrs;
static cudaError_t ensure_svd_attrs() {
  return g_svd_attrs.run([] {
    cudaError_t e = set_svd_attrs_t<double>();
    if (e == cudaSuccess) e = set_svd_attrs_t<double2>();
    if (e == cudaSuccess) e = set_tile_attrs_t<double>();
    if (e == cudaSuccess) e = set_tile_attrs_t<double2>();
    if (e == cudaSuccess) e = set_panel_attrs_t<double>();
    if (e == cudaSuccess) e = set_panel_attrs_t<double2>();
    return e;
  });
}

// launch classes: svd_jacobi_kernel (log2 CS) x (shared memory, workspace): 0..7;
// svd_jacobi_tile_kernel 8 + 6 log2 CS + index of RG in kTileRG: 8..31
// svd_jacobi_panel_kernel, 32 lanes per pair: 32 + 7 log2 CS + index of RH in kPanelRH (32..66);
// 16 lanes per pair (two pair slots per warp): 67 + 7 log2 CS + index of RH in kPanelRH16 (67..101)
constexpr int kSvdClasses = 102;
constexpr int kPanelNRH = 7;
constexpr int kPanelRH[kPanelNRH] = {1, 2, 3, 4, 5, 6, 7};
constexpr int kPanelRH16[kPanelNRH] = {2, 4, 6, 8, 10, 12, 14};
static int panel_rpl_index(int rh, int lp = 32) {
  for (int i = 0; i < kPanelNRH; ++i)
    if ((lp == 32 ? kPanelRH[i] : kPanelRH16[i]) == rh) return i;
  return kPanelNRH - 1;
}
static int panel_class(int cs, int rh, int lp) {
  int l2cs = 0;
  while ((1 << l2cs) < cs) ++l2cs;
  return (lp == 32 ? 32 : 67) + kPanelNRH * l2cs + panel_rpl_index(rh, lp);
}
constexpr int kTileRG[6] = {1, 2, 3, 4, 6, 8};
static int tile_rg_index(int rg) {
  for (int i = 0; i < 6; ++i)
    if (kTileRG[i] == rg) return i;
  return 5;
}
struct SvdPlan {
  Tensor* At = nullptr;
  bool cplx = false;
  PermPlan pa;
  PadLayout la;
  std::vector<SvdBlock> blocks;
  DevBuf d_blocks;
  std::vector<int32_t> lists[kSvdClasses];
  int class_smem[kSvdClasses] = {};
  int class_threads[kSvdClasses] = {};
  double class_t[kSvdClasses] = {};  // the longest estimated block time of the class (stream priority)
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

// svd_jacobi_tile_kernel at cluster size cs: registers per lane (RG), shared memory, and an estimate of
// the cycles of one sweep (K rounds): the slices read and written once per round at 128 B per cycle
// (+10 % for bank conflicts), the partial-sum exchange at ~20 B per cycle of DSMEM plus ~300 cycles of
// its latency, and ~400 cycles of dependent chain (shuffles, rotation, barrier).
struct TileCand {
  bool ok = false;
  int rg = 0, smem = 0;
  double t = 0.0;
};
static TileCand tile_cand(const SvdBlock& b, int cs, int es) {
  TileCand c;
  if (b.K < 1 || b.K > 2 * kTileMaxPairs) return c;
  const int Rl = (b.R + cs - 1) / cs, Kl = (b.K + cs - 1) / cs;
  const int tg = (Rl + 7) / 8, tv = (Kl + 7) / 8;
  int rg = 0;
  for (int x : kTileRG)
    if (x >= tg && (es == 8 || x <= 4)) {
      rg = x;
      break;
    }
  if (!rg) return c;
  const int npairs = (b.K + 1) / 2;
  const int64_t bytes = tile_smem_bytes(b.K, rg, tv, cs, es);
  if (bytes > 227 * 1024) return c;
  // per round: the busiest scheduler issues ~(warps / 4) x (~60 + 12 instructions per row of G and V a
  // lane holds) at ~1.5 cycles each; the exchange (bulk copies + mbarrier) ~600 cycles in a cluster
  const double warps = std::ceil(npairs * kTileL / 32.0);
  const double per_warp = 60.0 + 12.0 * (rg + tv) * (es == 8 ? 1.0 : 2.0);
  const double issue = std::ceil(warps / 4.0) * per_warp * 1.5;
  const double lat = 500.0 + 14.0 * (rg + tv);
  c.ok = true;
  c.rg = rg;
  c.smem = (int)bytes;
  c.t = (std::max(issue, lat) + (cs > 1 ? 600.0 : 0.0)) * (b.K + (b.K & 1) - 1);
  return c;
}

// svd_jacobi_panel_kernel at cluster size cs: m columns per half-panel, RPL rows per lane, shared memory, and
// an estimate of the cycles of one sweep: (2m - 1) stage-0 rounds and (P - 2) m outer-round rounds of
// ~700 cycles of dependent chain plus the warps' issue and shared-memory traffic, and P - 1 moves of two
// half-panels over DSMEM (~1500 cycles + bytes at ~50 B per cycle).
struct PanelCand {
  bool ok = false;
  int m = 0, rpl = 0, lp = 32, smem = 0, threads = 0;
  double t = 0.0;
};
static PanelCand panel_cand(const SvdBlock& b, int cs, int es) {
  PanelCand c;
  if (b.K < 1 || b.K > 192) return c;
  static const int lp_knob = (int)knob("TK_SVD_LP", 16);
  const int lp = es == 8 ? lp_knob : 32;  // two pair slots per warp (Float64)
  const int Rp = (b.R + 31) & ~31, Kv = (b.K + 31) & ~31, Lc = Rp + Kv;
  const int rh_need = std::max(Rp, Kv) / lp;
  int rh = 0;
  for (int i = 0; i < kPanelNRH; ++i) {
    const int x = lp == 32 ? kPanelRH[i] : kPanelRH16[i];
    if (x >= rh_need) {
      rh = x;
      break;
    }
  }
  if (!rh) return c;
  const int m = (b.K + 2 * cs - 1) / (2 * cs);
  const int ppw = 32 / lp;
  const int gw = (m + ppw - 1) / ppw;
  const int maxw = (lp == 16 ? kPanelThreads16 : es == 8 ? kPanelThreadsReal : kPanelThreadsCplx) / 64;
  if (gw > maxw) return c;  // (G-warps + V-warps)
  const int64_t bytes = panel_smem_bytes(m, Lc, cs, es);
  if (bytes > 227 * 1024) return c;
  // cycles per round: ~900 of dependent chain (loads, dots, reduction, rotation, update, barrier) plus
  // ~(20 + 12 rows) per pair for the issue of the G- and V-warps; per move ~1500 + the two half-panels at
  // ~30 B per cycle of DSMEM (fitted to B200 measurements of 181 x 181 at 8 and 16 CTAs, 32 lanes per
  // pair: 2100 / 1550 cycles per round, 4200 / 2800 per move)
  const int rows = std::max(Rp, Kv) / 32;
  const double t_in = 900.0 + m * (20.0 * lp / 32 + 12.0 * rows * (es == 8 ? 1.0 : 2.0));
  const double P = 2.0 * cs;
  double sweep = (2.0 * m) * t_in * 1.1;
  if (cs > 1) sweep += (P - 2) * (m + 1) * t_in + (P - 1) * (1500.0 + 2.0 * m * Lc * es / 30.0);
  c.ok = true;
  c.m = m;
  c.rpl = rh;
  c.lp = lp;
  c.smem = (int)bytes;
  c.threads = 64 * gw;
  c.t = sweep;
  return c;
}

// Cluster sizes of the tile-kernel blocks: all blocks run concurrently, so the step takes about
// max(longest block, total CTA-time / SMs). Start from the fastest CS of every block (bound Lb), then
// give every block the smallest CS that still finishes within the target, and raise the target to the
// area bound while that moves it.
static void assign_tile_blocks(SvdPlan& P, const std::vector<int>& tiles, int es) {
  if (tiles.empty()) return;
  static const int n_sm = [] {
    int d = 0, n = 0;
    if (cudaGetDevice(&d) == cudaSuccess && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) == cudaSuccess &&
        n > 0)
      return n;
    cudaGetLastError();
    return 148;
  }();
  static const int force_cs = (int)knob("TK_SVD_TILE_CS", 0);
  const int css[4] = {1, 2, 4, 8};
  double Lb = 0.0;
  for (int i : tiles) {
    double best = 1e300;
    for (int cs : css) {
      const TileCand c = tile_cand(P.blocks[i], cs, es);
      if (c.ok) best = std::min(best, c.t);
    }
    Lb = std::max(Lb, best);
  }
  std::vector<int> pick(tiles.size(), 8);
  double target = Lb;
  for (int it = 0; it < 6; ++it) {
    double area = 0.0;
    for (size_t k = 0; k < tiles.size(); ++k) {
      const SvdBlock& b = P.blocks[tiles[k]];
      int chosen = 0;
      double ct = 0.0;
      for (int cs : css) {
        const TileCand c = tile_cand(b, cs, es);
        if (!c.ok) continue;
        if (force_cs ? cs == force_cs : c.t <= target * 1.0001) {
          chosen = cs;
          ct = c.t;
          break;
        }
      }
      if (!chosen) {  // (force_cs not feasible) the fastest feasible
        double best = 1e300;
        for (int cs : css) {
          const TileCand c = tile_cand(b, cs, es);
          if (c.ok && c.t < best) best = c.t, chosen = cs;
        }
        ct = best;
      }
      pick[k] = chosen;
      area += chosen * ct;
    }
    const double nt = std::max(Lb, area / n_sm);
    if (nt <= target * 1.01) break;
    target = nt;
  }
  // longest blocks first inside every class
  std::vector<std::pair<double, int>> order;
  for (size_t k = 0; k < tiles.size(); ++k) {
    SvdBlock& b = P.blocks[tiles[k]];
    const TileCand c = tile_cand(b, pick[k], es);
    b.tile = 1;
    b.cs = pick[k];
    b.rg = c.rg;
    b.smem = 1;
    b.Rl = (b.R + b.cs - 1) / b.cs;
    b.Kl = (b.K + b.cs - 1) / b.cs;
    order.push_back({-c.t, tiles[k]});
    int l2cs = 0;
    while ((1 << l2cs) < b.cs) ++l2cs;
    const int cls = 8 + 6 * l2cs + tile_rg_index(b.rg);
    P.class_smem[cls] = std::max(P.class_smem[cls], c.smem);
    P.class_t[cls] = std::max(P.class_t[cls], c.t);
  }
  std::sort(order.begin(), order.end());
  for (auto& o : order) {
    const SvdBlock& b = P.blocks[o.second];
    int l2cs = 0;
    while ((1 << l2cs) < b.cs) ++l2cs;
    P.lists[8 + 6 * l2cs + tile_rg_index(b.rg)].push_back((int32_t)o.second);
  }
}

// Panel-kernel blocks: the blocks run concurrently, so the SVD takes about max(longest block, total
// CTA-time / SMs). Start from every block's fastest cluster size (bound Lb), give every block the
// smallest cluster size that finishes within the target, and raise the target to the area bound while
// that moves it (the largest blocks keep 8-16 CTAs, the many small ones 1-2).
static void assign_panel_blocks(SvdPlan& P, const std::vector<int>& panels, int es) {
  if (panels.empty()) return;
  static const int force_cs = (int)knob("TK_SVD_PANEL_CS", 0);
  static const int n_sm = [] {
    int d = 0, n = 0;
    if (cudaGetDevice(&d) == cudaSuccess && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) == cudaSuccess &&
        n > 0)
      return n;
    cudaGetLastError();
    return 148;
  }();
  const int css[5] = {1, 2, 4, 8, 16};
  double Lb = 0.0;
  for (int i : panels) {
    double best = 1e300;
    for (int cs : css) {
      const PanelCand c = panel_cand(P.blocks[i], cs, es);
      if (c.ok) best = std::min(best, c.t);
    }
    Lb = std::max(Lb, best);
  }
  std::vector<PanelCand> pick(panels.size());
  std::vector<int> pick_cs(panels.size(), 1);
  double target = Lb;
  for (int it = 0; it < 8; ++it) {
    double area = 0.0;
    for (size_t k = 0; k < panels.size(); ++k) {
      const SvdBlock& b = P.blocks[panels[k]];
      PanelCand ch;
      int chcs = 0;
      for (int cs : css) {
        const PanelCand c = panel_cand(b, cs, es);
        if (c.ok && (force_cs ? cs == force_cs : c.t <= target * 1.0001)) {
          ch = c;
          chcs = cs;
          break;
        }
      }
      if (!ch.ok) {  // the fastest feasible
        double best = 1e300;
        for (int cs : css) {
          const PanelCand c = panel_cand(b, cs, es);
          if (c.ok && c.t < best) best = c.t, ch = c, chcs = cs;
        }
      }
      pick[k] = ch;
      pick_cs[k] = chcs;
      area += chcs * ch.t;
    }
    const double nt = std::max(Lb, area / n_sm);
    if (force_cs || nt <= target * 1.01) break;
    target = nt;
  }
  std::vector<std::pair<double, int>> order;
  for (size_t k = 0; k < panels.size(); ++k) {
    SvdBlock& b = P.blocks[panels[k]];
    b.cs = pick_cs[k];
    b.tile = 2;
    b.rg = pick[k].rpl;
    b.lp = pick[k].lp;
    b.Kl = pick[k].m;
    b.Rl = pick[k].threads;  // (not read by the kernel: blockDim)
    b.smem = 1;
    const int cls = panel_class(b.cs, b.rg, b.lp);
    P.class_smem[cls] = std::max(P.class_smem[cls], pick[k].smem);
    P.class_threads[cls] = std::max(P.class_threads[cls], pick[k].threads);
    P.class_t[cls] = std::max(P.class_t[cls], pick[k].t);
    order.push_back({-pick[k].t, panels[k]});
  }
  std::sort(order.begin(), order.end());
  for (auto& o : order) {
    const SvdBlock& b = P.blocks[o.second];
    P.lists[panel_class(b.cs, b.rg, b.lp)].push_back((int32_t)o.second);
  }
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
  static const bool tile_enabled = knob("TK_SVD_NO_TILE", 0) == 0;
  static const bool panel_enabled = knob("TK_SVD_NO_PANEL", 0) == 0;
  std::vector<int> tiles, panels;
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
    b.tile = 0;
    b.rg = 0;
    if (panel_enabled && (panel_cand(b, 8, es).ok || panel_cand(b, 16, es).ok)) {  // decided below
      panels.push_back((int)P->blocks.size());
      P->blocks.push_back(b);
      continue;
    }
    if (tile_enabled && tile_cand(b, 8, es).ok) {  // decided below, over all blocks (after the panel kernel)
      tiles.push_back((int)P->blocks.size());
      P->blocks.push_back(b);
      continue;
    }
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
    P->class_t[cls] = 1e18;  // the blocks too large for the tile / panel kernels are the longest
    P->blocks.push_back(b);
  }
  assign_tile_blocks(*P, tiles, es);
  assign_panel_blocks(*P, panels, es);
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
        if (c >= 67)
          fprintf(stderr, " panel16 cs%d/rh%d x%zu (smem %d B, %d threads)", 1 << ((c - 67) / kPanelNRH),
                  kPanelRH16[(c - 67) % kPanelNRH], P->lists[c].size(), P->class_smem[c], P->class_threads[c]);
        else if (c >= 32)
          fprintf(stderr, " panel cs%d/rh%d x%zu (smem %d B, %d threads)", 1 << ((c - 32) / kPanelNRH),
                  kPanelRH[(c - 32) % kPanelNRH],
                  P->lists[c].size(), P->class_smem[c], P->class_threads[c]);
        else if (c < 8)
          fprintf(stderr, " cs%d/%s x%zu (smem %d B)", 1 << (c / 2), (c & 1) ? "ws" : "smem", P->lists[c].size(),
                  P->class_smem[c]);
        else
          fprintf(stderr, " tile cs%d/rg%d x%zu (smem %d B)", 1 << ((c - 8) / 6), kTileRG[(c - 8) % 6], P->lists[c].size(),
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
// Library-private streams, per device, slot and priority level (0 = the device's greatest priority).
// The SVD's launch classes run concurrently; the classes holding the longest blocks get the higher
// priorities, so their clusters are placed first and the many small blocks backfill the SMs left over
// (with equal priorities the small CTAs occupied the SMs an 8-CTA cluster needed and the longest block
// started late).
static cudaStream_t svd_aux_stream(int i, int level) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, cudaStream_t> st;
  const int d = current_device();
  std::lock_guard<std::mutex> g(mu);
  auto& s = st[{d, i, level}];
  if (!s) {
    int least = 0, greatest = 0;
    check_cuda(cudaDeviceGetStreamPriorityRange(&least, &greatest), "stream priorities");
    const int prio = std::min(least, greatest + level);  // greatest is numerically smallest
    check_cuda(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio), "svd stream");
  }
  return s;
}

template <int CS, typename T, int RG>
static cudaError_t launch_tile_class(const SvdPlan& P, int cls, void* ws, int32_t* idx, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P.lists[cls].size() * CS));
  cfg.blockDim = dim3(kTileThreads);
  cfg.dynamicSmemBytes = (size_t)P.class_smem[cls];
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
  return cudaLaunchKernelEx(&cfg, svd_jacobi_tile_kernel<CS, T, RG>, ws, idx, (const SvdBlock*)P.d_blocks.p,
                            (const int32_t*)P.d_lists[cls].p, debug);
}
template <int CS, typename T>
static cudaError_t launch_tile_cs(const SvdPlan& P, int cls, void* ws, int32_t* idx, cudaStream_t st) {
  switch ((cls - 8) % 6) {
    case 0: return launch_tile_class<CS, T, 1>(P, cls, ws, idx, st);
    case 1: return launch_tile_class<CS, T, 2>(P, cls, ws, idx, st);
    case 2: return launch_tile_class<CS, T, 3>(P, cls, ws, idx, st);
    case 3: return launch_tile_class<CS, T, 4>(P, cls, ws, idx, st);
    default:
      if constexpr (sizeof(T) == 8) {
        if ((cls - 8) % 6 == 4) return launch_tile_class<CS, T, 6>(P, cls, ws, idx, st);
        return launch_tile_class<CS, T, 8>(P, cls, ws, idx, st);
      }
      return cudaErrorInvalidValue;
  }
}

template <typename T, int RH, int LP>
static cudaError_t launch_panel_class(const SvdPlan& P, int cls, void* ws, int32_t* idx, cudaStream_t st) {
  const unsigned cs = 1u << ((cls - (LP == 32 ? 32 : 67)) / kPanelNRH);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P.lists[cls].size() * cs));
  cfg.blockDim = dim3((unsigned)P.class_threads[cls]);
  cfg.dynamicSmemBytes = (size_t)P.class_smem[cls];
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  static const int debug = std::getenv("TK_SVD_DEBUG") ? 1 : 0;  // diagnostic print only
  return cudaLaunchKernelEx(&cfg, svd_jacobi_panel_kernel<T, RH, LP>, ws, idx, (const SvdBlock*)P.d_blocks.p,
                            (const int32_t*)P.d_lists[cls].p, debug);
}

template <typename T>
static cudaError_t launch_svd_cls(const SvdPlan& P, int cls, void* ws, int32_t* idx, cudaStream_t st) {
  if (cls >= 67) {
    if constexpr (sizeof(T) == 8) {
      switch ((cls - 67) % kPanelNRH) {
        case 0: return launch_panel_class<T, 2, 16>(P, cls, ws, idx, st);
        case 1: return launch_panel_class<T, 4, 16>(P, cls, ws, idx, st);
        case 2: return launch_panel_class<T, 6, 16>(P, cls, ws, idx, st);
        case 3: return launch_panel_class<T, 8, 16>(P, cls, ws, idx, st);
        case 4: return launch_panel_class<T, 10, 16>(P, cls, ws, idx, st);
        case 5: return launch_panel_class<T, 12, 16>(P, cls, ws, idx, st);
        default: return launch_panel_class<T, 14, 16>(P, cls, ws, idx, st);
      }
    }
    return cudaErrorInvalidValue;
  }
  if (cls >= 32) {
    switch ((cls - 32) % kPanelNRH) {
      case 0: return launch_panel_class<T, 1, 32>(P, cls, ws, idx, st);
      case 1: return launch_panel_class<T, 2, 32>(P, cls, ws, idx, st);
      case 2: return launch_panel_class<T, 3, 32>(P, cls, ws, idx, st);
      case 3: return launch_panel_class<T, 4, 32>(P, cls, ws, idx, st);
      case 4: return launch_panel_class<T, 5, 32>(P, cls, ws, idx, st);
      case 5: return launch_panel_class<T, 6, 32>(P, cls, ws, idx, st);
      default: return launch_panel_class<T, 7, 32>(P, cls, ws, idx, st);
    }
  }
  if (cls >= 8) {
    switch ((cls - 8) / 6) {
      case 0: return launch_tile_cs<1, T>(P, cls, ws, idx, st);
      case 1: return launch_tile_cs<2, T>(P, cls, ws, idx, st);
      case 2: return launch_tile_cs<4, T>(P, cls, ws, idx, st);
      default: return launch_tile_cs<8, T>(P, cls, ws, idx, st);
    }
  }
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
  for (int c = kSvdClasses - 1; c >= 0; --c)
    if (!P.lists[c].empty()) cl.push_back(c);
  if (cl.empty()) return;
  // longest classes first: they take the higher-priority streams
  std::stable_sort(cl.begin(), cl.end(), [&](int a, int b) { return P.class_t[a] > P.class_t[b]; });
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> joins(cl.size(), nullptr);
  check_cuda(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "svd event");
  for (auto& e : joins) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "svd event");
  cudaError_t err = cudaEventRecord(fork, st);
  for (size_t i = 0; i < cl.size() && err == cudaSuccess; ++i) {
    cudaStream_t a = svd_aux_stream((int)i, std::min<int>((int)i, 5));
    err = cudaStreamWaitEvent(a, fork, 0);
    if (err == cudaSuccess) err = launch_svd_cls<T>(P, cl[i], ws, idx, a);
    if (err == cudaSuccess) err = cudaEventRecord(joins[i], a);
  }
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
