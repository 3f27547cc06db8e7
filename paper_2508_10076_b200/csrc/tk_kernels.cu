// sm_100a kernels of the symmetric-tensor contraction hot path.
//
//  permute_kernel  batched subblock permute (Alg. 6 / Alg. 10):
//                  every CTA takes one job (a slice of one recoupling group) from the planner's
//                  table; y_j = alpha * sum_i M[i][j] perm(x_i) + beta * y_j with the fermionic
//                  sign / SU(2) recoupling matrix M applied in flight. Two paths per group:
//                    rows  : destination leg 0 is also unit-stride in the source -> direct,
//                            coalesced on both sides; per-row base offsets staged in smem.
//                    tiled : 32x32 shared-memory transpose over (dst-fastest leg) x (src-fastest
//                            leg), so that both the loads and the stores are coalesced.
//  gemm_kernel     grouped FP64 GEMM over all coupled sectors in one launch (Alg. 8 P:1276-1300,
//                  composition = matmul P:591-609): DMMA (mma.sync m8n8k4 f64, the sm_100 FP64
//                  tensor-core path -- tcgen05 has no f64 kind), 3-stage cp.async pipeline, tiles
//                  of all groups listed by the planner (long-K first); K = 0 groups write
//                  beta*C (the zero fill of P:1271).
#include <cstdint>

#include "tk_kernels.hpp"

namespace tk {

// ---------------------------------------------------------------- helpers
struct FastDiv {  // unsigned 32-bit division by a runtime constant (round-up magic)
  uint32_t d, m, s;
  __device__ __forceinline__ void init(uint32_t dd) {
    d = dd;
    s = 0;
    while ((1u << s) < d) ++s;
    m = (d <= 1) ? 0u : (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << s) - d)) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (d <= 1) return n;
    uint32_t t = __umulhi(n, m);
    return (t + ((n - t) >> 1)) >> (s - 1);
  }
};

template <typename T>
struct Num;
template <>
struct Num<double> {
  static __device__ __forceinline__ double zero() { return 0.0; }
  static __device__ __forceinline__ double axpy(double a, double x, double y) { return fma(a, x, y); }
  static __device__ __forceinline__ double scale(double a, double x) { return a * x; }
};
template <>
struct Num<double2> {
  static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ double2 axpy(double a, double2 x, double2 y) {
    return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y));
  }
  static __device__ __forceinline__ double2 scale(double a, double2 x) { return make_double2(a * x.x, a * x.y); }
};

constexpr int kPermThreads = 256;
constexpr int kMaxRows = 256;

struct PermShared {
  int64_t rsa[kMaxRows], rsb[kMaxRows], rda[kMaxRows], rdb[kMaxRows];
  double coef[kMaxGroupMembers * kMaxGroupMembers];
  int64_t moff[2 * kMaxGroupMembers], mld[2 * kMaxGroupMembers];
};

template <typename T>
__device__ void permute_rows(const T* __restrict__ src, T* __restrict__ dst, const PermGroup& g, const PermJob& job,
                             PermShared& sh, double alpha, double beta) {
  const int tid = threadIdx.x;
  const int cnt = job.count;
  for (int r = tid; r < cnt; r += kPermThreads) {
    int64_t R = job.first + r;
    int64_t sa = 0, sb = 0, da = 0, db = 0;
#pragma unroll
    for (int l = 1; l < kMaxLegs; ++l) {
      if (l < g.ndim) {
        int64_t e = g.ext[l];
        int64_t i = R % e;
        R /= e;
        sa += i * g.sa[l];
        sb += i * g.sb[l];
        da += i * g.da[l];
        db += i * g.db[l];
      }
    }
    sh.rsa[r] = sa;
    sh.rsb[r] = sb;
    sh.rda[r] = da;
    sh.rdb[r] = db;
  }
  __syncthreads();
  const uint32_t n0 = (uint32_t)g.ext[0];
  FastDiv fd;
  fd.init(n0);
  const uint32_t total = (uint32_t)cnt * n0;
  const int ks = g.ksrc, kd = g.kdst;
  if (ks == 1 && kd == 1) {
    const int64_t so = sh.moff[0], sl = sh.mld[0], dof = sh.moff[kMaxGroupMembers], dl = sh.mld[kMaxGroupMembers];
    const int64_t s0 = g.sa[0] + sl * g.sb[0], d0 = g.da[0] + dl * g.db[0];
    const double c = alpha * sh.coef[0];
    for (uint32_t e = tid; e < total; e += kPermThreads) {
      uint32_t r = fd.div(e);
      uint32_t i0 = e - r * n0;
      T x = __ldg(src + so + sh.rsa[r] + sl * sh.rsb[r] + (int64_t)i0 * s0);
      T* yp = dst + dof + sh.rda[r] + dl * sh.rdb[r] + (int64_t)i0 * d0;
      T y = Num<T>::scale(c, x);
      if (beta != 0.0) y = Num<T>::axpy(beta, *yp, y);
      *yp = y;
    }
    return;
  }
  for (uint32_t e = tid; e < total; e += kPermThreads) {
    uint32_t r = fd.div(e);
    uint32_t i0 = e - r * n0;
    T x[kMaxGroupMembers];
#pragma unroll
    for (int i = 0; i < kMaxGroupMembers; ++i)
      if (i < ks) {
        int64_t ld = sh.mld[i];
        x[i] = __ldg(src + sh.moff[i] + sh.rsa[r] + ld * sh.rsb[r] + (int64_t)i0 * (g.sa[0] + ld * g.sb[0]));
      }
    for (int j = 0; j < kd; ++j) {
      T acc = Num<T>::zero();
#pragma unroll
      for (int i = 0; i < kMaxGroupMembers; ++i)
        if (i < ks) acc = Num<T>::axpy(sh.coef[i * kd + j], x[i], acc);
      int64_t ld = sh.mld[kMaxGroupMembers + j];
      T* yp = dst + sh.moff[kMaxGroupMembers + j] + sh.rda[r] + ld * sh.rdb[r] + (int64_t)i0 * (g.da[0] + ld * g.db[0]);
      T y = Num<T>::scale(alpha, acc);
      if (beta != 0.0) y = Num<T>::axpy(beta, *yp, y);
      *yp = y;
    }
  }
}

template <typename T>
__device__ void permute_tiled(const T* __restrict__ src, T* __restrict__ dst, const PermGroup& g, const PermJob& job,
                              PermShared& sh, T (*tile)[33], double alpha, double beta) {
  // single source / destination member (abelian groups); leg 0 = dst-fastest, leg t = src-fastest
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int t = g.tleg;
  const int n0 = g.ext[0], nt = g.ext[t];
  const int T0 = (n0 + 31) >> 5, Tt = (nt + 31) >> 5;
  const int64_t so = sh.moff[0], sl = sh.mld[0], dof = sh.moff[kMaxGroupMembers], dl = sh.mld[kMaxGroupMembers];
  const int64_t s0 = g.sa[0] + sl * g.sb[0], st = g.sa[t] + sl * g.sb[t];
  const int64_t d0 = g.da[0] + dl * g.db[0], dt = g.da[t] + dl * g.db[t];
  const double c = alpha * sh.coef[0];
  for (int u = 0; u < job.count; ++u) {
    int64_t U = job.first + u;
    int u0 = (int)(U % T0);
    U /= T0;
    int ut = (int)(U % Tt);
    int64_t R = U / Tt;
    int64_t sbase = so, dbase = dof;
    for (int l = 1; l < g.ndim; ++l) {
      if (l == t) continue;
      int64_t e = g.ext[l];
      int64_t i = R % e;
      R /= e;
      sbase += i * (g.sa[l] + sl * g.sb[l]);
      dbase += i * (g.da[l] + dl * g.db[l]);
    }
    const int i0base = u0 * 32, itbase = ut * 32;
    __syncthreads();
    // load: lanes run along the src-fastest leg (coalesced)
    if (itbase + tx < nt) {
      for (int b = ty; b < 32; b += kPermThreads / 32) {
        int i0 = i0base + b;
        if (i0 < n0) tile[b][tx] = __ldg(src + sbase + (int64_t)i0 * s0 + (int64_t)(itbase + tx) * st);
      }
    }
    __syncthreads();
    // store: lanes run along the dst-fastest leg (coalesced)
    if (i0base + tx < n0) {
      for (int a = ty; a < 32; a += kPermThreads / 32) {
        int it = itbase + a;
        if (it < nt) {
          T* yp = dst + dbase + (int64_t)(i0base + tx) * d0 + (int64_t)it * dt;
          T y = Num<T>::scale(c, tile[tx][a]);
          if (beta != 0.0) y = Num<T>::axpy(beta, *yp, y);
          *yp = y;
        }
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kPermThreads) permute_kernel(const T* __restrict__ src, T* __restrict__ dst,
                                                               const PermGroup* __restrict__ groups,
                                                               const PermMember* __restrict__ members,
                                                               const double* __restrict__ coefs,
                                                               const PermJob* __restrict__ jobs, double alpha,
                                                               double beta) {
  __shared__ PermShared sh;
  __shared__ T tile[32][33];
  const PermJob job = jobs[blockIdx.x];
  const PermGroup& g = groups[job.group];
  const int tid = threadIdx.x;
  if (tid < g.ksrc * g.kdst) sh.coef[tid] = coefs[g.coef_off + tid];
  if (tid < g.ksrc) {
    sh.moff[tid] = members[g.src_mem + tid].off;
    sh.mld[tid] = members[g.src_mem + tid].ld;
  }
  if (tid < g.kdst) {
    sh.moff[kMaxGroupMembers + tid] = members[g.dst_mem + tid].off;
    sh.mld[kMaxGroupMembers + tid] = members[g.dst_mem + tid].ld;
  }
  __syncthreads();
  if (g.mode == 1 && g.ksrc == 1 && g.kdst == 1)
    permute_tiled<T>(src, dst, g, job, sh, tile, alpha, beta);
  else
    permute_rows<T>(src, dst, g, job, sh, alpha, beta);
}

cudaError_t launch_permute(const double* src, double* dst, const PermGroup* groups, const PermMember* members,
                           const double* coefs, const PermJob* jobs, int njobs_rows, int njobs_tiled, double alpha,
                           double beta, int complex_, cudaStream_t st) {
  int n = njobs_rows + njobs_tiled;
  if (n == 0) return cudaSuccess;
  if (complex_)
    permute_kernel<double2><<<n, kPermThreads, 0, st>>>((const double2*)src, (double2*)dst, groups, members, coefs,
                                                         jobs, alpha, beta);
  else
    permute_kernel<double><<<n, kPermThreads, 0, st>>>(src, dst, groups, members, coefs, jobs, alpha, beta);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- grouped FP64 GEMM (DMMA)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
struct GemmCfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int MF = WM / 8, NF = WN / 8;
  static constexpr int LDA_S = BM + 8;  // As[k][m], padded: conflict-free fragment loads
  static constexpr int LDB_S = BK + 4;  // Bs[n][k]
  static constexpr int A_STAGE = BK * LDA_S, B_STAGE = BN * LDB_S;
  static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
};

template <int BM, int BN, int WM, int WN, int BK, int STAGES>
__device__ void gemm_tile(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                          const GemmGroup& g, int m0, int n0, double alpha, double beta, double* smem) {
  using Cfg = GemmCfg<BM, BN, WM, WN, BK, STAGES>;
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % Cfg::WARPS_M, wn = warp / Cfg::WARPS_M;
  const int gq = lane >> 2, tq = lane & 3;
  const double* Ag = A + g.a_off;
  const double* Bg = B + g.b_off;
  const int M = g.M, N = g.N, K = g.K;
  const int nk = (K + BK - 1) / BK;

  double acc[Cfg::MF][Cfg::NF][2];
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int kt, int s) {
    const int k0 = kt * BK;
    double* as = As + s * Cfg::A_STAGE;
    double* bs = Bs + s * Cfg::B_STAGE;
#pragma unroll
    for (int i = 0; i < (BM * BK) / Cfg::THREADS; ++i) {
      int idx = tid + i * Cfg::THREADS;
      int m = idx % BM, k = idx / BM;
      bool ok = (m0 + m < M) && (k0 + k < K);
      const double* gp = ok ? Ag + (int64_t)(m0 + m) + (int64_t)(k0 + k) * g.lda : A;
      cp_async8(as + k * Cfg::LDA_S + m, gp, ok);
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / Cfg::THREADS; ++i) {
      int idx = tid + i * Cfg::THREADS;
      int k = idx % BK, n = idx / BK;
      bool ok = (n0 + n < N) && (k0 + k < K);
      const double* gp = ok ? Bg + (int64_t)(k0 + k) + (int64_t)(n0 + n) * g.ldb : B;
      cp_async8(bs + n * Cfg::LDB_S + k, gp, ok);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt, nxt % STAGES);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * Cfg::A_STAGE;
    const double* bs = Bs + (kt % STAGES) * Cfg::B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::MF], bf[Cfg::NF];
#pragma unroll
      for (int i = 0; i < Cfg::MF; ++i) af[i] = as[(kk + tq) * Cfg::LDA_S + wm * WM + i * 8 + gq];
#pragma unroll
      for (int j = 0; j < Cfg::NF; ++j) bf[j] = bs[(wn * WN + j * 8 + gq) * Cfg::LDB_S + kk + tq];
#pragma unroll
      for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NF; ++j) dmma884(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // epilogue: C = alpha * acc + beta * C (column-major, ldc)
  double* Cg = C + g.c_off;
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i) {
    int m = m0 + wm * WM + i * 8 + gq;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        int n = n0 + wn * WN + j * 8 + 2 * tq + c;
        if (n < N) {
          double* p = Cg + (int64_t)m + (int64_t)n * g.ldc;
          double v = alpha * acc[i][j][c];
          if (beta != 0.0) v = fma(beta, *p, v);
          *p = v;
        }
      }
    }
  }
}

using BigCfg = GemmCfg<128, 128, 64, 32, 16, 3>;
using SmallCfg = GemmCfg<64, 64, 32, 32, 16, 3>;

__global__ void __launch_bounds__(BigCfg::THREADS, 1)
    gemm_big_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                    const GemmGroup* __restrict__ groups, const GemmTile* __restrict__ tiles, double alpha,
                    double beta) {
  extern __shared__ __align__(16) double smem[];
  const GemmTile t = tiles[blockIdx.x];
  const GemmGroup g = groups[t.group];
  gemm_tile<128, 128, 64, 32, 16, 3>(A, B, C, g, t.m0, t.n0, alpha, beta, smem);
}

__global__ void __launch_bounds__(SmallCfg::THREADS)
    gemm_small_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                      const GemmGroup* __restrict__ groups, const GemmTile* __restrict__ tiles, double alpha,
                      double beta) {
  extern __shared__ __align__(16) double smem[];
  const GemmTile t = tiles[blockIdx.x];
  const GemmGroup g = groups[t.group];
  gemm_tile<64, 64, 32, 32, 16, 3>(A, B, C, g, t.m0, t.n0, alpha, beta, smem);
}

cudaError_t launch_gemm(const double* A, const double* B, double* C, const GemmGroup* groups, const GemmTile* tiles,
                        int ntiles_big, int ntiles_small, double alpha, double beta, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BigCfg::SMEM);
    cudaFuncSetAttribute(gemm_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SmallCfg::SMEM);
    attr = true;
  }
  if (ntiles_big)
    gemm_big_kernel<<<ntiles_big, BigCfg::THREADS, BigCfg::SMEM, st>>>(A, B, C, groups, tiles, alpha, beta);
  if (ntiles_small)
    gemm_small_kernel<<<ntiles_small, SmallCfg::THREADS, SmallCfg::SMEM, st>>>(A, B, C, groups, tiles + ntiles_big,
                                                                               alpha, beta);
  return cudaGetLastError();
}

}  // namespace tk
