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
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "tk_device.cuh"
#include "tk_internal.hpp"
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

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Programmatic dependent launch (sm_90+): every kernel lets the next kernel in the stream start its
// launch early (launch_dependents) and reads/writes tensor data only after griddepcontrol.wait, which
// returns once the preceding grid has completed and its writes are visible. Descriptor tables (plan
// constants) are read before the wait, so job/group decoding overlaps the previous kernel's tail.

#ifndef TK_PERM_MINB
#define TK_PERM_MINB 4       // resident permute CTAs per SM (register budget: 64 / thread at 256 x 4)
#endif
#ifndef TK_ROWS_MINB
#define TK_ROWS_MINB 6  // Float64 rows-only permute: 6 CTAs/SM (<= 40 registers): cfg4 5.41 vs 5.24 TB/s at 5
#endif
#ifndef TK_ROWS_MINB_C
#define TK_ROWS_MINB_C TK_PERM_MINB  // ComplexF64 rows-only instances
#endif
#ifndef TK_ROWS_U
#define TK_ROWS_U 8  // loads in flight per thread in the rows path (Float64)
#endif

// Element I/O of the permute kernels per complex mode CM (see PermCM in tk_kernels.hpp). Offsets are in
// units of the pointer type: complex elements for interleaved buffers, doubles for planar ones. A
// planar member's imaginary part sits d1 doubles after its real part; the real representation of a
// B~ block stores [[re, im], [-im, re]] at +0, +d1, +d2, +d1+d2 (d1 = N ld, d2 = K).
template <int CM>
struct CIO {
  using V = typename std::conditional<CM == kPermReal, double, double2>::type;  // value in registers
  using S = typename std::conditional<CM == kPermReal || CM == kPermPlanarToC, double, double2>::type;
  using D = typename std::conditional<CM == kPermCToC || CM == kPermPlanarToC, double2, double>::type;
  static __device__ __forceinline__ V load(const S* __restrict__ src, int64_t o, int64_t d1) {
    if constexpr (CM == kPermPlanarToC)
      return make_double2(__ldg(src + o), __ldg(src + o + d1));
    else
      return __ldg(src + o);
  }
  // y already carries alpha * coefficient; ims = -1 conjugates (operand permutes of tk_contract)
  static __device__ __forceinline__ void store(D* __restrict__ dst, int64_t o, int64_t d1, int64_t d2, V y,
                                               double beta, double ims) {
    if constexpr (CM == kPermReal || CM == kPermCToC || CM == kPermPlanarToC) {
      if (beta != 0.0) y = Num<V>::axpy(beta, dst[o], y);
      dst[o] = y;
    } else if constexpr (CM == kPermCToPlanar) {  // workspace target: beta == 0 (host-checked)
      dst[o] = y.x;
      dst[o + d1] = ims * y.y;
    } else {  // kPermCToRealRep
      const double im = ims * y.y;
      dst[o] = y.x;
      dst[o + d1] = im;
      dst[o + d2] = -im;
      dst[o + d1 + d2] = y.x;
    }
  }
};

struct PermShared {
  int64_t rsa[kMaxRows], rsb[kMaxRows], rda[kMaxRows], rdb[kMaxRows];
  double coef[kMaxGroupMembers * kMaxGroupMembers];
  int64_t moff[2 * kMaxGroupMembers], mld[2 * kMaxGroupMembers];
  int64_t md1[2 * kMaxGroupMembers], md2[2 * kMaxGroupMembers];
};

// single-member rows job: destination leg 0 is also unit-stride in the source; the row starts of the
// job are decoded once into shared memory, then the job's elements are walked as one flat range with
// TK_ROWS_U loads in flight per thread
template <int CM>
__device__ void permute_rows(const typename CIO<CM>::S* __restrict__ src, typename CIO<CM>::D* __restrict__ dst,
                             const PermGroup& g, const PermJob& job, PermShared& sh, double alpha, double beta,
                             double ims) {
  using IO = CIO<CM>;
  using V = typename IO::V;
  const int tid = threadIdx.x;
  const int cnt = job.count;
  const int64_t sl = sh.mld[0], dl = sh.mld[kMaxGroupMembers];
  for (int r = tid; r < cnt; r += kPermThreads) {
    uint32_t R = (uint32_t)(job.first + r);  // group element counts are < 2^31 (host-checked)
    int64_t sa = 0, sb = 0, da = 0, db = 0;
#pragma unroll 1
    for (int l = 1; l < kMaxLegs; ++l) {
      if (l < g.ndim) {
        const uint32_t e = (uint32_t)g.ext[l];
        const uint32_t q = R / e;
        const int64_t i = R - q * e;
        R = q;
        sa += i * g.sa[l];
        sb += i * g.sb[l];
        da += i * g.da[l];
        db += i * g.db[l];
      }
    }
    sh.rsa[r] = sh.moff[0] + sa + sl * sb;  // final element offsets of the row start
    sh.rda[r] = sh.moff[kMaxGroupMembers] + da + dl * db;
  }
  __syncthreads();
  pdl_wait();
  const int n0 = g.ext[0];
  const int64_t s0 = g.sa[0] + sl * g.sb[0], d0 = g.da[0] + dl * g.db[0];
  const int64_t sd1 = sh.md1[0], dd1 = sh.md1[kMaxGroupMembers], dd2 = sh.md2[kMaxGroupMembers];
  const double c = alpha * sh.coef[0];
  // independent loads in flight per thread (64 bytes: bytes in flight hide DRAM latency)
  constexpr int U = sizeof(V) == 16 ? TK_ROWS_U / 2 : TK_ROWS_U;
  FastDiv fd;
  fd.init((uint32_t)n0);
  const uint32_t total = (uint32_t)cnt * (uint32_t)n0;
  for (uint32_t e0 = tid; e0 < total; e0 += U * kPermThreads) {
    V x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t e = e0 + u * kPermThreads;
      if (e < total) {
        uint32_t r = fd.div(e);
        uint32_t i0 = e - r * (uint32_t)n0;
        x[u] = IO::load(src, sh.rsa[r] + (int64_t)i0 * s0, sd1);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t e = e0 + u * kPermThreads;
      if (e < total) {
        uint32_t r = fd.div(e);
        uint32_t i0 = e - r * (uint32_t)n0;
        IO::store(dst, sh.rda[r] + (int64_t)i0 * d0, dd1, dd2, Num<V>::scale(c, x[u]), beta, ims);
      }
    }
  }
}

template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem) {
  uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
  else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// stage one source element into shared memory (planar sources: real and imaginary part separately)
template <int CM>
__device__ __forceinline__ void stage_elem(typename CIO<CM>::V* smem, const typename CIO<CM>::S* gmem, int64_t d1) {
  if constexpr (CM == kPermPlanarToC) {
    cp_async_elem<double>(&smem->x, gmem);
    cp_async_elem<double>(&smem->y, gmem + d1);
  } else {
    cp_async_elem<typename CIO<CM>::S>(smem, gmem);
  }
}

// Mixed-radix counter over a (za, zb, *) box, advanced by a fixed step: no divisions per element.
struct Walk3 {
  int x0, x1, x2, d0, d1, d2, za, zb;
  __device__ __forceinline__ void init(int start, int step, int za_, int zb_) {
    za = za_;
    zb = zb_;
    x0 = start % za;
    int q = start / za;
    x1 = q % zb;
    x2 = q / zb;
    d0 = step % za;
    q = step / za;
    d1 = q % zb;
    d2 = q / zb;
  }
  __device__ __forceinline__ void next() {
    x0 += d0;
    int c = x0 >= za;
    x0 -= c ? za : 0;
    x1 += d1 + c;
    c = x1 >= zb;
    x1 -= c ? zb : 0;
    x2 += d2 + c;
  }
};

// Tile phases, specialised on the load walk order (O0 fastest, O1, O2) over {0: i0, 1: it, 2: r}.
template <int CM, int O0, int O1, int O2>
__device__ __forceinline__ void tile_load(const typename CIO<CM>::S* __restrict__ src, typename CIO<CM>::V* __restrict__ Sb,
                                          const int64_t* __restrict__ rs, int c0, int ct, int R, int c0p, int nr,
                                          int m0, int mt, int64_t s0, int64_t st, int64_t sd1) {
  const int sz[3] = {c0, ct, R};
  const int n = c0 * ct * R;
  Walk3 w;
  w.init(threadIdx.x, kPermThreads, sz[O0], sz[O1]);
  for (int e = threadIdx.x; e < n; e += kPermThreads, w.next()) {
    int v[3];
    v[O0] = w.x0;
    v[O1] = w.x1;
    v[O2] = w.x2;
    const int i0 = v[0], it = v[1], r = v[2];
    if (r < nr && i0 < m0 && it < mt)
      stage_elem<CM>(Sb + (r * ct + it) * c0p + i0, src + rs[r] + (int64_t)i0 * s0 + (int64_t)it * st, sd1);
  }
}

template <int CM>
__device__ __forceinline__ void tile_store(typename CIO<CM>::D* __restrict__ dst, const typename CIO<CM>::V* __restrict__ Sb,
                                           const int64_t* __restrict__ rd, int c0, int ct, int R, int c0p, int nr,
                                           int m0, int mt, int64_t d0, int64_t dt, int64_t dd1, int64_t dd2, double c,
                                           double beta, double ims) {
  using V = typename CIO<CM>::V;
  const int n = c0 * ct * R;
  Walk3 w;
  w.init(threadIdx.x, kPermThreads, c0, ct);
  for (int e = threadIdx.x; e < n; e += kPermThreads, w.next()) {
    const int i0 = w.x0, it = w.x1, r = w.x2;
    if (r < nr && i0 < m0 && it < mt)
      CIO<CM>::store(dst, rd[r] + (int64_t)i0 * d0 + (int64_t)it * dt, dd1, dd2,
                     Num<V>::scale(c, Sb[(r * ct + it) * c0p + i0]), beta, ims);
  }
}

template <int CM>
__device__ void permute_tiled(const typename CIO<CM>::S* __restrict__ src, typename CIO<CM>::D* __restrict__ dst,
                              const PermGroup& g, const PermJob& job, PermShared& sh, typename CIO<CM>::V* __restrict__ S,
                              double alpha, double beta, double ims) {
  // One source / destination member (abelian groups). Leg 0 = dst-fastest, leg t = dst leg 1.
  // A tile holds chunk c0 of leg 0 x chunk ct of leg t x R consecutive "rest" indices (all other
  // legs). Loads walk the tile in source-stride order (coalesced reads) as cp.async straight into
  // shared memory, double-buffered so that tile u+1 streams in while tile u is stored; stores walk
  // the tile in destination order (leg 0 fastest: coalesced writes). S[r][it][i0] has an odd row
  // pitch so both phases are free of shared-memory bank conflicts.
  const int tid = threadIdx.x;
  const int t = g.tleg;
  const int n0 = g.ext[0], nt = g.ext[t];
  const int c0 = g.c0, ct = g.ct, R = g.R, c0p = c0 | 1;
  const int64_t so = sh.moff[0], sl = sh.mld[0], dof = sh.moff[kMaxGroupMembers], dl = sh.mld[kMaxGroupMembers];
  const int64_t s0 = g.sa[0] + sl * g.sb[0], st = g.sa[t] + sl * g.sb[t];
  const int64_t d0 = g.da[0] + dl * g.db[0], dt = g.da[t] + dl * g.db[t];
  const int64_t sd1 = sh.md1[0], dd1 = sh.md1[kMaxGroupMembers], dd2 = sh.md2[kMaxGroupMembers];
  const double c = alpha * sh.coef[0];
  const int lorder = g.lorder;
  const int half = kTileElems / 2;  // two tile buffers

  auto tile_geom = [&](int u, int& i0b, int& itb, int& nr, int& m0, int& mt, int64_t& rb) {
    int64_t U = job.first + u;
    const int u0 = (int)(U % g.T0);
    U /= g.T0;
    const int ut = (int)(U % g.Tt);
    rb = (U / g.Tt) * R;
    i0b = u0 * c0;
    itb = ut * ct;
    nr = (int)min((int64_t)R, g.nrest - rb);
    m0 = min(c0, n0 - i0b);
    mt = min(ct, nt - itb);
  };
  auto tables = [&](int u, int b) {  // per-rest-index base offsets of tile u into table buffer b
    int i0b, itb, nr, m0, mt;
    int64_t rb;
    tile_geom(u, i0b, itb, nr, m0, mt, rb);
    int64_t* rs = sh.rsa + b * (kMaxRows / 2);
    int64_t* rd = sh.rda + b * (kMaxRows / 2);
    for (int r = tid; r < nr; r += kPermThreads) {
      uint32_t Rr = (uint32_t)(rb + r);
      int64_t sbase = so, dbase = dof;
      for (int l = 1; l < g.ndim; ++l) {
        if (l == t) continue;
        const uint32_t e = (uint32_t)g.ext[l];
        const uint32_t q = Rr / e;
        const int64_t i = Rr - q * e;
        Rr = q;
        sbase += i * (g.sa[l] + sl * g.sb[l]);
        dbase += i * (g.da[l] + dl * g.db[l]);
      }
      rs[r] = sbase + (int64_t)i0b * s0 + (int64_t)itb * st;
      rd[r] = dbase + (int64_t)i0b * d0 + (int64_t)itb * dt;
    }
  };
  auto issue_loads = [&](int u, int b) {
    int i0b, itb, nr, m0, mt;
    int64_t rb;
    tile_geom(u, i0b, itb, nr, m0, mt, rb);
    typename CIO<CM>::V* Sb = S + b * half;
    const int64_t* rs = sh.rsa + b * (kMaxRows / 2);
    switch (lorder) {
      case 0 + 3 * 1 + 9 * 2: tile_load<CM, 0, 1, 2>(src, Sb, rs, c0, ct, R, c0p, nr, m0, mt, s0, st, sd1); break;
      case 0 + 3 * 2 + 9 * 1: tile_load<CM, 0, 2, 1>(src, Sb, rs, c0, ct, R, c0p, nr, m0, mt, s0, st, sd1); break;
      case 1 + 3 * 0 + 9 * 2: tile_load<CM, 1, 0, 2>(src, Sb, rs, c0, ct, R, c0p, nr, m0, mt, s0, st, sd1); break;
      case 1 + 3 * 2 + 9 * 0: tile_load<CM, 1, 2, 0>(src, Sb, rs, c0, ct, R, c0p, nr, m0, mt, s0, st, sd1); break;
      case 2 + 3 * 0 + 9 * 1: tile_load<CM, 2, 0, 1>(src, Sb, rs, c0, ct, R, c0p, nr, m0, mt, s0, st, sd1); break;
      default: tile_load<CM, 2, 1, 0>(src, Sb, rs, c0, ct, R, c0p, nr, m0, mt, s0, st, sd1); break;
    }
    cp_async_commit();
  };

  tables(0, 0);
  __syncthreads();
  pdl_wait();
  issue_loads(0, 0);
  for (int u = 0; u < job.count; ++u) {
    const int b = u & 1;
    if (u + 1 < job.count) {
      tables(u + 1, b ^ 1);
      __syncthreads();
      issue_loads(u + 1, b ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    int i0b, itb, nr, m0, mt;
    int64_t rb;
    tile_geom(u, i0b, itb, nr, m0, mt, rb);
    tile_store<CM>(dst, S + b * half, sh.rda + b * (kMaxRows / 2), c0, ct, R, c0p, nr, m0, mt, d0, dt, dd1, dd2, c,
                   beta, ims);
    __syncthreads();  // buffer b and its tables are reused by tile u+2
  }
}

__device__ __forceinline__ void load_job_header(const PermGroup& g, const PermMember* __restrict__ members,
                                                const double* __restrict__ coefs, PermShared& sh) {
  const int tid = threadIdx.x;
  for (int i = tid; i < g.ksrc * g.kdst; i += kPermThreads) sh.coef[i] = coefs[g.coef_off + i];
  if (tid < g.ksrc) {
    const PermMember m = members[g.src_mem + tid];
    sh.moff[tid] = m.off;
    sh.mld[tid] = m.ld;
    sh.md1[tid] = m.d1;
    sh.md2[tid] = m.d2;
  }
  if (tid < g.kdst) {
    const PermMember m = members[g.dst_mem + tid];
    sh.moff[kMaxGroupMembers + tid] = m.off;
    sh.mld[kMaxGroupMembers + tid] = m.ld;
    sh.md1[kMaxGroupMembers + tid] = m.d1;
    sh.md2[kMaxGroupMembers + tid] = m.d2;
  }
  __syncthreads();
}

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute (PDL); returns the launch's
// own status (never cudaGetLastError, which would also report and clear unrelated earlier errors)
template <typename... KArgs, typename... Args>
static cudaError_t launch_k2(void (*kern)(KArgs...), dim3 grid, int block, size_t smem, cudaStream_t st,
                             Args... args) {
  static const bool pdl = knob("TK_NO_PDL", 0) == 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args... args) {
  return launch_k2(kern, dim3((unsigned)grid), block, smem, st, args...);
}

// packed jobs of small single-member rows groups (see kPackGroups): per CTA, the groups' row tables
// are built once into shared memory, then all elements of the job are walked as one flat range with
// 64 bytes of loads in flight per thread; each thread advances its group index monotonically.
struct PackShared {
  int64_t rs[kPackRows], rd[kPackRows];
  int64_t s0[kPackGroups], d0[kPackGroups], sd1[kPackGroups], dd1[kPackGroups], dd2[kPackGroups];
  double c[kPackGroups];
  uint32_t fm[kPackGroups], fs[kPackGroups], n0[kPackGroups];
  int32_t rstart[kPackGroups + 1], estart[kPackGroups + 1];
};

template <int CM>
__device__ void permute_packed(const typename CIO<CM>::S* __restrict__ src, typename CIO<CM>::D* __restrict__ dst,
                               const PermGroup* __restrict__ groups, const PermMember* __restrict__ members,
                               const double* __restrict__ coefs, const PermJob& job, PackShared& sh, double alpha,
                               double beta, double ims) {
  using IO = CIO<CM>;
  using V = typename IO::V;
  const int ng = job.count;
  const int tid = threadIdx.x;
  // group headers + prefix sums of rows / elements (one warp)
  if (tid < 32) {
    int racc = 0, eacc = 0;
    for (int base = 0; base < ng; base += 32) {
      const int gi = base + tid;
      int rows = 0, el = 0;
      if (gi < ng) {
        const PermGroup& g = groups[job.group + gi];
        const PermMember ms = members[g.src_mem], md = members[g.dst_mem];
        const uint32_t n0 = (uint32_t)g.ext[0];
        el = (int)g.nelem;
        rows = el / (int)n0;
        sh.s0[gi] = g.sa[0] + ms.ld * g.sb[0];
        sh.d0[gi] = g.da[0] + md.ld * g.db[0];
        sh.sd1[gi] = ms.d1;
        sh.dd1[gi] = md.d1;
        sh.dd2[gi] = md.d2;
        sh.c[gi] = alpha * coefs[g.coef_off];
        FastDiv fd;
        fd.init(n0);
        sh.fm[gi] = fd.m;
        sh.fs[gi] = fd.s;
        sh.n0[gi] = n0;
      }
      int ri = rows, ei = el;  // inclusive warp scans
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int yr = __shfl_up_sync(0xffffffffu, ri, o), ye = __shfl_up_sync(0xffffffffu, ei, o);
        if (tid >= o) {
          ri += yr;
          ei += ye;
        }
      }
      if (gi < ng) {
        sh.rstart[gi] = racc + ri - rows;
        sh.estart[gi] = eacc + ei - el;
      }
      racc += __shfl_sync(0xffffffffu, ri, 31);
      eacc += __shfl_sync(0xffffffffu, ei, 31);
    }
    if (tid == 0) {
      sh.rstart[ng] = racc;
      sh.estart[ng] = eacc;
    }
  }
  __syncthreads();
  // row tables: final source / destination offsets of every row start
  const int nrows = sh.rstart[ng];
  for (int r = tid; r < nrows; r += kPermThreads) {
    int lo = 0, hi = ng - 1;  // last group with rstart <= r
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (sh.rstart[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const PermGroup& g = groups[job.group + lo];
    uint32_t R = (uint32_t)(r - sh.rstart[lo]);
    int64_t sa = 0, sb = 0, da = 0, db = 0;
#pragma unroll 1
    for (int l = 1; l < g.ndim; ++l) {
      const uint32_t e = (uint32_t)g.ext[l];
      const uint32_t q = R / e;
      const int64_t i = R - q * e;
      R = q;
      sa += i * g.sa[l];
      sb += i * g.sb[l];
      da += i * g.da[l];
      db += i * g.db[l];
    }
    const PermMember ms = members[g.src_mem], md = members[g.dst_mem];
    sh.rs[r] = ms.off + sa + ms.ld * sb;
    sh.rd[r] = md.off + da + md.ld * db;
  }
  __syncthreads();
  pdl_wait();
  const int total = sh.estart[ng];
  constexpr int U = sizeof(V) == 16 ? 4 : 8;
  int gi = 0;
  for (int e0 = tid; e0 < total; e0 += U * kPermThreads) {
    V x[U];
    int64_t od[U];
    int gu[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kPermThreads;
      gu[u] = -1;
      if (e < total) {
        while (sh.estart[gi + 1] <= e) ++gi;
        const uint32_t loc = (uint32_t)(e - sh.estart[gi]);
        FastDiv fd;
        fd.d = sh.n0[gi];
        fd.m = sh.fm[gi];
        fd.s = sh.fs[gi];
        const uint32_t r = fd.div(loc);
        const uint32_t i0 = loc - r * fd.d;
        const int row = sh.rstart[gi] + (int)r;
        x[u] = IO::load(src, sh.rs[row] + (int64_t)i0 * sh.s0[gi], sh.sd1[gi]);
        od[u] = sh.rd[row] + (int64_t)i0 * sh.d0[gi];
        gu[u] = gi;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (gu[u] >= 0) {
        const int g = gu[u];
        IO::store(dst, od[u], sh.dd1[g], sh.dd2[g], Num<V>::scale(sh.c[g], x[u]), beta, ims);
      }
  }
}

// kJobSeg (see SegGroup): with the job's blob in shared memory (sm), walk its elements as one flat
// range with 64 bytes of loads in flight per thread. Each thread's elements are kPermThreads apart, so
// (row, index in row) advance incrementally by (q, rem) of the current chunk; the division runs only
// when a thread enters a new chunk.
template <int CM>
__device__ __forceinline__ void seg_body(const typename CIO<CM>::S* __restrict__ src,
                                         typename CIO<CM>::D* __restrict__ dst, const int64_t* sm, double alpha,
                                         double beta, double ims) {
  using IO = CIO<CM>;
  using V = typename IO::V;
  const SegHeader h = *reinterpret_cast<const SegHeader*>(sm);
  const SegGroup* G = reinterpret_cast<const SegGroup*>(sm + 2);
  const int32_t* rs = reinterpret_cast<const int32_t*>(sm + 2 + 10 * h.ng);
  const int32_t* rd = rs + h.nrows;
  const int total = h.total, last = h.ng - 1;
  constexpr int U = sizeof(V) == 16 ? 4 : 8;
  int e = threadIdx.x;
  if (e >= total) return;
  int gi = 0, end = -1;  // end = -1: locate the chunk of the first element
  uint32_t n0 = 1, q = 0, rem = 0, r = 0, i0 = 0;
  int rst = 0, s0 = 0, d0 = 0;
  while (e < total) {
    V x[U];
    int od[U];
    int gu[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      gu[u] = -1;
      if (e < total) {
        if (e >= end) {  // entering a later chunk
          while (gi < last && G[gi + 1].estart <= e) ++gi;
          end = gi < last ? G[gi + 1].estart : total;
          n0 = G[gi].n0;
          q = G[gi].q;
          rem = G[gi].rem;
          rst = G[gi].rstart;
          s0 = (int)G[gi].s0;
          d0 = (int)G[gi].d0;
          FastDiv fd;
          fd.d = n0;
          fd.m = G[gi].fm;
          fd.s = G[gi].fs;
          const uint32_t loc = (uint32_t)(e - G[gi].estart);
          r = fd.div(loc);
          i0 = loc - r * n0;
        }
        const int row = rst + (int)r;
        x[u] = IO::load(src, (int64_t)(rs[row] + (int)i0 * s0), G[gi].sd1);
        od[u] = rd[row] + (int)i0 * d0;
        gu[u] = gi;
        e += kPermThreads;
        i0 += rem;
        r += q;
        if (i0 >= n0) {
          i0 -= n0;
          ++r;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (gu[u] >= 0) {
        const SegGroup& g = G[gu[u]];
        IO::store(dst, (int64_t)od[u], g.dd1, g.dd2, Num<V>::scale(alpha * g.c, x[u]), beta, ims);
      }
  }
}

// a seg job inside the general permute kernel (launches that mix seg with tiled / box jobs)
template <int CM>
__device__ void permute_seg(const typename CIO<CM>::S* __restrict__ src, typename CIO<CM>::D* __restrict__ dst,
                            const int64_t* __restrict__ blob, const PermJob& job, int64_t* sm, double alpha,
                            double beta, double ims) {
  const longlong2* g2 = reinterpret_cast<const longlong2*>(blob + job.first);
  longlong2* s2 = reinterpret_cast<longlong2*>(sm);
  const int n2 = job.group >> 1;
  for (int i = threadIdx.x; i < n2; i += kPermThreads) s2[i] = __ldg(g2 + i);
  __syncthreads();
  pdl_wait();
  seg_body<CM>(src, dst, sm, alpha, beta, ims);
}

// recoupling jobs: offsets of every row start relative to the member bases (legs 1..), in smem
__device__ __forceinline__ void recouple_row_tables(const PermGroup& g, const PermJob& job, PermShared& sh) {
  for (int r = threadIdx.x; r < job.count; r += kPermThreads) {
    uint32_t R = (uint32_t)(job.first + r);
    int64_t sa = 0, sb = 0, da = 0, db = 0;
#pragma unroll 1
    for (int l = 1; l < g.ndim; ++l) {
      const uint32_t e = (uint32_t)g.ext[l], q = R / e;
      const int64_t i = R - q * e;
      R = q;
      sa += i * g.sa[l];
      sb += i * g.sb[l];
      da += i * g.da[l];
      db += i * g.db[l];
    }
    sh.rsa[r] = sa;
    sh.rsb[r] = sb;
    sh.rda[r] = da;
    sh.rdb[r] = db;
  }
  __syncthreads();
}

// recoupling groups of <= kRecoupleDirect sources: all of an element's source loads are in flight at
// once from registers, then y_j = alpha sum_i M[i][j] x_i for every destination j
template <int CM>
__device__ void recouple_direct(const typename CIO<CM>::S* __restrict__ src, typename CIO<CM>::D* __restrict__ dst,
                                const PermGroup& g, const PermJob& job, const PermShared& sh, double alpha,
                                double beta, double ims) {
  using IO = CIO<CM>;
  using V = typename IO::V;
  const int ks = g.ksrc, kd = g.kdst, n0 = g.ext[0];
  const uint32_t E = (uint32_t)job.count * (uint32_t)n0;
  FastDiv fn0;
  fn0.init((uint32_t)n0);
  for (uint32_t e = threadIdx.x; e < E; e += kPermThreads) {
    const uint32_t r = fn0.div(e), i0 = e - r * (uint32_t)n0;
    V x[kRecoupleDirect];
#pragma unroll
    for (int i = 0; i < kRecoupleDirect; ++i)
      if (i < ks) {
        const int64_t ld = sh.mld[i];
        x[i] = IO::load(src, sh.moff[i] + sh.rsa[r] + ld * sh.rsb[r] + (int64_t)i0 * (g.sa[0] + ld * g.sb[0]),
                        sh.md1[i]);
      }
    for (int j = 0; j < kd; ++j) {
      V acc = Num<V>::zero();
#pragma unroll
      for (int i = 0; i < kRecoupleDirect; ++i)
        if (i < ks) acc = Num<V>::axpy(sh.coef[i * kd + j], x[i], acc);
      const int jm = kMaxGroupMembers + j;
      const int64_t ld = sh.mld[jm];
      IO::store(dst, sh.moff[jm] + sh.rda[r] + ld * sh.rdb[r] + (int64_t)i0 * (g.da[0] + ld * g.db[0]), sh.md1[jm],
                sh.md2[jm], Num<V>::scale(alpha, acc), beta, ims);
    }
  }
}

// One launch covers every abelian-style job of up to two permutes (A~ and B~ of a contraction, op 0/1):
// rows, smem-tiled and packed jobs share the grid, so small latency-bound permutes do not serialise
// over several launches. <= 64 registers so that 4 CTAs (32 warps) share an SM.
union PermSharedAll {
  PermShared p;
  PackShared k;
  int64_t seg[kSegWords];
};

// ROWS_ONLY: a launch whose jobs are all rows jobs (the large cfg4 permutes) uses a leaner instance
// (48 registers instead of 64; measured 5.0 vs 4.6 TB/s on cfg4).
template <int CM, bool ROWS_ONLY>
__global__ void __launch_bounds__(kPermThreads, ROWS_ONLY ? (CM == kPermReal ? TK_ROWS_MINB : TK_ROWS_MINB_C) : TK_PERM_MINB)
    permute_kernel(PermOp op0, PermOp op1, const PermJob* __restrict__ jobs) {
  using IO = CIO<CM>;
  __shared__ __align__(16) typename std::conditional<ROWS_ONLY, PermShared, PermSharedAll>::type sh_;
  PermShared& sh = *reinterpret_cast<PermShared*>(&sh_);
  extern __shared__ __align__(16) unsigned char perm_dyn[];
  pdl_trigger();
  const PermJob job = jobs[blockIdx.x];
  const PermOp& op = (ROWS_ONLY || !job.op) ? op0 : op1;  // rows-only launches carry a single permute
  const auto* src = (const typename IO::S*)op.src;
  auto* dst = (typename IO::D*)op.dst;
  if constexpr (!ROWS_ONLY) {
    if (job.type == kJobSeg) {
      permute_seg<CM>(src, dst, op.blob, job, reinterpret_cast<int64_t*>(&sh_), op.alpha, op.beta, op.ims);
      return;
    }
    if (job.type == kJobPacked) {
      permute_packed<CM>(src, dst, op.groups, op.members, op.coefs, job, *reinterpret_cast<PackShared*>(&sh_),
                         op.alpha, op.beta, op.ims);
      return;
    }
  }
  const PermGroup& g = op.groups[job.group];
  load_job_header(g, op.members, op.coefs, sh);
  if constexpr (!ROWS_ONLY) {
    if (job.type == kJobMulti) {  // a recoupling group of <= kRecoupleDirect sources (host-routed)
      recouple_row_tables(g, job, sh);
      pdl_wait();
      recouple_direct<CM>(src, dst, g, job, sh, op.alpha, op.beta, op.ims);
      return;
    }
  }
  if (!ROWS_ONLY && job.type == kJobTiled)
    permute_tiled<CM>(src, dst, g, job, sh, reinterpret_cast<typename IO::V*>(perm_dyn), op.alpha, op.beta, op.ims);
  else
    permute_rows<CM>(src, dst, g, job, sh, op.alpha, op.beta, op.ims);
}

// rows jobs of recoupling groups (SU(2): k_src x k_dst coefficient matrix in flight). The job's source
// elements of all k_src members are staged in shared memory with cp.async -- one round trip for the
// whole job instead of a chain of dependent loads per element (the sum over sources used to wait on
// each load in turn) -- then y_j = alpha sum_i M[i][j] x_i is formed from shared memory and stored.
// Jobs larger than the stage are walked in chunks.
template <int CM>
__global__ void __launch_bounds__(kPermThreads, 3)
    permute_recouple_kernel(PermOp op0, PermOp op1, const PermJob* __restrict__ jobs) {
  using IO = CIO<CM>;
  using V = typename IO::V;
  __shared__ PermShared sh;
  extern __shared__ __align__(16) unsigned char rc_dyn[];
  V* Xs = reinterpret_cast<V*>(rc_dyn);
  constexpr int kStage = kRecoupleStage * 8 / (int)sizeof(V);
  pdl_trigger();
  const PermJob job = jobs[blockIdx.x];
  const PermOp& op = job.op ? op1 : op0;
  const PermGroup& g = op.groups[job.group];
  load_job_header(g, op.members, op.coefs, sh);
  const auto* src = (const typename IO::S*)op.src;
  auto* dst = (typename IO::D*)op.dst;
  const int tid = threadIdx.x;
  const int cnt = job.count, ks = g.ksrc, kd = g.kdst;
  recouple_row_tables(g, job, sh);
  pdl_wait();
  if (ks <= kRecoupleDirect) {
    recouple_direct<CM>(src, dst, g, job, sh, op.alpha, op.beta, op.ims);
    return;
  }
  const int n0 = g.ext[0];
  const uint32_t E = (uint32_t)cnt * (uint32_t)n0;
  const uint32_t chunk = (uint32_t)(kStage / ks);
  FastDiv fn0;
  fn0.init((uint32_t)n0);
  for (uint32_t e0 = 0; e0 < E; e0 += chunk) {
    const uint32_t ec = min(chunk, E - e0);
    FastDiv fc;
    fc.init(ec);
    // stage: Xs[i * ec + e] = source member i, element e0 + e
    for (uint32_t idx = tid; idx < (uint32_t)ks * ec; idx += kPermThreads) {
      const uint32_t i = fc.div(idx), e = e0 + (idx - i * ec);
      const uint32_t r = fn0.div(e), i0 = e - r * (uint32_t)n0;
      const int64_t ld = sh.mld[i];
      stage_elem<CM>(Xs + idx, src + sh.moff[i] + sh.rsa[r] + ld * sh.rsb[r] + (int64_t)i0 * (g.sa[0] + ld * g.sb[0]),
                     sh.md1[i]);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (uint32_t e = tid; e < ec; e += kPermThreads) {
      const uint32_t ee = e0 + e, r = fn0.div(ee), i0 = ee - r * (uint32_t)n0;
      for (int j0 = 0; j0 < kd; j0 += kRegMembers) {
        V acc[kRegMembers];
#pragma unroll
        for (int jj = 0; jj < kRegMembers; ++jj) acc[jj] = Num<V>::zero();
        for (int i = 0; i < ks; ++i) {
          const V x = Xs[i * ec + e];
          const double* cr = sh.coef + i * kd + j0;
#pragma unroll
          for (int jj = 0; jj < kRegMembers; ++jj)
            if (j0 + jj < kd) acc[jj] = Num<V>::axpy(cr[jj], x, acc[jj]);
        }
#pragma unroll
        for (int jj = 0; jj < kRegMembers; ++jj)
          if (j0 + jj < kd) {
            const int jm = kMaxGroupMembers + j0 + jj;
            const int64_t ld = sh.mld[jm];
            IO::store(dst, sh.moff[jm] + sh.rda[r] + ld * sh.rdb[r] + (int64_t)i0 * (g.da[0] + ld * g.db[0]),
                      sh.md1[jm], sh.md2[jm], Num<V>::scale(op.alpha, acc[jj]), op.beta, op.ims);
          }
      }
    }
    __syncthreads();  // the stage is refilled by the next chunk
  }
}

template <int CM>
static cudaError_t set_permute_attrs() {
  cudaError_t e = cudaFuncSetAttribute(permute_kernel<CM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kTileElems * (int)sizeof(typename CIO<CM>::V));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(permute_recouple_kernel<CM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kRecoupleStage * 8);
  return e;
}

template <int CM>
static cudaError_t launch_permute_cm(PermOp op0, PermOp op1, const PermJob* jobs, int njobs, int njobs_multi,
                                     bool tiled, int variant, cudaStream_t st) {
  const int smem = tiled ? kTileElems * (int)sizeof(typename CIO<CM>::V) : 0;
  cudaError_t e = cudaSuccess;
  if (njobs && variant == kLaunchRowsOnly)
    e = launch_k(permute_kernel<CM, true>, njobs, kPermThreads, 0, st, op0, op1, jobs);
  if (e == cudaSuccess && njobs && variant == kLaunchGeneral)
    e = launch_k(permute_kernel<CM, false>, njobs, kPermThreads, smem, st, op0, op1, jobs);
  if (e == cudaSuccess && njobs_multi)
    e = launch_k(permute_recouple_kernel<CM>, njobs_multi, kPermThreads, kRecoupleStage * 8, st, op0, op1,
                 jobs + njobs);
  return e;
}

cudaError_t launch_permute(const PermOp& op0, const PermOp& op1, const PermJob* jobs, int njobs, int njobs_multi,
                           bool tiled, int variant, int cm, cudaStream_t st) {
  switch (cm) {
    case kPermReal: return launch_permute_cm<kPermReal>(op0, op1, jobs, njobs, njobs_multi, tiled, variant, st);
    case kPermCToC: return launch_permute_cm<kPermCToC>(op0, op1, jobs, njobs, njobs_multi, tiled, variant, st);
    case kPermCToPlanar:
      return launch_permute_cm<kPermCToPlanar>(op0, op1, jobs, njobs, njobs_multi, tiled, variant, st);
    case kPermCToRealRep:
      return launch_permute_cm<kPermCToRealRep>(op0, op1, jobs, njobs, njobs_multi, tiled, variant, st);
    case kPermPlanarToC:
      return launch_permute_cm<kPermPlanarToC>(op0, op1, jobs, njobs, njobs_multi, tiled, variant, st);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- grouped FP64 GEMM (DMMA)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}


// Shared-memory pitches: As[k][m] with pitch BM+4 and Bs[n][k] with pitch BK+4 (both = 4 mod 16
// doubles) make the m8n8k4 fragment loads conflict-free in each 16-lane phase of a 64-bit LDS.
template <int BM, int BN, int WM, int WN, int BK, int STAGES>
struct GemmCfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int MF = WM / 8, NF = WN / 8;
  static constexpr int LDA_S = BM + 4;
  static constexpr int LDB_S = BK + 4;
  static constexpr int A_STAGE = BK * LDA_S, B_STAGE = BN * LDB_S;
  static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
};

#ifndef TK_WARP_LATIN
#define TK_WARP_LATIN 1
#endif
// Warp -> sub-tile (wm, wn) of a WARPS_M x WARPS_N warp grid. A warp runs on SM sub-partition warp & 3, each
// with its own DMMA pipe; the fragment guards skip 8-row / 8-column fragments outside the block, so the
// skipped work should come off all four pipes evenly. 4 x 4 grids (128 x 128 tiles): a Latin square, every
// sub-partition holds one warp of each row band and one of each column band. 2 x 4 grids (64 x 64 tiles):
// both row bands on every sub-partition (warps w and w + 4 share one), so an edge tile with <= 32 rows
// keeps four pipes busy; with wm = warp % WARPS_M it idled sub-partitions 1 and 3.
template <int WARPS_M, int WARPS_N>
__device__ __forceinline__ void warp_subtile(int warp, int& wm, int& wn) {
  wm = warp % WARPS_M, wn = warp / WARPS_M;
#if TK_WARP_LATIN
  if constexpr (WARPS_M == 4 && WARPS_N == 4) {
    wm = warp >> 2, wn = ((warp & 3) + wm) & 3;
  } else if constexpr (WARPS_M == 2 && WARPS_N == 4) {
    wm = (warp + (warp >> 2)) & 1, wn = ((warp & 3) >> 1) + 2 * (warp >> 2);
  }
#endif
}

// k range [kb, ke) (split-K: ke - kb < K); part != nullptr: write the raw partial tile (BM x BN,
// column-major) for the split-K reduction instead of alpha * acc + beta * C.
template <int BM, int BN, int WM, int WN, int BK, int STAGES>
__device__ __forceinline__ void gemm_tile(const double* __restrict__ A, const double* __restrict__ B,
                                          double* __restrict__ C, const GemmGroup& g, int m0, int n0, double alpha,
                                          double beta, bool vec, double* smem, int kb, int ke,
                                          double* __restrict__ part) {
  using Cfg = GemmCfg<BM, BN, WM, WN, BK, STAGES>;
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int wm, wn;
  warp_subtile<Cfg::WARPS_M, Cfg::WARPS_N>(warp, wm, wn);
  const int gq = lane >> 2, tq = lane & 3;
  const double* Ag = A + g.a_off;
  const double* Bg = B + g.b_off;
  const int M = g.M, N = g.N, K = ke;
  const int nk = (ke - kb + BK - 1) / BK;

  double acc[Cfg::MF][Cfg::NF][2];
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Per-thread load geometry, hoisted out of the k loop: a thread copies the same (row, k-offset) pattern
  // of every stage, so its global pointers advance by a constant per k-step and only the k < K test
  // changes. (The straightforward per-element index -> (m, k) -> address form was ~140 of the ~300
  // instructions a warp issued per k-step, and these kernels are issue-bound: ncu, cfg3 T3.R.)
  constexpr int T = Cfg::THREADS;
  static_assert(T % BM == 0 && T % BK == 0 && T % (BM / 2) == 0 && T % (BK / 2) == 0, "load geometry");
  static_assert((BM * BK) % T == 0 && (BN * BK) % T == 0 && (BM / 2 * BK) % T == 0 && (BK / 2 * BN) % T == 0,
                "load geometry");
  // element (am, akq + i * AKS) of A's stage; element (bkk, bnq + i * BNS) of B's stage
  const int ev = vec ? 2 : 1;  // elements per copy (constant divisors below: shifts)
  const int am = vec ? 2 * (tid % (BM / 2)) : tid % BM, akq = vec ? tid / (BM / 2) : tid / BM;
  const int bkk = vec ? 2 * (tid % (BK / 2)) : tid % BK, bnq = vec ? tid / (BK / 2) : tid / BK;
  const int AKS = vec ? T / (BM / 2) : T / BM, BNS = vec ? T / (BK / 2) : T / BK;
  // bytes of a copy that lie inside the block along the contiguous dimension (A: rows; B: k, per stage)
  const int abytes = m0 + am + ev <= M ? 8 * ev : (m0 + am < M ? 8 : 0);
  const double* pa0 = Ag + (m0 + am) + (int64_t)(kb + akq) * g.lda;
  const double* pb0 = Bg + (kb + bkk) + (int64_t)(n0 + bnq) * g.ldb;
  const int64_t astep = (int64_t)AKS * g.lda, bstep = (int64_t)BNS * g.ldb;
  const int sa0 = akq * Cfg::LDA_S + am, sb0 = bnq * Cfg::LDB_S + bkk;
  // stages are loaded in k order, one call per k-step: the pointers and the k origin run along
  const double* pa = pa0;
  const double* pb = pb0;
  const int64_t akstep = (int64_t)BK * g.lda;
  int k0 = kb - BK;
  auto load_stage = [&](int s) {
    k0 += BK;
    double* as = As + s * Cfg::A_STAGE + sa0;
    double* bs = Bs + s * Cfg::B_STAGE + sb0;
    const int kbytes = k0 + bkk + ev <= K ? 8 * ev : (k0 + bkk < K ? 8 : 0);
    if (vec) {
#pragma unroll
      for (int i = 0; i < (BM / 2 * BK) / T; ++i) {
        const int nb = k0 + akq + i * AKS < K ? abytes : 0;
        cp_async16(as + i * AKS * Cfg::LDA_S, nb ? pa + i * astep : A, nb);
      }
#pragma unroll
      for (int i = 0; i < (BK / 2 * BN) / T; ++i) {
        const int nb = n0 + bnq + i * BNS < N ? kbytes : 0;
        cp_async16(bs + i * BNS * Cfg::LDB_S, nb ? pb + i * bstep : B, nb);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (BM * BK) / T; ++i) {
        const bool ok = abytes != 0 && k0 + akq + i * AKS < K;
        cp_async8(as + i * AKS * Cfg::LDA_S, ok ? pa + i * astep : A, ok);
      }
#pragma unroll
      for (int i = 0; i < (BN * BK) / T; ++i) {
        const bool ok = kbytes != 0 && n0 + bnq + i * BNS < N;
        cp_async8(bs + i * BNS * Cfg::LDB_S, ok ? pb + i * bstep : B, ok);
      }
    }
    pa += akstep;
    pb += BK;
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s);
    cp_async_commit();
  }
  // warp-uniform: the warp's WM x WN sub-tile lies inside the block (8-row / 8-column fragment units)
  const bool interior = m0 + wm * WM + (Cfg::MF - 1) * 8 < M && n0 + wn * WN + (Cfg::NF - 1) * 8 < N;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt % STAGES);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * Cfg::A_STAGE + wm * WM + gq;
    const double* bs = Bs + (kt % STAGES) * Cfg::B_STAGE + (wn * WN + gq) * Cfg::LDB_S + tq;
    // padding is never multiplied: k-steps past K, and 8-row / 8-column fragments outside the block
    // (warp-uniform guards; small sectors are mostly padding in 64 x 64 tiles)
    const int kend = min(BK, K - (kb + kt * BK));
    if (interior && kend == BK) {  // all of this warp's fragments inside the block, a full k-step: no guards
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double af[Cfg::MF], bf[Cfg::NF];
#pragma unroll
        for (int i = 0; i < Cfg::MF; ++i) af[i] = as[(kk + tq) * Cfg::LDA_S + i * 8];
#pragma unroll
        for (int j = 0; j < Cfg::NF; ++j) bf[j] = bs[j * 8 * Cfg::LDB_S + kk];
#pragma unroll
        for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::NF; ++j) dmma884(acc[i][j], af[i], bf[j]);
      }
      continue;
    }
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if (kk >= kend) break;
      double af[Cfg::MF], bf[Cfg::NF];
#pragma unroll
      for (int i = 0; i < Cfg::MF; ++i) af[i] = as[(kk + tq) * Cfg::LDA_S + i * 8];
#pragma unroll
      for (int j = 0; j < Cfg::NF; ++j) bf[j] = bs[j * 8 * Cfg::LDB_S + kk];
#pragma unroll
      for (int i = 0; i < Cfg::MF; ++i) {
        if (m0 + wm * WM + i * 8 >= M) break;
#pragma unroll
        for (int j = 0; j < Cfg::NF; ++j) {
          if (n0 + wn * WN + j * 8 >= N) break;
          dmma884(acc[i][j], af[i], bf[j]);
        }
      }
    }
  }
  cp_async_wait<0>();
  if (part) {  // split-K partial: raw accumulators, the reduction applies alpha / beta
#pragma unroll
    for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::NF; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int ml = wm * WM + i * 8 + gq, nl = wn * WN + j * 8 + 2 * tq + c;
          part[ml + nl * BM] = acc[i][j][c];
        }
    return;
  }
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

// ---- mbarrier-pipelined variant: no CTA-wide barrier in the main loop. Every thread issues its
// share of a stage's cp.async copies and signals them with cp.async.mbarrier.arrive.noinc on the
// stage's "full" barrier; each warp waits only for the data it needs and releases the stage on an
// "empty" barrier, so warps may drift up to STAGES-PD-1 stages apart without idling the DMMA pipe.
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(smem_u32(bar)));
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES, int PD>
__device__ __forceinline__ void gemm_tile_mbar(const double* __restrict__ A, const double* __restrict__ B,
                                               double* __restrict__ C, const GemmGroup& g, int m0, int n0,
                                               double alpha, double beta, bool vec, double* smem) {
  using Cfg = GemmCfg<BM, BN, WM, WN, BK, STAGES>;
  static_assert(PD >= 1 && PD <= STAGES - 1, "prefetch distance");
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * Cfg::B_STAGE);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int wm, wn;
  warp_subtile<Cfg::WARPS_M, Cfg::WARPS_N>(warp, wm, wn);
  const int gq = lane >> 2, tq = lane & 3;
  const double* Ag = A + g.a_off;
  const double* Bg = B + g.b_off;
  const int M = g.M, N = g.N, K = g.K;
  const int nk = (K + BK - 1) / BK;
  if (tid < STAGES) {
    mbar_init(&full[tid], Cfg::THREADS);
    mbar_init(&empty[tid], Cfg::THREADS / 32);
  }
  __syncthreads();

  double acc[Cfg::MF][Cfg::NF][2];
#pragma unroll
  for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int kt, int s) {
    const int k0 = kt * BK;
    double* as = As + s * Cfg::A_STAGE;
    double* bs = Bs + s * Cfg::B_STAGE;
    if (vec) {
#pragma unroll
      for (int i = 0; i < (BM / 2 * BK) / Cfg::THREADS; ++i) {
        int idx = tid + i * Cfg::THREADS;
        int m = 2 * (idx % (BM / 2)), k = idx / (BM / 2);
        int gm = m0 + m, gk = k0 + k;
        int nb = (gm < M && gk < K) ? (gm + 1 < M ? 16 : 8) : 0;
        const double* gp = nb ? Ag + (int64_t)gm + (int64_t)gk * g.lda : A;
        cp_async16(as + k * Cfg::LDA_S + m, gp, nb);
      }
#pragma unroll
      for (int i = 0; i < (BK / 2 * BN) / Cfg::THREADS; ++i) {
        int idx = tid + i * Cfg::THREADS;
        int k = 2 * (idx % (BK / 2)), n = idx / (BK / 2);
        int gk = k0 + k, gn = n0 + n;
        int nb = (gn < N && gk < K) ? (gk + 1 < K ? 16 : 8) : 0;
        const double* gp = nb ? Bg + (int64_t)gk + (int64_t)gn * g.ldb : B;
        cp_async16(bs + n * Cfg::LDB_S + k, gp, nb);
      }
    } else {
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
    }
    cp_async_mbar_arrive(&full[s]);
  };

  for (int s = 0; s < PD && s < nk; ++s) load_stage(s, s);
  for (int kt = 0; kt < nk; ++kt) {
    const int nxt = kt + PD;
    if (nxt < nk) {
      const int s2 = nxt % STAGES;
      if (nxt >= STAGES) mbar_wait(&empty[s2], (uint32_t)(((nxt - STAGES) / STAGES) & 1));
      load_stage(nxt, s2);
    }
    const int s = kt % STAGES;
    mbar_wait(&full[s], (uint32_t)((kt / STAGES) & 1));
    const double* as = As + s * Cfg::A_STAGE + wm * WM + gq;
    const double* bs = Bs + s * Cfg::B_STAGE + (wn * WN + gq) * Cfg::LDB_S + tq;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::MF], bf[Cfg::NF];
#pragma unroll
      for (int i = 0; i < Cfg::MF; ++i) af[i] = as[(kk + tq) * Cfg::LDA_S + i * 8];
#pragma unroll
      for (int j = 0; j < Cfg::NF; ++j) bf[j] = bs[j * 8 * Cfg::LDB_S + kk];
#pragma unroll
      for (int i = 0; i < Cfg::MF; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::NF; ++j) dmma884(acc[i][j], af[i], bf[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
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

#ifndef TK_MBAR_BK
#define TK_MBAR_BK 16
#endif
#ifndef TK_MBAR_STAGES
#define TK_MBAR_STAGES 6
#endif
#define TK_MBAR 128, 128, 32, 32, TK_MBAR_BK, TK_MBAR_STAGES
#ifndef TK_MBAR_PD
#define TK_MBAR_PD 2  // prefetch distance (k-steps) of the big-tile GEMM's stage ring
#endif
using MbarCfg = GemmCfg<TK_MBAR>;
constexpr size_t kMbarSmem = MbarCfg::SMEM + 2 * 6 * sizeof(uint64_t);

template <int PD>
__global__ void __launch_bounds__(MbarCfg::THREADS, 1)
    gemm_mbar_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                     const GemmGroup* __restrict__ groups, const GemmTile* __restrict__ tiles, double alpha,
                     double beta, int base_vec) {
  extern __shared__ __align__(16) double smem[];
  pdl_trigger();
  const GemmTile t = tiles[blockIdx.x];
  const GemmGroup& g = t.g;
  pdl_wait();
  gemm_tile_mbar<TK_MBAR, PD>(A, B, C, g, t.m0, t.n0, alpha, beta, base_vec && g.vec, smem);
}

// ---- skinny blocks (N, K <= kSkinnyMax; the MPO steps T.W of the DMRG chains, M up to 2e5): a
// streaming kernel, HBM-bound (AI = 2KN / 8(K+N) < 1 flop/B), so plain FMAs: the K x N operand sits in
// shared memory, each thread owns rows of A~ / C~, loads A~[m, 0..K) (coalesced across the warp for
// every k) and writes C~[m, 0..N). One CTA covers kSkinnyRows consecutive rows of one group.
constexpr int kSkinnyThreads = 256;
template <int KM, int NM>
__device__ __forceinline__ void skinny_rows(const double* __restrict__ Ag, double* __restrict__ Cg, const double* Bs,
                                            const GemmGroup& g, int m0, int mend, double beta) {
  // RW rows per thread per iteration: 16 A~ loads in flight per thread, each B value read once per k, n
  constexpr int RW = 16 / (KM > NM ? KM : NM);
  const int K = g.K, N = g.N;
  for (int mb = m0 + threadIdx.x; mb < mend; mb += RW * kSkinnyThreads) {
    double a[RW][KM], acc[RW][NM];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const int m = mb + r * kSkinnyThreads;
#pragma unroll
      for (int k = 0; k < KM; ++k) a[r][k] = (k < K && m < mend) ? __ldg(Ag + m + (int64_t)k * g.lda) : 0.0;
#pragma unroll
      for (int n = 0; n < NM; ++n) acc[r][n] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < KM; ++k)
#pragma unroll
      for (int n = 0; n < NM; ++n) {
        const double b = Bs[k * kSkinnyMax + n];
#pragma unroll
        for (int r = 0; r < RW; ++r) acc[r][n] = fma(a[r][k], b, acc[r][n]);
      }
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const int m = mb + r * kSkinnyThreads;
      if (m < mend) {
#pragma unroll
        for (int n = 0; n < NM; ++n)
          if (n < N) {
            double* cp = Cg + m + (int64_t)n * g.ldc;
            *cp = beta != 0.0 ? fma(beta, *cp, acc[r][n]) : acc[r][n];
          }
      }
    }
  }
}

// one skinny tile (t.pad rows of one group), Bs = kSkinnyMax^2 doubles of shared memory
__device__ __forceinline__ void skinny_tile(const double* __restrict__ A, const double* __restrict__ B,
                                            double* __restrict__ C, const GemmTile& t, double alpha, double beta,
                                            double* Bs) {
  const GemmGroup& g = t.g;
  const int K = g.K, N = g.N;
  for (int i = threadIdx.x; i < kSkinnyMax * kSkinnyMax; i += kSkinnyThreads) {
    const int k = i / kSkinnyMax, n = i % kSkinnyMax;
    Bs[i] = (k < K && n < N) ? alpha * B[g.b_off + k + (int64_t)n * g.ldb] : 0.0;
  }
  __syncthreads();
  const double* Ag = A + g.a_off;
  double* Cg = C + g.c_off;
  const int mend = min(g.M, t.m0 + t.pad);
  // unrolled FMA blocks sized to the group (the FP64 FMA rate must stay above the HBM rate)
  const int kc = K <= 4 ? 0 : (K <= 8 ? 1 : 2), nc = N <= 4 ? 0 : (N <= 8 ? 1 : 2);
  switch (kc * 3 + nc) {
    case 0: skinny_rows<4, 4>(Ag, Cg, Bs, g, t.m0, mend, beta); break;
    case 1: skinny_rows<4, 8>(Ag, Cg, Bs, g, t.m0, mend, beta); break;
    case 2: skinny_rows<4, 16>(Ag, Cg, Bs, g, t.m0, mend, beta); break;
    case 3: skinny_rows<8, 4>(Ag, Cg, Bs, g, t.m0, mend, beta); break;
    case 4: skinny_rows<8, 8>(Ag, Cg, Bs, g, t.m0, mend, beta); break;
    case 5: skinny_rows<8, 16>(Ag, Cg, Bs, g, t.m0, mend, beta); break;
    case 6: skinny_rows<16, 4>(Ag, Cg, Bs, g, t.m0, mend, beta); break;
    case 7: skinny_rows<16, 8>(Ag, Cg, Bs, g, t.m0, mend, beta); break;
    default: skinny_rows<16, 16>(Ag, Cg, Bs, g, t.m0, mend, beta); break;
  }
}

#ifndef TK_SMALL_STAGES
#define TK_SMALL_STAGES 3
#endif
#ifndef TK_SMALL_WN
#define TK_SMALL_WN 16  // warp tile 32 x WN (16: 8 warps per 64 x 64 tile)
#endif
#ifndef TK_SMALL_BK
#define TK_SMALL_BK 16
#endif
#define TK_SMALL 64, 64, 32, TK_SMALL_WN, TK_SMALL_BK, TK_SMALL_STAGES
#ifndef TK_SMALL_MINB
#define TK_SMALL_MINB 2
#endif
using SmallCfg = GemmCfg<TK_SMALL>;

__global__ void __launch_bounds__(SmallCfg::THREADS, TK_SMALL_MINB)
    gemm_small_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                      const GemmGroup* __restrict__ groups, const GemmTile* __restrict__ tiles, double alpha,
                      double beta, int base_vec, double* __restrict__ parts) {
  extern __shared__ __align__(16) double smem[];
  pdl_trigger();
  const GemmTile t = tiles[blockIdx.x];
  const GemmGroup& g = t.g;
  pdl_wait();
  if (t.tmap < 0) {  // a skinny tile riding in the small-tile launch (one launch fewer per contraction)
    skinny_tile(A, B, C, t, alpha, beta, smem);
    return;
  }
  double* part = t.slot >= 0 ? parts + (int64_t)t.slot * (64 * 64) : nullptr;
  gemm_tile<TK_SMALL>(A, B, C, g, t.m0, t.n0, alpha, beta, base_vec && g.vec, smem, t.k0, t.k1, part);
}

// split-K reduction of 64 x 64 tiles: C = alpha * sum_s partial_s + beta * C, summed in slot order
// (deterministic). gridDim.y = 4 quarters of a tile, one element per thread; all partial loads of an
// element are issued before the (ordered) sum, so the kernel costs about one L2 round trip.
constexpr int kSplitMax = 16;
__global__ void __launch_bounds__(256)
    gemm_splitk_reduce_kernel(double* __restrict__ C, const GemmGroup* __restrict__ groups,
                              const GemmTile* __restrict__ heads, const double* __restrict__ parts, double alpha,
                              double beta) {
  pdl_trigger();
  const GemmTile t = heads[blockIdx.x];
  const GemmGroup& g = t.g;
  pdl_wait();
  double* Cg = C + g.c_off;
  for (int e = blockIdx.y * 1024 + threadIdx.x; e < (blockIdx.y + 1) * 1024; e += 256) {
    const int ml = e % 64, nl = e / 64;
    const int m = t.m0 + ml, n = t.n0 + nl;
    if (m >= g.M || n >= g.N) continue;
    double x[kSplitMax];
#pragma unroll
    for (int sidx = 0; sidx < kSplitMax; ++sidx)
      x[sidx] = sidx < t.nsplit ? parts[(int64_t)(t.slot + sidx) * (64 * 64) + e] : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int sidx = 0; sidx < kSplitMax; ++sidx) acc += x[sidx];
    double* p = Cg + (int64_t)m + (int64_t)n * g.ldc;
    double v = alpha * acc;
    if (beta != 0.0) v = fma(beta, *p, v);
    *p = v;
  }
}

#ifdef TK_SKINNY_MINB  // A/B knob; the default leaves the register choice to ptxas (82 registers)
__global__ void __launch_bounds__(kSkinnyThreads, TK_SKINNY_MINB)
#else
__global__ void __launch_bounds__(kSkinnyThreads)
#endif
    gemm_skinny_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                       const GemmGroup* __restrict__ groups, const GemmTile* __restrict__ tiles, double alpha,
                       double beta) {
  __shared__ double Bs[kSkinnyMax * kSkinnyMax];
  pdl_trigger();
  const GemmTile t = tiles[blockIdx.x];
  pdl_wait();
  skinny_tile(A, B, C, t, alpha, beta, Bs);
}

// ---- gathered skinny GEMM (GatherSeg in tk_kernels.hpp): one thread per row (two for K <= 8) of
// A~^c. The tile's slot -- descriptor, subblock segments, B~ table -- is copied into shared memory
// before griddepcontrol.wait (plan data); each thread then issues its rows' K element loads from A with
// cp.async into As[k][row] (all in flight at once, no registers held) and the K x N block of B~ is
// gathered from B through the table; after one wait every thread computes its C~ rows.
#ifndef TK_GATHER_MINB
#define TK_GATHER_MINB 3
#endif
template <int KM, int NM>
__global__ void __launch_bounds__(kGatherRows, TK_GATHER_MINB)
    gather_skinny_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                         const int64_t* __restrict__ slots, const GatherSeg* __restrict__ segs,
                         const int32_t* __restrict__ btab, const GatherOut* __restrict__ gouts, double alpha,
                         double oalpha, double beta) {
  constexpr int RPT = gather_rows(KM) / kGatherRows;  // rows per thread
  __shared__ double Bs[kSkinnyMax * kSkinnyMax];
  extern __shared__ __align__(16) double gather_dyn[];
  double (*As)[gather_rows(KM)] = reinterpret_cast<double (*)[gather_rows(KM)]>(gather_dyn);  // [KM][rows]
  __shared__ __align__(16) GatherSeg sbig[gather_seg_cap(KM)];
  __shared__ __align__(16) int64_t slot[kGatherSlotWords];
  pdl_trigger();
  const int tid = threadIdx.x;
  {  // the tile's slot: descriptor, first segments, first B~ table entries -- one coalesced copy
    const int4* src4 = reinterpret_cast<const int4*>(slots + (int64_t)blockIdx.x * kGatherSlotWords);
    for (int i = tid; i < kGatherSlotWords / 2; i += kGatherRows) reinterpret_cast<int4*>(slot)[i] = __ldg(src4 + i);
  }
  for (int i = tid; i < kSkinnyMax * kSkinnyMax; i += kGatherRows) Bs[i] = 0.0;
  __syncthreads();
  const GatherTile& t = *reinterpret_cast<const GatherTile*>(slot);
  const GemmGroup& g = t.g;
  const GatherSeg* ss = reinterpret_cast<const GatherSeg*>(slot + 10);
  if (t.nseg > kGatherSlotSegs) {  // rare: more segments than the slot holds
    const int4* src4 = reinterpret_cast<const int4*>(segs + t.seg0);
    int4* dst4 = reinterpret_cast<int4*>(sbig);
    for (int i = tid; i < t.nseg * (int)(sizeof(GatherSeg) / 16); i += kGatherRows) dst4[i] = __ldg(src4 + i);
    __syncthreads();
    ss = sbig;
  }
  const int K = g.K, N = g.N;
  const int32_t* sbt = reinterpret_cast<const int32_t*>(slot + 10 + 16 * kGatherSlotSegs);
  const int be = tid < K * N ? (K * N <= kGatherSlotB ? sbt[tid] : __ldg(btab + t.bt + tid)) : -1;
  pdl_wait();
  // A~ rows first (cp.async, nothing held in registers), then the B~ block, then one wait for both
  uint32_t neg[RPT];
  int rlo[RPT];          // the row's first segment (its row tree): the output map's index
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    neg[j] = 0;
    rlo[j] = 0;
    const int lr = tid + j * kGatherRows;
    if (lr >= t.nrows) continue;
    const int m = t.m0 + lr;
    // this row's row tree: the last segment with r0 <= m (segments sorted by (r0, k0)); its column
    // subblocks are the run of segments sharing that r0
    int lo = 0, hi = t.nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ss[mid].r0 <= m) lo = mid; else hi = mid - 1;
    }
    const int r0 = ss[lo].r0;
    while (lo > 0 && ss[lo - 1].r0 == r0) --lo;
    rlo[j] = lo;
    // the row's mixed-radix digits over the row legs are the same for every column subblock of the row
    // tree unless a subblock merged its legs differently: decode once, re-decode only when (nrl, ext)
    // changes (the decode -- integer divisions -- dominated the kernel's instruction count)
    int cnrl = -1;
    int cext[4] = {0, 0, 0, 0};
    uint32_t dig[4] = {0, 0, 0, 0};
    for (int s = lo; s < t.nseg && ss[s].r0 == r0; ++s) {
      const GatherSeg& q = ss[s];
      const int nrl = q.nrl;
      bool same = nrl == cnrl;
#pragma unroll
      for (int l = 0; l < 4; ++l) same = same && (l >= nrl || q.ext[l] == cext[l]);
      if (!same) {
        uint32_t r = (uint32_t)(m - q.r0);
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          if (l < nrl) {
            const uint32_t e = (uint32_t)q.ext[l], qq = r / e;
            dig[l] = r - qq * e;
            cext[l] = (int)e;
            r = qq;
          }
        }
        cnrl = nrl;
      }
      int rs = 0;
#pragma unroll
      for (int l = 0; l < 4; ++l)
        if (l < nrl) rs += (int)dig[l] * q.str[l];
      const double* a = A + q.src + rs;
      for (int kk = 0; kk < q.nk; ++kk) cp_async8(&As[q.k0 + kk][lr], a + q.colsrc[kk], true);
      if (q.neg) neg[j] |= ((1u << q.nk) - 1u) << q.k0;
    }
  }
  cp_async_commit();
  if (be >= 0) {
    const double x = alpha * __ldg(B + (be >> 1));
    Bs[(tid / N) * kSkinnyMax + tid % N] = (be & 1) ? -x : x;
  }
  cp_async_wait<0>();
  __syncthreads();  // Bs (and, formally, every thread's own As columns) visible
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int lr = tid + j * kGatherRows;
    if (lr >= t.nrows) break;
    double acc[NM];
#pragma unroll
    for (int n = 0; n < NM; ++n) acc[n] = 0.0;
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      if (k < K) {
        const double x = As[k][lr];
        const double a = (neg[j] >> k) & 1u ? -x : x;
#pragma unroll
        for (int n = 0; n < NM; ++n) acc[n] = fma(a, Bs[k * kSkinnyMax + n], acc[n]);
      }
    }
    if (t.gout0 < 0) {
      double* Cg = C + g.c_off + t.m0 + lr;
#pragma unroll
      for (int n = 0; n < NM; ++n)
        if (n < N) {
          double* cp = Cg + (int64_t)n * g.ldc;
          *cp = beta != 0.0 ? fma(beta, *cp, acc[n]) : acc[n];
        }
    } else {  // the output permute folded in: C~ element (row, n) -> C[base + digits . str], sign
      const GatherOut* go = gouts + t.gout0 + rlo[j] * N;
      uint32_t r = (uint32_t)(t.m0 + lr - ss[rlo[j]].r0), e0 = (uint32_t)go[0].ext0, e1 = (uint32_t)go[0].ext1;
      const uint32_t d0 = r % e0;
      r /= e0;
      const uint32_t d1 = r % e1, d2 = r / e1;
#pragma unroll
      for (int n = 0; n < NM; ++n)
        if (n < N) {
          const GatherOut o = go[n];
          double* cp = C + o.base + ((int64_t)d0 * o.str[0] + (int64_t)d1 * o.str[1] + (int64_t)d2 * o.str[2]);
          double y = oalpha * acc[n];
          if (o.neg) y = -y;
          *cp = beta != 0.0 ? fma(beta, *cp, y) : y;
        }
    }
  }
}

template <int KM, int NM>
static cudaError_t set_gather_attr() {
  return cudaFuncSetAttribute(gather_skinny_kernel<KM, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              KM * gather_rows(KM) * 8);
}

cudaError_t launch_gather_gemm(const double* A, const double* B, double* C, const int64_t* slots, int ntiles,
                               const GatherSeg* segs, const int32_t* btab, const GatherOut* gouts, int kmax, int nmax,
                               double alpha, double oalpha, double beta, cudaStream_t st) {
  if (!ntiles) return cudaSuccess;
  const int kc = kmax <= 4 ? 0 : (kmax <= 8 ? 1 : 2), nc = nmax <= 4 ? 0 : (nmax <= 8 ? 1 : 2);
#define TK_GATHER(KM, NM)                                                                               \
  return launch_k(gather_skinny_kernel<KM, NM>, ntiles, kGatherRows, KM * gather_rows(KM) * 8, st, A, B, C, \
                  slots, segs, btab, gouts, alpha, oalpha, beta);
  switch (kc * 3 + nc) {
    case 0: TK_GATHER(4, 4)
    case 1: TK_GATHER(4, 8)
    case 2: TK_GATHER(4, 16)
    case 3: TK_GATHER(8, 4)
    case 4: TK_GATHER(8, 8)
    case 5: TK_GATHER(8, 16)
    case 6: TK_GATHER(16, 4)
    case 7: TK_GATHER(16, 8)
    default: TK_GATHER(16, 16)
  }
#undef TK_GATHER
}

cudaError_t launch_gemm(const double* A, const double* B, double* C, const GemmGroup* groups, const GemmTile* tiles,
                        int ntiles_big, int ntiles_small, int ntiles_skinny, const GemmTile* split_heads,
                        int nsplit_heads, double* parts, double alpha, double beta, cudaStream_t st) {
  // big tiles: mbarrier pipeline, 16 warps of 32x32 on 128x128, BK 16, 6 stages, prefetch distance 2
  const int base_vec = ((((uintptr_t)A) | ((uintptr_t)B)) & 15) == 0;
  cudaError_t e = cudaSuccess;
  if (ntiles_big)
    e = launch_k(gemm_mbar_kernel<TK_MBAR_PD>, ntiles_big, MbarCfg::THREADS, kMbarSmem, st, A, B, C, groups, tiles,
                 alpha, beta, base_vec);
  // skinny tiles (GemmTile::tmap == -1) ride in the small-tile launch when there is one: the tile
  // tables are contiguous ([big | small | skinny]) and both use 256-thread CTAs
  if (e == cudaSuccess && ntiles_small)
    e = launch_k(gemm_small_kernel, ntiles_small + ntiles_skinny, SmallCfg::THREADS, SmallCfg::SMEM, st, A, B, C,
                 groups, tiles + ntiles_big, alpha, beta, base_vec, parts);
  if (e == cudaSuccess && nsplit_heads)
    e = launch_k2(gemm_splitk_reduce_kernel, dim3(nsplit_heads, 4), 256, 0, st, C, groups, split_heads,
                  (const double*)parts, alpha, beta);
  if (e == cudaSuccess && ntiles_skinny && !ntiles_small)
    e = launch_k(gemm_skinny_kernel, ntiles_skinny, kSkinnyThreads, 0, st, A, B, C, groups,
                 tiles + ntiles_big + ntiles_small, alpha, beta);
  return e;
}

// ---- FP64 tensor-pipe probe (tk_dmma_probe): back-to-back independent DMMAs, no memory traffic
__global__ void __launch_bounds__(256) dmma_probe_kernel(double* __restrict__ sink, long long iters) {
  const double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (long long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma884(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) sink[0] = s;  // never true; keeps the chain live
}

cudaError_t launch_dmma_probe(int blocks, long long iters, cudaStream_t st) {
  return launch_k(dmma_probe_kernel, blocks, 256, 0, st, (double*)nullptr, iters);
}

// Kernel attributes (opt-in dynamic shared memory) are per device: set once per device, before the
// first launch on it (callers run this ahead of any launch of a tk_* call).
static PerDeviceOnce g_attrs;
cudaError_t ensure_kernel_attrs() {
  return g_attrs.run([] {
    cudaError_t e = set_permute_attrs<kPermReal>();
    if (e == cudaSuccess) e = set_permute_attrs<kPermCToC>();
    if (e == cudaSuccess) e = set_permute_attrs<kPermCToPlanar>();
    if (e == cudaSuccess) e = set_permute_attrs<kPermCToRealRep>();
    if (e == cudaSuccess) e = set_permute_attrs<kPermPlanarToC>();
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_mbar_kernel<TK_MBAR_PD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kMbarSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SmallCfg::SMEM);
    if (e == cudaSuccess) e = set_gather_attr<4, 4>();
    if (e == cudaSuccess) e = set_gather_attr<4, 8>();
    if (e == cudaSuccess) e = set_gather_attr<4, 16>();
    if (e == cudaSuccess) e = set_gather_attr<8, 4>();
    if (e == cudaSuccess) e = set_gather_attr<8, 8>();
    if (e == cudaSuccess) e = set_gather_attr<8, 16>();
    if (e == cudaSuccess) e = set_gather_attr<16, 4>();
    if (e == cudaSuccess) e = set_gather_attr<16, 8>();
    if (e == cudaSuccess) e = set_gather_attr<16, 16>();
    return e;
  });
}

}  // namespace tk
