// Latency microbenchmark (B200): dependent chains of DFMA, DADD, FFMA, SHFL (double), LDS->use,
// MUFU.RSQ64H-based rsqrt(double), bar.sync over N warps, and a 2-CTA cluster st.async + mbarrier ping.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, long long* cyc, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = fma(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 1024;
}
__global__ void k_dadd(double* out, long long* cyc, double a) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = x + a; }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 1024;
}
__global__ void k_ffma(float* out, long long* cyc, float a, float b) {
  float x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = fmaf(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 1024;
}
__global__ void k_shfl(double* out, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x += __shfl_xor_sync(0xffffffffu, x, 1); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 1024;
}
__global__ void k_lds(double* out, long long* cyc) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) % 1024;
  __syncthreads();
  int j = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { j = (int)s[j]; }
  long long t1 = clock64();
  out[threadIdx.x] = j;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 1024;
}
__global__ void k_rsqrt(double* out, long long* cyc, double a) {
  double x = 2.0 + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = rsqrt(x) + a; }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
}
__global__ void k_sqrt(double* out, long long* cyc, double a) {
  double x = 2.0 + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = sqrt(x) + a; }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
}
__global__ void k_rcp(double* out, long long* cyc, double a) {
  double x = 2.0 + threadIdx.x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = __drcp_rn(x) + a; }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
}
__global__ void k_bar(double* out, long long* cyc) {
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { __syncthreads(); }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 1024;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __cluster_dims__(2, 1, 1) k_ping(double* out, long long* cyc, int bytes_per_thread) {
  // every round: each thread pushes `bytes_per_thread/8` doubles to the peer (st.async), then waits on its own mbarrier
  __shared__ __align__(16) double buf[2][1024 * 2];
  __shared__ __align__(8) unsigned long long bar[2];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const uint32_t peer = rank ^ 1;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const int nd = bytes_per_thread / 8;
  const int total = nd * 8 * blockDim.x;
  long long t0 = clock64();
  uint32_t ph = 0;
#pragma unroll 1
  for (int r = 0; r < 256; ++r) {
    const int p = r & 1;
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[p])), "r"(total) : "memory");
    for (int k = 0; k < nd; ++k) {
      uint32_t la = smem_u32(&buf[p][threadIdx.x * 2 + k]), lb = smem_u32(&bar[p]), ra, rb;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(peer));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(peer));
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"((double)r), "r"(rb) : "memory");
    }
    asm volatile("{\n\t.reg .pred q;\n\tW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 q, [%0], %1;\n\t@!q bra W_%=;\n\t}" ::"r"(smem_u32(&bar[p])), "r"((ph >> p) & 1) : "memory");
    ph ^= 1u << p;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) cyc[0] = (t1 - t0) / 256;
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  out[threadIdx.x] = buf[0][threadIdx.x];
}

__device__ __forceinline__ void warp_sum4(double& a, double& b, double& c, double& d) {
  const int lane = threadIdx.x & 31;
  const bool hi16 = lane & 16;
  {
    const double s0 = hi16 ? a : c, s1 = hi16 ? b : d;
    const double r0 = __shfl_xor_sync(0xffffffffu, s0, 16), r1 = __shfl_xor_sync(0xffffffffu, s1, 16);
    if (hi16) { c += r0; d += r1; a = c; b = d; } else { a += r0; b += r1; }
  }
  const bool hi8 = lane & 8;
  {
    const double sx = hi8 ? a : b;
    const double r = __shfl_xor_sync(0xffffffffu, sx, 8);
    a = (hi8 ? b : a) + r;
  }
  a += __shfl_xor_sync(0xffffffffu, a, 4);
  a += __shfl_xor_sync(0xffffffffu, a, 2);
  a += __shfl_xor_sync(0xffffffffu, a, 1);
  const double t0 = __shfl_sync(0xffffffffu, a, 0), t1 = __shfl_sync(0xffffffffu, a, 8);
  const double t2 = __shfl_sync(0xffffffffu, a, 16), t3 = __shfl_sync(0xffffffffu, a, 24);
  a = t0; b = t1; c = t2; d = t3;
}
__device__ __forceinline__ double jacobi_tan(double al, double be, double ag) {
  const double d = be - al;
  if (fabs(d) > 1.152921504606847e18 * ag) return ag / d;
  const long long eb = (__double_as_longlong(ag) >> 52) & 0x7ff;
  const double sc = __longlong_as_double((2046LL - eb) << 52);
  const double num = d * (0.5 * sc), den = ag * sc;
  const float z = __double2float_rn(num) / __double2float_rn(den);
  const float tf = copysignf(1.0f, z) / (fabsf(z) + sqrtf(fmaf(z, z, 1.0f)));
  return (double)tf;
}
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
__global__ void k_ws4(double* out, long long* cyc) {
  double a = threadIdx.x, b = 1, c = 2, d = 3;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { warp_sum4(a, b, c, d); a *= 1e-3; }
  long long t1 = clock64();
  out[threadIdx.x] = a + b + c + d;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
}
__global__ void k_rotfast(double* out, long long* cyc, double al0) {
  double al = al0 + threadIdx.x, be = 2.0, ag = 0.5, c, s;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { jacobi_cs_fast(al, be, ag, c, s); al = 1.0 + c * 1e-3; ag = 0.5 + s * 1e-3; }
  long long t1 = clock64();
  out[threadIdx.x] = c + s;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
}
__global__ void k_rotexact(double* out, long long* cyc, double al0) {
  double al = al0 + threadIdx.x, be = 2.0, ag = 0.5, c = 0, sn = 0;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    const double zeta = 0.5 * (be - al) / ag;
    const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
    c = rsqrt(fma(tt, tt, 1.0)); sn = c * tt;
    al = 1.0 + c * 1e-3; ag = 0.5 + sn * 1e-3;
  }
  long long t1 = clock64();
  out[threadIdx.x] = c + sn;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
}
// DFMA throughput: 8 independent chains per thread, nw warps
__global__ void k_dfma_tp(double* out, long long* cyc, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < 1024; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
int main() {
  double* out; long long* cyc; float* fo;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64); cudaMalloc(&fo, 1 << 20);
  long long h;
#define RUN(name, ...) __VA_ARGS__; cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%-28s %lld cycles\n", name, h);
  RUN("dfma chain", k_dfma<<<1, 32>>>(out, cyc, 1.0000001, 1e-9));
  RUN("dadd chain", k_dadd<<<1, 32>>>(out, cyc, 1e-9));
  RUN("ffma chain", k_ffma<<<1, 32>>>(fo, cyc, 1.0000001f, 1e-9f));
  RUN("shfl(double)+dadd chain", k_shfl<<<1, 32>>>(out, cyc));
  RUN("lds->use chain", k_lds<<<1, 32>>>(out, cyc));
  RUN("rsqrt(double)+dadd", k_rsqrt<<<1, 32>>>(out, cyc, 1.0));
  RUN("sqrt(double)+dadd", k_sqrt<<<1, 32>>>(out, cyc, 1.0));
  RUN("__drcp_rn+dadd", k_rcp<<<1, 32>>>(out, cyc, 1.0));
  for (int w : {1, 4, 8, 16, 32}) { char nm[64]; sprintf(nm, "bar.sync %d warps", w); RUN(nm, k_bar<<<1, 32 * w>>>(out, cyc)); }
  for (int t : {32, 256, 1024}) for (int b : {8, 16}) { char nm[64]; sprintf(nm, "ping %d thr x %dB", t, b); RUN(nm, k_ping<<<2, t>>>(out, cyc, b)); }
  RUN("warp_sum4 chain", k_ws4<<<1, 32>>>(out, cyc));
  RUN("jacobi_cs_fast chain", k_rotfast<<<1, 32>>>(out, cyc, 1.0));
  RUN("exact rotation chain", k_rotexact<<<1, 32>>>(out, cyc, 1.0));
  for (int w : {4, 8, 16, 32}) { char nm[64]; k_dfma_tp<<<1, 32 * w>>>(out, cyc, 1.0000001, 1e-9); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("DFMA throughput %2d warps: %.2f lane-FMA/clk/SM\n", w, 32.0 * w * 8 * 1024 / h); }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
