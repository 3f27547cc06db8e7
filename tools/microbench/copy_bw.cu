// HBM copy microbenchmark: how close can 8-byte (vs 16-byte) element copies get to the copy roofline,
// plain and software-pipelined, and a row-structured copy (rows of n0 doubles, the cfg4 permute shape).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o copy_bw copy_bw.cu && ./copy_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int T = 256;

template <int U>
__global__ void __launch_bounds__(T) copy8(const double* __restrict__ s, double* __restrict__ d, int64_t n) {
  for (int64_t b = (int64_t)blockIdx.x * T * U + threadIdx.x; b < n; b += (int64_t)gridDim.x * T * U) {
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = b + u * T < n ? __ldg(s + b + u * T) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + u * T < n) d[b + u * T] = x[u];
  }
}

template <int U>
__global__ void __launch_bounds__(T) copy16(const double2* __restrict__ s, double2* __restrict__ d, int64_t n) {
  for (int64_t b = (int64_t)blockIdx.x * T * U + threadIdx.x; b < n; b += (int64_t)gridDim.x * T * U) {
    double2 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = b + u * T < n ? __ldg(s + b + u * T) : make_double2(0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + u * T < n) d[b + u * T] = x[u];
  }
}

// software pipelined: loads of chunk i+1 are issued before the stores of chunk i
template <int U>
__global__ void __launch_bounds__(T) copy8p(const double* __restrict__ s, double* __restrict__ d, int64_t n) {
  const int64_t step = (int64_t)gridDim.x * T * U;
  int64_t b = (int64_t)blockIdx.x * T * U + threadIdx.x;
  double x[U], y[U];
#pragma unroll
  for (int u = 0; u < U; ++u) x[u] = b + u * T < n ? __ldg(s + b + u * T) : 0.0;
  for (; b < n; b += 2 * step) {
    const int64_t c = b + step;
#pragma unroll
    for (int u = 0; u < U; ++u) y[u] = c + u * T < n ? __ldg(s + c + u * T) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + u * T < n) d[b + u * T] = x[u];
    const int64_t e = c + step;
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = e + u * T < n ? __ldg(s + e + u * T) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c + u * T < n) d[c + u * T] = y[u];
  }
}

// rows: element e of a job -> (row r = e / n0, i0); src row start rs[r], dst row start rd[r]
// (here: a permutation of row slots with arbitrary 8-byte alignment), U loads in flight
template <int U>
__global__ void __launch_bounds__(T) rows8(const double* __restrict__ s, double* __restrict__ d,
                                           const int64_t* __restrict__ rs, const int64_t* __restrict__ rd,
                                           int n0, int64_t nrows, int rows_per_job) {
  __shared__ int64_t ss[1024], sd[1024];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_job;
  const int nr = (int)(nrows - r0 < rows_per_job ? nrows - r0 : rows_per_job);
  for (int r = threadIdx.x; r < nr; r += T) {
    ss[r] = rs[r0 + r];
    sd[r] = rd[r0 + r];
  }
  __syncthreads();
  const int total = nr * n0;
  for (int e0 = threadIdx.x; e0 < total; e0 += T * U) {
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * T;
      if (e < total) {
        const int r = e / n0, i = e - r * n0;
        x[u] = __ldg(s + ss[r] + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * T;
      if (e < total) {
        const int r = e / n0, i = e - r * n0;
        d[sd[r] + i] = x[u];
      }
    }
  }
}

template <typename F>
float timeit(F f, int reps = 10) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  const int64_t n = 1110720212;  // cfg4 operand elements (Float64)
  double *s, *d;
  cudaMalloc(&s, n * 8);
  cudaMalloc(&d, n * 8);
  cudaMemset(s, 0, n * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = 2.0 * n * 8;
  auto rep = [&](const char* name, float ms) { printf("%-28s %8.3f ms  %7.1f GB/s\n", name, ms, bytes / (ms * 1e6)); };
  rep("cudaMemcpy D2D", timeit([&] { cudaMemcpy(d, s, n * 8, cudaMemcpyDeviceToDevice); }));
  for (int waves : {4, 8, 32}) {
    char nm[64];
    snprintf(nm, 64, "copy8<8> grid %dx", waves);
    rep(nm, timeit([&] { copy8<8><<<sms * waves, T>>>(s, d, n); }));
    snprintf(nm, 64, "copy8<16> grid %dx", waves);
    rep(nm, timeit([&] { copy8<16><<<sms * waves, T>>>(s, d, n); }));
    snprintf(nm, 64, "copy8p<8> grid %dx", waves);
    rep(nm, timeit([&] { copy8p<8><<<sms * waves, T>>>(s, d, n); }));
    snprintf(nm, 64, "copy16<4> grid %dx", waves);
    rep(nm, timeit([&] { copy16<4><<<sms * waves, T>>>((const double2*)s, (double2*)d, n / 2); }));
    snprintf(nm, 64, "copy16<8> grid %dx", waves);
    rep(nm, timeit([&] { copy16<8><<<sms * waves, T>>>((const double2*)s, (double2*)d, n / 2); }));
  }
  // rows of 18 doubles (cfg4 median), row slots permuted in blocks of 64 (dst), identity src
  const int n0 = 18;
  const int64_t nrows = n / n0;
  int64_t *rs, *rd;
  cudaMalloc(&rs, nrows * 8);
  cudaMalloc(&rd, nrows * 8);
  {
    int64_t* h = (int64_t*)malloc(nrows * 8);
    for (int64_t r = 0; r < nrows; ++r) h[r] = r * n0;
    cudaMemcpy(rs, h, nrows * 8, cudaMemcpyHostToDevice);
    for (int64_t r = 0; r < nrows; ++r) {  // transpose rows within 32 x 32 blocks
      const int64_t blk = r / 1024, w = r % 1024;
      const int64_t t = blk * 1024 + (w % 32) * 32 + w / 32;
      h[r] = (t < nrows ? t : r) * n0;
    }
    cudaMemcpy(rd, h, nrows * 8, cudaMemcpyHostToDevice);
    free(h);
  }
  for (int rpj : {256, 455}) {
    char nm[64];
    const int64_t jobs = (nrows + rpj - 1) / rpj;
    snprintf(nm, 64, "rows8<8> %d rows/job", rpj);
    rep(nm, timeit([&] { rows8<8><<<(unsigned)jobs, T>>>(s, d, rs, rd, n0, nrows, rpj); }));
    snprintf(nm, 64, "rows8<16> %d rows/job", rpj);
    rep(nm, timeit([&] { rows8<16><<<(unsigned)jobs, T>>>(s, d, rs, rd, n0, nrows, rpj); }));
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
