// Host planner internals shared by the contraction (tk_plan.cpp) and decomposition (tk_svd.cpp) code.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "tk_internal.hpp"
#include "tk_kernels.hpp"

namespace tk {

// ------------------------------------------------------------------ device buffers
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  void upload(const std::vector<T>& v) {
    n = v.size() * sizeof(T);
    if (n == 0) return;
    if (cudaMalloc(&p, n) != cudaSuccess) TK_THROW(TK_ERR_CUDA, "cudaMalloc of plan table failed");
    if (cudaMemcpy(p, v.data(), n, cudaMemcpyHostToDevice) != cudaSuccess)
      TK_THROW(TK_ERR_CUDA, "upload of plan table failed");
  }
};

// ------------------------------------------------------------------ permute plan
struct PermPlan {
  bool identity = false;
  std::vector<PermGroup> groups;
  std::vector<PermMember> members;
  std::vector<double> coefs;
  std::vector<PermJob> jobs;
  std::vector<int64_t> blob;  // kJobSeg job blobs (SegHeader | SegGroup[ng] | rs | rd per job)
  int njobs = 0, njobs_multi = 0, njobs_rows = 0, njobs_box = 0;  // jobs = [rows | box | seg/tiled/packed | recoupling]
  bool tiled = false, rows_only = false;
  bool split = false;  // large permute: rows jobs in their own (leaner) launch
  DevBuf d_groups, d_members, d_coefs, d_jobs, d_blob;
  int elem_bytes = 8;  // 8 Float64, 16 ComplexF64
  double bytes = 0;  // algorithmic bytes (each stored element read once and written once)
  int64_t n_src = 0, n_dst = 0;
  bool uploaded = false;
  void upload() {
    if (uploaded) return;
    d_groups.upload(groups);
    d_members.upload(members);
    d_coefs.upload(coefs);
    d_jobs.upload(jobs);
    d_blob.upload(blob);
    uploaded = true;
  }
};

// Internal (workspace) layout of A~, B~, C~: same blocks and subblock order as the canonical
// layout, but every block's leading dimension is padded to a multiple of 4 doubles and every block
// starts 32-byte aligned, so the GEMM can use 16-byte cp.async and columns start on sector bounds.
// ComplexF64 blocks are stored as their real representation (PermCM in tk_kernels.hpp):
// planar   (A~, C~): rows x 2cols, [re | im], imaginary part d1 = cols * ld doubles after the real part;
// real rep (B~):     2rows x 2cols, [[re, im], [-im, re]], d1 = cols * ld, d2 = rows.
enum class PadKind { Real, Planar, RealRep };
struct PadLayout {
  PadKind kind = PadKind::Real;
  std::vector<int64_t> off, ld, d1, d2;  // in doubles
  int64_t total = 0;                     // doubles
};

PadLayout pad_layout(const Tensor& t, PadKind kind = PadKind::Real);
void validate_perm(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q);
// Alg. 2 selection rule: spaces of permute(A, (p, q)) (new references, release after use)
void permuted_spaces(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q,
                     std::vector<Space*>& cod, std::vector<Space*>& dom);
void trace_cache_clear();
void permute_transfer_matrix(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q, const Tensor& C,
                             double* out);
void check_target(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q, const Tensor& C);
void build_perm_plan(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q, const Tensor& C,
                     PermPlan& P, int elem_bytes, const PadLayout* spl = nullptr, const PadLayout* dpl = nullptr);
Tensor* permuted_tensor(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q, tk_dtype dt);
void check_cuda(cudaError_t e, const char* what);
void run_permute(PermPlan& P, const void* src, void* dst, double alpha, double beta, int cm, double ims,
                 cudaStream_t st);
size_t align256(size_t x);
void add_launches(int n);
void reset_launches();
void svd_cache_clear();

}  // namespace tk
