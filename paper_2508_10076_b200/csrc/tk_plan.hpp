// Host planner internals shared by the contraction (tk_plan.cpp) and decomposition (tk_svd.cpp) code.
#pragma once
#include <cuda_runtime.h>

#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "tk_gemm_tma.hpp"
#include "tk_internal.hpp"
#include "tk_kernels.hpp"

namespace tk {

// ------------------------------------------------------------------ device context
int current_device();  // cudaGetDevice, or -1 without a usable device (host-only layout / workspace queries)
void check_cuda(cudaError_t e, const char* what);

// ------------------------------------------------------------------ device buffers
// Library-owned device memory: the descriptor tables of a plan, uploaded ONCE per plan (std::call_once
// in Plan::ensure_uploaded; the plan cache does it inside its lock right after building the plan, so the
// plan pointer never escapes without its tables; only host-only queries made without a device defer it
// to the first device-side call). The upload is capture-safe: it runs in relaxed capture mode on a
// library-private non-blocking stream and is waited for before returning, so a cold plan built while
// the caller's stream is being captured into a CUDA graph neither joins the capture nor breaks it.
// Frees are deferred (free_deferred()) to a point where no capture is in progress on the calling
// stream, because cudaFree synchronises the device.
void upload_bytes(void** p, const void* host, size_t n);
void free_later(void* p, int device);
void free_deferred(cudaStream_t caller);  // no-op while `caller` is capturing
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  int dev = -1;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) free_later(p, dev);
  }
  template <typename T>
  void upload(const std::vector<T>& v) {
    if (p) TK_THROW(TK_ERR_CUDA, "internal: plan table uploaded twice");
    n = v.size() * sizeof(T);
    if (n == 0) return;
    dev = current_device();
    upload_bytes(&p, v.data(), n);
  }
};

// ------------------------------------------------------------------ plan cache
// Memoised plans ("crucial for performance"). The key always carries the device
// ordinal, because a plan's tables live on the device it was built on. Plans are handed out as
// shared_ptr taken under the lock, so tk_cache_clear / eviction never frees a plan another thread is
// still launching from. Bounded LRU (kPlanCacheCap entries per cache): a DMRG sweep creates new bond
// spaces after every truncation. A plan's tables must outlive any CUDA graph captured from it: do not
// clear the cache (or let it evict) while such a graph is still replayed.
constexpr size_t kPlanCacheCap = 512;
template <class Plan>
class PlanCache {
 public:
  explicit PlanCache(size_t cap = kPlanCacheCap) : cap_(cap) {}
  template <class Build>
  std::shared_ptr<Plan> get(const std::string& key0, Build build) {
    const std::string key = key0 + "@dev" + std::to_string(current_device());
    std::lock_guard<std::mutex> g(mu_);
    auto it = map_.find(key);
    if (it != map_.end()) {
      lru_.splice(lru_.begin(), lru_, it->second);
      return it->second->second;
    }
    std::shared_ptr<Plan> P = build();  // throws: nothing cached
    if (current_device() >= 0) P->ensure_uploaded();
    lru_.emplace_front(key, P);
    map_[key] = lru_.begin();
    while (lru_.size() > cap_) {
      map_.erase(lru_.back().first);
      lru_.pop_back();
    }
    return P;
  }
  void clear() {
    std::lock_guard<std::mutex> g(mu_);
    map_.clear();
    lru_.clear();
  }
  size_t size() {
    std::lock_guard<std::mutex> g(mu_);
    return lru_.size();
  }

 private:
  size_t cap_;
  std::mutex mu_;
  std::list<std::pair<std::string, std::shared_ptr<Plan>>> lru_;
  std::unordered_map<std::string, typename std::list<std::pair<std::string, std::shared_ptr<Plan>>>::iterator> map_;
};

// ------------------------------------------------------------------ permute plan
struct PermPlan {
  bool identity = false;
  std::vector<PermGroup> groups;
  std::vector<PermMember> members;
  std::vector<double> coefs;
  std::vector<PermJob> jobs;
  std::vector<int64_t> blob;  // kJobSeg job blobs (SegHeader | SegGroup[ng] | rs | rd per job)
  int njobs = 0, njobs_multi = 0, njobs_rows = 0;  // jobs = [rows | seg/tiled/packed | recoupling]
  bool tiled = false, rows_only = false;
  bool split = false;  // large permute: rows jobs in their own (leaner) launch
  DevBuf d_groups, d_members, d_coefs, d_jobs, d_blob;
  int elem_bytes = 8;  // 8 Float64, 16 ComplexF64
  double bytes = 0;  // algorithmic bytes (each stored element read once and written once)
  int64_t n_src = 0, n_dst = 0;
  bool uploaded = false;
  std::once_flag up_once;
  void ensure_uploaded() {
    std::call_once(up_once, [&] {
      check_cuda(ensure_kernel_attrs(), "kernel attributes");
      d_groups.upload(groups);
      d_members.upload(members);
      d_coefs.upload(coefs);
      d_jobs.upload(jobs);
      d_blob.upload(blob);
      uploaded = true;
    });
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
void fused_cache_clear();
void ncon_cache_clear();  // tk_ncon.cpp: planned networks

// Abelian output permute as an element map (tk_plan.cpp): a C~ row tree of F rows starting at padded
// offset src (column n folded into src) lands in one C subblock with sign +-1; map() fills the GatherOut
// (its own radix: the permute's row legs of extent > 1, at most 3), or returns false.
class OutMap {
 public:
  OutMap(const PermPlan& pc, const PadLayout& lc);
  bool ok() const { return ok_; }
  bool map(int64_t src, int F, GatherOut& o) const;

 private:
  struct Box {
    int32_t r0, nr, c0, nc;
    int g;
  };
  const PermPlan& pc_;
  const PadLayout& lc_;
  std::map<int64_t, std::vector<Box>> boxes_;
  bool ok_ = true;
};

// ------------------------------------------------------------------ contraction plan (tk_plan.cpp)
struct ContractPlan {
  Tensor* At = nullptr;  // A~ (canonical layout, reading C2 tuples)
  Tensor* Bt = nullptr;
  Tensor* Ct = nullptr;
  PermPlan pa, pb, pc;
  PadLayout la, lb, lc;  // workspace layouts of A~, B~, C~
  std::vector<GemmGroup> ggroups;
  std::vector<GemmTile> tiles;
  int ntiles_big = 0, ntiles_small = 0, ntiles_skinny = 0;
  std::vector<GemmTile> split_heads;  // split-K reduction targets
  int nslots = 0;
  size_t off_parts = 0;
  DevBuf d_heads;
  bool cplx = false;  // ComplexF64: workspace in the real representation (PermCM), one real GEMM
  // small Float64 contractions: both operand permutes in ONE launch (jobs of A~ = op 0, B~ = op 1)
  bool merged_ab = false;
  std::vector<PermJob> jobs_ab;
  int njobs_ab = 0, njobs_ab_multi = 0;
  bool ab_tiled = false;
  DevBuf d_ggroups, d_tiles, d_jobs_ab;
  // gathered skinny GEMM (build_gather): the A~ permute folded into the GEMM's loads
  bool gather = false;
  std::vector<GatherSeg> gsegs;
  std::vector<GatherTile> gtiles;
  std::vector<int32_t> btab;
  std::vector<int64_t> gslots;
  int g_kmax = 0, g_nmax = 0;
  DevBuf d_gsegs, d_btab, d_gslots;
  bool gout = false;  // the output permute folded into the gathered GEMM's stores (GatherOut)
  std::vector<GatherOut> gouts;
  DevBuf d_gouts;
  size_t off_a = 0, off_b = 0, off_c = 0, off_counter = 0, ws_bytes = 0;
  double flops = 0;
  // persistent TMA GEMM for the big tiles (tk_gemm_tma.cu): groups with a tensor-map pair, and the
  // maps encoded for the last (A~, B~) workspace pointers seen (re-encoded when they change)
  bool tma = false;
  std::vector<int> tma_groups;
  std::mutex tma_mu;
  std::unique_ptr<GemmTmaParams> tma_params;
  const void* tma_a = nullptr;
  const void* tma_b = nullptr;
  bool uploaded = false;
  std::once_flag up_once;
  ~ContractPlan() {
    if (At) tk_tensor_release((tk_tensor*)At);
    if (Bt) tk_tensor_release((tk_tensor*)Bt);
    if (Ct) tk_tensor_release((tk_tensor*)Ct);
  }
  void ensure_uploaded() {
    std::call_once(up_once, [&] { upload(); });
  }
  void upload() {
    check_cuda(ensure_kernel_attrs(), "kernel attributes");
    if (!pa.identity) pa.ensure_uploaded();
    if (!pb.identity) pb.ensure_uploaded();
    if (!pc.identity) pc.ensure_uploaded();
    d_ggroups.upload(ggroups);
    d_tiles.upload(tiles);
    d_heads.upload(split_heads);
    d_jobs_ab.upload(jobs_ab);
    d_gsegs.upload(gsegs);
    d_btab.upload(btab);
    d_gslots.upload(gslots);
    d_gouts.upload(gouts);
    uploaded = true;
  }
};

// memoised plan of tk_contract (labels, reading C2) and its execution (operand permutes, grouped GEMM,
// output permute); `stream` is the caller's tk_stream
std::shared_ptr<ContractPlan> get_contract_plan(const Tensor& A, const int32_t* labA, const Tensor& B,
                                                const int32_t* labB, const Tensor& C, const int32_t* labC);
void run_contract(ContractPlan* P, const void* a, const void* b, void* c, int32_t conjA, int32_t conjB,
                  double alpha, double beta, void* ws, size_t ws_bytes, tk_stream stream);
int sm_count();

}  // namespace tk
