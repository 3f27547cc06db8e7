// Partial traces of symmetric tensor maps (Alg. 3, Alg. 7 "Abelian Tensor Trace" P:1225-1257,
// fusion-tree traces P:1880-1904).
//
// C = alpha * permute(trace(A, (pt, qt)), (p, q)) + beta * C: legs pt[i] (read as codomain legs, Alg. 3's
// "(a_1 ...; b_1^* ...)") are contracted with legs qt[i] (read as domain legs), the remaining legs are
// arranged as (p ; q). Planner: permute A to A~ = (p..., pt_1..pt_n ; q..., qt_1..qt_n) with the
// library's permute (any kind; planar kinds need the pairs to be nested in the cyclic order), then
// peel the traced pairs from the ends of the trees: the last splitting leg and the last fusion leg
// (same tree label a) are closed into a loop, which leaves the splitting and fusion trees without that
// leg -- their new coupled labels must agree (e) -- with the bubble factor d_c / d_e ("recoupling the
// result to a tadpole"; for SU(2) the CG identity sum_{m_a, m_c} C C = (2c+1)/(2e+1)).
// Kernel: one CTA per output subblock, each output element sums its source subblocks' diagonals.
// Fermionic kinds are refused (the supertrace needs the twist, which the unitary
// convention of reading C13 does not carry).
#include <algorithm>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>

#include "tk_plan.hpp"

namespace tk {

constexpr int kTraceMaxPairs = 4;

struct TraceDst {
  int64_t off;
  int32_t ld, rows, cols;
  int32_t src_begin, src_count;
  int32_t pad_;
};

struct TraceSrc {
  int64_t off;  // in the A~ workspace (doubles)
  int32_t ld, nt;
  int32_t T[kTraceMaxPairs];
  int64_t dstride[kTraceMaxPairs];
  double coef;
};

// V = double (Float64) or double2 (ComplexF64, interleaved; the coefficients are real)
__device__ __forceinline__ double tr_zero(double) { return 0.0; }
__device__ __forceinline__ double2 tr_zero(double2) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double tr_add(double a, double b) { return a + b; }
__device__ __forceinline__ double2 tr_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double tr_axpy(double c, double x, double y) { return fma(c, x, y); }
__device__ __forceinline__ double2 tr_axpy(double c, double2 x, double2 y) {
  return make_double2(fma(c, x.x, y.x), fma(c, x.y, y.y));
}

template <typename V>
__global__ void __launch_bounds__(256) trace_kernel(const V* __restrict__ At, V* __restrict__ C,
                                                    const TraceDst* __restrict__ dsts,
                                                    const TraceSrc* __restrict__ srcs, double alpha, double beta) {
  const TraceDst d = dsts[blockIdx.x];
  const int64_t n = (int64_t)d.rows * d.cols;
  for (int64_t e = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.y * blockDim.x) {
    const int64_t r = e % d.rows, cc = e / d.rows;
    V acc = tr_zero(V{});
    for (int k = 0; k < d.src_count; ++k) {
      const TraceSrc s = srcs[d.src_begin + k];
      const int64_t base = s.off + r + (int64_t)s.ld * cc;
      int ntot = 1;
      for (int q = 0; q < s.nt; ++q) ntot *= s.T[q];
      V part = tr_zero(V{});
      for (int u = 0; u < ntot; ++u) {  // the diagonal of the traced pairs (mixed radix)
        int rem = u;
        int64_t o = 0;
        for (int q = 0; q < s.nt; ++q) {
          const int t = rem % s.T[q];
          rem /= s.T[q];
          o += (int64_t)t * s.dstride[q];
        }
        part = tr_add(part, At[base + o]);
      }
      acc = tr_axpy(s.coef, part, acc);
    }
    V* p = C + d.off + r + (int64_t)d.ld * cc;
    V v = tr_axpy(alpha, acc, tr_zero(V{}));
    if (beta != 0.0) v = tr_axpy(beta, *p, v);
    *p = v;
  }
}

namespace {

struct TracePlan {
  Tensor* At = nullptr;
  PermPlan pa;
  PadLayout la;
  std::vector<TraceDst> dsts;
  std::vector<TraceSrc> srcs;
  std::vector<std::pair<int, std::pair<int, double>>> transfer;  // (A~ sub, (C sub, coef)) for tests
  DevBuf d_dsts, d_srcs;
  size_t ws_bytes = 0;
  std::once_flag up_once;
  void ensure_uploaded() {
    std::call_once(up_once, [&] {
      pa.ensure_uploaded();
      d_dsts.upload(dsts);
      d_srcs.upload(srcs);
    });
  }
  ~TracePlan() {
    if (At) tk_tensor_release((tk_tensor*)At);
  }
};

PlanCache<TracePlan> g_trace_cache;

// drop the last leg of a canonical left-to-right tree
Tree peel(Kind k, const Tree& t) {
  Tree u = t;
  const size_t n = t.unc.size();
  u.unc.pop_back();
  u.dims.pop_back();
  if (n == 1) {
    u.coupled = sector_unit(k);
  } else if (n == 2) {
    u.coupled = t.unc[0];
  } else {
    u.coupled = t.inner.back();
    u.inner.pop_back();
  }
  return u;
}

const Space* leg_as_cod(const Tensor& A, int i, Space** tmp) {  // Alg. 3: (a_1 ...; b_1^* ...)
  if (i < A.n_cod()) return A.cod[i];
  *tmp = dual_space(A.dom[i - A.n_cod()]);
  return *tmp;
}
const Space* leg_as_dom(const Tensor& A, int i, Space** tmp) {  // (a_1^* ...; b_1 ...)
  if (i >= A.n_cod()) return A.dom[i - A.n_cod()];
  *tmp = dual_space(A.cod[i]);
  return *tmp;
}

std::shared_ptr<TracePlan> build_trace_plan(const Tensor& A, const std::vector<int>& pp, const std::vector<int>& qq,
                                            size_t npairs, const std::vector<int>& p, const std::vector<int>& q,
                                            const Tensor* C);

std::shared_ptr<TracePlan> get_trace_plan(const Tensor& A, const std::vector<int>& pt, const std::vector<int>& qt,
                          const std::vector<int>& p, const std::vector<int>& q, const Tensor* C) {
  if (kind_fermionic(A.kind)) TK_THROW(TK_ERR_UNSUPPORTED, "tk_trace: fermionic kinds (supertrace) not supported");
  if (pt.size() != qt.size() || pt.size() > (size_t)kTraceMaxPairs)
    TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_trace: 1..4 traced pairs, |pt| == |qt|");
  std::vector<int> pp(p), qq(q);
  pp.insert(pp.end(), pt.begin(), pt.end());
  qq.insert(qq.end(), qt.begin(), qt.end());
  validate_perm(A, pp, qq);
  for (size_t i = 0; i < pt.size(); ++i) {
    Space *t1 = nullptr, *t2 = nullptr;
    bool ok = same_space(leg_as_cod(A, pt[i], &t1), leg_as_dom(A, qt[i], &t2));
    if (t1) tk_space_release((tk_space*)t1);
    if (t2) tk_space_release((tk_space*)t2);
    if (!ok) TK_THROW(TK_ERR_SPACE_MISMATCH, "tk_trace: traced legs are not a ket/bra pair of one space");
  }
  std::ostringstream os;
  os << A.sig << "#";
  for (int x : pp) os << x << ",";
  os << "#";
  for (int x : qq) os << x << "," ;
  os << "#" << pt.size() << "#" << (C ? C->sig : std::string("-"));
  return g_trace_cache.get(os.str(), [&] { return build_trace_plan(A, pp, qq, pt.size(), p, q, C); });
}

std::shared_ptr<TracePlan> build_trace_plan(const Tensor& A, const std::vector<int>& pp, const std::vector<int>& qq,
                                            size_t npairs, const std::vector<int>& p, const std::vector<int>& q,
                                            const Tensor* C) {
  auto P = std::make_shared<TracePlan>();
  // A~ in the workspace in A's own element type (ComplexF64: interleaved, offsets in complex elements)
  const int eb = A.dtype == TK_C64 ? 16 : 8;
  P->At = permuted_tensor(A, pp, qq, A.dtype);
  P->la = pad_layout(*P->At);
  build_perm_plan(A, pp, qq, *P->At, P->pa, eb, nullptr, &P->la);
  P->pa.identity = false;
  P->ws_bytes = align256((size_t)P->la.total * eb);
  if (C) {
    check_target(A, p, q, *C);
    const Tensor& At = *P->At;
    const int nt = (int)npairs;
    std::vector<std::vector<std::pair<int, double>>> per_dst(C->subs.size());
    for (int i = 0; i < (int)At.subs.size(); ++i) {
      Tree s = At.s_tree(i), f = At.f_tree(i);
      double coef = 1.0;
      bool ok = true;
      for (int r = 0; r < nt && ok; ++r) {
        if (s.unc.back() != f.unc.back()) {
          ok = false;
          break;
        }
        const Sector c = s.coupled;
        s = peel(A.kind, s);
        f = peel(A.kind, f);
        if (s.coupled != f.coupled) ok = false;
        else coef *= sector_dim(A.kind, c) / sector_dim(A.kind, s.coupled);
      }
      if (!ok) continue;
      auto jt = C->sub_index.find(tree_pair_key(s, f));
      if (jt == C->sub_index.end()) TK_THROW(TK_ERR_SPACE_MISMATCH, "internal: traced tree pair not in the output");
      per_dst[jt->second].push_back({i, coef});
      P->transfer.push_back({i, {jt->second, coef}});
    }
    for (int j = 0; j < (int)C->subs.size(); ++j) {
      const Subblock& sb = C->subs[j];
      const Tree& cs = C->s_tree(j);
      const Tree& cf = C->f_tree(j);
      TraceDst d{};
      d.off = sb.off;
      d.ld = (int32_t)C->ld(j);
      d.rows = (int32_t)cs.size;
      d.cols = (int32_t)cf.size;
      d.src_begin = (int32_t)P->srcs.size();
      d.src_count = (int32_t)per_dst[j].size();
      for (auto& pr : per_dst[j]) {
        const int i = pr.first;
        const Subblock& asb = At.subs[i];
        const Tree& as = At.s_tree(i);
        const Tree& af = At.f_tree(i);
        TraceSrc t{};
        const int b = asb.block;
        t.off = P->la.off[b] + asb.row_off + P->la.ld[b] * asb.col_off;
        t.ld = (int32_t)P->la.ld[b];
        t.nt = nt;
        t.coef = pr.second;
        // traced legs are the last nt legs of both trees, in the order pt_1..pt_n / qt_1..qt_n
        const int n1 = (int)as.unc.size(), n2 = (int)af.unc.size();
        int64_t sc = 1, sd = 1;
        for (int l = 0; l < n1 - nt; ++l) sc *= as.dims[l];
        for (int l = 0; l < n2 - nt; ++l) sd *= af.dims[l];
        for (int r = 0; r < nt; ++r) {
          t.T[r] = (int32_t)as.dims[n1 - nt + r];
          t.dstride[r] = sc + (int64_t)t.ld * sd;
          sc *= as.dims[n1 - nt + r];
          sd *= af.dims[n2 - nt + r];
        }
        P->srcs.push_back(t);
      }
      P->dsts.push_back(d);
    }
  }
  return P;
}

std::vector<int> ivec(const int32_t* v, int n) { return std::vector<int>(v, v + n); }

}  // namespace

void trace_cache_clear() { g_trace_cache.clear(); }
size_t trace_cache_size() { return g_trace_cache.size(); }

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

tk_status tk_trace_output(const tk_tensor* A_, const int32_t* pt, const int32_t* qt, int32_t nt, const int32_t* p,
                          int32_t np, const int32_t* q, int32_t nq, tk_tensor** out) {
  TK_API_BEGIN
  if (!A_ || !out || nt < 1) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  get_trace_plan(A, ivec(pt, nt), ivec(qt, nt), ivec(p, np), ivec(q, nq), nullptr);  // validation
  *out = (tk_tensor*)permuted_tensor(A, ivec(p, np), ivec(q, nq), A.dtype);
  TK_API_END
}

tk_status tk_trace_workspace(const tk_tensor* A, const int32_t* pt, const int32_t* qt, int32_t nt, const int32_t* p,
                             int32_t np, const int32_t* q, int32_t nq, const tk_tensor* C, size_t* bytes) {
  TK_API_BEGIN
  if (!A || !C || !bytes || nt < 1) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  *bytes = get_trace_plan(*(const Tensor*)A, ivec(pt, nt), ivec(qt, nt), ivec(p, np), ivec(q, nq),
                          (const Tensor*)C)->ws_bytes;
  TK_API_END
}

tk_status tk_trace(const tk_tensor* A_, const void* a, const int32_t* pt, const int32_t* qt, int32_t nt,
                   const int32_t* p, int32_t np, const int32_t* q, int32_t nq, const tk_tensor* C_, void* c,
                   double alpha, double beta, void* ws, size_t ws_bytes, tk_stream stream) {
  TK_API_BEGIN
  if (!A_ || !C_ || nt < 1) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  const Tensor& C = *(const Tensor*)C_;
  if ((!a && A.nelems) || (!c && C.nelems)) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null data pointer");
  auto P = get_trace_plan(A, ivec(pt, nt), ivec(qt, nt), ivec(p, np), ivec(q, nq), &C);
  if (ws_bytes < P->ws_bytes || (P->ws_bytes && !ws)) TK_THROW(TK_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
  if (((uintptr_t)ws & 255) != 0) TK_THROW(TK_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  P->ensure_uploaded();
  cudaStream_t st = (cudaStream_t)stream;
  free_deferred(st);
  reset_launches();
  const bool cx = A.dtype == TK_C64;
  run_permute(P->pa, a, ws, 1.0, 0.0, cx ? kPermCToC : kPermReal, 1.0, st);
  if (!P->dsts.empty()) {
    const dim3 grid((unsigned)P->dsts.size(), 4);
    if (cx)
      trace_kernel<double2><<<grid, 256, 0, st>>>((const double2*)ws, (double2*)c, (const TraceDst*)P->d_dsts.p,
                                                 (const TraceSrc*)P->d_srcs.p, alpha, beta);
    else
      trace_kernel<double><<<grid, 256, 0, st>>>((const double*)ws, (double*)c, (const TraceDst*)P->d_dsts.p,
                                                (const TraceSrc*)P->d_srcs.p, alpha, beta);
    check_cuda(cudaPeekAtLastError(), "trace launch");
    add_launches(1);
  }
  TK_API_END
}

// host transfer matrix of the trace map on tree pairs (A subblocks x C subblocks), tests / §4.3
tk_status tk_trace_transfer(const tk_tensor* A_, const int32_t* pt, const int32_t* qt, int32_t nt, const int32_t* p,
                            int32_t np, const int32_t* q, int32_t nq, const tk_tensor* C_, double* out) {
  TK_API_BEGIN
  if (!A_ || !C_ || !out || nt < 1) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  const Tensor& C = *(const Tensor*)C_;
  auto P = get_trace_plan(A, ivec(pt, nt), ivec(qt, nt), ivec(p, np), ivec(q, nq), &C);
  // compose: A subblocks -> A~ subblocks (permute transfer) -> C subblocks (trace map)
  const Tensor& At = *P->At;
  std::vector<double> Tpa(A.subs.size() * At.subs.size());
  std::vector<int> pp = ivec(p, np), qq = ivec(q, nq);
  pp.insert(pp.end(), pt, pt + nt);
  qq.insert(qq.end(), qt, qt + nt);
  permute_transfer_matrix(A, pp, qq, At, Tpa.data());
  const size_t nc = C.subs.size(), na = At.subs.size();
  std::fill(out, out + A.subs.size() * nc, 0.0);
  for (size_t i = 0; i < A.subs.size(); ++i)
    for (auto& tr : P->transfer) out[i * nc + tr.second.first] += Tpa[i * na + tr.first] * tr.second.second;
  TK_API_END
}

}  // extern "C"
