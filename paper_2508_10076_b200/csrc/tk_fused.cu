// Two consecutive contractions in one pass: C = (A . B1 -> T) . B2 (tk_contract2, include/tk.h).
//
// The DMRG two-site update applies the two MPO tensors one after the other (Alg. 12: the
// chain L.theta -> .W1 -> .W2 -> .R in its fixed pairwise order). Both MPO steps are skinny contractions
// (K, N <= 16) whose operand permutes the planner already folds into gathered GEMMs (build_gather in
// tk_plan.cpp). Run as two tk_contract calls, the intermediate T (cfg3: 6.7 M doubles) makes a full HBM
// round trip. Here the pair runs as ONE kernel with the SAME pairwise arithmetic -- the two steps' own
// plans (reading C2 tuples, C13 signs) define every coefficient -- and T never leaves the SM:
//
//  * A "fiber" is one row of step 2's gathered operand A~2 within its row tree. When A~2's rows are
//    contiguous in T (checked: its row legs have strides 1, ext0, ext0 ext1, ...) and each row tree of A~2 reads, for every
//    one of its columns, a whole row tree of step 1's output block (checked), a fiber's step-2 inputs are
//    T values of the SAME row index in a handful of step-1 row trees. Connected row trees form a class
//    (for the MPO chain: one pair of bond sectors (alpha', beta) -- a class's fibers are its
//    deg(alpha') x deg(beta) index pairs); all row trees of a class have the same number of rows F.
//  * Per class the planner writes a program: the step-1 inputs (T1 offsets as base + digits(f) . strides,
//    the A~1 gather of step 1), the T elements as sparse sums over inputs with B1 coefficients (step 1's
//    GEMM, B~1 gathered from B1 with its sign), and the outputs as sparse sums over T elements with B2
//    coefficients (step 2's GEMM). A thread runs the program for one fiber: loads its inputs (coalesced
//    across fibers: consecutive f are consecutive T1 addresses), forms its T values in shared memory and
//    writes its outputs (consecutive C addresses).
//  * B1 / B2 values are read at run time (the program holds their offsets and signs), so a plan serves
//    any data; only the structure is baked in.
// Anything else (non-gathered steps, an output permute on either step, ComplexF64, oversized fibers)
// runs the two contractions as they are, with T in the workspace.
#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <sstream>

#include "tk_device.cuh"
#include "tk_plan.hpp"

namespace tk {

namespace {
constexpr int kFusedThreads = 128;  // 4 warps, each its own chunk of <= 32 fibers
constexpr int kFusedWarps = kFusedThreads / 32;
constexpr int kFusedMaxIn = 64;     // inputs per class (the sign mask is 64 bits)
constexpr int kFusedMaxMid = 64;    // T elements per fiber
constexpr int kFusedMaxCoef = 1024; // coefficient entries per class (shared-memory doubles per warp)

// A class program, in 8-byte words: header | ins[n_in] | t1[n_t1] | t2[n_t2] | outs[n_out] | midref[] | coef[]
// (everything between the header and coef[] is staged in shared memory by the kernel)
struct FusedHeader {
  int32_t F, nrl, n_in, n_t1, n_t2, n_mid, n_ref, n_coef1, n_coef;
  int32_t n_out;
  int32_t ext[4];        // mixed radix of the fiber index f over step 1's row legs (first fastest)
  uint64_t neg_in;       // bit j: input j enters negated (its subblock's coefficient -1, C13)
};
struct FusedIn {         // a step-1 input: T1 offset = base + sum_l digit_l(f) * str[l] (32-bit: T1 < 2^31 elements)
  int32_t base, str[3];
};
struct FusedT1 {         // a step-1 row tree: T values mid0 + n (n < N) = sum_k in(in0 + k) coef[c0 + k NM + n]
  int32_t in0, K, N, mid0, c0, pad[3];
};
struct FusedT2 {         // a step-2 row tree: output n = sum_k mid(midref[r0 + k]) coef[c0 + k NM + n] -> outs[o0 + n]
  int32_t K, N, r0, c0, o0, pad;
};
// midref: 2 * T-value index + (subblock coefficient < 0); coef: B~ table entry (2 * offset into W + sign,
// -1 = structural zero) of each distinct GEMM group of the class, step 1's first (n_coef1 of them)
struct FusedChunk {      // fibers [f0, f0 + nf) of the class whose program starts at word `prog`
  int64_t prog;
  int32_t f0, nf;
};
static_assert(sizeof(FusedHeader) == 64 && sizeof(FusedIn) == 16 && sizeof(FusedT1) == 32 &&
                  sizeof(FusedT2) == 24,
              "fused layout");
}  // namespace

// ------------------------------------------------------------------ device side
__device__ __forceinline__ void fused_cp8(double* smem, const double* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

// One warp per chunk of <= 32 fibers of one class (many classes are smaller than a CTA); 4 independent
// warps per CTA. Per warp, BEFORE griddepcontrol.wait (plan data only): the class program (input table,
// row trees, output maps, T-value references) is copied into the warp's shared memory in one batch of
// independent loads, and the class's coefficients are resolved into shared memory (W value, sign, alpha
// for step 2 without an output permute: exactly the B~ value the gathered GEMM forms), each K x N table
// stored as K rows of NM (zero-padded, 16-byte aligned: read as double2 broadcasts). After the wait the
// only global loads are the fiber's T1 inputs: per step-1 row tree its K inputs (loaded together), its N
// T values to shared memory
// ([slot][thread], conflict-free); then each step-2 row tree reads its K T values and writes its N outputs
// (through the output permute's map when step 2 has one). Every product is the gathered GEMM's own:
// acc_n = fma(+-a_k, b~_kn, acc_n) over k ascending from zero, zeros included, so the fused result is
// bitwise that of the two tk_contract calls. NM (4 / 6 / 8 / 16) bounds K and N of both steps (the
// coefficient rows are NM wide: NM = 6 for the D_W = 10 MPOs of cfg3, whose K, N <= 6, computes no padding).
// (Measured alternatives, cfg3: all inputs fetched by cp.async and T values recomputed where consumed,
// 101 us; two fibers per thread, 86 us; next tree's inputs prefetched, 89 us; program read from global
// memory, one dependent load chain per row tree, 77-90 us; program staged and all of a fiber's inputs
// issued at once (registers), 12 us slower than per tree -- see DESIGN.md §6.4.)
template <int NM>
__global__ void __launch_bounds__(kFusedThreads)
    fused_pair_kernel(const double* __restrict__ T1, const double* __restrict__ W1, const double* __restrict__ W2,
                      double* __restrict__ C, const int64_t* __restrict__ progs, const FusedChunk* __restrict__ chunks,
                      int nchunks, int max_mid, int max_coef, int max_stage, double calpha, double oalpha,
                      double beta) {
  extern __shared__ __align__(16) double fsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tid = threadIdx.x;
  pdl_trigger();
  const int ci = blockIdx.x * kFusedWarps + warp;
  if (ci >= nchunks) return;
  const FusedChunk ch = chunks[ci];
  const int64_t* prog = progs + ch.prog;
  FusedHeader h;
  {
    const int4* p4 = reinterpret_cast<const int4*>(prog);
    int4* h4 = reinterpret_cast<int4*>(&h);
#pragma unroll
    for (int i = 0; i < 4; ++i) h4[i] = __ldg(p4 + i);
  }
  double* vmid = fsm;
  double* cf = vmid + max_mid * kFusedThreads + warp * (max_coef + max_stage);
  int64_t* sp = reinterpret_cast<int64_t*>(cf + max_coef);  // the staged program (after the header)
  const int nst = 2 * h.n_in + 4 * h.n_t1 + 3 * h.n_t2 + 4 * h.n_out + ((h.n_ref + 1) >> 1);
  {
    const longlong2* g2 = reinterpret_cast<const longlong2*>(prog + 8);
    longlong2* s2 = reinterpret_cast<longlong2*>(sp);
    for (int e = lane; e < (nst >> 1); e += 32) s2[e] = __ldg(g2 + e);
    if ((nst & 1) && lane == 0) sp[nst - 1] = __ldg(prog + 8 + nst - 1);
  }
  const int4* sin = reinterpret_cast<const int4*>(sp);  // FusedIn[n_in]
  const int4* t1 = sin + h.n_in;                         // FusedT1[n_t1] (2 x int4 each)
  const FusedT2* t2 = reinterpret_cast<const FusedT2*>(sp + 2 * h.n_in + 4 * h.n_t1);
  const GatherOut* outs = reinterpret_cast<const GatherOut*>(sp + 2 * h.n_in + 4 * h.n_t1 + 3 * h.n_t2);
  const int32_t* midref = reinterpret_cast<const int32_t*>(sp + 2 * h.n_in + 4 * h.n_t1 + 3 * h.n_t2 + 4 * h.n_out);
  const int32_t* coefs = reinterpret_cast<const int32_t*>(prog + 8 + nst);
  const int f = ch.f0 + lane;
  int d0 = 0, d1 = 0, d2 = 0;  // f's digits over step 1's row legs (first fastest)
  {
    int r = f;
    if (h.nrl > 0) { d0 = r % h.ext[0]; r /= h.ext[0]; }
    if (h.nrl > 1) { d1 = r % h.ext[1]; r /= h.ext[1]; }
    if (h.nrl > 2) d2 = r % h.ext[2];
  }
  // the class's B~ values, one lane per entry
  for (int e = lane; e < h.n_coef; e += 32) {
    const int be = __ldg(coefs + e);
    double v = 0.0;
    if (be >= 0) {
      v = e < h.n_coef1 ? __ldg(W1 + (be >> 1)) : calpha * __ldg(W2 + (be >> 1));
      if (be & 1) v = -v;
    }
    cf[e] = v;
  }
  pdl_wait();
  __syncwarp();
  if (lane >= ch.nf) return;
  const double2* cf2 = reinterpret_cast<const double2*>(cf);
  // step 1's GEMM per row tree: the tree's K inputs (gathered from T1) -> its N T values
  for (int t = 0; t < h.n_t1; ++t) {
    const int4 q = t1[2 * t];  // in0, K, N, mid0
    const int c0 = t1[2 * t + 1].x;
    double a[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      a[k] = 0.0;
      if (k < q.y) {
        const int4 x = sin[q.x + k];
        a[k] = __ldg(T1 + (x.x + d0 * x.y + d1 * x.z + d2 * x.w));
      }
    }
    double acc[NM];
#pragma unroll
    for (int n = 0; n < NM; ++n) acc[n] = 0.0;
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      if (k < q.y) {
        const double ak = ((h.neg_in >> (q.x + k)) & 1) ? -a[k] : a[k];
        const double2* w = cf2 + (c0 + k * NM) / 2;
#pragma unroll
        for (int j = 0; j < NM / 2; ++j) {
          const double2 b = w[j];
          acc[2 * j] = fma(ak, b.x, acc[2 * j]);
          acc[2 * j + 1] = fma(ak, b.y, acc[2 * j + 1]);
        }
      }
    }
#pragma unroll
    for (int n = 0; n < NM; ++n)
      if (n < q.z) vmid[(q.w + n) * kFusedThreads + tid] = acc[n];
  }
  // step 2's GEMM per row tree: the fiber's outputs, C = alpha * (...) + beta * C
  for (int t = 0; t < h.n_t2; ++t) {
    const FusedT2 q = t2[t];
    double acc2[NM];
#pragma unroll
    for (int n = 0; n < NM; ++n) acc2[n] = 0.0;
#pragma unroll
    for (int k = 0; k < NM; ++k) {
      if (k < q.K) {
        const int r = midref[q.r0 + k];
        double ak = vmid[(r >> 1) * kFusedThreads + tid];
        if (r & 1) ak = -ak;
        const double2* w = cf2 + (q.c0 + k * NM) / 2;
#pragma unroll
        for (int j = 0; j < NM / 2; ++j) {
          const double2 b = w[j];
          acc2[2 * j] = fma(ak, b.x, acc2[2 * j]);
          acc2[2 * j + 1] = fma(ak, b.y, acc2[2 * j + 1]);
        }
      }
    }
    uint32_t e0 = (uint32_t)outs[q.o0].ext0, e1 = (uint32_t)outs[q.o0].ext1, r = (uint32_t)f;
    const uint32_t o0 = r % e0;
    r /= e0;
    const uint32_t o1 = r % e1, o2 = r / e1;  // f's digits in the output map's radix
#pragma unroll
    for (int n = 0; n < NM; ++n)
      if (n < q.N) {
        const GatherOut o = outs[q.o0 + n];
        double* pn = C + o.base + ((int64_t)o0 * o.str[0] + (int64_t)o1 * o.str[1] + (int64_t)o2 * o.str[2]);
        double y = oalpha * acc2[n];
        if (o.neg) y = -y;
        *pn = beta != 0.0 ? fma(beta, *pn, y) : y;
      }
  }
}

// ------------------------------------------------------------------ host side
namespace {

struct RowTree {  // a row tree of a gathered GEMM: rows [r0, r0 + nrows) of group `grp`, its segments
  int grp;
  int32_t r0, nrows;
  std::vector<const GatherSeg*> segs;  // sorted by k0, covering [0, K)
};

// row trees of a gather plan, per group (deduplicated: a tile boundary may copy a tree's segments)
struct GatherIndex {
  std::vector<GemmGroup> groups;  // by group index
  std::vector<int> bt;            // btab offset per group
  std::vector<RowTree> trees;
  std::map<std::pair<int, int32_t>, int> tree_of;  // (group, r0) -> tree
};

bool index_gather(const ContractPlan& P, GatherIndex& X) {
  std::map<int64_t, int> grp_of_coff;
  for (const GatherTile& t : P.gtiles) {
    auto it = grp_of_coff.find(t.g.c_off);
    int gi;
    if (it == grp_of_coff.end()) {
      gi = (int)X.groups.size();
      grp_of_coff[t.g.c_off] = gi;
      X.groups.push_back(t.g);
      X.bt.push_back(t.bt);
    } else {
      gi = it->second;
    }
    for (int s = t.seg0; s < t.seg0 + t.nseg; ++s) {
      const GatherSeg& q = P.gsegs[s];
      auto key = std::make_pair(gi, q.r0);
      auto jt = X.tree_of.find(key);
      int ti;
      if (jt == X.tree_of.end()) {
        ti = (int)X.trees.size();
        X.tree_of[key] = ti;
        X.trees.push_back(RowTree{gi, q.r0, q.nrows, {}});
      } else {
        ti = jt->second;
      }
      RowTree& rt = X.trees[ti];
      if (rt.nrows != q.nrows) return false;
      bool dup = false;
      for (const GatherSeg* o : rt.segs) dup = dup || o->k0 == q.k0;
      if (!dup) rt.segs.push_back(&q);
    }
  }
  for (RowTree& rt : X.trees) {
    std::sort(rt.segs.begin(), rt.segs.end(), [](const GatherSeg* a, const GatherSeg* b) { return a->k0 < b->k0; });
    int k = 0;
    for (const GatherSeg* q : rt.segs) {
      if (q->k0 != k) return false;  // columns must be covered exactly once, in order
      k += q->nk;
    }
    if (k != X.groups[rt.grp].K) return false;
  }
  return true;
}

int find_union(std::vector<int>& p, int x) {
  while (p[x] != x) x = p[x] = p[p[x]];
  return x;
}

}  // namespace

struct FusedPlan {
  bool fused = false;
  std::shared_ptr<ContractPlan> p1, p2;
  std::vector<int64_t> progs;
  std::vector<FusedChunk> chunks;
  int smem = 0, max_in = 0, max_mid = 0, max_coef = 0, max_stage = 0, nm = 0;
  DevBuf d_progs, d_chunks;
  size_t ws_bytes = 0, off_t = 0, off_ws = 0;  // unfused: T | the larger of the two steps' workspaces
  std::once_flag up_once;
  void ensure_uploaded() {
    std::call_once(up_once, [&] {
      d_progs.upload(progs);
      d_chunks.upload(chunks);
    });
  }
};

// Builds the fused program; returns false (unfused) when any structural condition fails.
static bool build_fused(FusedPlan& F) {
  const ContractPlan& P1 = *F.p1;
  const ContractPlan& P2 = *F.p2;
  // both steps entirely gathered (no other GEMM tiles: K = 0 blocks of C would need their beta pass)
  // step 1's output is T itself (C~1 canonical); step 2 may carry an output permute (abelian: each C~2
  // subblock lands in one C subblock with a sign), folded into the fused kernel's stores
  if (!P1.gather || !P2.gather || !P1.pc.identity || P1.cplx || P2.cplx) return false;
  if (!P1.tiles.empty() || !P2.tiles.empty()) return false;
  GatherIndex X1, X2;
  if (!index_gather(P1, X1) || !index_gather(P2, X2)) return false;
  {  // the kernel instance: K and N (both steps) <= NM
    int nmax = 0;
    for (const GemmGroup& g : X1.groups) nmax = std::max(nmax, (int)g.N);
    for (const GemmGroup& g : X2.groups) nmax = std::max(nmax, (int)g.N);
    for (const GemmGroup& g : X1.groups) nmax = std::max(nmax, (int)g.K);
    for (const GemmGroup& g : X2.groups) nmax = std::max(nmax, (int)g.K);
    F.nm = nmax <= 4 ? 4 : nmax <= 6 ? 6 : nmax <= 8 ? 8 : 16;
    if (nmax > 16) return false;  // (T1 < 2^31 elements: build_gather's own condition)
  }
  // T offsets of step 1's output blocks: group by c_off (T is C~1 in its canonical layout)
  std::vector<std::pair<int64_t, int>> t_blocks;  // (c_off, group of step 1)
  for (int g = 0; g < (int)X1.groups.size(); ++g) t_blocks.push_back({X1.groups[g].c_off, g});
  std::sort(t_blocks.begin(), t_blocks.end());
  auto locate = [&](int64_t off, int& g, int32_t& r, int32_t& c) {  // T offset -> (step-1 group, row, col)
    auto it = std::upper_bound(t_blocks.begin(), t_blocks.end(), std::make_pair(off, INT32_MAX));
    if (it == t_blocks.begin()) return false;
    --it;
    g = it->second;
    const GemmGroup& G = X1.groups[g];
    const int64_t rel = off - G.c_off;
    r = (int32_t)(rel % G.ldc);
    c = (int32_t)(rel / G.ldc);
    return c < G.N && r < G.M;
  };
  // edges: step-2 row tree -> the step-1 row trees its columns read
  const int n1 = (int)X1.trees.size(), n2 = (int)X2.trees.size();
  std::vector<int> parent(n1 + n2);
  std::iota(parent.begin(), parent.end(), 0);
  struct Ref {
    int tree1;    // step-1 row tree
    int32_t col;  // column of T (step 1's output column) = step 1's GEMM column
    int neg;
  };
  std::vector<std::vector<Ref>> refs(n2);  // per step-2 tree, per step-2 column k: the T element
  for (int t2 = 0; t2 < n2; ++t2) {
    const RowTree& rt = X2.trees[t2];
    refs[t2].resize(X2.groups[rt.grp].K);
    for (const GatherSeg* q : rt.segs) {
      // A~2's rows of the tree are contiguous in T: row legs of strides 1, ext0, ext0 ext1, ...
      int64_t run = 1;
      for (int l = 0; l < q->nrl; ++l) {
        if (q->str[l] != run) return false;
        run *= q->ext[l];
      }
      if (run != rt.nrows) return false;
      for (int kk = 0; kk < q->nk; ++kk) {
        int g;
        int32_t r, c;
        if (!locate(q->src + q->colsrc[kk], g, r, c)) return false;
        auto jt = X1.tree_of.find({g, r});
        if (jt == X1.tree_of.end() || X1.trees[jt->second].nrows != rt.nrows) return false;
        refs[t2][q->k0 + kk] = Ref{jt->second, c, q->neg};
        parent[find_union(parent, n1 + t2)] = find_union(parent, jt->second);
      }
    }
  }
  // output permute of step 2 (C~2 -> C), abelian: folded into the stores (OutMap, tk_plan.cpp)
  std::unique_ptr<OutMap> om;
  if (!P2.pc.identity) {
    om = std::make_unique<OutMap>(P2.pc, P2.lc);
    if (!om->ok()) return false;
  }
  // classes, each one program
  std::map<int, std::vector<int>> cls;  // root -> members (step-1 trees < n1 <= step-2 trees)
  for (int i = 0; i < n1 + n2; ++i) cls[find_union(parent, i)].push_back(i);
  for (auto& kv : cls) {
    std::vector<int> t1s, t2s;
    for (int i : kv.second) (i < n1 ? t1s : t2s).push_back(i < n1 ? i : i - n1);
    if (t2s.empty()) return false;  // a step-1 row tree no step-2 tree reads (unreachable for a pair plan)
    const int Fr = X2.trees[t2s[0]].nrows;
    FusedHeader h{};
    h.F = Fr;
    {  // step-1 digit radix: every input subblock of the class must decompose f the same way
      const GatherSeg* s0 = X1.trees[t1s[0]].segs[0];
      if (s0->nrl > 3) return false;
      h.nrl = s0->nrl;
      for (int l = 0; l < 4; ++l) h.ext[l] = l < s0->nrl ? s0->ext[l] : 1;
    }
    std::vector<FusedIn> ins;
    std::vector<FusedT1> v1;
    std::vector<FusedT2> v2;
    std::vector<int32_t> midref, coef1, coef2;
    std::map<int, int> c1_of, c2_of;  // group -> its B~ table in coef1 / coef2
    std::map<int, int> mid0_of;       // step-1 tree -> its first T value
    for (int t : t1s) {
      const RowTree& rt = X1.trees[t];
      if (rt.nrows != Fr) return false;
      const GemmGroup& G = X1.groups[rt.grp];
      FusedT1 q{};
      q.in0 = (int32_t)ins.size();
      q.K = G.K;
      q.N = G.N;
      q.mid0 = h.n_mid;
      h.n_mid += G.N;
      for (const GatherSeg* s : rt.segs) {
        if (s->nrl != h.nrl) return false;
        for (int l = 0; l < s->nrl; ++l)
          if (s->ext[l] != h.ext[l]) return false;
        for (int kk = 0; kk < s->nk; ++kk) {
          if (ins.size() >= (size_t)kFusedMaxIn) return false;
          FusedIn x{};
          x.base = (int32_t)(s->src + s->colsrc[kk]);
          for (int l = 0; l < 3; ++l) x.str[l] = l < s->nrl ? s->str[l] : 0;
          if (s->neg) h.neg_in |= uint64_t(1) << ins.size();
          ins.push_back(x);
        }
      }
      auto it = c1_of.find(rt.grp);
      if (it == c1_of.end()) {
        it = c1_of.emplace(rt.grp, (int)coef1.size()).first;
        for (int k = 0; k < G.K; ++k)
          for (int n = 0; n < F.nm; ++n) coef1.push_back(n < G.N ? P1.btab[X1.bt[rt.grp] + k * G.N + n] : -1);
      }
      q.c0 = it->second;
      mid0_of[t] = q.mid0;
      v1.push_back(q);
    }
    std::vector<GatherOut> outs;
    for (int t : t2s) {
      const RowTree& rt = X2.trees[t];
      if (rt.nrows != Fr) return false;
      const GemmGroup& G = X2.groups[rt.grp];
      FusedT2 q{};
      q.o0 = (int32_t)outs.size();
      for (int n = 0; n < G.N; ++n) {
        GatherOut o{};
        if (P2.pc.identity) {  // C~2 is C: the tree's rows are contiguous
          o.base = G.c_off + rt.r0 + (int64_t)n * G.ldc;
          o.str[0] = 1;
          o.ext0 = Fr;
          o.ext1 = 1;
        } else if (!om->map(G.c_off + rt.r0 + (int64_t)n * G.ldc, Fr, o) ||
                   (n > 0 && (o.ext0 != outs[q.o0].ext0 || o.ext1 != outs[q.o0].ext1))) {
          return false;
        }
        outs.push_back(o);
      }
      q.K = G.K;
      q.N = G.N;
      q.r0 = (int32_t)midref.size();
      for (int k = 0; k < G.K; ++k) {
        const Ref& rf = refs[t][k];
        midref.push_back(2 * (mid0_of.at(rf.tree1) + rf.col) + (rf.neg ? 1 : 0));
      }
      auto it = c2_of.find(rt.grp);
      if (it == c2_of.end()) {
        it = c2_of.emplace(rt.grp, (int)coef2.size()).first;
        for (int k = 0; k < G.K; ++k)
          for (int n = 0; n < F.nm; ++n) coef2.push_back(n < G.N ? P2.btab[X2.bt[rt.grp] + k * G.N + n] : -1);
      }
      q.c0 = it->second;  // offset by n_coef1 below
      v2.push_back(q);
    }
    if (h.n_mid > kFusedMaxMid) return false;
    h.n_in = (int32_t)ins.size();
    h.n_t1 = (int32_t)v1.size();
    h.n_t2 = (int32_t)v2.size();
    h.n_ref = (int32_t)midref.size();
    h.n_out = (int32_t)outs.size();
    h.n_coef1 = (int32_t)coef1.size();
    h.n_coef = (int32_t)(coef1.size() + coef2.size());
    if (h.n_coef > kFusedMaxCoef) return false;
    for (FusedT2& q : v2) q.c0 += h.n_coef1;
    // serialise (8-byte words; programs 16-byte aligned: the header is read as int4)
    if (F.progs.size() & 1) F.progs.push_back(0);
    const int64_t prog = (int64_t)F.progs.size();
    auto put = [&](const void* p, size_t bytes) {
      const size_t w = (bytes + 7) / 8;
      const size_t at = F.progs.size();
      F.progs.resize(at + w, 0);
      if (bytes) std::memcpy(F.progs.data() + at, p, bytes);
    };
    put(&h, sizeof h);
    put(ins.data(), ins.size() * sizeof(FusedIn));
    put(v1.data(), v1.size() * sizeof(FusedT1));
    put(v2.data(), v2.size() * sizeof(FusedT2));
    put(outs.data(), outs.size() * sizeof(GatherOut));
    if (midref.size() & 1) midref.push_back(0);
    put(midref.data(), midref.size() * 4);
    coef1.insert(coef1.end(), coef2.begin(), coef2.end());
    put(coef1.data(), coef1.size() * 4);
    F.max_in = std::max(F.max_in, h.n_in);
    F.max_stage = std::max(F.max_stage, 2 * h.n_in + 4 * h.n_t1 + 3 * h.n_t2 + 4 * h.n_out + ((h.n_ref + 1) >> 1));
    F.max_mid = std::max(F.max_mid, h.n_mid);
    F.max_coef = std::max(F.max_coef, h.n_coef);
    if (plan_debug() && getenv("TK_FUSED_ALL"))
      fprintf(stderr, "[tk fused] class: F %d, trees %zu + %zu, n_in %d, n_mid %d, n_coef %d\n", Fr, t1s.size(),
              t2s.size(), h.n_in, h.n_mid, h.n_coef);
    for (int f0 = 0; f0 < Fr; f0 += 32) F.chunks.push_back(FusedChunk{prog, f0, std::min(32, Fr - f0)});
  }
  F.max_coef = (F.max_coef + 1) & ~1;
  // vmid [max_mid][threads] | per warp: coefficients [max_coef] + the staged program [max_stage] words
  F.max_stage = (F.max_stage + 1) & ~1;
  F.smem = (F.max_mid * kFusedThreads + (F.max_coef + F.max_stage) * kFusedWarps) * 8;
  if (plan_debug())
    fprintf(stderr, "[tk fused] %zu classes, max n_in %d, max n_mid %d, max n_coef %d, max staged words %d\n",
            cls.size(), F.max_in, F.max_mid, F.max_coef, F.max_stage);
  return F.smem <= 200 * 1024;
}

static PlanCache<FusedPlan> g_fused_cache;
size_t fused_cache_size() { return g_fused_cache.size(); }
void fused_cache_clear() { g_fused_cache.clear(); }

static std::shared_ptr<FusedPlan> get_fused_plan(const Tensor& A, const int32_t* labA, const Tensor& B1,
                                                 const int32_t* labB1, const Tensor& T, const int32_t* labT,
                                                 const Tensor& B2, const int32_t* labB2, const Tensor& C,
                                                 const int32_t* labC) {
  auto P1 = get_contract_plan(A, labA, B1, labB1, T, labT);
  auto P2 = get_contract_plan(T, labT, B2, labB2, C, labC);
  std::ostringstream os;
  os << (const void*)P1.get() << "#" << (const void*)P2.get();
  return g_fused_cache.get(os.str(), [&] {
    auto F = std::make_shared<FusedPlan>();
    F->p1 = P1;
    F->p2 = P2;
    static const bool off = knob("TK_NO_FUSE", 0) != 0;
    F->fused = !off && build_fused(*F);
    if (!F->fused) {
      F->progs.clear();
      F->chunks.clear();
      F->off_t = 0;
      F->off_ws = align256((size_t)T.nelems * 8);
      F->ws_bytes = F->off_ws + std::max(P1->ws_bytes, P2->ws_bytes);
    }
    if (plan_debug())
      fprintf(stderr, "[tk fused] %s: %zu chunks, %zu program words, %d B shared memory\n",
              F->fused ? "fused" : "two contractions", F->chunks.size(), F->progs.size(), F->smem);
    return F;
  });
}

static PerDeviceOnce g_fused_attr;

using FusedKern = void (*)(const double*, const double*, const double*, double*, const int64_t*, const FusedChunk*,
                           int, int, int, int, double, double, double);
static FusedKern fused_kernel_for(int nm) {
  return nm == 4 ? fused_pair_kernel<4> : nm == 6 ? fused_pair_kernel<6> : nm == 8 ? fused_pair_kernel<8>
                                                                   : fused_pair_kernel<16>;
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

tk_status tk_contract2_workspace(const tk_tensor* A, const int32_t* labA, const tk_tensor* B1, const int32_t* labB1,
                                 const tk_tensor* T, const int32_t* labT, const tk_tensor* B2, const int32_t* labB2,
                                 const tk_tensor* C, const int32_t* labC, size_t* bytes, int32_t* fused) {
  TK_API_BEGIN
  if (!A || !B1 || !T || !B2 || !C || !labA || !labB1 || !labT || !labB2 || !bytes)
    TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  auto F = get_fused_plan(*(const Tensor*)A, labA, *(const Tensor*)B1, labB1, *(const Tensor*)T, labT,
                          *(const Tensor*)B2, labB2, *(const Tensor*)C, labC);
  *bytes = F->ws_bytes;
  if (fused) *fused = F->fused ? 1 : 0;
  TK_API_END
}

tk_status tk_contract2(const tk_tensor* A_, const void* a, const int32_t* labA, const tk_tensor* B1_, const void* b1,
                       const int32_t* labB1, const tk_tensor* T_, const int32_t* labT, const tk_tensor* B2_,
                       const void* b2, const int32_t* labB2, const tk_tensor* C_, void* c, const int32_t* labC,
                       double alpha, double beta, void* ws, size_t ws_bytes, tk_stream stream) {
  TK_API_BEGIN
  if (!A_ || !B1_ || !T_ || !B2_ || !C_ || !labA || !labB1 || !labT || !labB2)
    TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  const Tensor& B1 = *(const Tensor*)B1_;
  const Tensor& T = *(const Tensor*)T_;
  const Tensor& B2 = *(const Tensor*)B2_;
  const Tensor& C = *(const Tensor*)C_;
  if ((!a && A.nelems) || (!b1 && B1.nelems) || (!b2 && B2.nelems) || (!c && C.nelems))
    TK_THROW(TK_ERR_INVALID_ARGUMENT, "null data pointer");
  if (A.dtype != T.dtype || T.dtype != C.dtype) TK_THROW(TK_ERR_INVALID_ARGUMENT, "dtypes differ");
  auto F = get_fused_plan(A, labA, B1, labB1, T, labT, B2, labB2, C, labC);
  if (ws_bytes < F->ws_bytes || (F->ws_bytes && !ws)) TK_THROW(TK_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
  if (((uintptr_t)ws & 255) != 0) TK_THROW(TK_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  if (!F->fused) {  // the two contractions as they are, T in the workspace
    char* w = (char*)ws;
    void* t = w + F->off_t;
    run_contract(F->p1.get(), a, b1, t, 0, 0, 1.0, 0.0, w + F->off_ws, ws_bytes - F->off_ws, stream);
    const int n1 = tk_last_launch_count();
    run_contract(F->p2.get(), t, b2, c, 0, 0, alpha, beta, w + F->off_ws, ws_bytes - F->off_ws, stream);
    add_launches(n1);
    return TK_OK;
  }
  F->ensure_uploaded();
  check_cuda(g_fused_attr.run([&] {
               cudaError_t e = cudaSuccess;
               for (int nm : {4, 6, 8, 16})
                 if (e == cudaSuccess)
                   e = cudaFuncSetAttribute(fused_kernel_for(nm), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            200 * 1024);
               return e;
             }),
             "fused kernel attribute");
  free_deferred(st);
  reset_launches();
  static const bool pdl = knob("TK_NO_PDL", 0) == 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((F->chunks.size() + kFusedWarps - 1) / kFusedWarps));
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = (size_t)F->smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  if (!F->chunks.empty()) {
    auto kern = fused_kernel_for(F->nm);
    check_cuda(cudaLaunchKernelEx(&cfg, kern, (const double*)a, (const double*)b1, (const double*)b2,
                                  (double*)c, (const int64_t*)F->d_progs.p, (const FusedChunk*)F->d_chunks.p,
                                  (int)F->chunks.size(), F->max_mid, F->max_coef, F->max_stage,
                                  F->p2->pc.identity ? alpha : 1.0, F->p2->pc.identity ? 1.0 : alpha, beta),
               "fused launch");
    add_launches(1);
  }
  TK_API_END
}

}  // extern "C"
