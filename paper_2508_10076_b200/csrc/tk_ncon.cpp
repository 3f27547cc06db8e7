// ncon-style network contraction (@tensor networks) on top of the pairwise
// entry points: the network is contracted pair by pair in the caller's order, every step one
// tk_contract (Alg. 4) whose intermediate lands in the caller's workspace. See include/tk.h.
//
// Intermediates are the library's own, so their leg order is chosen here (the arithmetic does not
// depend on it: A~, B~ and C~ of every step are the same matrices whatever order an intermediate is
// stored in). Default: the producer's C~ order (open legs of A, then of B: no output permute). When the
// consumer would have to permute the intermediate in a separate pass (its A~ / B~ is not gathered) and
// the producer is a gathered GEMM that can store straight into that order (GatherOut: the abelian output
// permute folded into its stores), the intermediate is stored in the consumer's operand order instead:
// the consumer's permute pass disappears. Consecutive steps whose pair tk_contract2 fuses run as one
// call.
#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "tk_plan.hpp"

using namespace tk;

namespace {

struct Item {
  const tk_tensor* t;       // the tensor (borrowed input or owned intermediate)
  bool owned;
  std::vector<int32_t> lab;
  const void* data;         // input pointer, or nullptr for an intermediate (at ws + off)
  size_t off;
  bool pair_result = false; // output of a pairwise step (a partial trace of an input stands for the input)
};

struct Step {
  int a, b;                 // items contracted (b = -1: a partial trace of item a)
  std::vector<int32_t> labA, labB, labC;
  int32_t ncod;
  bool last;                // writes the network's output (alpha / beta, caller's buffer)
  std::vector<int32_t> pt, qt, p, q;  // trace steps: tk_trace arguments
};

// Walks the network: validates the labels, decides the pairwise steps, creates the intermediate
// HomSpaces and their workspace offsets. The final tensor's HomSpace is returned in *out (new
// reference) when `out` is non-null; the workspace size in *bytes.
void ncon_plan(int32_t n, const tk_tensor* const* T, const int32_t* const* labels, const int32_t* order, int32_t norder,
               int32_t n_cod_out, std::vector<Item>& items, std::vector<Step>& steps, size_t* bytes,
               tk_tensor** out) {
  if (n < 1 || !T || !labels) TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_ncon: no tensors");
  std::map<int32_t, int> count;
  int nneg = 0;
  for (int i = 0; i < n; ++i) {
    if (!T[i]) TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_ncon: null tensor");
    const Tensor& t = *(const Tensor*)T[i];
    if (t.nlegs() > 0 && !labels[i]) TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_ncon: null label list");
    Item it{T[i], false, {}, nullptr, 0};
    for (int l = 0; l < t.nlegs(); ++l) {
      const int32_t x = labels[i][l];
      if (x == 0) TK_THROW(TK_ERR_MALFORMED_NETWORK, "tk_ncon: label 0");
      if (x < 0) ++nneg;
      if (++count[x] > (x > 0 ? 2 : 1)) TK_THROW(TK_ERR_MALFORMED_NETWORK, "tk_ncon: label used too often");
      it.lab.push_back(x);
    }
    items.push_back(it);
  }
  for (auto& e : count) {
    if (e.first > 0 && e.second != 2) TK_THROW(TK_ERR_MALFORMED_NETWORK, "tk_ncon: a positive label must appear twice");
    if (e.first < -nneg) TK_THROW(TK_ERR_MALFORMED_NETWORK, "tk_ncon: open labels must be -1 .. -m");
  }
  if (n_cod_out < 0 || n_cod_out > nneg) TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_ncon: bad output codomain count");
  std::vector<int32_t> seq(order, order + std::max(norder, 0));
  for (int32_t x : seq)
    if (x <= 0 || !count.count(x)) TK_THROW(TK_ERR_UNKNOWN_LABEL, "tk_ncon: order names an unknown label");
  for (auto& e : count)
    if (e.first > 0 && std::find(seq.begin(), seq.end(), e.first) == seq.end())
      TK_THROW(TK_ERR_MALFORMED_NETWORK, "tk_ncon: order must list every contracted label");
  std::vector<int32_t> outlab;
  for (int k = 1; k <= nneg; ++k) outlab.push_back(-k);

  std::vector<bool> alive(items.size(), true);
  size_t off = 0, wsmax = 0;
  // a label twice on one tensor is a partial trace (Alg. 3): done first, by tk_trace, into
  // an intermediate that keeps the remaining legs in order (codomain legs stay codomain)
  for (int i = 0; i < n; ++i) {
    const Tensor& t = *(const Tensor*)items[i].t;
    Step s{i, -1, items[i].lab, {}, {}, 0, false, {}, {}, {}, {}};
    std::vector<bool> used(t.nlegs(), false);
    for (int x = 0; x < t.nlegs(); ++x)
      for (int y = x + 1; y < t.nlegs(); ++y)
        if (items[i].lab[x] == items[i].lab[y]) {
          // the ket leg is read as the codomain leg of the pair (include/tk.h, tk_trace)
          const Space* sx = x < t.n_cod() ? t.cod[x] : t.dom[x - t.n_cod()];
          const bool ket_x = !(sx->dual ^ (x >= t.n_cod()));
          s.pt.push_back(ket_x ? x : y);
          s.qt.push_back(ket_x ? y : x);
          used[x] = used[y] = true;
        }
    if (s.pt.empty()) continue;
    int nalive = 0;
    for (bool al : alive) nalive += al;
    for (int l = 0; l < t.nlegs(); ++l)
      if (!used[l]) (l < t.n_cod() ? s.p : s.q).push_back(l);
    for (int l : s.p) s.labC.push_back(items[i].lab[l]);
    for (int l : s.q) s.labC.push_back(items[i].lab[l]);
    s.ncod = (int32_t)s.p.size();
    if (nalive == 1 && n == 1) TK_THROW(TK_ERR_UNSUPPORTED, "tk_ncon: a single tensor (use tk_trace)");
    tk_tensor* C = nullptr;
    tk_status st = tk_trace_output(items[i].t, s.pt.data(), s.qt.data(), (int32_t)s.pt.size(), s.p.data(),
                                   (int32_t)s.p.size(), s.q.data(), (int32_t)s.q.size(), &C);
    if (st != TK_OK) TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
    size_t w = 0;
    st = tk_trace_workspace(items[i].t, s.pt.data(), s.qt.data(), (int32_t)s.pt.size(), s.p.data(),
                            (int32_t)s.p.size(), s.q.data(), (int32_t)s.q.size(), C, &w);
    if (st != TK_OK) {
      tk_tensor_release(C);
      TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
    }
    wsmax = std::max(wsmax, w);
    const Tensor& c = *(const Tensor*)C;
    items.push_back(Item{C, true, s.labC, nullptr, off});
    off = align256(off + (size_t)c.nelems * (c.dtype == TK_C64 ? 16 : 8));
    alive[i] = false;
    alive.push_back(true);
    steps.push_back(s);
  }
  auto contract_pair = [&](int a, int b) {
    Step s{a, b, items[a].lab, items[b].lab, {}, 0, false, {}, {}, {}, {}};
    std::vector<int32_t> oa, ob;
    for (int32_t x : s.labA)
      if (std::find(s.labB.begin(), s.labB.end(), x) == s.labB.end()) oa.push_back(x);
    for (int32_t x : s.labB)
      if (std::find(s.labA.begin(), s.labA.end(), x) == s.labA.end()) ob.push_back(x);
    int nalive = 0;
    for (bool al : alive) nalive += al;
    s.last = nalive == 2;
    if (s.last) {  // the network's output: legs -1, -2, ... with n_cod_out codomain legs
      s.labC = outlab;
      s.ncod = n_cod_out;
    } else {  // intermediates keep C~'s own order (open A ; open B): no output permute
      s.labC = oa;
      s.labC.insert(s.labC.end(), ob.begin(), ob.end());
      s.ncod = (int32_t)oa.size();
    }
    tk_tensor* C = nullptr;
    tk_status st = tk_contract_output(items[a].t, s.labA.data(), items[b].t, s.labB.data(), s.labC.data(), s.ncod, &C);
    if (st != TK_OK) TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
    size_t w = 0;
    st = tk_contract_workspace(items[a].t, s.labA.data(), items[b].t, s.labB.data(), C, s.labC.data(), &w);
    if (st != TK_OK) {
      tk_tensor_release(C);
      TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
    }
    wsmax = std::max(wsmax, w);
    const Tensor& c = *(const Tensor*)C;
    Item it{C, true, s.labC, nullptr, off, true};
    if (!s.last) off = align256(off + (size_t)c.nelems * (c.dtype == TK_C64 ? 16 : 8));
    alive[a] = alive[b] = false;
    items.push_back(it);
    alive.push_back(true);
    steps.push_back(s);
  };
  for (int32_t x : seq) {
    int a = -1, b = -1;
    for (int i = 0; i < (int)items.size(); ++i)
      if (alive[i] && std::find(items[i].lab.begin(), items[i].lab.end(), x) != items[i].lab.end())
        (a < 0 ? a : b) = i;
    if (a < 0) continue;  // contracted already (shared with an earlier label of the same pair)
    if (b < 0) TK_THROW(TK_ERR_MALFORMED_NETWORK, "tk_ncon: internal label bookkeeping");
    // a left fold: the running intermediate is the left operand A (two inputs: list order)
    if (items[b].pair_result && !items[a].pair_result) std::swap(a, b);
    contract_pair(a, b);
  }
  // disconnected pieces: outer products, left to right
  for (;;) {
    std::vector<int> al;
    for (int i = 0; i < (int)items.size(); ++i)
      if (alive[i]) al.push_back(i);
    if (al.size() < 2) break;
    contract_pair(al[0], al[1]);
  }
  if (steps.empty()) TK_THROW(TK_ERR_UNSUPPORTED, "tk_ncon: a single tensor (use tk_permute)");
  // intermediate leg orders (see the file comment): X = output of step k, consumed by step j > k. Last
  // step first: a decision reads the consumer's final output order, and only changes step k's.
  static const bool no_relabel = knob("TK_NCON_NO_RELABEL", 0) != 0;
  for (size_t k = steps.size(); k-- > 0 && !no_relabel;) {
    if (steps[k].last || steps[k].b < 0) continue;
    const int x = n + (int)k;
    size_t j = k + 1;
    while (j < steps.size() && steps[j].a != x && steps[j].b != x) ++j;
    if (j == steps.size() || steps[j].b < 0) continue;
    Step& c = steps[j];
    const bool isA = c.a == x;
    const Item& o = items[isA ? c.b : c.a];
    const Tensor& tx = *(const Tensor*)items[x].t;
    const Tensor& to = *(const Tensor*)o.t;
    {  // the consumer as planned now: nothing to do when its operand is gathered or already in place
      auto P = get_contract_plan(isA ? tx : to, c.labA.data(), isA ? to : tx, c.labB.data(),
                                 *(const Tensor*)items[n + (int)j].t, c.labC.data());
      if (P->gather || (isA ? P->pa.identity : P->pb.identity)) continue;
    }
    // the operand order of reading C2: A~ = (open legs in C's order | contracted legs in B's order),
    // B~ = (contracted legs in A's order | open legs in C's order)
    const std::vector<int32_t>& lx = items[x].lab;
    const std::vector<int32_t>& lo = o.lab;
    std::vector<int32_t> open, con;
    for (int32_t l : c.labC)
      if (std::find(lx.begin(), lx.end(), l) != lx.end()) open.push_back(l);
    for (int32_t l : lo)
      if (std::find(lx.begin(), lx.end(), l) != lx.end()) con.push_back(l);
    std::vector<int32_t> nl = isA ? open : con;
    nl.insert(nl.end(), (isA ? con : open).begin(), (isA ? con : open).end());
    if (nl.size() != lx.size()) continue;
    const int32_t ncod = (int32_t)(isA ? open.size() : con.size());
    Step& p = steps[k];
    tk_tensor* X = nullptr;
    tk_status st = tk_contract_output(items[p.a].t, p.labA.data(), items[p.b].t, p.labB.data(), nl.data(), ncod, &X);
    if (st != TK_OK) TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
    {  // only where the producer absorbs the moved permute (a gathered GEMM storing through the map):
       // anywhere else it would just move a pass (non-abelian recoupling permutes cost the same or more)
      auto Pp = get_contract_plan(*(const Tensor*)items[p.a].t, p.labA.data(), *(const Tensor*)items[p.b].t,
                                  p.labB.data(), *(const Tensor*)X, nl.data());
      if (!(Pp->gather && (Pp->gout || Pp->pc.identity))) {
        tk_tensor_release(X);
        continue;
      }
    }
    size_t w = 0;
    st = tk_contract_workspace(items[p.a].t, p.labA.data(), items[p.b].t, p.labB.data(), X, nl.data(), &w);
    if (st != TK_OK) {
      tk_tensor_release(X);
      TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
    }
    tk_tensor_release(const_cast<tk_tensor*>(items[x].t));
    items[x].t = X;  // same element count: the workspace offset stays
    items[x].lab = nl;
    p.labC = nl;
    p.ncod = ncod;
    (isA ? c.labA : c.labB) = nl;
    wsmax = std::max(wsmax, w);
    size_t w2 = 0;
    st = tk_contract_workspace(items[c.a].t, c.labA.data(), items[c.b].t, c.labB.data(), items[n + (int)j].t,
                               c.labC.data(), &w2);
    if (st != TK_OK) TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
    wsmax = std::max(wsmax, w2);
  }
  *bytes = off + wsmax;
  if (plan_debug())
    for (const Step& st : steps) {
      fprintf(stderr, "[tk ncon] step %d x %d ->", st.a, st.b);
      for (int32_t l : st.labC) fprintf(stderr, " %d", l);
      fprintf(stderr, " (ncod %d)\n", st.ncod);
    }
  if (out) {
    *out = const_cast<tk_tensor*>(items.back().t);
    items.back().owned = false;  // ownership moves to the caller
  }
}

// A planned network: the pairwise steps, the intermediate HomSpaces (owned) with their workspace offsets,
// the output HomSpace (owned) and the workspace size. Planning walks every intermediate's fusion-tree
// layout (cfg3's Alg. 12 chain: ~1 s of host time for a 190 us chain), so plans are cached like the
// pairwise plans: keyed by the inputs' structure signatures, the labels, the order and n_cod_out; the
// inputs of a cached plan are slots (the caller's tensors of the current call stand in for them).
struct NconPlan {
  std::vector<Item> items;
  std::vector<Step> steps;
  size_t bytes = 0;
  tk_tensor* out = nullptr;
  void ensure_uploaded() {}  // no device tables of its own (the pairwise plans hold them)
  ~NconPlan() {
    for (Item& it : items)
      if (it.owned) tk_tensor_release(const_cast<tk_tensor*>(it.t));
    if (out) tk_tensor_release(out);
  }
};

// a planned network owns its intermediates' block layouts (tens of MB of host memory for cfg3-sized
// chains), so this cache is kept much smaller than the pairwise ones
PlanCache<NconPlan> g_ncon_cache(64);

std::shared_ptr<NconPlan> get_ncon_plan(int32_t n, const tk_tensor* const* T, const int32_t* const* labels,
                                        const int32_t* order, int32_t norder, int32_t n_cod_out) {
  if (n < 1 || !T || !labels) TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_ncon: no tensors");
  if (norder > 0 && !order) TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_ncon: null order");
  std::string key = "N";
  for (int i = 0; i < n; ++i) {
    if (!T[i]) TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_ncon: null tensor");
    const Tensor& t = *(const Tensor*)T[i];
    if (t.nlegs() > 0 && !labels[i]) TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_ncon: null label list");
    key += "#" + t.sig + "#";
    for (int l = 0; l < t.nlegs(); ++l) key += std::to_string(labels[i][l]) + ",";
  }
  key += "#o";
  for (int i = 0; i < norder; ++i) key += std::to_string(order[i]) + ",";
  key += "#" + std::to_string(n_cod_out);
  return g_ncon_cache.get(key, [&] {
    auto P = std::make_shared<NconPlan>();  // a throw below frees the intermediates made so far
    ncon_plan(n, T, labels, order, norder, n_cod_out, P->items, P->steps, &P->bytes, &P->out);
    for (int i = 0; i < n; ++i) P->items[i].t = nullptr;  // input slots: never dereferenced from the cache
    return P;
  });
}

}  // namespace

namespace tk {
void ncon_cache_clear() { g_ncon_cache.clear(); }
size_t ncon_cache_size() { return g_ncon_cache.size(); }
}  // namespace tk

#define TK_API_BEGIN try {
#define TK_API_END                  \
  return TK_OK;                     \
  }                                 \
  catch (const tk::Error& e) {      \
    set_last_error(e.what());       \
    return e.code;                  \
  }                                 \
  catch (const std::exception& e) { \
    set_last_error(e.what());       \
    return TK_ERR_INVALID_ARGUMENT; \
  }

extern "C" {

tk_status tk_ncon_output(int32_t n, const tk_tensor* const* T, const int32_t* const* labels, const int32_t* order,
                         int32_t norder, int32_t n_cod_out, tk_tensor** out) {
  TK_API_BEGIN
  if (!out) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  auto P = get_ncon_plan(n, T, labels, order, norder, n_cod_out);
  tk_tensor_retain(P->out);  // the caller's own reference
  *out = P->out;
  TK_API_END
}

tk_status tk_ncon_workspace(int32_t n, const tk_tensor* const* T, const int32_t* const* labels, const int32_t* order,
                            int32_t norder, int32_t n_cod_out, size_t* bytes) {
  TK_API_BEGIN
  if (!bytes) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  *bytes = get_ncon_plan(n, T, labels, order, norder, n_cod_out)->bytes;
  TK_API_END
}

tk_status tk_ncon(int32_t n, const tk_tensor* const* T, const void* const* data, const int32_t* const* labels,
                  const int32_t* order, int32_t norder, int32_t n_cod_out, const tk_tensor* C, void* c, double alpha,
                  double beta, void* ws, size_t ws_bytes, tk_stream stream) {
  TK_API_BEGIN
  if (!data || !C) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  auto P = get_ncon_plan(n, T, labels, order, norder, n_cod_out);
  if (((const Tensor*)P->out)->sig != ((const Tensor*)C)->sig)
    TK_THROW(TK_ERR_SPACE_MISMATCH, "tk_ncon: C does not have the network's output HomSpace");
  const size_t bytes = P->bytes;
  if (ws_bytes < bytes || (bytes && !ws)) TK_THROW(TK_ERR_WORKSPACE_TOO_SMALL, "tk_ncon: workspace too small");
  if (((uintptr_t)ws & 255) != 0) TK_THROW(TK_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  std::vector<Item> items(P->items);  // this call's view: the caller's tensors and data in the input slots
  const std::vector<Step>& steps = P->steps;
  for (int i = 0; i < n; ++i) items[i].t = T[i];
  for (int i = 0; i < n; ++i) items[i].data = data[i];
  size_t inter = 0;  // intermediates occupy [0, inter) of the workspace, the pairwise scratch the rest
  for (const Item& it : items)
    if (it.owned && it.data == nullptr) {
      const Tensor& t = *(const Tensor*)it.t;
      inter = std::max(inter, align256(it.off + (size_t)t.nelems * (t.dtype == TK_C64 ? 16 : 8)));
    }
  char* w = (char*)ws;
  int launches = 0;
  for (size_t k = 0; k < steps.size(); ++k) {
    const Step& s = steps[k];
    Item& ia = items[s.a];
    if (s.b < 0) {  // partial trace of an input tensor
      Item& ic = items[n + k];
      const void* a = ia.data ? ia.data : (const void*)(w + ia.off);
      tk_status st = tk_trace(ia.t, a, s.pt.data(), s.qt.data(), (int32_t)s.pt.size(), s.p.data(), (int32_t)s.p.size(),
                              s.q.data(), (int32_t)s.q.size(), ic.t, w + ic.off, 1.0, 0.0, w + inter, ws_bytes - inter,
                              stream);
      if (st != TK_OK) TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
      launches += tk_last_launch_count();
      continue;
    }
    Item& ib = items[s.b];
    const void* a = ia.data ? ia.data : (const void*)(w + ia.off);
    const void* b = ib.data ? ib.data : (const void*)(w + ib.off);
    Item& ic = items[n + k];
    static const bool use_pair = knob("TK_NCON_FUSE", 1) != 0;
    if (use_pair && !s.last && k + 1 < steps.size() && steps[k + 1].a == n + (int)k && steps[k + 1].b >= 0) {
      // the pair (this step, the next) through tk_contract2: one kernel when it fuses
      const Step& s2 = steps[k + 1];
      Item& i2 = items[s2.b];
      Item& io = items[n + k + 1];
      const tk_tensor* C2 = s2.last ? C : io.t;
      size_t w2 = 0;
      int32_t fused = 0;
      tk_status st = tk_contract2_workspace(ia.t, s.labA.data(), ib.t, s.labB.data(), ic.t, s.labC.data(), i2.t,
                                            s2.labB.data(), C2, s2.labC.data(), &w2, &fused);
      if (st != TK_OK) TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
      if (fused && w2 <= ws_bytes - inter) {
        const void* b2 = i2.data ? i2.data : (const void*)(w + i2.off);
        void* c2 = s2.last ? c : (void*)(w + io.off);
        st = tk_contract2(ia.t, a, s.labA.data(), ib.t, b, s.labB.data(), ic.t, s.labC.data(), i2.t, b2,
                          s2.labB.data(), C2, c2, s2.labC.data(), s2.last ? alpha : 1.0, s2.last ? beta : 0.0,
                          w + inter, ws_bytes - inter, stream);
        if (st != TK_OK) TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
        launches += tk_last_launch_count();
        ++k;
        continue;
      }
    }
    void* cc = s.last ? c : (void*)(w + ic.off);
    const tk_tensor* Ct = s.last ? C : ic.t;
    tk_status st = tk_contract(ia.t, a, s.labA.data(), 0, ib.t, b, s.labB.data(), 0, Ct, cc, s.labC.data(),
                               s.last ? alpha : 1.0, s.last ? beta : 0.0, w + inter, ws_bytes - inter, stream);
    if (st != TK_OK) TK_THROW(st, std::string("tk_ncon: ") + tk_last_error());
    launches += tk_last_launch_count();
  }
  reset_launches();  // tk_last_launch_count: the whole network
  add_launches(launches);
  TK_API_END
}

}  // extern "C"
