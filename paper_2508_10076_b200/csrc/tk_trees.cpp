// Fusion-tree-pair transformations for permute (Alg. 10): the planner's
// "transform", computed by localized moves -- never by fusion-tensor overlaps:
//
//   1. bend every domain leg, last first, to the end of the splitting tree
//      (bend along the right, eq. ftbendright: coefficient sqrt(d_c/d_e) B^{eb}_c,
//       times chi_b when the bent leg carried a Z);
//   2. braid to the target order by adjacent swaps found by bubble sort (footnote P:425-428):
//      swap of the first two legs = R-move (eq. Rmove); deeper swaps use the
//      F-R-F sequence (the alternative named in the footnote of P:1728-1730):
//        coef(e -> e') = sum_f F^{l a b}_t[e,f] R^{ab}_f F^{l b a}_t[e',f]
//   3. bend the trailing legs back to the domain.
// For abelian kinds all F, B, d, chi are 1 and this reduces to the Koszul sign of reading C13
// (koszul_sign below is the fast path the planner uses; tests check the two agree).
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <sstream>
#include <unordered_map>

#include "tk_internal.hpp"

namespace tk {

namespace {

struct State {
  Tree s, f;                 // dims unused here
  std::vector<int> s_ids, f_ids;    // original leg ids carried by each tree leg
  std::vector<bool> s_dual, f_dual;
};

std::vector<Sector> chain_of(const Tree& t) {
  // chain[k] = coupled label of the first k+1 legs
  size_t n = t.unc.size();
  std::vector<Sector> c;
  if (n == 0) return c;
  c.push_back(t.unc[0]);
  for (size_t k = 1; k + 1 < n; ++k) c.push_back(t.inner[k - 1]);
  if (n >= 2) c.push_back(t.coupled);
  return c;
}

void set_chain(Tree& t, const std::vector<Sector>& chain, Kind k) {
  size_t n = t.unc.size();
  t.inner.clear();
  if (n == 0) {
    t.coupled = sector_unit(k);
    return;
  }
  for (size_t i = 1; i + 1 < n; ++i) t.inner.push_back(chain[i]);
  t.coupled = chain[n - 1];
}

std::string state_key(const State& st) { return tree_pair_key(st.s, st.f); }

using Combo = std::map<std::string, std::pair<State, double>>;

void add_term(Combo& out, State&& st, double c) {
  if (c == 0.0) return;
  std::string key = state_key(st);
  auto it = out.find(key);
  if (it == out.end())
    out.emplace(key, std::make_pair(std::move(st), c));
  else
    it->second.second += c;
}

// move the last leg of `from` to the end of `to` (both trees share the coupled label c);
// the new coupled label e is the chain value of `from` before its last leg.
void bend_last(Kind k, Tree& from, std::vector<int>& from_ids, std::vector<bool>& from_dual, Tree& to,
               std::vector<int>& to_ids, std::vector<bool>& to_dual, double& coef) {
  size_t n = from.unc.size();
  Sector c = from.coupled;
  Sector b = from.unc[n - 1];
  bool was_dual = from_dual[n - 1];
  std::vector<Sector> ch = chain_of(from);
  Sector e = (n >= 2) ? ch[n - 2] : sector_unit(k);
  // shrink `from`
  from.unc.pop_back();
  std::vector<Sector> fch(ch.begin(), ch.end() - (n >= 1 ? 1 : 0));
  set_chain(from, fch, k);
  if (from.unc.empty()) from.coupled = sector_unit(k);
  int id = from_ids.back();
  from_ids.pop_back();
  from_dual.pop_back();
  // grow `to`: new leg label dual(b), new coupled e
  std::vector<Sector> tch = chain_of(to);
  to.unc.push_back(sector_dual(k, b));
  if (to.unc.size() == 1) {
    tch.assign(1, to.unc[0]);
  } else {
    tch.push_back(e);
  }
  set_chain(to, tch, k);
  if (to.unc.size() >= 2) to.coupled = e;
  to_ids.push_back(id);
  to_dual.push_back(!was_dual);
  double dc = sector_dim(k, c), de = sector_dim(k, e);
  coef *= std::sqrt(dc / de) * bsymbol(k, e, b, c);
  if (was_dual) coef *= sector_fs(k, b);
}

void braid(Kind k, const Combo& in, int i, Combo& out) {
  out.clear();
  std::vector<Sector> opts;
  for (auto& kv : in) {
    const State& st = kv.second.first;
    double c0 = kv.second.second;
    const Tree& t = st.s;
    std::vector<Sector> ch = chain_of(t);
    Sector a = t.unc[i], b = t.unc[i + 1];
    State ns = st;
    std::swap(ns.s.unc[i], ns.s.unc[i + 1]);
    std::swap(ns.s_ids[i], ns.s_ids[i + 1]);
    { bool tmpd = ns.s_dual[i]; ns.s_dual[i] = ns.s_dual[i + 1]; ns.s_dual[i + 1] = tmpd; }
    if (i == 0) {
      Sector e = ch[1];  // label fusing legs 0 and 1
      std::vector<Sector> nch = ch;
      nch[0] = b;
      set_chain(ns.s, nch, k);
      add_term(out, std::move(ns), c0 * rsymbol(k, a, b, e));
    } else {
      Sector l = ch[i - 1], e = ch[i], top = ch[i + 1];
      sector_fuse(k, l, b, opts);
      for (const Sector& ep : opts) {
        if (!sector_admissible(k, ep, a, top)) continue;
        double c = 0.0;
        std::vector<Sector> fs;
        sector_fuse(k, a, b, fs);
        for (const Sector& f : fs) {
          if (!sector_admissible(k, l, f, top)) continue;
          c += fsymbol(k, l, a, b, top, e, f) * rsymbol(k, a, b, f) * fsymbol(k, l, b, a, top, ep, f);
        }
        if (std::abs(c) < 1e-15) continue;
        State nn = ns;
        std::vector<Sector> nch = ch;
        nch[i] = ep;
        set_chain(nn.s, nch, k);
        add_term(out, std::move(nn), c0 * c);
      }
    }
  }
}

// Planar cyclic rotation of a codomain-only tree with unit coupled charge (all legs bent into the
// codomain): (a1, a2, ..., aN) -> (a2, ..., aN, a1), the planar move of Alg. 1/5 that needs
// no braiding. Two steps: (i) recouple a1 to the top, ((a1 a2)e2 a3)e3... = sum_f prod_k
// F^{a1 f_{k-1} a_k}_{e_k}[e_{k-1}, f_k] (a1 (a2 ... aN)_y)_I with y = dual(a1) (P:1117-1123 F-moves);
// (ii) carry a1 around the unit vertex to the right end, (a1 Y)_I -> (Y a1)_I, coefficient kappa(a1)
// (the left fold followed by a right bend): kappa = chi_{a1}, the Frobenius-Schur
// indicator -- the only choice that reproduces the dense SU(2) oracle for every cyclic transpose with
// dual legs, integer and half-integer spins (tests/test_library_host.py::test_planar_route_su2).
double g_rot_kappa_mode = 1;  // 0: 1, 1: chi_{a1}, 2: chi_{y} (validation knob for the test hook)

void rotate_left(Kind k, const Combo& in, Combo& out) {
  out.clear();
  for (auto& kv : in) {
    const State& st = kv.second.first;
    double c0 = kv.second.second;
    const Tree& t = st.s;
    const int n = (int)t.unc.size();
    State ns = st;
    std::rotate(ns.s.unc.begin(), ns.s.unc.begin() + 1, ns.s.unc.end());
    std::rotate(ns.s_ids.begin(), ns.s_ids.begin() + 1, ns.s_ids.end());
    { std::vector<bool> d(st.s_dual.begin() + 1, st.s_dual.end()); d.push_back(st.s_dual[0]); ns.s_dual = d; }
    if (n <= 1) {
      add_term(out, std::move(ns), c0);
      continue;
    }
    const Sector a1 = t.unc[0];
    const std::vector<Sector> ech = chain_of(t);  // e[0] = a1, e[k] = label of legs 0..k
    // paths over the chain of (a2 ... aN): f[0] = a2, f[k-1] fuses a2..a_{k+1}
    struct Path {
      std::vector<Sector> f;
      double c;
    };
    std::vector<Path> paths{{{t.unc[1]}, 1.0}};
    std::vector<Sector> opts;
    for (int kk = 2; kk < n; ++kk) {  // attach leg a_kk (0-based) to the right-hand subtree
      std::vector<Path> nx;
      for (auto& P : paths) {
        sector_fuse(k, P.f.back(), t.unc[kk], opts);
        for (const Sector& fnew : opts) {
          // ((a1 Y)_{e_{kk-1}} a_kk)_{e_kk} -> (a1 (Y a_kk)_{fnew})_{e_kk}
          double c = fsymbol(k, a1, P.f.back(), t.unc[kk], ech[kk], ech[kk - 1], fnew);
          if (std::abs(c) < 1e-15) continue;
          Path q = P;
          q.f.push_back(fnew);
          q.c *= c;
          nx.push_back(std::move(q));
        }
      }
      paths.swap(nx);
    }
    for (auto& P : paths) {
      const Sector y = P.f.back();
      if (!sector_admissible(k, a1, y, ech[n - 1])) continue;
      double kap = 1.0;
      if (g_rot_kappa_mode == 1) kap = sector_fs(k, a1);
      if (g_rot_kappa_mode == 2) kap = sector_fs(k, y);
      std::vector<Sector> nch = P.f;  // chain of (a2 ... aN a1): f..., then the unit
      nch.push_back(ech[n - 1]);
      State nn = ns;
      set_chain(nn.s, nch, k);
      add_term(out, std::move(nn), c0 * P.c * kap);
    }
  }
}

std::mutex g_memo_mu;
std::unordered_map<std::string, std::vector<TPTerm>> g_memo;  // memoised transforms
thread_local bool g_force_planar = false;

}  // namespace

void set_force_planar(bool on) { g_force_planar = on; }
void set_rotation_kappa_mode(int m) { g_rot_kappa_mode = m; }

bool is_planar_perm(int n1, const std::vector<int>& p, const std::vector<int>& q) {
  const int N = n1 + (int)(p.size() + q.size()) - n1;
  std::vector<int> S, T(p.begin(), p.end());
  for (int i = 0; i < n1; ++i) S.push_back(i);
  for (int i = N - 1; i >= n1; --i) S.push_back(i);
  for (int j = (int)q.size() - 1; j >= 0; --j) T.push_back(q[j]);
  if (N == 0) return true;
  for (int r = 0; r < N; ++r) {
    bool ok = true;
    for (int i = 0; i < N && ok; ++i) ok = T[i] == S[(i + r) % N];
    if (ok) return true;
  }
  return false;
}

void permute_tree_pair(Kind k, const Tree& s, const Tree& f, const std::vector<int>& p,
                       const std::vector<int>& q, const std::vector<bool>& isdual, std::vector<TPTerm>& out) {
  int n1 = (int)s.unc.size(), n2 = (int)f.unc.size(), N = n1 + n2;
  // planar route (cyclic rotations, no braiding): kinds without a real braiding, or forced (tests)
  const bool planar = !kind_braided(k) || g_force_planar;
  if (planar && !is_planar_perm(n1, p, q))
    TK_THROW(TK_ERR_BRAIDING_UNAVAILABLE, "non-planar permutation of a kind without (real) braiding");
  std::ostringstream mk;
  mk << (int)k << (planar ? "P" : "B") << g_rot_kappa_mode << "#" << tree_pair_key(s, f) << "#";
  for (int x : p) mk << x << ",";
  mk << "#";
  for (int x : q) mk << x << ",";
  mk << "#";
  for (bool d : isdual) mk << (d ? 1 : 0);
  std::string memo_key = mk.str();
  {
    std::lock_guard<std::mutex> g(g_memo_mu);
    auto it = g_memo.find(memo_key);
    if (it != g_memo.end()) {
      out = it->second;
      return;
    }
  }
  State st;
  st.s = s;
  st.f = f;
  for (int i = 0; i < n1; ++i) {
    st.s_ids.push_back(i);
    st.s_dual.push_back(isdual[i]);
  }
  for (int j = 0; j < n2; ++j) {
    st.f_ids.push_back(n1 + j);
    st.f_dual.push_back(isdual[n1 + j]);
  }
  double coef = 1.0;
  // 1. bend all domain legs to the codomain (last first)
  while (!st.f.unc.empty())
    bend_last(k, st.f, st.f_ids, st.f_dual, st.s, st.s_ids, st.s_dual, coef);
  Combo cur, nxt;
  add_term(cur, std::move(st), coef);
  // 2. braid into T = (p..., reversed q)
  std::vector<int> T(p.begin(), p.end());
  for (int j = (int)q.size() - 1; j >= 0; --j) T.push_back(q[j]);
  std::vector<int> pos(N);
  for (int i = 0; i < N; ++i) pos[T[i]] = i;
  std::vector<int> order = cur.begin()->second.first.s_ids;
  if (planar && N > 0) {  // rotate until the codomain order is T (a cyclic shift of S)
    int r = 0;
    while (r < N && order[r] != T[0]) ++r;
    for (int i = 0; i < r; ++i) {
      rotate_left(k, cur, nxt);
      std::swap(cur, nxt);
    }
    std::rotate(order.begin(), order.begin() + r, order.end());
  }
  for (int sweep = 0; sweep < N && !planar; ++sweep) {
    bool any = false;
    for (int i = 0; i + 1 < N; ++i) {
      if (pos[order[i]] > pos[order[i + 1]]) {
        braid(k, cur, i, nxt);
        std::swap(cur, nxt);
        std::swap(order[i], order[i + 1]);
        any = true;
      }
    }
    if (!any) break;
  }
  // 3. bend the trailing legs back: domain = (q_1, ..., q_N2')
  int n2p = (int)q.size();
  out.clear();
  for (auto& kv : cur) {
    State x = kv.second.first;
    double c = kv.second.second;
    for (int j = 0; j < n2p; ++j) bend_last(k, x.s, x.s_ids, x.s_dual, x.f, x.f_ids, x.f_dual, c);
    if (std::abs(c) < 1e-15) continue;
    TPTerm term;
    term.s = x.s;
    term.f = x.f;
    term.coef = c;
    out.push_back(std::move(term));
  }
  std::lock_guard<std::mutex> g(g_memo_mu);
  g_memo[memo_key] = out;
}

int koszul_sign(Kind k, const std::vector<Sector>& labels, int n1, const std::vector<int>& p,
                const std::vector<int>& q) {
  if (!kind_fermionic(k)) return 1;
  int N = (int)labels.size();
  int S[16], T[16], ps[16], pt[16];
  int idx = 0;
  for (int i = 0; i < n1; ++i) S[idx++] = i;
  for (int i = N - 1; i >= n1; --i) S[idx++] = i;
  idx = 0;
  for (int x : p) T[idx++] = x;
  for (int j = (int)q.size() - 1; j >= 0; --j) T[idx++] = q[j];
  for (int i = 0; i < N; ++i) {
    ps[S[i]] = i;
    pt[T[i]] = i;
  }
  int odd = 0;
  for (int x = 0; x < N; ++x) {
    if (!sector_parity(k, labels[x])) continue;
    for (int y = x + 1; y < N; ++y)
      if (sector_parity(k, labels[y]) && ((ps[x] < ps[y]) != (pt[x] < pt[y]))) odd ^= 1;
  }
  return odd ? -1 : 1;
}

}  // namespace tk
