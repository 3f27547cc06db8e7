// Graded spaces, canonical fusion trees and the block layout of a tensor map (host).
//
// Spaces: V = (+)_a C^{N_a} (x) V^(a); a dual leg's trees carry the dual label
// ("use the sector as if it were a normal space"; reading C6).
// Trees: canonical left-to-right fusion/splitting trees: uncoupled a_1..a_N,
// inner e_2..e_{N-1}, coupled e_N; for N = 0 the coupled label is the unit.
// Layout (readings C4/C5; eq. abeliangrouping; embedding P:1786-1790): blocks by
// coupled label ascending; trees in a block by (uncoupled tuple, first leg most significant;
// then inner labels); block c is a column-major rows(c) x cols(c) matrix; blocks concatenated.
#include <algorithm>
#include <cstring>
#include <sstream>

#include "tk_internal.hpp"

namespace tk {

void Space::finalize() {
  std::vector<std::pair<Sector, int64_t>> tl;
  for (size_t i = 0; i < sectors.size(); ++i)
    tl.push_back({dual ? sector_dual(kind, sectors[i]) : sectors[i], degs[i]});
  std::sort(tl.begin(), tl.end(), [](auto& x, auto& y) { return x.first < y.first; });
  tree_labels.clear();
  tree_degs.clear();
  for (auto& p : tl) {
    tree_labels.push_back(p.first);
    tree_degs.push_back(p.second);
  }
}

int64_t Space::deg_of_tree_label(const Sector& l) const {
  auto it = std::lower_bound(tree_labels.begin(), tree_labels.end(), l);
  if (it == tree_labels.end() || *it != l) return 0;
  return tree_degs[it - tree_labels.begin()];
}

std::string Space::signature() const {
  std::ostringstream os;
  os << kind_name(kind) << (dual ? "*" : "") << "[";
  for (size_t i = 0; i < sectors.size(); ++i) os << sectors[i].v[0] << "," << sectors[i].v[1] << ":" << degs[i] << ";";
  os << "]";
  return os.str();
}

Space* make_space(Kind k, std::vector<Sector> secs, std::vector<int64_t> degs, bool dual) {
  std::vector<std::pair<Sector, int64_t>> v;
  for (size_t i = 0; i < secs.size(); ++i) {
    sector_validate(k, secs[i]);
    if (degs[i] < 0) TK_THROW(TK_ERR_INVALID_ARGUMENT, "negative degeneracy");
    if (degs[i] > 0) v.push_back({secs[i], degs[i]});
  }
  std::sort(v.begin(), v.end(), [](auto& x, auto& y) { return x.first < y.first; });
  for (size_t i = 1; i < v.size(); ++i)
    if (v[i].first == v[i - 1].first) TK_THROW(TK_ERR_INVALID_ARGUMENT, "duplicate sector label");
  Space* s = new Space();
  s->kind = k;
  for (auto& p : v) {
    s->sectors.push_back(p.first);
    s->degs.push_back(p.second);
  }
  s->dual = dual;
  s->finalize();
  return s;
}

Space* dual_space(const Space* s) { return make_space(s->kind, s->sectors, s->degs, !s->dual); }

bool same_space(const Space* a, const Space* b) {
  return a->kind == b->kind && a->dual == b->dual && a->sectors == b->sectors && a->degs == b->degs;
}

// ---------------------------------------------------------------- trees
static void inner_sequences(Kind k, const std::vector<Sector>& unc,
                            std::vector<std::pair<std::vector<Sector>, Sector>>& out) {
  out.clear();
  size_t n = unc.size();
  if (n == 0) {
    out.push_back({{}, sector_unit(k)});
    return;
  }
  if (n == 1) {
    out.push_back({{}, unc[0]});
    return;
  }
  std::vector<Sector> chain;
  std::vector<Sector> tmp;
  // iterative DFS in lexicographic order of (e_2, ..., e_N)
  struct Frame {
    std::vector<Sector> opts;
    size_t i;
  };
  std::vector<Frame> st;
  sector_fuse(k, unc[0], unc[1], tmp);
  st.push_back({tmp, 0});
  while (!st.empty()) {
    Frame& fr = st.back();
    if (fr.i >= fr.opts.size()) {
      st.pop_back();
      if (!chain.empty()) chain.pop_back();
      continue;
    }
    Sector e = fr.opts[fr.i++];
    chain.push_back(e);
    size_t depth = chain.size();  // number of inner+coupled labels so far: e_2..e_{depth+1}
    if (depth + 1 == n) {
      out.push_back({std::vector<Sector>(chain.begin(), chain.end() - 1), chain.back()});
      chain.pop_back();
    } else {
      sector_fuse(k, e, unc[depth + 1], tmp);
      st.push_back({tmp, 0});
    }
  }
}

void enumerate_trees(Kind k, const std::vector<Space*>& legs, std::map<Sector, std::vector<Tree>>& out) {
  out.clear();
  size_t n = legs.size();
  std::vector<size_t> idx(n, 0);
  for (auto* s : legs)
    if (s->tree_labels.empty()) return;  // empty space: no trees
  std::vector<std::pair<std::vector<Sector>, Sector>> seqs;
  while (true) {
    Tree t;
    for (size_t i = 0; i < n; ++i) {
      t.unc.push_back(legs[i]->tree_labels[idx[i]]);
      t.dims.push_back(legs[i]->tree_degs[idx[i]]);
      t.size *= legs[i]->tree_degs[idx[i]];
    }
    inner_sequences(k, t.unc, seqs);
    for (auto& sq : seqs) {
      Tree u = t;
      u.inner = sq.first;
      u.coupled = sq.second;
      out[u.coupled].push_back(std::move(u));
    }
    // advance: last leg fastest => first leg most significant
    int i = (int)n - 1;
    while (i >= 0) {
      if (++idx[i] < legs[i]->tree_labels.size()) break;
      idx[i] = 0;
      --i;
    }
    if (i < 0) break;
  }
}

// Binary key of a tree pair (uncoupled | inner | coupled | uncoupled | inner labels, 8 bytes per sector, a
// marker between the lists): built per subblock of every tensor and per planner lookup, so no streams here.
static inline void put_sector(std::string& k, const Sector& s) { k.append(reinterpret_cast<const char*>(s.v), 8); }

std::string tree_pair_key(const Tree& s, const Tree& f) {
  static const int32_t bar[2] = {INT32_MIN, INT32_MIN};
  std::string k;
  k.reserve(8 * (s.unc.size() + s.inner.size() + f.unc.size() + f.inner.size() + 5));
  for (auto& x : s.unc) put_sector(k, x);
  k.append(reinterpret_cast<const char*>(bar), 8);
  for (auto& x : s.inner) put_sector(k, x);
  k.append(reinterpret_cast<const char*>(bar), 8);
  put_sector(k, s.coupled);
  k.append(reinterpret_cast<const char*>(bar), 8);
  for (auto& x : f.unc) put_sector(k, x);
  k.append(reinterpret_cast<const char*>(bar), 8);
  for (auto& x : f.inner) put_sector(k, x);
  return k;
}

Tensor::~Tensor() {
  for (auto* s : cod) tk_space_release((tk_space*)s);
  for (auto* s : dom) tk_space_release((tk_space*)s);
}

int Tensor::key_len() const {
  int n1 = n_cod(), n2 = n_dom();
  return kind_width(kind) * (n1 + std::max(n1 - 2, 0) + 1 + n2 + std::max(n2 - 2, 0));
}

void Tensor::write_key(int sub, int32_t* out) const {
  int w = kind_width(kind);
  const Tree& s = s_tree(sub);
  const Tree& f = f_tree(sub);
  auto put = [&](const Sector& x) {
    for (int i = 0; i < w; ++i) *out++ = x.v[i];
  };
  for (auto& x : s.unc) put(x);
  for (auto& x : s.inner) put(x);
  put(s.coupled);
  for (auto& x : f.unc) put(x);
  for (auto& x : f.inner) put(x);
}

Tensor* make_tensor(tk_dtype dtype, const std::vector<Space*>& cod, const std::vector<Space*>& dom,
                    int kind_if_rank0) {
  if (cod.empty() && dom.empty() && kind_if_rank0 < 0)
    TK_THROW(TK_ERR_INVALID_ARGUMENT, "tensor with no legs (its sector kind is unknown)");
  Kind k = !cod.empty() ? cod[0]->kind : (!dom.empty() ? dom[0]->kind : (Kind)kind_if_rank0);
  for (auto* s : cod)
    if (s->kind != k) TK_THROW(TK_ERR_SECTOR_MISMATCH, "legs of different sector kinds");
  for (auto* s : dom)
    if (s->kind != k) TK_THROW(TK_ERR_SECTOR_MISMATCH, "legs of different sector kinds");
  if (cod.size() + dom.size() > 8) TK_THROW(TK_ERR_UNSUPPORTED, "at most 8 legs");
  Tensor* t = new Tensor();
  t->dtype = dtype;
  t->kind = k;
  t->cod = cod;
  t->dom = dom;
  for (auto* s : cod) tk_space_retain((tk_space*)s);
  for (auto* s : dom) tk_space_retain((tk_space*)s);
  std::map<Sector, std::vector<Tree>> ct, dt;
  enumerate_trees(k, cod, ct);
  enumerate_trees(k, dom, dt);
  int64_t off = 0;
  for (auto& kv : ct) {
    auto it = dt.find(kv.first);
    if (it == dt.end()) continue;
    Block b;
    b.coupled = kv.first;
    b.cod_trees = std::move(kv.second);  // each coupled sector makes one block: the lists move
    b.dom_trees = std::move(it->second);
    for (auto& tr : b.cod_trees) {
      b.row_off.push_back(b.rows);
      b.rows += tr.size;
    }
    for (auto& tr : b.dom_trees) {
      b.col_off.push_back(b.cols);
      b.cols += tr.size;
    }
    b.off = off;
    off += b.rows * b.cols;
    t->blocks.push_back(std::move(b));
  }
  t->nelems = off;
  for (int bi = 0; bi < (int)t->blocks.size(); ++bi) {
    const Block& b = t->blocks[bi];
    for (int f = 0; f < (int)b.dom_trees.size(); ++f)
      for (int s = 0; s < (int)b.cod_trees.size(); ++s) {
        Subblock sb;
        sb.block = bi;
        sb.s = s;
        sb.f = f;
        sb.row_off = b.row_off[s];
        sb.col_off = b.col_off[f];
        sb.off = b.off + sb.row_off + b.rows * sb.col_off;
        t->sub_index[tree_pair_key(b.cod_trees[s], b.dom_trees[f])] = (int)t->subs.size();
        t->subs.push_back(sb);
      }
  }
  std::ostringstream os;
  os << (int)dtype << "|" << kind_name(k) << "|" << cod.size() << "|";
  for (auto* s : cod) os << s->signature();
  os << "|";
  for (auto* s : dom) os << s->signature();
  t->sig = os.str();
  return t;
}

}  // namespace tk
