// C ABI: spaces, tensors, topological data (host only). See include/tk.h for the contract.
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <string>

#include "tk_internal.hpp"

namespace tk {
static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace tk

using namespace tk;

#define TK_API_BEGIN try {
#define TK_API_END                \
  return TK_OK;                   \
  }                               \
  catch (const tk::Error& e) {    \
    set_last_error(e.what());     \
    return e.code;                \
  }                               \
  catch (const std::exception& e) { \
    set_last_error(e.what());     \
    return TK_ERR_INVALID_ARGUMENT; \
  }

static Sector read_label(Kind k, const int32_t* p) {
  Sector s;
  s.v[0] = p[0];
  s.v[1] = kind_width(k) == 2 ? p[1] : 0;
  return s;
}

extern "C" {

const char* tk_last_error(void) { return g_last_error.c_str(); }
const char* tk_version(void) { return "tk_b200 0.1 (sm_100a)"; }

tk_status tk_space_create(const char* kind, int32_t n, const int32_t* labels, const int64_t* degs, int32_t is_dual,
                          tk_space** out) {
  TK_API_BEGIN
  if (!kind || !out || n < 0 || (n > 0 && (!labels || !degs))) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  Kind k = parse_kind(kind);
  int w = kind_width(k);
  std::vector<Sector> secs;
  std::vector<int64_t> d;
  for (int i = 0; i < n; ++i) {
    secs.push_back(read_label(k, labels + w * i));
    d.push_back(degs[i]);
  }
  *out = (tk_space*)make_space(k, secs, d, is_dual != 0);
  TK_API_END
}

// "U1[-2:3, 0:5]'", "SU2[0:1, 1/2:2]", "U1xU1[(1,-1):2, (0,0):1]"
tk_status tk_space_parse(const char* text, tk_space** out) {
  TK_API_BEGIN
  if (!text || !out) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  std::string s(text);
  std::string t;
  for (char ch : s)
    if (!std::isspace((unsigned char)ch)) t += ch;
  size_t lb = t.find('['), rb = t.rfind(']');
  if (lb == std::string::npos || rb == std::string::npos || rb < lb) TK_THROW(TK_ERR_INVALID_ARGUMENT, "bad space text");
  Kind k = parse_kind(t.substr(0, lb));
  bool dual = rb + 1 < t.size() && t[rb + 1] == '\'';
  std::string body = t.substr(lb + 1, rb - lb - 1);
  std::vector<Sector> secs;
  std::vector<int64_t> degs;
  size_t i = 0;
  // integer, or j / p/2 for a spin component (SU2 labels, the second entry of fU1xSU2): returns doubled
  auto parse_num = [&](size_t& j, bool spin) -> int32_t {
    size_t st = j;
    if (j < body.size() && (body[j] == '-' || body[j] == '+')) ++j;
    while (j < body.size() && std::isdigit((unsigned char)body[j])) ++j;
    long v = std::strtol(body.substr(st, j - st).c_str(), nullptr, 10);
    if (spin) {
      if (j < body.size() && body[j] == '/') {
        ++j;
        size_t st2 = j;
        while (j < body.size() && std::isdigit((unsigned char)body[j])) ++j;
        long den = std::strtol(body.substr(st2, j - st2).c_str(), nullptr, 10);
        if (den != 2) TK_THROW(TK_ERR_UNKNOWN_LABEL, "SU2 spins are j or j/2");
        return (int32_t)v;
      }
      return (int32_t)(2 * v);
    }
    return (int32_t)v;
  };
  while (i < body.size()) {
    Sector sc;
    if (body[i] == '(') {
      ++i;
      sc.v[0] = parse_num(i, k == Kind::FSU2SU2);
      if (i >= body.size() || body[i] != ',') TK_THROW(TK_ERR_INVALID_ARGUMENT, "bad tuple label");
      ++i;
      sc.v[1] = parse_num(i, k == Kind::FU1SU2 || k == Kind::FSU2SU2);
      if (i >= body.size() || body[i] != ')') TK_THROW(TK_ERR_INVALID_ARGUMENT, "bad tuple label");
      ++i;
    } else {
      sc.v[0] = parse_num(i, k == Kind::SU2);
    }
    if (i >= body.size() || body[i] != ':') TK_THROW(TK_ERR_INVALID_ARGUMENT, "expected ':'");
    ++i;
    size_t st = i;
    while (i < body.size() && std::isdigit((unsigned char)body[i])) ++i;
    degs.push_back(std::strtoll(body.substr(st, i - st).c_str(), nullptr, 10));
    secs.push_back(sc);
    if (i < body.size() && body[i] == ',') ++i;
  }
  *out = (tk_space*)make_space(k, secs, degs, dual);
  TK_API_END
}

tk_status tk_space_info(const tk_space* s_, int32_t* n, int64_t* dim, int32_t* is_dual, int32_t* width) {
  TK_API_BEGIN
  if (!s_) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null space");
  const Space* s = (const Space*)s_;
  if (n) *n = (int32_t)s->sectors.size();
  if (dim) {
    int64_t d = 0;
    for (size_t i = 0; i < s->sectors.size(); ++i) d += s->degs[i] * (int64_t)sector_dim(s->kind, s->sectors[i]);
    *dim = d;
  }
  if (is_dual) *is_dual = s->dual;
  if (width) *width = kind_width(s->kind);
  TK_API_END
}

tk_status tk_space_sectors(const tk_space* s_, int32_t* labels, int64_t* degs) {
  TK_API_BEGIN
  if (!s_) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null space");
  const Space* s = (const Space*)s_;
  int w = kind_width(s->kind);
  for (size_t i = 0; i < s->sectors.size(); ++i) {
    if (labels)
      for (int c = 0; c < w; ++c) labels[w * i + c] = s->sectors[i].v[c];
    if (degs) degs[i] = s->degs[i];
  }
  TK_API_END
}

tk_status tk_space_dual(const tk_space* s, tk_space** out) {
  TK_API_BEGIN
  if (!s || !out) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  *out = (tk_space*)dual_space((const Space*)s);
  TK_API_END
}

void tk_space_retain(tk_space* s) {
  if (s) ((Space*)s)->refs.fetch_add(1);
}
void tk_space_release(tk_space* s) {
  if (s && ((Space*)s)->refs.fetch_sub(1) == 1) delete (Space*)s;
}

tk_status tk_tensor_create(tk_dtype dtype, int32_t n_cod, tk_space* const* cod, int32_t n_dom, tk_space* const* dom,
                           tk_tensor** out) {
  TK_API_BEGIN
  if (!out || n_cod < 0 || n_dom < 0 || (n_cod && !cod) || (n_dom && !dom))
    TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  if (dtype != TK_F64 && dtype != TK_C64) TK_THROW(TK_ERR_INVALID_ARGUMENT, "bad dtype");
  std::vector<Space*> c, d;
  for (int i = 0; i < n_cod; ++i) {
    if (!cod[i]) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null space");
    c.push_back((Space*)cod[i]);
  }
  for (int i = 0; i < n_dom; ++i) {
    if (!dom[i]) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null space");
    d.push_back((Space*)dom[i]);
  }
  *out = (tk_tensor*)make_tensor(dtype, c, d);
  TK_API_END
}

tk_status tk_tensor_nelems(const tk_tensor* t, int64_t* n) {
  TK_API_BEGIN
  if (!t || !n) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  *n = ((const Tensor*)t)->nelems;
  TK_API_END
}

tk_status tk_tensor_info(const tk_tensor* t_, int32_t* n_cod, int32_t* n_dom, int32_t* dtype, int32_t* width,
                         int32_t* n_blocks, int32_t* n_sub, int32_t* key_len) {
  TK_API_BEGIN
  if (!t_) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null tensor");
  const Tensor* t = (const Tensor*)t_;
  if (n_cod) *n_cod = t->n_cod();
  if (n_dom) *n_dom = t->n_dom();
  if (dtype) *dtype = (int32_t)t->dtype;
  if (width) *width = kind_width(t->kind);
  if (n_blocks) *n_blocks = (int32_t)t->blocks.size();
  if (n_sub) *n_sub = (int32_t)t->subs.size();
  if (key_len) *key_len = t->key_len();
  TK_API_END
}

tk_status tk_tensor_blocks(const tk_tensor* t_, int32_t* coupled, int64_t* rows, int64_t* cols, int64_t* offset) {
  TK_API_BEGIN
  if (!t_) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null tensor");
  const Tensor* t = (const Tensor*)t_;
  int w = kind_width(t->kind);
  for (size_t i = 0; i < t->blocks.size(); ++i) {
    const Block& b = t->blocks[i];
    if (coupled)
      for (int c = 0; c < w; ++c) coupled[w * i + c] = b.coupled.v[c];
    if (rows) rows[i] = b.rows;
    if (cols) cols[i] = b.cols;
    if (offset) offset[i] = b.off;
  }
  TK_API_END
}

tk_status tk_tensor_subblocks(const tk_tensor* t_, int32_t* keys, int32_t* block, int64_t* row_off, int64_t* col_off,
                              int64_t* extents8, int64_t* offset) {
  TK_API_BEGIN
  if (!t_) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null tensor");
  const Tensor* t = (const Tensor*)t_;
  int kl = t->key_len();
  for (size_t i = 0; i < t->subs.size(); ++i) {
    const Subblock& sb = t->subs[i];
    if (keys) t->write_key((int)i, keys + kl * i);
    if (block) block[i] = sb.block;
    if (row_off) row_off[i] = sb.row_off;
    if (col_off) col_off[i] = sb.col_off;
    if (offset) offset[i] = sb.off;
    if (extents8) {
      int64_t* e = extents8 + 8 * i;
      int k = 0;
      for (auto d : t->s_tree((int)i).dims) e[k++] = d;
      for (auto d : t->f_tree((int)i).dims) e[k++] = d;
      while (k < 8) e[k++] = 0;
    }
  }
  TK_API_END
}

void tk_tensor_retain(tk_tensor* t) {
  if (t) ((Tensor*)t)->refs.fetch_add(1);
}
void tk_tensor_release(tk_tensor* t) {
  if (t && ((Tensor*)t)->refs.fetch_sub(1) == 1) delete (Tensor*)t;
}

tk_status tk_fsymbol(const char* kind, const int32_t* a, const int32_t* b, const int32_t* c, const int32_t* d,
                     const int32_t* e, const int32_t* f, double* out) {
  TK_API_BEGIN
  if (!kind || !a || !b || !c || !d || !e || !f || !out) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  Kind k = parse_kind(kind);
  *out = fsymbol(k, read_label(k, a), read_label(k, b), read_label(k, c), read_label(k, d), read_label(k, e),
                 read_label(k, f));
  TK_API_END
}

tk_status tk_rsymbol(const char* kind, const int32_t* a, const int32_t* b, const int32_t* c, double* out) {
  TK_API_BEGIN
  if (!kind || !a || !b || !c || !out) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  Kind k = parse_kind(kind);
  *out = rsymbol(k, read_label(k, a), read_label(k, b), read_label(k, c));
  TK_API_END
}

}  // extern "C"
