// Internal types of libtk_b200 (host planner side). Not part of the ABI.
#pragma once
#include <array>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <unordered_map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tk.h"

namespace tk {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  tk_status code;
  Error(tk_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void set_last_error(const std::string& m);
#define TK_THROW(code, msg) throw ::tk::Error((code), (msg))

// Tuning knobs used for A/B experiments (job sizes, kernel-class thresholds). A product build compiles
// them to their defaults; only a build with -DTK_DEBUG_KNOBS (tools/build_variant.sh) reads the
// environment, so no environment variable can silently change kernel selection in the shipped library.
#ifdef TK_DEBUG_KNOBS
inline long long knob(const char* name, long long dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoll(v) : dflt;
}
#else
inline constexpr long long knob(const char*, long long dflt) { return dflt; }
#endif
// Diagnostic output only (plan statistics on stderr; never changes what runs): TK_PLAN_DEBUG=1.
inline bool plan_debug() {
  static const bool on = std::getenv("TK_PLAN_DEBUG") != nullptr;
  return on;
}

// ------------------------------------------------------------------ sectors
// Sector kinds (P:1011-1022 Z2; P:2347-2362 SVect; U1 S:138; Deligne products P:2380-2412;
// SU(2) P:2303-2332). Labels are up to two int32: Z2/fZ2 {g}, U1 {q}, U1xU1 {N, 2Sz}, SU2 {2j},
// fU1xSU2 {N, 2j}, fSU2xSU2 {2j_charge, 2j_spin}, Fib {0: I, 1: tau}, Ising {0: I, 1: sigma, 2: psi}.
enum class Kind : int { Z2 = 0, FZ2 = 1, U1 = 2, U1U1 = 3, FU1U1 = 4, SU2 = 5, FU1SU2 = 6, FSU2SU2 = 7, FIB = 8, ISING = 9 };

struct Sector {
  int32_t v[2] = {0, 0};
  bool operator<(const Sector& o) const { return v[0] != o.v[0] ? v[0] < o.v[0] : v[1] < o.v[1]; }
  bool operator==(const Sector& o) const { return v[0] == o.v[0] && v[1] == o.v[1]; }
  bool operator!=(const Sector& o) const { return !(*this == o); }
};

Kind parse_kind(const std::string& s);
const char* kind_name(Kind k);
int kind_width(Kind k);
bool kind_abelian(Kind k);
bool kind_fermionic(Kind k);
bool kind_braided(Kind k);  // false: planar operations only (Fib, Ising: complex R)
Sector sector_unit(Kind k);
Sector sector_dual(Kind k, const Sector& a);
void sector_validate(Kind k, const Sector& a);          // throws UNKNOWN_LABEL
void sector_fuse(Kind k, const Sector& a, const Sector& b, std::vector<Sector>& out);  // ascending
bool sector_admissible(Kind k, const Sector& a, const Sector& b, const Sector& c);
double sector_dim(Kind k, const Sector& a);
int sector_parity(Kind k, const Sector& a);
double sector_fs(Kind k, const Sector& a);                // Frobenius-Schur chi_a
// F^{abc}_d[e,f], R^{ab}_c and B^{ab}_c = sqrt(d_a d_b / d_c) F^{a b bbar}_a[c, I]
double fsymbol(Kind k, const Sector& a, const Sector& b, const Sector& c, const Sector& d,
               const Sector& e, const Sector& f);
double rsymbol(Kind k, const Sector& a, const Sector& b, const Sector& c);
double bsymbol(Kind k, const Sector& a, const Sector& b, const Sector& c);

// ------------------------------------------------------------------ spaces
struct Space {
  std::atomic<int> refs{1};
  Kind kind;
  std::vector<Sector> sectors;  // underlying V's sectors, ascending
  std::vector<int64_t> degs;
  bool dual = false;
  // tree labels (dual(a) for a dual space) with degeneracies, ascending by tree label
  std::vector<Sector> tree_labels;
  std::vector<int64_t> tree_degs;
  void finalize();
  int64_t deg_of_tree_label(const Sector& l) const;  // 0 if absent
  std::string signature() const;
};

// ------------------------------------------------------------------ trees / layout
struct Tree {
  std::vector<Sector> unc;    // uncoupled (tree labels)
  std::vector<Sector> inner;  // e_2 .. e_{N-1}
  Sector coupled;
  std::vector<int64_t> dims;
  int64_t size = 1;
};

struct Block {
  Sector coupled;
  int64_t rows = 0, cols = 0, off = 0;
  std::vector<Tree> cod_trees, dom_trees;
  std::vector<int64_t> row_off, col_off;  // per tree
};

struct Subblock {
  int block;
  int s, f;  // tree indices within the block
  int64_t row_off, col_off, off;
};

struct Tensor {
  std::atomic<int> refs{1};
  tk_dtype dtype;
  Kind kind;
  std::vector<Space*> cod, dom;
  std::vector<Block> blocks;
  std::vector<Subblock> subs;
  int64_t nelems = 0;
  std::string sig;                      // structural signature (plan-cache key part)
  std::unordered_map<std::string, int> sub_index; // tree-pair key -> subblock index
  ~Tensor();
  int n_cod() const { return (int)cod.size(); }
  int n_dom() const { return (int)dom.size(); }
  int nlegs() const { return n_cod() + n_dom(); }
  int key_len() const;
  void write_key(int sub, int32_t* out) const;
  const Tree& s_tree(int sub) const { return blocks[subs[sub].block].cod_trees[subs[sub].s]; }
  const Tree& f_tree(int sub) const { return blocks[subs[sub].block].dom_trees[subs[sub].f]; }
  int64_t ld(int sub) const { return blocks[subs[sub].block].rows; }
};

std::string tree_pair_key(const Tree& s, const Tree& f);
void enumerate_trees(Kind k, const std::vector<Space*>& legs, std::map<Sector, std::vector<Tree>>& out);
// rank 0 (no legs, a scalar: one 1 x 1 block at the unit sector) needs the kind from the caller
Tensor* make_tensor(tk_dtype dtype, const std::vector<Space*>& cod, const std::vector<Space*>& dom,
                    int kind_if_rank0 = -1);
Space* make_space(Kind k, std::vector<Sector> sectors, std::vector<int64_t> degs, bool dual);
Space* dual_space(const Space* s);
bool same_space(const Space* a, const Space* b);

// ------------------------------------------------------------------ tree transforms
// One term of a tree-pair transformation (Alg. 10 "transform"): destination tree pair and coefficient.
struct TPTerm {
  Tree s, f;
  double coef;
};
// Transform the tree pair (s, f) of a rank-(N1, N2) tensor under permute (p, q) with the given
// leg spaces' duality flags (isdual of A's legs in cod..dom order). Generic path: bend all domain
// legs to the codomain (B-symbols), braid by adjacent swaps (R-move P:1717-1726,
// F-R-F move P:1728-1743 footnote), bend back.
void permute_tree_pair(Kind k, const Tree& s, const Tree& f, const std::vector<int>& p,
                       const std::vector<int>& q, const std::vector<bool>& isdual,
                       std::vector<TPTerm>& out);
// Planar route (Alg. 1/5 cyclic transposes): used for kinds without a real braiding (Fib, Ising) and,
// through the test hook, to validate the rotation against SU(2)'s dense oracle.
bool is_planar_perm(int n1, const std::vector<int>& p, const std::vector<int>& q);
void set_force_planar(bool on);
void set_rotation_kappa_mode(int m);
// Reading C13 sign for abelian kinds (fast path; equals the generic path, tested).
int koszul_sign(Kind k, const std::vector<Sector>& labels, int n1, const std::vector<int>& p,
                const std::vector<int>& q);

}  // namespace tk
