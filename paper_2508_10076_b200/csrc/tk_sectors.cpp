// Sector algebra and topological data for the planner (host).
//
// Kinds and their data:
//   Z2       P:1011-1022 fusion table; bosonic (F = R = 1)
//   fZ2      SVect: F trivial (eq. trivialF), R^{JJ}_I = -1, chi = d = 1
//   U1       charge addition, dual = negation; bosonic
//   U1xU1    Deligne product U1 x U1: componentwise
//   fU1xU1   U1xU1 with fermion parity N mod 2 (BASELINE cfg3), i.e. fZ2 (x) U1 (x) U1 restricted;
//            R = (-1)^{p_a p_b} (Deligne product of R-symbols)
//   SU2      N^{j1j2}_{j3}, F via 6j (eq. SU2FSymbol, reading C9),
//            R^{j1j2}_{j3} = (-1)^{j1+j2-j3} (reading C8), chi_j = (-1)^{2j}
//   fU1xSU2  Hubbard fZ2 (x) U1 (x) SU2, labels (N, 2j), fermion parity N mod 2 (reading C14
//            as for fU1xU1): Deligne product data -- fusion componentwise, d = 2j+1,
//            F = F_SU2 on the spins (U1 and SVect F are trivial), R = R_SU2 * (-1)^{p_a p_b},
//            chi = (-1)^{2j} (SVect chi = 1)
//   fSU2xSU2 Hubbard at half filling, fZ2 (x) SU2 (x) SU2 (charge and spin SU(2)): labels
//            (2j_charge, 2j_spin), fermion parity 2j_spin mod 2 (the singly occupied spin-1/2 site is odd,
//            the empty/doubly occupied charge doublet even); Deligne product data: F = F(charge) F(spin),
//            R = R(charge) R(spin) (-1)^{p_a p_b}, d = (2jc+1)(2js+1), chi = (-1)^{2jc+2js}
//   Fib      {I, tau}: tau x tau = I + tau, d_tau = phi, F^{tau tau tau}_tau =
//            [[1/phi, 1/sqrt(phi)], [1/sqrt(phi), -1/phi]] over {I, tau}; R complex -> planar only
//   Ising    {I, sigma, psi}: sigma x sigma = I + psi, sigma x psi = sigma, psi x psi = I,
//            d_sigma = sqrt 2, F^{sss}_s = [[1, 1], [1, -1]] / sqrt 2 over {I, psi}, F^{s psi s}_psi[s, s] =
//            F^{psi s psi}_s[s, s] = -1; R complex -> planar only. chi = 1 for every anyon label.
// B-symbol: B^{ab}_c = sqrt(d_a d_b / d_c) F^{a b bbar}_a[c, I].
#include <cmath>
#include <cstring>

#include "tk_internal.hpp"

namespace tk {

Kind parse_kind(const std::string& s) {
  if (s == "Z2") return Kind::Z2;
  if (s == "fZ2") return Kind::FZ2;
  if (s == "U1") return Kind::U1;
  if (s == "U1xU1") return Kind::U1U1;
  if (s == "fU1xU1") return Kind::FU1U1;
  if (s == "SU2") return Kind::SU2;
  if (s == "fU1xSU2") return Kind::FU1SU2;
  if (s == "fSU2xSU2") return Kind::FSU2SU2;
  if (s == "Fib") return Kind::FIB;
  if (s == "Ising") return Kind::ISING;
  // the Deligne-product spellings of the fermionic kinds (reading C14: parity = N mod 2,
  // resp. 2 j_spin mod 2 -- the restricted products these kinds are)
  if (s == "fZ2xU1xU1") return Kind::FU1U1;
  if (s == "fZ2xU1xSU2") return Kind::FU1SU2;
  if (s == "fZ2xSU2xSU2") return Kind::FSU2SU2;
  TK_THROW(TK_ERR_UNKNOWN_LABEL, "unknown sector kind '" + s + "'");
}

const char* kind_name(Kind k) {
  static const char* names[] = {"Z2", "fZ2", "U1", "U1xU1", "fU1xU1", "SU2", "fU1xSU2", "fSU2xSU2", "Fib", "Ising"};
  return names[(int)k];
}

int kind_width(Kind k) {
  return (k == Kind::U1U1 || k == Kind::FU1U1 || k == Kind::FU1SU2 || k == Kind::FSU2SU2) ? 2 : 1;
}
bool kind_abelian(Kind k) {
  return k != Kind::SU2 && k != Kind::FU1SU2 && k != Kind::FSU2SU2 && k != Kind::FIB && k != Kind::ISING;
}
static bool kind_anyon(Kind k) { return k == Kind::FIB || k == Kind::ISING; }
bool kind_braided(Kind k) { return !kind_anyon(k); }
bool kind_fermionic(Kind k) {
  return k == Kind::FZ2 || k == Kind::FU1U1 || k == Kind::FU1SU2 || k == Kind::FSU2SU2;
}
// doubled spins of the SU(2) factors of a label (n = number of factors: 0, 1 or 2)
static int spins2(Kind k, const Sector& a, int* j) {
  switch (k) {
    case Kind::SU2: j[0] = a.v[0]; return 1;
    case Kind::FU1SU2: j[0] = a.v[1]; return 1;
    case Kind::FSU2SU2: j[0] = a.v[0]; j[1] = a.v[1]; return 2;
    default: return 0;
  }
}
Sector sector_unit(Kind) { return Sector{}; }

Sector sector_dual(Kind k, const Sector& a) {
  switch (k) {
    case Kind::Z2:
    case Kind::FZ2:
    case Kind::SU2:
    case Kind::FSU2SU2:
    case Kind::FIB:
    case Kind::ISING:
      return a;  // self-dual (SU2: "all irreps are self-dual"; Fib, Ising: P:2420)
    case Kind::U1:
      return Sector{{-a.v[0], 0}};
    case Kind::FU1SU2:
      return Sector{{-a.v[0], a.v[1]}};
    default:
      return Sector{{-a.v[0], -a.v[1]}};
  }
}

void sector_validate(Kind k, const Sector& a) {
  bool ok = true;
  switch (k) {
    case Kind::Z2:
    case Kind::FZ2:
      ok = (a.v[0] == 0 || a.v[0] == 1) && a.v[1] == 0;
      break;
    case Kind::U1:
      ok = a.v[1] == 0;
      break;
    case Kind::SU2:
      ok = a.v[0] >= 0 && a.v[1] == 0;
      break;
    case Kind::FU1SU2:
      ok = a.v[1] >= 0;
      break;
    case Kind::FSU2SU2:
      ok = a.v[0] >= 0 && a.v[1] >= 0;
      break;
    case Kind::FIB:
      ok = (a.v[0] == 0 || a.v[0] == 1) && a.v[1] == 0;
      break;
    case Kind::ISING:
      ok = a.v[0] >= 0 && a.v[0] <= 2 && a.v[1] == 0;
      break;
    default:
      break;
  }
  if (!ok) TK_THROW(TK_ERR_UNKNOWN_LABEL, std::string("invalid ") + kind_name(k) + " label");
}

void sector_fuse(Kind k, const Sector& a, const Sector& b, std::vector<Sector>& out) {
  out.clear();
  switch (k) {
    case Kind::Z2:
    case Kind::FZ2:
      out.push_back(Sector{{(a.v[0] + b.v[0]) & 1, 0}});
      break;
    case Kind::U1:
      out.push_back(Sector{{a.v[0] + b.v[0], 0}});
      break;
    case Kind::U1U1:
    case Kind::FU1U1:
      out.push_back(Sector{{a.v[0] + b.v[0], a.v[1] + b.v[1]}});
      break;
    case Kind::SU2: {
      int lo = std::abs(a.v[0] - b.v[0]), hi = a.v[0] + b.v[0];
      for (int j = lo; j <= hi; j += 2) out.push_back(Sector{{j, 0}});
      break;
    }
    case Kind::FU1SU2: {
      int lo = std::abs(a.v[1] - b.v[1]), hi = a.v[1] + b.v[1];
      for (int j = lo; j <= hi; j += 2) out.push_back(Sector{{a.v[0] + b.v[0], j}});
      break;
    }
    case Kind::FSU2SU2: {
      for (int jc = std::abs(a.v[0] - b.v[0]); jc <= a.v[0] + b.v[0]; jc += 2)
        for (int js = std::abs(a.v[1] - b.v[1]); js <= a.v[1] + b.v[1]; js += 2) out.push_back(Sector{{jc, js}});
      break;
    }
    case Kind::FIB:
      if (a.v[0] == 0) out.push_back(b);
      else if (b.v[0] == 0) out.push_back(a);
      else { out.push_back(Sector{{0, 0}}); out.push_back(Sector{{1, 0}}); }
      break;
    case Kind::ISING: {
      const int x = a.v[0], y = b.v[0];
      if (x == 0) out.push_back(b);
      else if (y == 0) out.push_back(a);
      else if (x == 1 && y == 1) { out.push_back(Sector{{0, 0}}); out.push_back(Sector{{2, 0}}); }
      else if (x == 2 && y == 2) out.push_back(Sector{{0, 0}});
      else out.push_back(Sector{{1, 0}});  // sigma x psi = psi x sigma = sigma
      break;
    }
  }
}

static bool su2_tri(int a, int b, int c) { return std::abs(a - b) <= c && c <= a + b && ((a + b + c) & 1) == 0; }

bool sector_admissible(Kind k, const Sector& a, const Sector& b, const Sector& c) {
  if (kind_anyon(k)) {
    std::vector<Sector> tmp;
    sector_fuse(k, a, b, tmp);
    for (auto& x : tmp)
      if (x == c) return true;
    return false;
  }
  if (k == Kind::SU2) return su2_tri(a.v[0], b.v[0], c.v[0]);
  if (k == Kind::FU1SU2) return c.v[0] == a.v[0] + b.v[0] && su2_tri(a.v[1], b.v[1], c.v[1]);
  if (k == Kind::FSU2SU2) return su2_tri(a.v[0], b.v[0], c.v[0]) && su2_tri(a.v[1], b.v[1], c.v[1]);
  std::vector<Sector> tmp;
  sector_fuse(k, a, b, tmp);
  return tmp[0] == c;
}

static const double kPhi = 0.5 * (1.0 + std::sqrt(5.0));
double sector_dim(Kind k, const Sector& a) {
  if (k == Kind::FIB) return a.v[0] == 1 ? kPhi : 1.0;
  if (k == Kind::ISING) return a.v[0] == 1 ? std::sqrt(2.0) : 1.0;
  int j[2] = {0, 0};
  int n = spins2(k, a, j);
  double d = 1.0;
  for (int i = 0; i < n; ++i) d *= (double)(j[i] + 1);
  return d;
}

int sector_parity(Kind k, const Sector& a) {
  if (k == Kind::FZ2) return a.v[0] & 1;
  if (k == Kind::FU1U1 || k == Kind::FU1SU2) return a.v[0] & 1;  // N mod 2 (two's complement: also N < 0)
  if (k == Kind::FSU2SU2) return a.v[1] & 1;                       // 2 j_spin mod 2
  return 0;
}

double sector_fs(Kind k, const Sector& a) {
  int j[2] = {0, 0};
  int n = spins2(k, a, j), t = 0;
  for (int i = 0; i < n; ++i) t += j[i];
  return (t & 1) ? -1.0 : 1.0;  // prod (-1)^{2j}; 1 for the abelian kinds and SVect
}

// ---- SU(2) 6j symbol via the Racah sum, long double factorials (doubled spins).
static long double lfact(int n) {
  static long double tab[256];
  static bool init = false;
  if (!init) {
    tab[0] = 1.0L;
    for (int i = 1; i < 256; ++i) tab[i] = tab[i - 1] * (long double)i;
    init = true;
  }
  if (n < 0 || n >= 256) TK_THROW(TK_ERR_UNSUPPORTED, "SU2 spin too large for the 6j table");
  return tab[n];
}

static long double tri_delta(int a, int b, int c) {
  return std::sqrt(lfact((a + b - c) / 2) * lfact((a - b + c) / 2) * lfact((-a + b + c) / 2) /
                   lfact((a + b + c) / 2 + 1));
}

static double sixj(int j1, int j2, int j3, int j4, int j5, int j6) {
  if (!su2_tri(j1, j2, j3) || !su2_tri(j1, j5, j6) || !su2_tri(j4, j2, j6) || !su2_tri(j4, j5, j3))
    return 0.0;
  long double pre = tri_delta(j1, j2, j3) * tri_delta(j1, j5, j6) * tri_delta(j4, j2, j6) * tri_delta(j4, j5, j3);
  int a1 = (j1 + j2 + j3) / 2, a2 = (j1 + j5 + j6) / 2, a3 = (j4 + j2 + j6) / 2, a4 = (j4 + j5 + j3) / 2;
  int b1 = (j1 + j2 + j4 + j5) / 2, b2 = (j2 + j3 + j5 + j6) / 2, b3 = (j3 + j1 + j6 + j4) / 2;
  int lo = std::max(std::max(a1, a2), std::max(a3, a4));
  int hi = std::min(b1, std::min(b2, b3));
  long double s = 0;
  for (int t = lo; t <= hi; ++t) {
    long double term = lfact(t + 1) / (lfact(t - a1) * lfact(t - a2) * lfact(t - a3) * lfact(t - a4) *
                                       lfact(b1 - t) * lfact(b2 - t) * lfact(b3 - t));
    s += (t & 1) ? -term : term;
  }
  return (double)(pre * s);
}

double fsymbol(Kind k, const Sector& a, const Sector& b, const Sector& c, const Sector& d,
               const Sector& e, const Sector& f) {
  if (!sector_admissible(k, a, b, e) || !sector_admissible(k, e, c, d) || !sector_admissible(k, b, c, f) ||
      !sector_admissible(k, a, f, d))
    return 0.0;
  if (kind_abelian(k)) return 1.0;  // abelian / SVect: trivial F (eq. trivialF)
  if (k == Kind::FIB) {
    if (a.v[0] == 1 && b.v[0] == 1 && c.v[0] == 1 && d.v[0] == 1) {
      const int i = e.v[0], j = f.v[0];  // basis order {I, tau}
      if (i == 0 && j == 0) return 1.0 / kPhi;
      if (i == 1 && j == 1) return -1.0 / kPhi;
      return 1.0 / std::sqrt(kPhi);
    }
    return 1.0;
  }
  if (k == Kind::ISING) {
    const int A = a.v[0], B = b.v[0], C = c.v[0], D = d.v[0];
    if (A == 1 && B == 1 && C == 1 && D == 1) {  // e, f in {I, psi}
      const double r = 1.0 / std::sqrt(2.0);
      return (e.v[0] == 2 && f.v[0] == 2) ? -r : r;
    }
    if (A == 1 && B == 2 && C == 1 && D == 2) return -1.0;  // F^{s psi s}_psi[s, s]
    if (A == 2 && B == 1 && C == 2 && D == 1) return -1.0;  // F^{psi s psi}_s[s, s]
    return 1.0;
  }
  // SU(2) factors (Deligne product: F is the product of the factors' F)
  int ja[2], jb[2], jc[2], jd[2], je[2], jf[2];
  int n = spins2(k, a, ja);
  spins2(k, b, jb);
  spins2(k, c, jc);
  spins2(k, d, jd);
  spins2(k, e, je);
  spins2(k, f, jf);
  double r = 1.0;
  for (int i = 0; i < n; ++i) {
    double sg = (((ja[i] + jb[i] + jc[i] + jd[i]) / 2) & 1) ? -1.0 : 1.0;
    r *= std::sqrt((double)(je[i] + 1) * (double)(jf[i] + 1)) * sg * sixj(ja[i], jb[i], je[i], jc[i], jd[i], jf[i]);
  }
  return r;
}

double rsymbol(Kind k, const Sector& a, const Sector& b, const Sector& c) {
  if (kind_anyon(k)) TK_THROW(TK_ERR_BRAIDING_UNAVAILABLE, "Fib / Ising R-symbols are complex phases (P:2426, P:2447)");
  if (!sector_admissible(k, a, b, c)) return 0.0;
  double r = 1.0;
  int ja[2], jb[2], jc[2];
  int n = spins2(k, a, ja);
  spins2(k, b, jb);
  spins2(k, c, jc);
  for (int i = 0; i < n; ++i)  // SU(2) factors, reading C8
    if (((ja[i] + jb[i] - jc[i]) / 2) & 1) r = -r;
  if (kind_fermionic(k) && (sector_parity(k, a) & sector_parity(k, b))) r = -r;  // SVect factor
  return r;  // Deligne product of R-symbols
}

double bsymbol(Kind k, const Sector& a, const Sector& b, const Sector& c) {
  if (!sector_admissible(k, a, b, c)) return 0.0;
  if (kind_abelian(k)) return 1.0;
  Sector bb = sector_dual(k, b);
  double da = sector_dim(k, a), db = sector_dim(k, b), dc = sector_dim(k, c);
  return std::sqrt(da * db / dc) * fsymbol(k, a, b, bb, a, c, sector_unit(k));
}

}  // namespace tk
