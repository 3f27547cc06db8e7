// Host planner: permute plans (Alg. 6 / Alg. 10) and contraction plans (Alg. 4 / Alg. 8),
// memoised in a mutex-guarded cache, plus the device-side C ABI calls.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>

#include <cuda_runtime.h>

#include "tk_internal.hpp"
#include "tk_kernels.hpp"
#include "tk_plan.hpp"
#include "tk_gemm_tma.hpp"

namespace tk {

static std::vector<int> dst_from_src_legs(const std::vector<int>& p, const std::vector<int>& q) {
  std::vector<int> v(p.begin(), p.end());
  v.insert(v.end(), q.begin(), q.end());
  return v;
}

void validate_perm(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q) {
  int N = A.nlegs();
  if ((int)(p.size() + q.size()) != N) TK_THROW(TK_ERR_INVALID_PERMUTATION, "|p| + |q| != number of legs");
  std::vector<int> seen(N, 0);
  for (int x : p) {
    if (x < 0 || x >= N || seen[x]++) TK_THROW(TK_ERR_INVALID_PERMUTATION, "(p, q) is not a permutation");
  }
  for (int x : q) {
    if (x < 0 || x >= N || seen[x]++) TK_THROW(TK_ERR_INVALID_PERMUTATION, "(p, q) is not a permutation");
  }
}

// Space selection rule of Alg. 2.
void permuted_spaces(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q,
                            std::vector<Space*>& cod, std::vector<Space*>& dom) {
  int n1 = A.n_cod();
  auto leg = [&](int i) -> Space* { return i < n1 ? A.cod[i] : A.dom[i - n1]; };
  cod.clear();
  dom.clear();
  for (int i : p) cod.push_back(i < n1 ? tk::make_space(leg(i)->kind, leg(i)->sectors, leg(i)->degs, leg(i)->dual)
                                       : dual_space(leg(i)));
  for (int j : q) dom.push_back(j < n1 ? dual_space(leg(j))
                                       : tk::make_space(leg(j)->kind, leg(j)->sectors, leg(j)->degs, leg(j)->dual));
}

void check_target(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q, const Tensor& C) {
  if (C.n_cod() != (int)p.size() || C.n_dom() != (int)q.size())
    TK_THROW(TK_ERR_SPACE_MISMATCH, "output tensor has the wrong number of codomain/domain legs");
  if (C.kind != A.kind) TK_THROW(TK_ERR_SECTOR_MISMATCH, "sector kinds differ");
  std::vector<Space*> cod, dom;
  permuted_spaces(A, p, q, cod, dom);
  bool ok = true;
  for (size_t i = 0; i < cod.size(); ++i) ok = ok && same_space(cod[i], C.cod[i]);
  for (size_t j = 0; j < dom.size(); ++j) ok = ok && same_space(dom[j], C.dom[j]);
  for (auto* s : cod) tk_space_release((tk_space*)s);
  for (auto* s : dom) tk_space_release((tk_space*)s);
  if (!ok) TK_THROW(TK_ERR_SPACE_MISMATCH, "output spaces differ from the permuted spaces (Alg. 2 selection rule)");
}

static Tree abelian_tree(Kind k, const std::vector<Sector>& unc) {
  Tree t;
  t.unc = unc;
  std::vector<Sector> tmp;
  Sector e = unc.empty() ? sector_unit(k) : unc[0];
  std::vector<Sector> chain;
  if (!unc.empty()) chain.push_back(e);
  for (size_t i = 1; i < unc.size(); ++i) {
    sector_fuse(k, e, unc[i], tmp);
    e = tmp[0];
    chain.push_back(e);
  }
  for (size_t i = 1; i + 1 < unc.size(); ++i) t.inner.push_back(chain[i]);
  t.coupled = unc.empty() ? sector_unit(k) : e;
  return t;
}

// per-leg strides (a, b) of a subblock: codomain legs (a = prod of previous cod extents, b = 0),
// domain legs (a = 0, b = prod of previous dom extents); element stride = a + b * ld.
static void leg_strides(const std::vector<int64_t>& ext, int n1, std::vector<int64_t>& a, std::vector<int64_t>& b) {
  int N = (int)ext.size();
  a.assign(N, 0);
  b.assign(N, 0);
  int64_t s = 1;
  for (int i = 0; i < n1; ++i) {
    a[i] = s;
    s *= ext[i];
  }
  s = 1;
  for (int i = n1; i < N; ++i) {
    b[i] = s;
    s *= ext[i];
  }
}

static void finish_group_geometry(PermGroup& g, const std::vector<int64_t>& src_ext, int src_n1,
                                  const std::vector<int>& src_leg, int dst_n1, int elem_bytes) {
  int N = (int)src_leg.size();
  std::vector<int64_t> sa, sb, da, db, dext(N);
  leg_strides(src_ext, src_n1, sa, sb);
  for (int k = 0; k < N; ++k) dext[k] = src_ext[src_leg[k]];
  leg_strides(dext, dst_n1, da, db);
  // dst order, drop extent-1 legs, merge contiguous neighbours
  struct L {
    int64_t e, sa, sb, da, db;
  };
  std::vector<L> legs;
  for (int k = 0; k < N; ++k) {
    if (dext[k] == 1) continue;
    L l{dext[k], sa[src_leg[k]], sb[src_leg[k]], da[k], db[k]};
    if (!legs.empty()) {
      L& pv = legs.back();
      if (l.sa == pv.sa * pv.e && l.sb == pv.sb * pv.e && l.da == pv.da * pv.e && l.db == pv.db * pv.e) {
        pv.e *= l.e;
        continue;
      }
    }
    legs.push_back(l);
  }
  if (legs.empty()) legs.push_back(L{1, 0, 0, 0, 0});
  if ((int)legs.size() > kMaxLegs) TK_THROW(TK_ERR_UNSUPPORTED, "too many legs after merging");
  g.ndim = (int)legs.size();
  int64_t ne = 1;
  for (auto& l : legs) ne *= l.e;
  if (ne >= (int64_t(1) << 31)) TK_THROW(TK_ERR_UNSUPPORTED, "a single subblock with >= 2^31 elements");
  g.nelem = 1;
  for (int i = 0; i < kMaxLegs; ++i) {
    if (i < g.ndim) {
      g.ext[i] = (int32_t)legs[i].e;
      g.sa[i] = legs[i].sa;
      g.sb[i] = legs[i].sb;
      g.da[i] = legs[i].da;
      g.db[i] = legs[i].db;
      g.nelem *= legs[i].e;
    } else {
      g.ext[i] = 1;
      g.sa[i] = g.sb[i] = g.da[i] = g.db[i] = 0;
    }
  }
  // mode 1 (smem tile): leg 0 (dst-fastest) x leg 1 (dst-next) x a block of the remaining legs, loaded
  // in source-stride order and stored in destination order, so both sides stream long contiguous
  // runs. Mode 0 (direct rows) for single-leg groups and for recoupling groups (k_src, k_dst > 1).
  g.mode = 0;
  g.tleg = 0;
  g.c0 = g.ct = g.R = g.T0 = g.Tt = 1;
  g.lorder = 0 + 3 * 1 + 9 * 2;
  g.nrest = 1;
  static const bool tile_all = knob("TK_PERM_TILE_ALL", 0) != 0;
  bool lead_unit = (g.sa[0] == 1 && g.sb[0] == 0);
  if (g.ndim >= 2 && g.ksrc == 1 && g.kdst == 1 && (!lead_unit || tile_all)) {
    g.mode = 1;
    g.tleg = 1;
    int64_t n0 = g.ext[0], nt = g.ext[1];
    g.c0 = (int32_t)std::min<int64_t>(n0, 64);
    int64_t c0p = g.c0 | 1;
    g.ct = (int32_t)std::min<int64_t>(nt, std::max<int64_t>(1, 1024 / c0p));
    g.nrest = g.nelem / (n0 * nt);
    g.R = (int32_t)std::max<int64_t>(1, std::min<int64_t>({128, g.nrest, (kTileElems / 2) / (g.ct * c0p)}));
    g.T0 = (int32_t)((n0 + g.c0 - 1) / g.c0);
    g.Tt = (int32_t)((nt + g.ct - 1) / g.ct);
    // load order: the three tile dimensions sorted by source stride (column-major: b-part dominates)
    auto key = [&](int leg) -> std::pair<int64_t, int64_t> {
      if (leg < 0) return {INT64_MAX, INT64_MAX};
      return {g.sb[leg], g.sa[leg]};
    };
    int rest0 = g.ndim >= 3 ? 2 : -1;
    std::pair<std::pair<int64_t, int64_t>, int> d[3] = {{key(0), 0}, {key(1), 1}, {key(rest0), 2}};
    std::sort(d, d + 3);
    g.lorder = d[0].second + 3 * d[1].second + 9 * d[2].second;
  }
}

// small single-member groups of either geometry (the packed path takes any leg-0 strides, so tiny
// transposing groups need no shared-memory tile)
static bool packable(const PermGroup& g) {
  return g.ksrc == 1 && g.kdst == 1 && g.nelem <= 2048 && g.nelem / g.ext[0] <= kPackRows;
}

// Builds kJobSeg blobs (SegHeader in tk_kernels.hpp): row ranges of single-member groups are packed
// greedily into jobs of <= job_elems elements, <= kPackGroups chunks and <= kPackRows rows; the row
// start offsets are the same index arithmetic the rows kernel does per job (legs 1.. of the group).
struct SegBuilder {
  PermPlan& P;
  std::vector<PermJob>& jobs;
  int64_t job_elems;
  std::vector<SegGroup> cg;
  std::vector<int32_t> rs, rd;
  int64_t elems = 0;
  SegBuilder(PermPlan& P_, std::vector<PermJob>& j, int64_t je) : P(P_), jobs(j), job_elems(je) {}
  static void fastdiv(uint32_t d, uint32_t& m, uint32_t& s) {  // = FastDiv::init (tk_kernels.cu)
    s = 0;
    while ((1u << s) < d) ++s;
    m = (d <= 1) ? 0u : (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << s) - d)) / d + 1);
  }
  void flush() {
    if (cg.empty()) return;
    const int64_t first = (int64_t)P.blob.size();
    SegHeader h{(int32_t)cg.size(), (int32_t)rs.size(), (int32_t)elems, 0};
    const int64_t* hw = reinterpret_cast<const int64_t*>(&h);
    P.blob.insert(P.blob.end(), hw, hw + 2);
    for (const SegGroup& g : cg) {
      const int64_t* w = reinterpret_cast<const int64_t*>(&g);
      P.blob.insert(P.blob.end(), w, w + 10);
    }
    std::vector<int32_t> rr(rs);
    rr.insert(rr.end(), rd.begin(), rd.end());
    if (rr.size() & 1) rr.push_back(0);
    const int64_t* rw = reinterpret_cast<const int64_t*>(rr.data());
    P.blob.insert(P.blob.end(), rw, rw + rr.size() / 2);
    if (P.blob.size() & 1) P.blob.push_back(0);
    jobs.push_back(PermJob{(int32_t)(P.blob.size() - first), (int16_t)cg.size(), kJobSeg, 0, first});
    cg.clear();
    rs.clear();
    rd.clear();
    elems = 0;
  }
  void add(int gi) {
    const PermGroup& g = P.groups[gi];
    const PermMember ms = P.members[g.src_mem], md = P.members[g.dst_mem];
    // the row leg: destination leg 0 for rows groups (unit stride on both sides); for transposing
    // groups the source-fastest leg, so loads stay coalesced and the stores scatter (TK_SEG_DSTLEG=1:
    // always destination leg 0)
    static const bool dst_leg = knob("TK_SEG_DSTLEG", 0) != 0;
    int L = 0;
    if (g.mode == 1 && !dst_leg)
      for (int l = 1; l < g.ndim; ++l)
        if (std::make_pair(g.sb[l], g.sa[l]) < std::make_pair(g.sb[L], g.sa[L])) L = l;
    const int64_t n0 = g.ext[L], nrows = g.nelem / n0;
    if (n0 > INT32_MAX / 2) TK_THROW(TK_ERR_UNSUPPORTED, "row too long for a seg job");
    for (int64_t r0 = 0; r0 < nrows;) {
      int64_t room = std::min<int64_t>((job_elems - elems) / n0, kPackRows - (int64_t)rs.size());
      if ((int)cg.size() == kPackGroups || room <= 0) {
        if (!cg.empty()) {
          flush();
          continue;
        }
        room = 1;  // one row longer than job_elems: a job of its own
      }
      const int64_t nr = std::min(room, nrows - r0);
      SegGroup sg{};
      sg.estart = (int32_t)elems;
      sg.rstart = (int32_t)rs.size();
      sg.n0 = (uint32_t)n0;
      fastdiv(sg.n0, sg.fm, sg.fs);
      sg.q = (uint32_t)(kPermThreads / n0);
      sg.rem = (uint32_t)(kPermThreads % n0);
      sg.s0 = g.sa[L] + ms.ld * g.sb[L];
      sg.d0 = g.da[L] + md.ld * g.db[L];
      sg.c = P.coefs[g.coef_off];
      sg.sd1 = ms.d1;
      sg.dd1 = md.d1;
      sg.dd2 = md.d2;
      cg.push_back(sg);
      for (int64_t r = r0; r < r0 + nr; ++r) {
        int64_t R = r, sa = 0, sbb = 0, da = 0, db = 0;
        for (int l = 0; l < g.ndim; ++l) {
          if (l == L) continue;
          const int64_t i = R % g.ext[l];
          R /= g.ext[l];
          sa += i * g.sa[l];
          sbb += i * g.sb[l];
          da += i * g.da[l];
          db += i * g.db[l];
        }
        const int64_t os = ms.off + sa + ms.ld * sbb, od = md.off + da + md.ld * db;
        // int32 offsets: the last element of the row (and its complex-mode partners) must fit
        const int64_t reach = 2 * ((n0 - 1) * std::max<int64_t>(std::abs(sg.s0), std::abs(sg.d0)) + std::max(os, od)) +
                              2 * (ms.d1 + md.d1 + md.d2);
        if (reach >= INT32_MAX) TK_THROW(TK_ERR_UNSUPPORTED, "seg job offsets exceed int32");
        rs.push_back((int32_t)os);
        rd.push_back((int32_t)od);
      }
      elems += nr * n0;
      r0 += nr;
    }
  }
  void finish() { flush(); }
};

static void make_jobs(PermPlan& P) {
  // small single-member groups go last and are packed several per CTA (permute_packed_kernel)
  std::stable_partition(P.groups.begin(), P.groups.end(), [](const PermGroup& g) { return !packable(g); });
  std::vector<PermJob> rows, multi, dmulti, tiles, packed;
  // elements per CTA job: 8192 for large permutes, smaller for small ones so that a latency-bound
  // permute still spreads over about two waves of the 148 SMs x 4 resident CTAs
  int64_t total = 0;
  for (const PermGroup& g : P.groups) total += g.nelem;
  static const int64_t job_div = knob("TK_JOB_DIV", 2 * 148 * 4);
  static const int64_t job_max = knob("TK_JOB_MAX", kPackElems);
  const int64_t job_elems = std::max<int64_t>(512, std::min<int64_t>(job_max, total / job_div));
  int64_t pack_elems = 0, pack_rows = 0;
  // latency regime: single-member rows / packable groups become kJobSeg blobs (TK_NO_SEG=1 disables)
  static const bool no_seg = knob("TK_NO_SEG", 0) != 0;
  // large-permute threshold: below it the latency regime (seg jobs, one launch), at or above it the
  // bandwidth regime (rows-only launch + a launch for the rest)
  static const int split_log2 = (int)knob("TK_SPLIT_LOG2", 24);
  const bool seg = !no_seg && total < (int64_t(1) << split_log2);
  std::vector<PermJob> segs;
  // seg job size: about total / 296 elements (measured against 1184 / 592 / 148 jobs per permute: fewer,
  // larger jobs amortise each CTA's blob copy and tail -- cfg7 124 -> 112 us, cfg3 219 -> 213 us;
  // tools/gpu_ab17.sh), within [256, TK_SEG_MAX = 8192] elements (the row table holds 1024 rows)
  static const int64_t seg_div = knob("TK_SEG_DIV", 2 * 148);
  static const int64_t seg_max = knob("TK_SEG_MAX", kPackElems);
  SegBuilder sb(P, segs, std::max<int64_t>(256, std::min<int64_t>(seg_max, total / seg_div)));
  for (int gi = 0; gi < (int)P.groups.size(); ++gi) {
    const PermGroup& g = P.groups[gi];
    if (seg && g.ksrc == 1 && g.kdst == 1) {
      sb.add(gi);
      continue;
    }
    if (packable(g)) {
      int64_t nrow = g.nelem / g.ext[0];
      if (!packed.empty() && packed.back().count < kPackGroups && pack_elems + g.nelem <= job_elems &&
          pack_rows + nrow <= kPackRows) {
        packed.back().count += 1;
        pack_elems += g.nelem;
        pack_rows += nrow;
      } else {
        packed.push_back(PermJob{gi, 1, kJobPacked, 0, 0});
        pack_elems = g.nelem;
        pack_rows = nrow;
      }
      continue;
    }
    if (g.mode == 0) {
      int64_t nrows = g.nelem / g.ext[0];
      const bool single = g.ksrc == 1 && g.kdst == 1;
      // recoupling jobs: the job's k_src source rows must fit the kernel's shared-memory stage
      const int64_t budget = single ? job_elems : std::min<int64_t>(job_elems, kRecoupleStage * 8 / P.elem_bytes / g.ksrc);
      int64_t per = std::max<int64_t>(1, std::min<int64_t>(kMaxRows, budget / std::max(1, g.ext[0])));
      // recoupling groups of few sources run inside the general launch (no second, serialised launch)
      static const bool direct_ok = knob("TK_NO_DIRECT_MULTI", 0) == 0;
      auto& dst = single ? rows : (direct_ok && g.ksrc <= kRecoupleDirect ? dmulti : multi);
      for (int64_t r = 0; r < nrows; r += per)
        dst.push_back(PermJob{gi, (int16_t)std::min(per, nrows - r), (int8_t)(single ? kJobRows : kJobMulti), 0, r});
    } else {
      int64_t ntiles = (int64_t)g.T0 * g.Tt * ((g.nrest + g.R - 1) / g.R);
      int64_t per = std::max<int64_t>(1, std::min<int64_t>(4096, 2 * job_elems / ((int64_t)g.R * g.ct * g.c0)));
      for (int64_t r = 0; r < ntiles; r += per)
        tiles.push_back(PermJob{gi, (int16_t)std::min(per, ntiles - r), kJobTiled, 0, r});
    }
  }
  // small permutes: one launch for rows, tiled and packed jobs (+ one for recoupling jobs); large ones
  // (>= 2^24 elements) run the rows jobs in a rows-only kernel instance and the rest in a second launch
  sb.finish();
  rows.insert(rows.begin(), segs.begin(), segs.end());    // seg jobs lead the non-rows-only launch
  P.njobs = (int)(tiles.size() + rows.size() + packed.size() + dmulti.size());
  P.njobs_rows = (int)(rows.size() - segs.size());
  P.njobs_multi = (int)multi.size();
  P.tiled = !tiles.empty();  // tiled jobs need the dynamic shared-memory tile
  P.rows_only = tiles.empty() && packed.empty() && segs.empty() && dmulti.empty();
  // large permutes (>= 2^24 elements) launch one kernel per job class: rows-only, the rest
  P.split = total >= (int64_t(1) << split_log2);
  const bool dbg = plan_debug();
  if (dbg) {
    int64_t er = 0, et = 0, ep = 0, em = 0, gr = 0, gt = 0, gp = 0;
    for (const PermGroup& g : P.groups) {
      if (packable(g)) ep += g.nelem, ++gp;
      else if (g.mode == 1) et += g.nelem, ++gt;
      else if (g.ksrc == 1 && g.kdst == 1) er += g.nelem, ++gr;
      else em += g.nelem;
    }
    std::map<int, std::pair<int, int64_t>> kh;  // k_src -> (groups, elements) of recoupling groups
    for (const PermGroup& g : P.groups)
      if (g.ksrc > 1 || g.kdst > 1) kh[g.ksrc].first++, kh[g.ksrc].second += g.nelem * g.ksrc;
    if (!kh.empty()) {
      fprintf(stderr, "[tk plan] recoupling k_src histogram (groups, source elements):");
      for (auto& e : kh) fprintf(stderr, " %d:(%d, %lld)", e.first, e.second.first, (long long)e.second.second);
      fprintf(stderr, "\n");
    }
    int sg_ng = 0, sg_rows = 0, sg_el = 0;
    for (const PermJob& j : segs) {
      const SegHeader* h = reinterpret_cast<const SegHeader*>(P.blob.data() + j.first);
      sg_ng = std::max(sg_ng, h->ng), sg_rows = std::max(sg_rows, h->nrows), sg_el = std::max(sg_el, h->total);
    }
    if (!segs.empty())
      fprintf(stderr, "[tk plan] seg: %zu jobs, max %d chunks / %d rows / %d elements per job\n", segs.size(), sg_ng,
              sg_rows, sg_el);
    fprintf(stderr, "[tk plan] %lld elems, job_elems %lld: rows %zu jobs (%lld groups, %lld el) | tiled %zu (%lld, %lld el) | "
            "packed %zu (%lld, %lld el) | multi %zu (%lld el)\n", (long long)total, (long long)job_elems, rows.size(),
            (long long)gr, (long long)er, tiles.size(), (long long)gt, (long long)et, packed.size(), (long long)gp,
            (long long)ep, multi.size(), (long long)em);
  }
  P.jobs = rows;
  P.jobs.insert(P.jobs.end(), tiles.begin(), tiles.end());
  P.jobs.insert(P.jobs.end(), packed.begin(), packed.end());
  P.jobs.insert(P.jobs.end(), dmulti.begin(), dmulti.end());
  P.jobs.insert(P.jobs.end(), multi.begin(), multi.end());
}

PadLayout pad_layout(const Tensor& t, PadKind kind) {
  PadLayout pl;
  pl.kind = kind;
  int64_t o = 0;
  for (const Block& b : t.blocks) {
    int64_t r = kind == PadKind::RealRep ? 2 * b.rows : b.rows;
    int64_t c = kind == PadKind::Real ? b.cols : 2 * b.cols;
    int64_t ld = (r + 3) & ~int64_t(3);
    pl.off.push_back(o);
    pl.ld.push_back(ld);
    pl.d1.push_back(kind == PadKind::Real ? 0 : b.cols * ld);
    pl.d2.push_back(kind == PadKind::RealRep ? b.rows : 0);
    o += ld * c;
  }
  pl.total = o;
  return pl;
}

// permute-table member of subblock i: canonical layout (pl == nullptr; offsets in elements of the
// tensor's dtype) or a workspace layout (offsets in doubles)
static PermMember sub_member(const Tensor& t, const PadLayout* pl, int i) {
  const Subblock& sb = t.subs[i];
  if (!pl) return PermMember{sb.off, t.ld(i), 0, 0};
  int b = sb.block;
  return PermMember{pl->off[b] + sb.row_off + pl->ld[b] * sb.col_off, pl->ld[b], pl->d1[b], pl->d2[b]};
}

static bool is_identity_perm(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q) {
  if ((int)p.size() != A.n_cod()) return false;
  for (int i = 0; i < (int)p.size(); ++i)
    if (p[i] != i) return false;
  for (int j = 0; j < (int)q.size(); ++j)
    if (q[j] != A.n_cod() + j) return false;
  return true;
}

void build_perm_plan(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q, const Tensor& C,
                     PermPlan& P, int elem_bytes, const PadLayout* spl, const PadLayout* dpl) {
  Kind k = A.kind;
  int n1 = A.n_cod(), N = A.nlegs();
  std::vector<int> src_leg = dst_from_src_legs(p, q);
  bool ident = C.n_cod() == n1;
  for (int i = 0; i < N && ident; ++i) ident = src_leg[i] == i;
  P.identity = ident;
  P.n_src = A.nelems;
  P.n_dst = C.nelems;
  P.bytes = (double)(A.nelems + C.nelems) * elem_bytes;
  P.elem_bytes = elem_bytes;
  std::vector<bool> isdual;
  for (auto* s : A.cod) isdual.push_back(s->dual);
  for (auto* s : A.dom) isdual.push_back(s->dual);
  std::vector<char> dst_done(C.subs.size(), 0);

  if (kind_abelian(k)) {
    // Alg. 6: one destination per source, coefficient = Koszul sign (reading C13)
    for (int i = 0; i < (int)A.subs.size(); ++i) {
      const Tree& s = A.s_tree(i);
      const Tree& f = A.f_tree(i);
      std::vector<Sector> lab(s.unc);
      lab.insert(lab.end(), f.unc.begin(), f.unc.end());
      std::vector<int64_t> ext(s.dims);
      ext.insert(ext.end(), f.dims.begin(), f.dims.end());
      std::vector<Sector> cu, du;
      for (int kk = 0; kk < (int)src_leg.size(); ++kk) {
        int l = src_leg[kk];
        bool was_cod = l < n1, now_cod = kk < C.n_cod();
        Sector x = (was_cod == now_cod) ? lab[l] : sector_dual(k, lab[l]);
        (now_cod ? cu : du).push_back(x);
      }
      Tree ts = abelian_tree(k, cu), tf = abelian_tree(k, du);
      auto it = C.sub_index.find(tree_pair_key(ts, tf));
      if (it == C.sub_index.end()) TK_THROW(TK_ERR_SPACE_MISMATCH, "internal: permuted channel not in output layout");
      int j = it->second;
      dst_done[j] = 1;
      PermGroup g{};
      g.ksrc = 1;
      g.kdst = 1;
      g.coef_off = (int)P.coefs.size();
      P.coefs.push_back((double)koszul_sign(k, lab, n1, p, q));
      g.src_mem = (int)P.members.size();
      P.members.push_back(sub_member(A, spl, i));
      g.dst_mem = (int)P.members.size();
      P.members.push_back(sub_member(C, dpl, j));
      finish_group_geometry(g, ext, n1, src_leg, C.n_cod(), elem_bytes);
      P.groups.push_back(g);
    }
  } else {
    // Alg. 10: group tree pairs by their uncoupled labels; per group a k_src x k_dst matrix
    std::map<std::string, std::vector<int>> by_unc;
    for (int i = 0; i < (int)A.subs.size(); ++i) {
      const Tree& s = A.s_tree(i);
      const Tree& f = A.f_tree(i);
      std::ostringstream os;
      for (auto& x : s.unc) os << x.v[0] << "," << x.v[1] << ";";
      os << "|";
      for (auto& x : f.unc) os << x.v[0] << "," << x.v[1] << ";";
      by_unc[os.str()].push_back(i);
    }
    std::vector<TPTerm> terms;
    for (auto& kv : by_unc) {
      const std::vector<int>& srcs = kv.second;
      std::vector<int> dsts;
      std::map<int, int> dpos;
      std::vector<std::vector<std::pair<int, double>>> rows(srcs.size());
      for (size_t a = 0; a < srcs.size(); ++a) {
        permute_tree_pair(k, A.s_tree(srcs[a]), A.f_tree(srcs[a]), p, q, isdual, terms);
        for (auto& t : terms) {
          auto it = C.sub_index.find(tree_pair_key(t.s, t.f));
          if (it == C.sub_index.end()) TK_THROW(TK_ERR_SPACE_MISMATCH, "internal: transformed tree pair not in output");
          int j = it->second;
          if (!dpos.count(j)) {
            dpos[j] = (int)dsts.size();
            dsts.push_back(j);
          }
          rows[a].push_back({dpos[j], t.coef});
        }
      }
      // also include every C tree pair with the permuted uncoupled labels (zero columns are written too)
      {
        const Tree& s0 = A.s_tree(srcs[0]);
        const Tree& f0 = A.f_tree(srcs[0]);
        std::vector<Sector> lab(s0.unc);
        lab.insert(lab.end(), f0.unc.begin(), f0.unc.end());
        std::vector<Sector> cu, du;
        for (int kk = 0; kk < (int)src_leg.size(); ++kk) {
          int l = src_leg[kk];
          bool was_cod = l < n1, now_cod = kk < C.n_cod();
          (now_cod ? cu : du).push_back((was_cod == now_cod) ? lab[l] : sector_dual(k, lab[l]));
        }
        for (int j = 0; j < (int)C.subs.size(); ++j) {
          if (dpos.count(j)) continue;
          if (C.s_tree(j).unc == cu && C.f_tree(j).unc == du) {
            dpos[j] = (int)dsts.size();
            dsts.push_back(j);
          }
        }
      }
      if ((int)srcs.size() > kMaxGroupMembers || (int)dsts.size() > kMaxGroupMembers)
        TK_THROW(TK_ERR_UNSUPPORTED, "recoupling group larger than 32 tree pairs");
      PermGroup g{};
      g.ksrc = (int)srcs.size();
      g.kdst = (int)dsts.size();
      g.coef_off = (int)P.coefs.size();
      std::vector<double> M(g.ksrc * g.kdst, 0.0);
      for (size_t a = 0; a < srcs.size(); ++a)
        for (auto& e : rows[a]) M[a * g.kdst + e.first] += e.second;
      P.coefs.insert(P.coefs.end(), M.begin(), M.end());
      g.src_mem = (int)P.members.size();
      for (int i : srcs) P.members.push_back(sub_member(A, spl, i));
      g.dst_mem = (int)P.members.size();
      for (int j : dsts) {
        P.members.push_back(sub_member(C, dpl, j));
        dst_done[j] = 1;
      }
      const Tree& s0 = A.s_tree(srcs[0]);
      const Tree& f0 = A.f_tree(srcs[0]);
      std::vector<int64_t> ext(s0.dims);
      ext.insert(ext.end(), f0.dims.begin(), f0.dims.end());
      finish_group_geometry(g, ext, n1, src_leg, C.n_cod(), elem_bytes);
      P.groups.push_back(g);
    }
  }
  for (size_t j = 0; j < dst_done.size(); ++j)
    if (!dst_done[j]) TK_THROW(TK_ERR_SPACE_MISMATCH, "internal: output subblock not covered by the permute plan");
  make_jobs(P);
}

// host-side transfer matrix (tests, §4.3 examples)
void permute_transfer_matrix(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q, const Tensor& C,
                             double* out) {
  validate_perm(A, p, q);
  check_target(A, p, q, C);
  PermPlan P;
  build_perm_plan(A, p, q, C, P, 8);
  size_t nc = C.subs.size();
  std::fill(out, out + A.subs.size() * nc, 0.0);
  // map member offsets back to subblock indices
  std::map<int64_t, int> aoff, coff;
  for (int i = 0; i < (int)A.subs.size(); ++i) aoff[A.subs[i].off] = i;
  for (int j = 0; j < (int)C.subs.size(); ++j) coff[C.subs[j].off] = j;
  for (auto& g : P.groups)
    for (int a = 0; a < g.ksrc; ++a)
      for (int b = 0; b < g.kdst; ++b) {
        int i = aoff.at(P.members[g.src_mem + a].off);
        int j = coff.at(P.members[g.dst_mem + b].off);
        out[i * nc + j] += P.coefs[g.coef_off + a * g.kdst + b];
      }
}

int sm_count();

struct Tuples {
  std::vector<int> pA, qA, pB, qB, pAB, qAB;
};

// contracted legs qA[c] <-> pB[c] must be a ket/bra pair: normalised spaces (cod: X, dom: X*) dual
// to each other
static void check_contracted_pairs(const Tensor& A, const Tensor& B, const Tuples& t) {
  for (size_t c = 0; c < t.qA.size(); ++c) {
    int ia = t.qA[c], jb = t.pB[c];
    const Space* sa = ia < A.n_cod() ? A.cod[ia] : A.dom[ia - A.n_cod()];
    const Space* sb = jb < B.n_cod() ? B.cod[jb] : B.dom[jb - B.n_cod()];
    bool da = sa->dual ^ (ia >= A.n_cod()), db = sb->dual ^ (jb >= B.n_cod());
    if (sa->kind != sb->kind || sa->sectors != sb->sectors || sa->degs != sb->degs || da == db)
      TK_THROW(TK_ERR_SPACE_MISMATCH, "contracted legs are not a ket/bra pair of the same space");
  }
}

// Explicit Alg. 4 tuples (reading C1: B~ = permute(B, (pB, qB))): (pA, qA) and (pB, qB)
// permutations of A's and B's legs, |qA| == |pB|, (pAB, qAB) a permutation of C~'s |pA| + |qB| legs.
static Tuples tuples_from_arrays(const Tensor& A, const Tensor& B, const int32_t* tup, const int32_t* ntup) {
  if (!ntup) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null tuple counts");
  int64_t tot = 0;
  for (int i = 0; i < 6; ++i) {
    if (ntup[i] < 0) TK_THROW(TK_ERR_INVALID_PERMUTATION, "negative tuple length");
    tot += ntup[i];
  }
  if (tot && !tup) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null tuples");
  Tuples t;
  std::vector<int>* dst[6] = {&t.pA, &t.qA, &t.pB, &t.qB, &t.pAB, &t.qAB};
  int64_t o = 0;
  for (int i = 0; i < 6; ++i)
    for (int k = 0; k < ntup[i]; ++k) dst[i]->push_back(tup[o++]);
  auto is_perm = [](const std::vector<int>& p, const std::vector<int>& q, int n) {
    if ((int)(p.size() + q.size()) != n) return false;
    std::vector<int> seen(n, 0);
    for (const auto* v : {&p, &q})
      for (int x : *v) {
        if (x < 0 || x >= n || seen[x]) return false;
        seen[x] = 1;
      }
    return true;
  };
  if (!is_perm(t.pA, t.qA, A.nlegs()) || !is_perm(t.pB, t.qB, B.nlegs()))
    TK_THROW(TK_ERR_INVALID_PERMUTATION, "(pA, qA) / (pB, qB) must permute the operand's legs");
  if (t.qA.size() != t.pB.size()) TK_THROW(TK_ERR_INVALID_PERMUTATION, "|qA| != |pB|");
  if (!is_perm(t.pAB, t.qAB, (int)(t.pA.size() + t.qB.size())))
    TK_THROW(TK_ERR_INVALID_PERMUTATION, "(pAB, qAB) must permute the |pA| + |qB| legs of A~ B~");
  check_contracted_pairs(A, B, t);
  return t;
}

// Reading C2: A~ = (open A in A order ; contracted in A order), B~ = (contracted ; open B),
// C~ = (open A ; open B), then permute C~ to labC. Validates labels.
static Tuples tuples_from_labels(const Tensor& A, const int32_t* labA, const Tensor& B, const int32_t* labB,
                                 const int32_t* labC, int nC, int nC_cod) {
  int NA = A.nlegs(), NB = B.nlegs();
  auto has = [](const int32_t* v, int n, int32_t x) {
    int c = 0;
    for (int i = 0; i < n; ++i) c += v[i] == x;
    return c;
  };
  for (int i = 0; i < NA; ++i)
    if (has(labA, NA, labA[i]) != 1) TK_THROW(TK_ERR_MALFORMED_NETWORK, "repeated label in A (traces unsupported)");
  for (int i = 0; i < NB; ++i)
    if (has(labB, NB, labB[i]) != 1) TK_THROW(TK_ERR_MALFORMED_NETWORK, "repeated label in B (traces unsupported)");
  Tuples t;
  std::vector<int32_t> openA, openB;
  for (int i = 0; i < NA; ++i) {
    if (has(labB, NB, labA[i])) {
      t.qA.push_back(i);
      int j = 0;
      while (labB[j] != labA[i]) ++j;
      t.pB.push_back(j);
    } else {
      t.pA.push_back(i);
      openA.push_back(labA[i]);
    }
  }
  for (int j = 0; j < NB; ++j)
    if (!has(labA, NA, labB[j])) {
      t.qB.push_back(j);
      openB.push_back(labB[j]);
    }
  std::vector<int32_t> ct(openA);
  ct.insert(ct.end(), openB.begin(), openB.end());
  if ((int)ct.size() != nC) TK_THROW(TK_ERR_MALFORMED_NETWORK, "labC must list exactly the open labels");
  if (nC_cod < 0 || nC_cod > nC) TK_THROW(TK_ERR_INVALID_ARGUMENT, "bad codomain count for C");
  for (int i = 0; i < nC; ++i) {
    int pos = -1;
    for (int j = 0; j < nC; ++j)
      if (ct[j] == labC[i]) pos = j;
    if (has(labC, nC, labC[i]) != 1) TK_THROW(TK_ERR_MALFORMED_NETWORK, "repeated label in labC");
    if (pos < 0) TK_THROW(TK_ERR_UNKNOWN_LABEL, "labC has a label that is not open");
    (i < nC_cod ? t.pAB : t.qAB).push_back(pos);
  }
  check_contracted_pairs(A, B, t);
  return t;
}

// Bosonic kinds: the order of the contracted legs inside A~ / B~ is free (the permutes are plain
// basis changes, reading C2), so pick the order (A's or B's) that makes the operand permutes cheapest:
// identity (no pass) < leading leg kept (coalesced rows path) < leading leg changes (smem transpose).
// Fermionic kinds keep reading C2 literally, because there the tuples fix the signs (C13).
static double perm_cost(const Tensor& X, const std::vector<int>& p, const std::vector<int>& q) {
  if (is_identity_perm(X, p, q)) return 0.0;
  int lead = p.empty() ? q[0] : p[0];
  return (double)X.nelems * (lead == 0 ? 1.0 : 2.0);
}

static void choose_contracted_order(const Tensor& A, const Tensor& B, Tuples& t) {
  // fermionic kinds: the tuples fix the signs; kinds without braiding: the reorder could break planarity
  if (kind_fermionic(A.kind) || !kind_braided(A.kind) || t.qA.size() < 2) return;
  std::vector<int> idx(t.qA.size());
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int)i;
  std::sort(idx.begin(), idx.end(), [&](int x, int y) { return t.pB[x] < t.pB[y]; });
  std::vector<int> qA2, pB2;
  for (int i : idx) {
    qA2.push_back(t.qA[i]);
    pB2.push_back(t.pB[i]);
  }
  double c1 = perm_cost(A, t.pA, t.qA) + perm_cost(B, t.pB, t.qB);
  double c2 = perm_cost(A, t.pA, qA2) + perm_cost(B, pB2, t.qB);
  if (c2 < c1) {
    t.qA = qA2;
    t.pB = pB2;
  }
}

Tensor* permuted_tensor(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q, tk_dtype dt) {
  std::vector<Space*> cod, dom;
  permuted_spaces(A, p, q, cod, dom);
  Tensor* t = make_tensor(dt, cod, dom, (int)A.kind);
  for (auto* s : cod) tk_space_release((tk_space*)s);
  for (auto* s : dom) tk_space_release((tk_space*)s);
  return t;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Gathered skinny GEMM (GatherSeg, tk_kernels.hpp). Applies when every GEMM block with K > 0 is skinny
// (K, N <= kSkinnyMax: the MPO steps T.W of the DMRG chains), the kind is abelian (single-member permute
// groups, coefficient +-1), Float64, and A~ is a genuine permute of A: then the A -> A~ pass (read A,
// write A~, read A~ again in the GEMM) becomes the GEMM's own gather from A. TK_NO_GATHER=1 disables.
static void build_gather(const Tensor& A, ContractPlan& P) {
  static const bool off = knob("TK_NO_GATHER", 0) != 0;
  if (off || P.cplx || P.pa.identity || P.ntiles_skinny == 0 || A.nelems >= INT32_MAX) return;
  for (const GemmGroup& g : P.ggroups)
    if (g.K > 0 && (g.K > kSkinnyMax || g.N > kSkinnyMax)) return;
  for (const PermGroup& g : P.pa.groups)
    if (g.ksrc != 1 || g.kdst != 1) return;
  // A~ subblocks per block of the padded layout, from the permute plan's destination members
  const PadLayout& la = P.la;
  const int nblk = (int)la.off.size();
  std::vector<std::vector<GatherSeg>> per(nblk);
  for (const PermGroup& g : P.pa.groups) {
    const PermMember ms = P.pa.members[g.src_mem], md = P.pa.members[g.dst_mem];
    const int b = (int)(std::upper_bound(la.off.begin(), la.off.end(), md.off) - la.off.begin()) - 1;
    const int64_t rel = md.off - la.off[b];
    GatherSeg q{};
    q.r0 = (int32_t)(rel % la.ld[b]);
    q.k0 = (int32_t)(rel / la.ld[b]);
    q.src = ms.off;
    const double c = P.pa.coefs[g.coef_off];
    if (c != 1.0 && c != -1.0) return;  // only signs in flight
    q.neg = c < 0;
    int64_t nr = 1, nc = 1;
    std::vector<std::pair<int64_t, int64_t>> cl;  // column legs (ext, source stride), fastest first
    for (int l = 0; l < g.ndim; ++l) {
      const int64_t str = g.sa[l] + ms.ld * g.sb[l];
      if (g.db[l] == 0) {  // a row leg of A~ (destination rows)
        if (q.nrl == 4) return;
        q.ext[q.nrl] = g.ext[l];
        q.str[q.nrl] = (int32_t)str;
        ++q.nrl;
        nr *= g.ext[l];
      } else {
        cl.push_back({g.ext[l], str});
        nc *= g.ext[l];
      }
    }
    if (nc > kSkinnyMax) return;
    q.nrows = (int32_t)nr;
    q.nk = (int32_t)nc;
    for (int64_t kk = 0; kk < nc; ++kk) {
      int64_t r = kk, o = 0;
      for (auto& e : cl) {
        o += (r % e.first) * e.second;
        r /= e.first;
      }
      q.colsrc[kk] = (int32_t)o;
    }
    per[b].push_back(q);
  }
  // GEMM group of each A~ block (same coupled sector), coverage check, tiles of whole row trees
  std::map<Sector, int> a_blk;
  for (int i = 0; i < (int)P.At->blocks.size(); ++i) a_blk[P.At->blocks[i].coupled] = i;
  std::vector<GatherSeg> segs;
  std::vector<GatherTile> tiles;
  int kmax = 0, nmax = 0;
  for (const GemmGroup& g : P.ggroups)
    if (g.K > 0) kmax = std::max(kmax, (int)g.K), nmax = std::max(nmax, (int)g.N);
  // the kernel instance is chosen by the launch's K class (4 / 8 / 16), which fixes its segment capacity
  const int kcls = kmax <= 4 ? 4 : kmax <= 8 ? 8 : 16;
  // 2 rows per thread only when that still leaves >= 2 tiles per resident CTA slot (148 SMs x 4):
  // measured cfg3 (1.95 M rows) 63 -> 47 us per T.W step, while cfg2 (0.2 M rows) prefers 256
  int64_t rows_total = 0;
  for (const GemmGroup& g : P.ggroups)
    if (g.K > 0) rows_total += g.M;
  const int cap = gather_seg_cap(kcls);
  static const int force_rows = (int)knob("TK_GATHER_ROWS", 0);
  int tile_rows = rows_total >= (int64_t)gather_rows(kcls) * 2 * 148 * 4 ? gather_rows(kcls) : kGatherRows;
  if (force_rows > 0) tile_rows = std::min(force_rows, gather_rows(kcls));
  for (int ci = 0; ci < (int)P.Ct->blocks.size(); ++ci) {
    const GemmGroup& gg = P.ggroups[ci];
    if (gg.K == 0) continue;
    auto ia = a_blk.find(P.Ct->blocks[ci].coupled);
    if (ia == a_blk.end()) return;
    std::vector<GatherSeg>& v = per[ia->second];
    std::sort(v.begin(), v.end(), [](const GatherSeg& x, const GatherSeg& y) {
      return x.r0 != y.r0 ? x.r0 < y.r0 : x.k0 < y.k0;
    });
    int64_t cover = 0;
    for (const GatherSeg& q : v) cover += (int64_t)q.nrows * q.nk;
    if (cover != (int64_t)gg.M * gg.K) return;  // every A~ element from exactly one subblock
    // row trees = runs of segments with equal r0 (they partition the block's rows); tiles are dense
    // kGatherRows-row ranges, each carrying the segments of every row tree it overlaps (a row tree cut
    // by a tile boundary has its segments copied into both tiles); fewer rows if that exceeds kGatherSegs
    std::vector<size_t> run;  // start index of each row tree in v
    for (size_t i = 0; i < v.size(); ++i)
      if (i == 0 || v[i].r0 != v[i - 1].r0) run.push_back(i);
    run.push_back(v.size());
    size_t rt = 0;  // first row tree overlapping the current tile
    for (int m0 = 0; m0 < gg.M;) {
      while (v[run[rt]].r0 + v[run[rt]].nrows <= m0) ++rt;
      int end = std::min(gg.M, m0 + tile_rows);
      size_t last = rt, nseg = 0;
      while (last < run.size() - 1 && v[run[last]].r0 < end) {
        const size_t cnt = run[last + 1] - run[last];
        if (nseg + cnt > (size_t)cap) {
          if (last == rt) return;  // one row tree with too many column subblocks
          end = v[run[last]].r0;   // stop before this row tree
          break;
        }
        nseg += cnt;
        ++last;
      }
      GatherTile t{};
      t.gout0 = -1;
      t.g = gg;
      t.m0 = m0;
      t.nrows = end - m0;
      t.seg0 = (int32_t)segs.size();
      for (size_t x = run[rt]; x < run[last]; ++x) segs.push_back(v[x]);
      t.nseg = (int32_t)(segs.size() - t.seg0);
      tiles.push_back(t);
      m0 = end;
    }
  }
  // B~ gather tables (GatherTile::bt): entry (k, n) of each group's K x N block of B~
  std::vector<int32_t> btab;
  std::vector<int> bt_of(P.ggroups.size(), -1);
  for (size_t ci = 0; ci < P.ggroups.size(); ++ci) {
    const GemmGroup& gg = P.ggroups[ci];
    if (gg.K == 0) continue;
    bt_of[ci] = (int)btab.size();
    btab.resize(btab.size() + (size_t)gg.K * gg.N, -1);
    if (P.pb.identity)  // B~ is B itself (canonical layout)
      for (int k = 0; k < gg.K; ++k)
        for (int n = 0; n < gg.N; ++n) {
          const int64_t o = gg.b_off + k + (int64_t)n * gg.ldb;
          if (o >= (int64_t(1) << 30)) return;
          btab[bt_of[ci] + k * gg.N + n] = (int32_t)(2 * o);
        }
  }
  if (!P.pb.identity) {
    std::map<Sector, int> c_of;  // coupled sector -> GEMM group
    for (int ci = 0; ci < (int)P.Ct->blocks.size(); ++ci) c_of[P.Ct->blocks[ci].coupled] = ci;
    const PadLayout& lb = P.lb;
    for (const PermGroup& g : P.pb.groups) {
      if (g.ksrc != 1 || g.kdst != 1) return;
      const double c = P.pb.coefs[g.coef_off];
      if (c != 1.0 && c != -1.0) return;
      const PermMember ms = P.pb.members[g.src_mem], md = P.pb.members[g.dst_mem];
      for (int64_t e = 0; e < g.nelem; ++e) {
        int64_t r = e, so = ms.off, dof = md.off;
        for (int l = 0; l < g.ndim; ++l) {
          const int64_t i = r % g.ext[l];
          r /= g.ext[l];
          so += i * (g.sa[l] + ms.ld * g.sb[l]);
          dof += i * (g.da[l] + md.ld * g.db[l]);
        }
        const int b = (int)(std::upper_bound(lb.off.begin(), lb.off.end(), dof) - lb.off.begin()) - 1;
        const int64_t rel = dof - lb.off[b];
        const int k = (int)(rel % lb.ld[b]), n = (int)(rel / lb.ld[b]);
        auto it = c_of.find(P.Bt->blocks[b].coupled);
        if (it == c_of.end() || bt_of[it->second] < 0 || so >= (int64_t(1) << 30)) return;
        const GemmGroup& gg = P.ggroups[it->second];
        if (k >= gg.K || n >= gg.N) return;
        btab[bt_of[it->second] + k * gg.N + n] = (int32_t)(2 * so + (c < 0));
      }
    }
  }
  // tiles -> their group's table (tiles were built group by group in GEMM-group order)
  {
    size_t ti = 0;
    for (size_t ci = 0; ci < P.ggroups.size(); ++ci) {
      const GemmGroup& gg = P.ggroups[ci];
      if (gg.K == 0) continue;
      for (int m0 = 0; ti < tiles.size() && m0 < gg.M; ++ti) {
        tiles[ti].bt = bt_of[ci];
        m0 = tiles[ti].m0 + tiles[ti].nrows;
      }
    }
    if (ti != tiles.size()) return;
  }
  // per-tile slots (GatherTile | first kGatherSlotSegs segments | first kGatherSlotB table entries)
  std::vector<int64_t> slots((size_t)tiles.size() * kGatherSlotWords, 0);
  for (size_t ti = 0; ti < tiles.size(); ++ti) {
    const GatherTile& t = tiles[ti];
    int64_t* w = slots.data() + ti * kGatherSlotWords;
    std::memcpy(w, &t, sizeof(GatherTile));
    std::memcpy(w + 10, segs.data() + t.seg0, sizeof(GatherSeg) * std::min(t.nseg, kGatherSlotSegs));
    int32_t* bw = reinterpret_cast<int32_t*>(w + 10 + 16 * kGatherSlotSegs);
    for (int e = 0; e < std::min(t.g.K * t.g.N, kGatherSlotB); ++e) bw[e] = btab[t.bt + e];
  }
  P.gslots = std::move(slots);
  P.gather = true;
  P.btab = std::move(btab);
  P.gsegs = std::move(segs);
  P.gtiles = std::move(tiles);
  P.g_kmax = kmax;
  P.g_nmax = nmax;
  // the skinny tiles are replaced; the A~ permute and its workspace are not used
  P.tiles.resize(P.ntiles_big + P.ntiles_small);
  P.ntiles_skinny = 0;
  P.merged_ab = false;
  if (plan_debug())
    fprintf(stderr, "[tk gather] %zu tiles, %zu subblocks, K <= %d, N <= %d\n", P.gtiles.size(), P.gsegs.size(), kmax,
            nmax);
}

OutMap::OutMap(const PermPlan& pc, const PadLayout& lc) : pc_(pc), lc_(lc) {
  for (int gi = 0; gi < (int)pc.groups.size(); ++gi) {
    const PermGroup& g = pc.groups[gi];
    const double cf = g.ksrc == 1 && g.kdst == 1 ? pc.coefs[g.coef_off] : 0.0;
    if (cf != 1.0 && cf != -1.0) {  // recoupling (non-abelian) or a non-sign coefficient
      ok_ = false;
      return;
    }
    const PermMember ms = pc.members[g.src_mem];
    const int b = (int)(std::upper_bound(lc.off.begin(), lc.off.end(), ms.off) - lc.off.begin()) - 1;
    if (b < 0) {
      ok_ = false;
      return;
    }
    const int64_t rel = ms.off - lc.off[b];
    int64_t nr = 1, nc = 1;
    for (int l = 0; l < g.ndim; ++l) (g.sb[l] == 0 ? nr : nc) *= g.ext[l];
    boxes_[lc.off[b]].push_back(Box{(int32_t)(rel % lc.ld[b]), (int32_t)nr, (int32_t)(rel / lc.ld[b]), (int32_t)nc, gi});
  }
}

bool OutMap::map(int64_t src, int F, GatherOut& o) const {
  if (!ok_) return false;
  const int b = (int)(std::upper_bound(lc_.off.begin(), lc_.off.end(), src) - lc_.off.begin()) - 1;
  if (b < 0) return false;
  auto it = boxes_.find(lc_.off[b]);
  if (it == boxes_.end()) return false;
  const int64_t rel = src - lc_.off[b];
  const int32_t r = (int32_t)(rel % lc_.ld[b]), c = (int32_t)(rel / lc_.ld[b]);
  const Box* x = nullptr;
  for (const Box& q : it->second)
    if (q.r0 == r && c >= q.c0 && c < q.c0 + q.nc) x = &q;
  if (!x || x->nr != F) return false;
  const PermGroup& g = pc_.groups[x->g];
  const PermMember md = pc_.members[g.dst_mem];
  // row legs (sb = 0, extent > 1) by ascending source row stride: the radix of the row index
  std::vector<int> rl, cl;
  for (int l = 0; l < g.ndim; ++l)
    if (g.ext[l] > 1) (g.sb[l] == 0 ? rl : cl).push_back(l);
  std::sort(rl.begin(), rl.end(), [&](int u, int v) { return g.sa[u] < g.sa[v]; });
  std::sort(cl.begin(), cl.end(), [&](int u, int v) { return g.sb[u] < g.sb[v]; });
  if (rl.size() > 3) return false;
  int64_t run = 1;
  for (int l : rl) {
    if (g.sa[l] != run) return false;
    run *= g.ext[l];
  }
  o = GatherOut{};
  o.ext0 = rl.size() > 0 ? g.ext[rl[0]] : 1;
  o.ext1 = rl.size() > 1 ? g.ext[rl[1]] : 1;
  for (size_t j = 0; j < rl.size(); ++j) {
    const int64_t st = g.da[rl[j]] + md.ld * g.db[rl[j]];
    if (st > INT32_MAX) return false;
    o.str[j] = (int32_t)st;
  }
  int64_t crun = 1;  // the column's digits over the column legs (ascending source column stride)
  for (int l : cl) {
    if (g.sb[l] != crun) return false;
    crun *= g.ext[l];
  }
  int64_t cc = c - x->c0;
  o.base = md.off;
  for (int l : cl) {
    o.base += (cc % g.ext[l]) * (g.da[l] + md.ld * g.db[l]);
    cc /= g.ext[l];
  }
  o.neg = pc_.coefs[g.coef_off] < 0;
  return true;
}

// The output permute of a gathered plan folded into the gathered GEMM's stores (GatherTile::gout0): a
// per-(row tree, column) map from the C~ row's digits to C. All-or-nothing per plan.
static void fold_gather_output(ContractPlan& P) {
  static const bool off = knob("TK_NO_GATHER_OUT", 0) != 0;
  if (off || !P.gather || P.pc.identity || P.cplx) return;
  if (!P.tiles.empty()) {
    if (plan_debug()) fprintf(stderr, "[tk gather] output permute not folded: other GEMM tiles\n");
    return;
  }
  OutMap om(P.pc, P.lc);
  if (!om.ok()) {
    if (plan_debug()) fprintf(stderr, "[tk gather] output permute not folded: not a signed map\n");
    return;
  }
  std::vector<GatherOut> gouts;
  std::vector<int32_t> g0(P.gtiles.size());
  for (size_t ti = 0; ti < P.gtiles.size(); ++ti) {
    const GatherTile& t = P.gtiles[ti];
    g0[ti] = (int32_t)gouts.size();
    gouts.resize(gouts.size() + (size_t)t.nseg * t.g.N);
    for (int s = 0; s < t.nseg; ++s) {
      const GatherSeg& q = P.gsegs[t.seg0 + s];
      if (s > 0 && P.gsegs[t.seg0 + s - 1].r0 == q.r0) continue;  // not the first segment of its row tree
      for (int n = 0; n < t.g.N; ++n) {
        GatherOut& o = gouts[g0[ti] + (size_t)s * t.g.N + n];
        if (!om.map(t.g.c_off + q.r0 + (int64_t)n * t.g.ldc, q.nrows, o) ||
            (n > 0 && (o.ext0 != gouts[g0[ti] + (size_t)s * t.g.N].ext0 ||
                       o.ext1 != gouts[g0[ti] + (size_t)s * t.g.N].ext1))) {
          if (plan_debug())
            fprintf(stderr, "[tk gather] output permute not folded: tile %zu seg %d col %d (r0 %d, %d rows, nrl %d)\n",
                    ti, s, n, q.r0, q.nrows, q.nrl);
          return;
        }
      }
    }
  }
  for (size_t ti = 0; ti < P.gtiles.size(); ++ti) {
    P.gtiles[ti].gout0 = g0[ti];
    std::memcpy(P.gslots.data() + ti * kGatherSlotWords, &P.gtiles[ti], sizeof(GatherTile));
  }
  P.gouts = std::move(gouts);
  P.gout = true;
  if (plan_debug()) fprintf(stderr, "[tk gather] output permute folded in (%zu maps)\n", P.gouts.size());
}

static void build_contract_plan(const Tensor& A, const Tensor& B, const Tensor& C, const Tuples& t, ContractPlan& P) {
  if (A.kind != B.kind || A.kind != C.kind) TK_THROW(TK_ERR_SECTOR_MISMATCH, "sector kinds differ");
  if (A.dtype != B.dtype || A.dtype != C.dtype) TK_THROW(TK_ERR_INVALID_ARGUMENT, "tk_contract: dtypes differ");
  P.cplx = A.dtype == TK_C64;
  P.At = permuted_tensor(A, t.pA, t.qA, A.dtype);
  P.Bt = permuted_tensor(B, t.pB, t.qB, B.dtype);
  {
    std::vector<Space*> cod(P.At->cod), dom(P.Bt->dom);
    P.Ct = make_tensor(C.dtype, cod, dom, (int)A.kind);
  }
  check_target(*P.Ct, t.pAB, t.qAB, C);
  // ComplexF64 always passes through the workspace (the permutes also change the representation)
  bool ia_id = !P.cplx && is_identity_perm(A, t.pA, t.qA), ib_id = !P.cplx && is_identity_perm(B, t.pB, t.qB);
  bool ic_id = !P.cplx && is_identity_perm(*P.Ct, t.pAB, t.qAB);
  P.la = pad_layout(*P.At, P.cplx ? PadKind::Planar : PadKind::Real);
  P.lb = pad_layout(*P.Bt, P.cplx ? PadKind::RealRep : PadKind::Real);
  P.lc = pad_layout(*P.Ct, P.cplx ? PadKind::Planar : PadKind::Real);
  const PadLayout* pla = ia_id ? nullptr : &P.la;
  const PadLayout* plb = ib_id ? nullptr : &P.lb;
  const PadLayout* plc = ic_id ? nullptr : &P.lc;
  const int eb = P.cplx ? 16 : 8;
  build_perm_plan(A, t.pA, t.qA, *P.At, P.pa, eb, nullptr, pla);
  build_perm_plan(B, t.pB, t.qB, *P.Bt, P.pb, eb, nullptr, plb);
  build_perm_plan(*P.Ct, t.pAB, t.qAB, C, P.pc, eb, plc, nullptr);
  P.pa.identity = ia_id;
  P.pb.identity = ib_id;
  P.pc.identity = ic_id;
  static const bool no_merge = knob("TK_NO_MERGE", 0) != 0;
  if (!no_merge && !P.cplx && !ia_id && !ib_id && !P.pa.split && !P.pb.split) {
    P.merged_ab = true;
    auto take = [&](const PermPlan& pp, int8_t op, bool multi) {
      int b = multi ? pp.njobs : 0, e = multi ? pp.njobs + pp.njobs_multi : pp.njobs;
      for (int i = b; i < e; ++i) {
        PermJob j = pp.jobs[i];
        j.op = op;
        P.jobs_ab.push_back(j);
      }
    };
    take(P.pa, 0, false);
    take(P.pb, 1, false);
    take(P.pa, 0, true);
    take(P.pb, 1, true);
    P.njobs_ab = P.pa.njobs + P.pb.njobs;
    P.njobs_ab_multi = P.pa.njobs_multi + P.pb.njobs_multi;
    P.ab_tiled = P.pa.tiled || P.pb.tiled;
  }
  // workspace: A~ | B~ | C~ (skipped when the permute is the identity)
  size_t off = 0;
  if (!P.pa.identity) {
    P.off_a = off;
    off = align256(off + (size_t)P.la.total * 8);
  }
  if (!P.pb.identity) {
    P.off_b = off;
    off = align256(off + (size_t)P.lb.total * 8);
  }
  if (!P.pc.identity) {
    P.off_c = off;
    off = align256(off + (size_t)P.lc.total * 8);
  }
  P.ws_bytes = off;
  // Alg. 8: one GEMM per coupled sector of C~; K = 0 blocks are zero-filled.
  // ComplexF64: the real GEMM of the real representation, M x 2K times 2K x 2N (= 8MKN real flops,
  // the useful complex flop count of reading C21).
  const int cm = P.cplx ? 2 : 1;
  std::map<Sector, int> a_blk, b_blk;
  for (int i = 0; i < (int)P.At->blocks.size(); ++i) a_blk[P.At->blocks[i].coupled] = i;
  for (int i = 0; i < (int)P.Bt->blocks.size(); ++i) b_blk[P.Bt->blocks[i].coupled] = i;
  std::vector<GemmTile> big, small, skinny;
  for (int ci = 0; ci < (int)P.Ct->blocks.size(); ++ci) {
    const Block& cb = P.Ct->blocks[ci];
    GemmGroup g{};
    g.M = (int32_t)cb.rows;
    g.N = (int32_t)(cm * cb.cols);
    g.c_off = plc ? plc->off[ci] : cb.off;
    g.ldc = (int32_t)(plc ? plc->ld[ci] : cb.rows);
    auto ia = a_blk.find(cb.coupled);
    auto ib = b_blk.find(cb.coupled);
    if (ia != a_blk.end() && ib != b_blk.end()) {
      const Block& ab = P.At->blocks[ia->second];
      const Block& bb = P.Bt->blocks[ib->second];
      if (ab.rows != cb.rows || bb.cols != cb.cols || ab.cols != bb.rows)
        TK_THROW(TK_ERR_SPACE_MISMATCH, "internal: block shapes of A~, B~, C~ disagree");
      g.K = (int32_t)(cm * ab.cols);
      g.a_off = pla ? pla->off[ia->second] : ab.off;
      g.b_off = plb ? plb->off[ib->second] : bb.off;
      g.lda = (int32_t)(pla ? pla->ld[ia->second] : ab.rows);
      g.ldb = (int32_t)(plb ? plb->ld[ib->second] : bb.rows);
      g.vec = (g.a_off % 2 == 0) && (g.lda % 2 == 0) && (g.b_off % 2 == 0) && (g.ldb % 2 == 0);
    } else {
      g.K = 0;
      g.lda = g.ldb = 1;
    }
    P.flops += 2.0 * g.M * (double)g.N * g.K;
    int gi = (int)P.ggroups.size();
    P.ggroups.push_back(g);
    if (g.K > 0 && g.K <= kSkinnyMax && g.N <= kSkinnyMax) {  // streaming path (HBM-bound block)
      static const int srows = (int)knob("TK_SKINNY_ROWS", kSkinnyRows);
      for (int m = 0; m < g.M; m += srows)
        skinny.push_back(GemmTile{gi, m, 0, std::min(srows, g.M - m), 0, g.K, -1, 0, -1});  // tmap -1: skinny
      continue;
    }
    // short-K blocks (K <= 128: the L.theta steps of the DMRG chains) take 64 x 64 tiles: 4x the CTAs,
    // 3 CTAs per SM, so tile epilogues overlap other tiles' main loops (measured cfg2 step 1: 30 -> 15 us)
    static const int small_k = (int)knob("TK_GEMM_SMALL_K", 128);
    bool isbig = g.M >= 96 && g.N >= 96 && g.K > small_k;
    int bm = isbig ? 128 : 64, bn = isbig ? 128 : 64;
    // L2-friendly rasterisation: bands of G tile-rows, walked column by column, so that the ~148
    // co-resident tiles share the A and B k-slices in L2 (row-major order re-read all of B from DRAM
    // once per tile-row). Big tiles: G = 4, the measured DRAM minimum of the cfg4 GEMM (ncu, D_leg 384:
    // 615 / 342 / 264 / 231 / 238 / 318 / 463 / 502 GB per launch at G = 1 / 2 / 3 / 4 / 6 / 12 / 24 / 48,
    // the same 535 ms for every G -- the kernel is DMMA-bound either way); small tiles keep G = 12.
    static const int band = (int)knob("TK_GEMM_BAND", 0);
    const int ntm = (g.M + bm - 1) / bm, ntn = (g.N + bn - 1) / bn, G = band > 0 ? band : (isbig ? 4 : 12);
    for (int mb = 0; mb < ntm; mb += G)
      for (int nt = 0; nt < ntn; ++nt)
        for (int mt = mb; mt < std::min(ntm, mb + G); ++mt)
          (isbig ? big : small).push_back(GemmTile{gi, mt * bm, nt * bn, g.K, 0, g.K, -1, 0});
  }
  // split-K for under-filled launches (fewer than two tiles per SM): long-K small tiles are cut into
  // S slices of 64-multiples, each writing a partial tile; one reduction CTA per tile sums them in a
  // fixed order (deterministic) and applies alpha / beta.
  const int ntot = (int)(big.size() + small.size());
  static const bool no_split = knob("TK_NO_SPLITK", 0) != 0;
  // tiles/SM below which long-K tiles are split (re-measured after the seg / gather changes: target 2
  // gives cfg3 T3.R 47.5 us vs 52.7 at 4, cfg2 / cfg7 unchanged; tools/gpu_ab14.sh)
  static const int split_target = (int)knob("TK_SPLIT_TARGET", 2);
  if (!no_split && ntot > 0 && ntot < split_target * 148) {
    const int want = (split_target * 148 + ntot - 1) / ntot;
    std::vector<GemmTile> out;
    int slot = 0;
    for (const GemmTile& t : small) {
      const int K = t.k1;
      static const int min_chunk = (int)knob("TK_SPLIT_CHUNK", 64);
      const int S = std::min(std::min(want, K / min_chunk), 16);  // kSplitMax in the reduction kernel
      if (S < 2) {
        out.push_back(t);
        continue;
      }
      const int chunk = ((K + S - 1) / S + 15) & ~15;
      int ns = 0;
      for (int k = 0; k < K; k += chunk, ++ns)
        out.push_back(GemmTile{t.group, t.m0, t.n0, std::min(chunk, K - k), k, std::min(K, k + chunk), slot + ns, 0});
      P.split_heads.push_back(GemmTile{t.group, t.m0, t.n0, K, 0, K, slot, ns});
      slot += ns;
    }
    small = out;
    P.nslots = slot;
  }
  auto by_k = [](const GemmTile& x, const GemmTile& y) { return x.pad > y.pad; };  // LPT: long K first
  std::stable_sort(big.begin(), big.end(), by_k);
  std::stable_sort(small.begin(), small.end(), by_k);
  if (P.nslots) {
    P.off_parts = P.ws_bytes;
    P.ws_bytes = align256(P.ws_bytes + (size_t)P.nslots * 64 * 64 * 8);
  }
  P.ntiles_big = (int)big.size();
  P.ntiles_small = (int)small.size();
  P.ntiles_skinny = (int)skinny.size();
  if (plan_debug()) {
    int mM = 0, mN = 0, mK = 0, nz = 0;
    double fpad = 0;
    for (const GemmGroup& g : P.ggroups) {
      mM = std::max(mM, g.M), mN = std::max(mN, g.N), mK = std::max(mK, g.K), nz += g.K > 0;
    }
    for (const GemmTile& t : big) fpad += 2.0 * 128 * 128 * (t.k1 - t.k0);
    double fdmma = 0;  // what the small kernel's fragment guards actually issue (8-row / 8-col / 4-k units)
    for (const GemmTile& t : small) {
      fpad += 2.0 * 64 * 64 * (t.k1 - t.k0);
      const GemmGroup& g = P.ggroups[t.group];
      auto up = [](int x, int q) { return (x + q - 1) / q * q; };
      fdmma += 2.0 * up(std::min(64, g.M - t.m0), 8) * up(std::min(64, g.N - t.n0), 8) * up(t.k1 - t.k0, 4);
    }
    fprintf(stderr, "[tk gemm] small-tile DMMA flops issued %.3g\n", fdmma);
    fprintf(stderr, "[tk gemm] %zu groups (%d with K>0), %.3g flops, max M %d N %d K %d | big %zu small %zu skinny %zu "
            "tiles, split slots %d | tile flops %.3g\n", P.ggroups.size(), nz, P.flops, mM, mN, mK, big.size(),
            small.size(), skinny.size(), P.nslots, fpad);
  }
  // big tiles run on the persistent TMA kernel when both operands live in the padded workspace layout
  // (TMA needs 16-byte aligned bases and strides; a caller's buffer used in place may not satisfy that)
  static const bool no_tma = knob("TK_NO_TMA", 0) != 0;
  if (!no_tma && !big.empty() && pla && plb) {
    std::map<int, int> mi;
    for (GemmTile& t : big) {
      auto it = mi.find(t.group);
      if (it == mi.end()) it = mi.emplace(t.group, (int)mi.size()).first;
      t.tmap = it->second;
    }
    if ((int)mi.size() <= kTmaMaxGroups) {
      P.tma = true;
      P.tma_groups.resize(mi.size());
      for (auto& kv : mi) P.tma_groups[kv.second] = kv.first;
      P.off_counter = P.ws_bytes;  // the dynamic tile scheduler's counter (zeroed before each launch)
      P.ws_bytes = align256(P.ws_bytes + 4);
    }
  }
  P.tiles = big;
  P.tiles.insert(P.tiles.end(), small.begin(), small.end());
  P.tiles.insert(P.tiles.end(), skinny.begin(), skinny.end());
  for (GemmTile& t : P.tiles) t.g = P.ggroups[t.group];
  for (GemmTile& t : P.split_heads) t.g = P.ggroups[t.group];
  build_gather(A, P);
  fold_gather_output(P);
}

// ------------------------------------------------------------------ device memory of plans
int sm_count() {  // multiprocessors of the current device (cached per device)
  static std::mutex mu;
  static std::map<int, int> n;
  const int d = current_device();
  std::lock_guard<std::mutex> g(mu);
  auto it = n.find(d);
  if (it != n.end()) return it->second;
  int c = 148;
  if (d < 0 || cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) {
    (void)cudaGetLastError();
    c = 148;
  }
  n[d] = c;
  return c;
}

int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    (void)cudaGetLastError();
    return -1;
  }
  return d;
}

namespace {
struct UploadStreams {  // one library-private non-blocking stream per device, for table uploads
  std::mutex mu;
  std::map<int, cudaStream_t> st;
};
UploadStreams& upload_streams() {
  static UploadStreams* u = new UploadStreams();  // intentionally leaked: usable during static destruction
  return *u;
}
struct Graveyard {  // device memory of evicted / cleared plans, freed when no capture can be disturbed
  std::mutex mu;
  std::vector<std::pair<void*, int>> v;
};
Graveyard& graveyard() {
  static Graveyard* g = new Graveyard();
  return *g;
}
// relaxed capture mode for the calling thread while in scope (a cold plan may be built while the
// caller's stream is capturing; the upload must neither join nor invalidate that capture)
struct RelaxedCapture {
  cudaStreamCaptureMode old = cudaStreamCaptureModeRelaxed;
  RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&old); }
  ~RelaxedCapture() { cudaThreadExchangeStreamCaptureMode(&old); }
};
}  // namespace

void upload_bytes(void** p, const void* host, size_t n) {
  RelaxedCapture rc;
  const int dev = current_device();
  cudaStream_t s = nullptr;
  {
    UploadStreams& u = upload_streams();
    std::lock_guard<std::mutex> g(u.mu);
    auto it = u.st.find(dev);
    if (it == u.st.end()) {
      check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "upload stream");
      u.st[dev] = s;
    } else {
      s = it->second;
    }
  }
  if (dev < 0) TK_THROW(TK_ERR_CUDA, "no CUDA device: plan tables cannot be uploaded");
  check_cuda(cudaMalloc(p, n), "cudaMalloc of plan table");
  cudaError_t e = cudaMemcpyAsync(*p, host, n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFree(*p);
    *p = nullptr;
    check_cuda(e, "upload of plan table");
  }
}

void free_later(void* p, int device) {
  Graveyard& g = graveyard();
  std::lock_guard<std::mutex> l(g.mu);
  g.v.emplace_back(p, device);
}

static void free_now(std::vector<std::pair<void*, int>>& v) {
  if (v.empty()) return;
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& x : v) {
    if (x.second >= 0) cudaSetDevice(x.second);
    cudaFree(x.first);
  }
  cudaSetDevice(cur);
  v.clear();
}

void free_deferred(cudaStream_t caller) {
  Graveyard& g = graveyard();
  std::vector<std::pair<void*, int>> v;
  {
    std::lock_guard<std::mutex> l(g.mu);
    if (g.v.empty()) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(caller, &cs) != cudaSuccess) {
      (void)cudaGetLastError();  // the query's own error; frees wait for a later call
      return;
    }
    if (cs != cudaStreamCaptureStatusNone) return;
    v.swap(g.v);
  }
  free_now(v);
}

// ------------------------------------------------------------------ plan cache
static PlanCache<ContractPlan> g_contract_cache;
static PlanCache<PermPlan> g_perm_cache;

static std::string labels_key(const int32_t* v, int n) {
  std::ostringstream os;
  for (int i = 0; i < n; ++i) os << v[i] << ",";
  return os.str();
}

static std::shared_ptr<ContractPlan> new_contract_plan(const Tensor& A, const Tensor& B, const Tensor& C,
                                                       const Tuples& t) {
  auto P = std::make_shared<ContractPlan>();
  build_contract_plan(A, B, C, t, *P);
  return P;
}

std::shared_ptr<ContractPlan> get_contract_plan(const Tensor& A, const int32_t* labA, const Tensor& B,
                                                const int32_t* labB, const Tensor& C, const int32_t* labC) {
  std::string key = A.sig + "#" + labels_key(labA, A.nlegs()) + "#" + B.sig + "#" + labels_key(labB, B.nlegs()) +
                    "#" + C.sig + "#" + labels_key(labC, C.nlegs());
  return g_contract_cache.get(key, [&] {
    if (A.kind != B.kind || A.kind != C.kind) TK_THROW(TK_ERR_SECTOR_MISMATCH, "sector kinds differ");
    Tuples t = tuples_from_labels(A, labA, B, labB, labC, C.nlegs(), C.n_cod());
    choose_contracted_order(A, B, t);
    return new_contract_plan(A, B, C, t);
  });
}

static std::shared_ptr<ContractPlan> get_contract_plan_tuples(const Tensor& A, const Tensor& B, const Tensor& C,
                                                              const int32_t* tup, const int32_t* ntup) {
  if (A.kind != B.kind || A.kind != C.kind) TK_THROW(TK_ERR_SECTOR_MISMATCH, "sector kinds differ");
  Tuples t = tuples_from_arrays(A, B, tup, ntup);
  std::ostringstream os;
  os << "T#" << A.sig << "#" << B.sig << "#" << C.sig;
  for (const auto* v : {&t.pA, &t.qA, &t.pB, &t.qB, &t.pAB, &t.qAB}) {
    os << "#";
    for (int x : *v) os << x << ",";
  }
  return g_contract_cache.get(os.str(), [&] { return new_contract_plan(A, B, C, t); });
}

static std::shared_ptr<PermPlan> get_perm_plan(const Tensor& A, const std::vector<int>& p, const std::vector<int>& q,
                                               const Tensor& C) {
  std::ostringstream os;
  os << A.sig << "#";
  for (int x : p) os << x << ",";
  os << "#";
  for (int x : q) os << x << ",";
  os << "#" << C.sig;
  return g_perm_cache.get(os.str(), [&] {
    validate_perm(A, p, q);
    check_target(A, p, q, C);
    auto P = std::make_shared<PermPlan>();
    build_perm_plan(A, p, q, C, *P, A.dtype == TK_C64 ? 16 : 8);
    return P;
  });
}

void cache_clear() {
  ncon_cache_clear();  // first: network plans hold intermediate HomSpaces, not pairwise plans
  fused_cache_clear();
  g_contract_cache.clear();
  g_perm_cache.clear();
  svd_cache_clear();
  trace_cache_clear();
  Graveyard& g = graveyard();
  std::vector<std::pair<void*, int>> v;
  {
    std::lock_guard<std::mutex> l(g.mu);
    v.swap(g.v);
  }
  free_now(v);
}

size_t cache_size() { return g_contract_cache.size() + g_perm_cache.size(); }
size_t svd_cache_size();
size_t trace_cache_size();
size_t fused_cache_size();
size_t ncon_cache_size();

// ------------------------------------------------------------------ profiling state
struct Prof {
  bool on = false;
  cudaEvent_t ev[5] = {};
  bool have = false;
  float ms[4] = {0, 0, 0, 0};
  double bytes[4] = {0, 0, 0, 0};
  double flops = 0;
};
static thread_local Prof g_prof;
static thread_local int g_launches = 0;
void add_launches(int n) { g_launches += n; }
void reset_launches() { g_launches = 0; }

static void prof_record(int i, cudaStream_t st) {
  if (!g_prof.on) return;
  if (!g_prof.ev[0])
    for (auto& e : g_prof.ev) cudaEventCreate(&e);
  cudaEventRecord(g_prof.ev[i], st);
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) TK_THROW(TK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static PermOp perm_op(PermPlan& P, const void* src, void* dst, double alpha, double beta, double ims) {
  if (!P.uploaded) TK_THROW(TK_ERR_CUDA, "internal: plan tables not uploaded");
  return PermOp{src, dst, (const PermGroup*)P.d_groups.p, (const PermMember*)P.d_members.p, (const double*)P.d_coefs.p,
                (const int64_t*)P.d_blob.p, alpha, beta, ims};
}

void run_permute(PermPlan& P, const void* src, void* dst, double alpha, double beta, int cm, double ims,
                 cudaStream_t st) {
  PermOp op = perm_op(P, src, dst, alpha, beta, ims);
  if (P.jobs.empty()) return;
  const PermJob* jobs = (const PermJob*)P.d_jobs.p;
  if (P.split) {
    const int nrest = P.njobs - P.njobs_rows;
    if (P.njobs_rows)
      check_cuda(launch_permute(op, op, jobs, P.njobs_rows, 0, false, kLaunchRowsOnly, cm, st), "permute launch");
    check_cuda(launch_permute(op, op, jobs + P.njobs_rows, nrest, P.njobs_multi, P.tiled, kLaunchGeneral, cm, st),
               "permute launch");
    g_launches += (P.njobs_rows > 0) + (nrest > 0) + (P.njobs_multi > 0);
  } else {
    const int variant = P.rows_only ? kLaunchRowsOnly : kLaunchGeneral;
    check_cuda(launch_permute(op, op, jobs, P.njobs, P.njobs_multi, P.tiled, variant, cm, st), "permute launch");
    g_launches += (P.njobs > 0) + (P.njobs_multi > 0);
  }
}

// one contraction through a plan: operand permutes, grouped GEMM, output permute (Alg. 4)
void run_contract(ContractPlan* P, const void* a, const void* b, void* c, int32_t conjA, int32_t conjB,
                         double alpha, double beta, void* ws, size_t ws_bytes, tk_stream stream) {
  if (ws_bytes < P->ws_bytes || (P->ws_bytes && !ws)) TK_THROW(TK_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
  if (((uintptr_t)ws & 255) != 0) TK_THROW(TK_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  P->ensure_uploaded();
  cudaStream_t st = (cudaStream_t)stream;
  free_deferred(st);
  char* w = (char*)ws;
  const double* At = P->pa.identity ? (const double*)a : (const double*)(w + P->off_a);
  const double* Bt = P->pb.identity ? (const double*)b : (const double*)(w + P->off_b);
  double* Ct = P->pc.identity ? (double*)c : (double*)(w + P->off_c);
  g_launches = 0;
  prof_record(0, st);
  const bool cx = P->cplx;
  if (P->gather) {  // A~ and B~ are gathered inside the GEMM: no permute pass
    prof_record(1, st);
  } else if (P->merged_ab) {
    PermOp oa = perm_op(P->pa, a, (double*)At, 1.0, 0.0, 1.0), ob = perm_op(P->pb, b, (double*)Bt, 1.0, 0.0, 1.0);
    check_cuda(launch_permute(oa, ob, (const PermJob*)P->d_jobs_ab.p, P->njobs_ab, P->njobs_ab_multi, P->ab_tiled,
                              kLaunchGeneral, kPermReal, st),
               "permute launch");
    g_launches += (P->njobs_ab > 0) + (P->njobs_ab_multi > 0);
  } else if (!P->pa.identity) {
    run_permute(P->pa, a, (double*)At, 1.0, 0.0, cx ? kPermCToPlanar : kPermReal, conjA ? -1.0 : 1.0, st);
  }
  if (!P->gather) prof_record(1, st);
  if (!P->gather && !P->merged_ab && !P->pb.identity)
    run_permute(P->pb, b, (double*)Bt, 1.0, 0.0, cx ? kPermCToRealRep : kPermReal, conjB ? -1.0 : 1.0, st);
  prof_record(2, st);
  double ga = P->pc.identity ? alpha : 1.0, gb = P->pc.identity ? beta : 0.0;
  if (!P->tiles.empty()) {
    int nbig = P->ntiles_big;
    const GemmTile* d_tiles = (const GemmTile*)P->d_tiles.p;
    if (P->tma && nbig > 0) {
      GemmTmaParams* prm = nullptr;
      {
        std::lock_guard<std::mutex> g(P->tma_mu);
        if (!P->tma_params || P->tma_a != At || P->tma_b != Bt) {
          if (!P->tma_params) P->tma_params = std::make_unique<GemmTmaParams>();
          P->tma_a = P->tma_b = nullptr;
          if (gemm_tma_encode(*P->tma_params, P->ggroups, P->tma_groups, At, Bt)) {
            P->tma_a = At;
            P->tma_b = Bt;
          }
        }
        if (P->tma_a == At && P->tma_b == Bt) {
          prm = new GemmTmaParams(*P->tma_params);  // per-call copy: output and scalars differ
        }
      }
      if (prm) {
        std::unique_ptr<GemmTmaParams> q(prm);
        q->C = Ct;
        q->tiles = d_tiles;
        q->counter = (int*)(w + P->off_counter);
        check_cuda(cudaMemsetAsync(q->counter, 0, sizeof(int), st), "tile counter reset");
        q->ntiles = nbig;
        q->alpha = ga;
        q->beta = gb;
        check_cuda(launch_gemm_tma(*q, std::min(nbig, sm_count()), st), "tma gemm launch");
        ++g_launches;
        d_tiles += nbig;
        nbig = 0;
      }
    }
    check_cuda(launch_gemm(At, Bt, Ct, (const GemmGroup*)P->d_ggroups.p, d_tiles, nbig, P->ntiles_small,
                           P->ntiles_skinny, (const GemmTile*)P->d_heads.p, (int)P->split_heads.size(),
                           (double*)(w + P->off_parts), ga, gb, st),
               "gemm launch");
    g_launches += (nbig > 0) + (P->ntiles_small > 0) + (P->ntiles_skinny > 0 && P->ntiles_small == 0) +
                  !P->split_heads.empty();
  }
  if (P->gather) {  // with the output permute folded in, the stores go to C itself (alpha, sign, beta there)
    check_cuda(launch_gather_gemm((const double*)a, (const double*)b, P->gout ? (double*)c : Ct,
                                  (const int64_t*)P->d_gslots.p, (int)P->gtiles.size(), (const GatherSeg*)P->d_gsegs.p,
                                  (const int32_t*)P->d_btab.p, (const GatherOut*)P->d_gouts.p, P->g_kmax, P->g_nmax,
                                  ga, alpha, P->gout ? beta : gb, st),
               "gather gemm launch");
    g_launches += !P->gtiles.empty();
  }
  prof_record(3, st);
  if (!P->pc.identity && !P->gout)
    run_permute(P->pc, Ct, c, alpha, beta, cx ? kPermPlanarToC : kPermReal, 1.0, st);
  prof_record(4, st);
  if (g_prof.on) {
    g_prof.have = true;
    // merged operand permutes: phase 0 covers both A~ and B~, phase 1 is empty
    g_prof.bytes[0] = (P->pa.identity ? 0 : P->pa.bytes) + (P->merged_ab ? P->pb.bytes : 0);
    g_prof.bytes[1] = (P->pb.identity || P->merged_ab) ? 0 : P->pb.bytes;
    g_prof.bytes[2] = 0;
    g_prof.bytes[3] = P->pc.identity ? 0 : P->pc.bytes;
    g_prof.flops = P->flops;
  }
}

}  // namespace tk

using namespace tk;

#define TK_API_BEGIN try {
#define TK_API_END                                    \
  return TK_OK;                                       \
  }                                                   \
  catch (const tk::Error& e) {                        \
    tk::set_last_error(e.what());                     \
    return e.code;                                    \
  }                                                   \
  catch (const std::exception& e) {                   \
    tk::set_last_error(e.what());                     \
    return TK_ERR_INVALID_ARGUMENT;                   \
  }

extern "C" {

tk_status tk_permute_workspace(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                               const tk_tensor* C, size_t* bytes) {
  TK_API_BEGIN
  if (!A || !C || !bytes) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  std::vector<int> pv(p, p + np), qv(q, q + nq);
  get_perm_plan(*(const Tensor*)A, pv, qv, *(const Tensor*)C);
  *bytes = 0;
  TK_API_END
}

tk_status tk_permute(const tk_tensor* A_, const void* a, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                     const tk_tensor* C_, void* c, double alpha, double beta, void*, size_t, tk_stream stream) {
  TK_API_BEGIN
  if (!A_ || !C_ || (!a && ((const Tensor*)A_)->nelems) || (!c && ((const Tensor*)C_)->nelems))
    TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  if (np < 0 || nq < 0 || (np && !p) || (nq && !q)) TK_THROW(TK_ERR_INVALID_ARGUMENT, "bad permutation arrays");
  const Tensor& A = *(const Tensor*)A_;
  const Tensor& C = *(const Tensor*)C_;
  if (A.dtype != C.dtype) TK_THROW(TK_ERR_INVALID_ARGUMENT, "dtype mismatch");
  std::vector<int> pv(p, p + np), qv(q, q + nq);
  std::shared_ptr<PermPlan> P = get_perm_plan(A, pv, qv, C);
  P->ensure_uploaded();
  free_deferred((cudaStream_t)stream);
  g_launches = 0;
  run_permute(*P, a, c, alpha, beta, A.dtype == TK_C64 ? kPermCToC : kPermReal, 1.0, (cudaStream_t)stream);
  TK_API_END
}

tk_status tk_permute_transfer_planar(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q,
                                     int32_t nq, const tk_tensor* C, int32_t kappa_mode, double* out) {
  TK_API_BEGIN
  if (!A || !C || !out) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  std::vector<int> pv(p, p + np), qv(q, q + nq);
  set_force_planar(true);
  if (kappa_mode >= 0) set_rotation_kappa_mode(kappa_mode);
  try {
    permute_transfer_matrix(*(const Tensor*)A, pv, qv, *(const Tensor*)C, out);
  } catch (...) {
    set_force_planar(false);
    throw;
  }
  set_force_planar(false);
  TK_API_END
}

tk_status tk_permute_transfer(const tk_tensor* A, const int32_t* p, int32_t np, const int32_t* q, int32_t nq,
                              const tk_tensor* C, double* out) {
  TK_API_BEGIN
  if (!A || !C || !out) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  std::vector<int> pv(p, p + np), qv(q, q + nq);
  permute_transfer_matrix(*(const Tensor*)A, pv, qv, *(const Tensor*)C, out);
  TK_API_END
}

tk_status tk_contract_output(const tk_tensor* A_, const int32_t* labA, const tk_tensor* B_, const int32_t* labB,
                             const int32_t* labC, int32_t n_cod_C, tk_tensor** out) {
  TK_API_BEGIN
  if (!A_ || !B_ || !labA || !labB || !out) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  const Tensor& B = *(const Tensor*)B_;
  if (A.kind != B.kind) TK_THROW(TK_ERR_SECTOR_MISMATCH, "sector kinds differ");
  // number of open labels
  int nopen = 0;
  for (int i = 0; i < A.nlegs(); ++i) {
    bool in = false;
    for (int j = 0; j < B.nlegs(); ++j) in |= labA[i] == labB[j];
    nopen += !in;
  }
  for (int j = 0; j < B.nlegs(); ++j) {
    bool in = false;
    for (int i = 0; i < A.nlegs(); ++i) in |= labA[i] == labB[j];
    nopen += !in;
  }
  if (nopen > 0 && !labC) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null labC");
  Tuples t = tuples_from_labels(A, labA, B, labB, labC, nopen, n_cod_C);
  Tensor* At = permuted_tensor(A, t.pA, t.qA, A.dtype);
  Tensor* Bt = permuted_tensor(B, t.pB, t.qB, B.dtype);
  std::vector<Space*> cod(At->cod), dom(Bt->dom);
  Tensor* Ct = make_tensor(A.dtype, cod, dom, (int)A.kind);
  Tensor* C = permuted_tensor(*Ct, t.pAB, t.qAB, A.dtype);
  tk_tensor_release((tk_tensor*)At);
  tk_tensor_release((tk_tensor*)Bt);
  tk_tensor_release((tk_tensor*)Ct);
  *out = (tk_tensor*)C;
  TK_API_END
}

tk_status tk_contract_workspace(const tk_tensor* A, const int32_t* labA, const tk_tensor* B, const int32_t* labB,
                                const tk_tensor* C, const int32_t* labC, size_t* bytes) {
  TK_API_BEGIN
  if (!A || !B || !C || !labA || !labB || !bytes) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  auto P = get_contract_plan(*(const Tensor*)A, labA, *(const Tensor*)B, labB, *(const Tensor*)C, labC);
  *bytes = P->ws_bytes;
  TK_API_END
}

tk_status tk_contract(const tk_tensor* A_, const void* a, const int32_t* labA, int32_t conjA, const tk_tensor* B_,
                      const void* b, const int32_t* labB, int32_t conjB, const tk_tensor* C_, void* c,
                      const int32_t* labC, double alpha, double beta, void* ws, size_t ws_bytes, tk_stream stream) {
  TK_API_BEGIN
  if (!A_ || !B_ || !C_ || !labA || !labB) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  const Tensor& B = *(const Tensor*)B_;
  const Tensor& C = *(const Tensor*)C_;
  if ((conjA || conjB) && A.dtype == TK_F64) TK_THROW(TK_ERR_INVALID_ARGUMENT, "conj flags need ComplexF64");
  if ((!a && A.nelems) || (!b && B.nelems) || (!c && C.nelems)) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null data pointer");
  auto P = get_contract_plan(A, labA, B, labB, C, labC);
  run_contract(P.get(), a, b, c, conjA, conjB, alpha, beta, ws, ws_bytes, stream);
  TK_API_END
}

tk_status tk_contract_tuples_output(const tk_tensor* A_, const tk_tensor* B_, const int32_t* tup,
                                   const int32_t* ntup, tk_tensor** out) {
  TK_API_BEGIN
  if (!A_ || !B_ || !out) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  const Tensor& B = *(const Tensor*)B_;
  if (A.kind != B.kind) TK_THROW(TK_ERR_SECTOR_MISMATCH, "sector kinds differ");
  if (A.dtype != B.dtype) TK_THROW(TK_ERR_INVALID_ARGUMENT, "dtypes differ");
  Tuples t = tuples_from_arrays(A, B, tup, ntup);
  Tensor* At = permuted_tensor(A, t.pA, t.qA, A.dtype);
  Tensor* Bt = permuted_tensor(B, t.pB, t.qB, B.dtype);
  std::vector<Space*> cod(At->cod), dom(Bt->dom);
  Tensor* Ct = make_tensor(A.dtype, cod, dom, (int)A.kind);
  Tensor* C = permuted_tensor(*Ct, t.pAB, t.qAB, A.dtype);
  tk_tensor_release((tk_tensor*)At);
  tk_tensor_release((tk_tensor*)Bt);
  tk_tensor_release((tk_tensor*)Ct);
  *out = (tk_tensor*)C;
  TK_API_END
}

tk_status tk_contract_tuples_workspace(const tk_tensor* A, const tk_tensor* B, const tk_tensor* C, const int32_t* tup,
                                       const int32_t* ntup, size_t* bytes) {
  TK_API_BEGIN
  if (!A || !B || !C || !bytes) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  auto P = get_contract_plan_tuples(*(const Tensor*)A, *(const Tensor*)B, *(const Tensor*)C, tup, ntup);
  *bytes = P->ws_bytes;
  TK_API_END
}

tk_status tk_contract_tuples(const tk_tensor* A_, const void* a, int32_t conjA, const tk_tensor* B_, const void* b,
                             int32_t conjB, const tk_tensor* C_, void* c, const int32_t* tup, const int32_t* ntup,
                             double alpha, double beta, void* ws, size_t ws_bytes, tk_stream stream) {
  TK_API_BEGIN
  if (!A_ || !B_ || !C_) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  const Tensor& A = *(const Tensor*)A_;
  const Tensor& B = *(const Tensor*)B_;
  const Tensor& C = *(const Tensor*)C_;
  if ((conjA || conjB) && A.dtype == TK_F64) TK_THROW(TK_ERR_INVALID_ARGUMENT, "conj flags need ComplexF64");
  if ((!a && A.nelems) || (!b && B.nelems) || (!c && C.nelems)) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null data pointer");
  auto P = get_contract_plan_tuples(A, B, C, tup, ntup);
  run_contract(P.get(), a, b, c, conjA, conjB, alpha, beta, ws, ws_bytes, stream);
  TK_API_END
}

tk_status tk_profile_enable(int32_t on) {
  g_prof.on = on != 0;
  return TK_OK;
}

tk_status tk_phase_times(float* ms4, double* bytes4, double* flops) {
  TK_API_BEGIN
  if (!g_prof.have) TK_THROW(TK_ERR_INVALID_ARGUMENT, "no profiled tk_contract call");
  for (int i = 0; i < 4; ++i) {
    float m = 0;
    check_cuda(cudaEventElapsedTime(&m, g_prof.ev[i], g_prof.ev[i + 1]), "event timing");
    if (ms4) ms4[i] = m;
    if (bytes4) bytes4[i] = g_prof.bytes[i];
  }
  if (flops) *flops = g_prof.flops;
  TK_API_END
}

int32_t tk_last_launch_count(void) { return g_launches; }

tk_status tk_contract_roofline(const tk_tensor* A, const int32_t* labA, const tk_tensor* B, const int32_t* labB,
                               const tk_tensor* C, const int32_t* labC, double peak_flops, double peak_bytes_per_s,
                               double* out4) {
  TK_API_BEGIN
  if (!A || !B || !C || !labA || !labB || !out4) TK_THROW(TK_ERR_INVALID_ARGUMENT, "null argument");
  if (!(peak_flops > 0) || !(peak_bytes_per_s > 0)) TK_THROW(TK_ERR_INVALID_ARGUMENT, "peaks must be positive");
  auto P = get_contract_plan(*(const Tensor*)A, labA, *(const Tensor*)B, labB, *(const Tensor*)C, labC);
  const double cm = P->cplx ? 2.0 : 1.0, s = P->cplx ? 16.0 : 8.0;
  double flops = 0, gbytes = 0, t = 0;
  for (const GemmGroup& g : P->ggroups) {  // the real-representation GEMM: M x cm K x cm N
    const double M = g.M, K = g.K / cm, N = g.N / cm;
    const double f = (P->cplx ? 8.0 : 2.0) * M * K * N;
    const double by = s * (M * K + K * N + M * N);
    flops += f;
    gbytes += by;
    t += std::max(f / peak_flops, by / peak_bytes_per_s);
  }
  const double pbytes = (P->pa.identity ? 0.0 : P->pa.bytes) + (P->pb.identity ? 0.0 : P->pb.bytes) +
                        (P->pc.identity ? 0.0 : P->pc.bytes);
  out4[0] = flops;
  out4[1] = gbytes;
  out4[2] = pbytes;
  out4[3] = t + pbytes / peak_bytes_per_s;
  TK_API_END
}

tk_status tk_dmma_probe(int32_t blocks, int64_t iters, tk_stream stream, double* flops) {
  TK_API_BEGIN
  if (blocks < 1 || iters < 1) TK_THROW(TK_ERR_INVALID_ARGUMENT, "blocks and iters must be >= 1");
  check_cuda(launch_dmma_probe(blocks, (long long)iters, (cudaStream_t)stream), "dmma probe launch");
  if (flops) *flops = (double)blocks * 8.0 * (double)iters * 8.0 * (2.0 * 8 * 8 * 4);
  TK_API_END
}

void tk_cache_clear(void) { tk::cache_clear(); }

int64_t tk_cache_size(void) { return (int64_t)(tk::cache_size() + tk::svd_cache_size() + tk::trace_cache_size() +
                                          tk::fused_cache_size() + tk::ncon_cache_size()); }

}  // extern "C"
