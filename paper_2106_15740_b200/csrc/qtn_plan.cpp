// Plan compiler: (sliced network structure, elimination order) -> bucket
// program for the sm_100a executors.  Pure host code (no GPU needed), so the
// reference's argument errors and the rank cap fire before any allocation.
//
// Semantics follow the reference bucket loop
//   _contract_with_ranks  /root/reference/pkg/src/qtnsim/contraction.py:57-111
// step by step: the order must be a permutation of the unfixed variables
// (60-62); bucket = ascending ids of the live tensors holding v (76); an empty
// bucket multiplies by 2 (77-81); the union rank is checked against the cap
// before anything is materialised (82-88); consumed tensors leave the live
// set and the result enters it with a fresh id (98-106); rank-0 tensors fold
// into the scalar at the end (108-110).  What differs is only HOW a bucket is
// evaluated: one fused pass (product of all operands and the v-sum) instead
// of the pairwise `_product` chain, with an output layout chosen so that the
// largest operand streams contiguously.
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "qtn_internal.h"
#include "qtn_stream.h"

namespace qtn {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

void make_runs(const std::vector<std::pair<int, int>>& src_dst, std::vector<uint32_t>& runs) {
  // src_dst: (bit in source index, bit in destination index); merge runs
  // where both advance by one.
  std::vector<std::pair<int, int>> p = src_dst;
  std::sort(p.begin(), p.end(), [](auto a, auto b) { return a.second < b.second; });
  runs.clear();
  size_t i = 0;
  while (i < p.size()) {
    int s = p[i].first, d = p[i].second, len = 1;
    while (i + len < p.size() && p[i + len].first == s + len && p[i + len].second == d + len) ++len;
    runs.push_back(pack_run((uint32_t)s, (uint32_t)d, (uint32_t)len));
    i += len;
  }
}

namespace {

// Split runs of the output index into the tile-local part (bits < tile_bits)
// and the per-tile part (bits >= tile_bits).
void split_runs(const std::vector<std::pair<int, int>>& src_dst, int tile_bits,
                std::vector<uint32_t>& lo, std::vector<uint32_t>& hi) {
  std::vector<std::pair<int, int>> a, b;
  for (auto& x : src_dst) (x.first < tile_bits ? a : b).push_back(x);
  make_runs(a, lo);
  make_runs(b, hi);
}

struct Block {
  int64_t off, size;
  int32_t start, end;  // inclusive lifetime in bucket steps
};

// First-fit placement on a (time x address) plane.
int64_t place(std::vector<Block>& blocks, int64_t size, int32_t start, int32_t end,
              int64_t align) {
  std::vector<std::pair<int64_t, int64_t>> busy;
  for (auto& b : blocks)
    if (!(b.end < start || b.start > end)) busy.push_back({b.off, b.off + b.size});
  std::sort(busy.begin(), busy.end());
  int64_t off = 0;
  for (auto& iv : busy) {
    if (iv.first >= off + size) break;
    off = std::max(off, (iv.second + align - 1) / align * align);
  }
  blocks.push_back({off, size, start, end});
  return off;
}

int64_t elem_bytes(bool c64) { return c64 ? 8 : 16; }

}  // namespace

// Output layout rule: primary = first operand of maximal rank; variables
// the primary lacks go on the most significant bits (union order), then the
// primary's own variables minus v in the primary's order on the low bits.
static void choose_layout(const std::vector<std::vector<int32_t>>& opvars, int32_t v,
                          int32_t& primary, std::vector<int32_t>& out_vars) {
  primary = 0;
  for (size_t i = 1; i < opvars.size(); ++i)
    if (opvars[i].size() > opvars[primary].size()) primary = (int32_t)i;
  const auto& pv = opvars[primary];
  std::vector<int32_t> uni;
  for (auto& vs : opvars)
    for (int32_t u : vs)
      if (std::find(uni.begin(), uni.end(), u) == uni.end()) uni.push_back(u);
  out_vars.clear();
  for (int32_t u : uni)
    if (u != v && std::find(pv.begin(), pv.end(), u) == pv.end()) out_vars.push_back(u);
  for (int32_t u : pv)
    if (u != v) out_vars.push_back(u);
}

// Operand index as (src bit in o, dst bit in operand) pairs + v's bit.
static void operand_map(const std::vector<int32_t>& vars, const std::vector<int32_t>& out_vars,
                        int32_t v, std::vector<std::pair<int, int>>& sd, int& vshift) {
  const int R = (int)out_vars.size(), r = (int)vars.size();
  sd.clear();
  vshift = -1;
  for (int k = 0; k < r; ++k) {
    int dst = r - 1 - k;
    if (vars[k] == v) {
      vshift = dst;
      continue;
    }
    int idx = (int)(std::find(out_vars.begin(), out_vars.end(), vars[k]) - out_vars.begin());
    sd.push_back({R - 1 - idx, dst});
  }
}

// Build the HBM-executor launch template of one bucket.  Operands: the
// primary first (streamed), small ones folded into shared-memory lookup
// tables, the rest gathered from global memory.
static int build_bucket_args(const std::vector<std::vector<int32_t>>& opvars,
                             const std::vector<uint8_t>& opc64, int32_t primary, int32_t v,
                             const std::vector<int32_t>& out_vars, bool out_c64,
                             bool primary_aligned, BucketArgs& a,
                             std::vector<int32_t>& g_ops, std::vector<int32_t>& t_ops) {
  std::memset(&a, 0, sizeof(a));
  const int R = (int)out_vars.size();
  a.R = (uint32_t)R;
  a.n_out = 1ull << R;
  a.out_c64 = out_c64;
  a.primary = primary_aligned ? 1u : 0u;
  g_ops.clear();
  t_ops.clear();
  std::vector<std::pair<int, int>> sd;
  int vshift;
  std::vector<uint32_t> lo, hi;
  auto add_g = [&](int i) -> bool {
    if ((int)a.ng >= kMaxG) return false;
    operand_map(opvars[i], out_vars, v, sd, vshift);
    split_runs(sd, kTileBits, lo, hi);
    if ((int)lo.size() > kMaxRuns || (int)hi.size() > kMaxRuns) return false;
    GOpArg& g = a.g[a.ng++];
    g.vshift = (uint32_t)vshift;
    g.c64 = opc64[i];
    g.n_lo = (uint32_t)lo.size();
    g.n_hi = (uint32_t)hi.size();
    std::copy(lo.begin(), lo.end(), g.lo);
    std::copy(hi.begin(), hi.end(), g.hi);
    g_ops.push_back(i);
    return true;
  };
  if (primary_aligned) {
    add_g(primary);
    // v's bit inside the primary operand
    const auto& pv = opvars[primary];
    a.p_k = (uint32_t)(pv.size() - 1 - (std::find(pv.begin(), pv.end(), v) - pv.begin()));
  }
  // candidates for tables: non-primary operands with <= kTBits non-v bits
  std::vector<int> cand, rest;
  for (int i = 0; i < (int)opvars.size(); ++i) {
    if (primary_aligned && i == primary) continue;
    if ((int)opvars[i].size() - 1 <= kTBits) cand.push_back(i);
    else rest.push_back(i);
  }
  std::stable_sort(cand.begin(), cand.end(),
                   [&](int x, int y) { return opvars[x].size() > opvars[y].size(); });
  // bits of o per candidate
  auto obits = [&](int i) {
    std::vector<int> b;
    for (int32_t u : opvars[i]) {
      if (u == v) continue;
      int idx = (int)(std::find(out_vars.begin(), out_vars.end(), u) - out_vars.begin());
      b.push_back(R - 1 - idx);
    }
    return b;
  };
  std::vector<std::vector<int>> tbits;       // o bits per table
  std::vector<std::vector<int>> tmembers;    // operand indices per table
  for (int i : cand) {
    auto b = obits(i);
    int best = -1, best_overlap = -1;
    for (int t = 0; t < (int)tbits.size(); ++t) {
      std::vector<int> u = tbits[t];
      int overlap = 0;
      for (int x : b) {
        if (std::find(u.begin(), u.end(), x) == u.end()) u.push_back(x);
        else ++overlap;
      }
      if ((int)u.size() <= kTBits && overlap > best_overlap) {
        best = t;
        best_overlap = overlap;
      }
    }
    int total_members = 0;
    for (auto& m : tmembers) total_members += (int)m.size();
    if (total_members >= kMaxTOps) {
      rest.push_back(i);
      continue;
    }
    if (best < 0) {
      if ((int)tbits.size() >= kMaxT) {
        rest.push_back(i);
        continue;
      }
      tbits.push_back({});
      tmembers.push_back({});
      best = (int)tbits.size() - 1;
    }
    for (int x : b)
      if (std::find(tbits[best].begin(), tbits[best].end(), x) == tbits[best].end())
        tbits[best].push_back(x);
    tmembers[best].push_back(i);
  }
  uint32_t smem_off = 0;
  for (int t = 0; t < (int)tbits.size(); ++t) {
    auto& bits = tbits[t];
    std::sort(bits.begin(), bits.end());
    TableArg& ta = a.t[a.nt++];
    ta.nbits = (uint32_t)bits.size();
    std::vector<std::pair<int, int>> osd;
    for (int b = 0; b < (int)bits.size(); ++b) osd.push_back({bits[b], b});
    split_runs(osd, kTileBits, lo, hi);
    ta.n_lo = (uint32_t)lo.size();
    ta.n_hi = (uint32_t)hi.size();
    std::copy(lo.begin(), lo.end(), ta.lo);
    std::copy(hi.begin(), hi.end(), ta.hi);
    ta.first_op = a.ntop;
    ta.n_ops = (uint32_t)tmembers[t].size();
    ta.smem_off = smem_off;
    smem_off += 2u << bits.size();
    for (int i : tmembers[t]) {
      TOpArg& to = a.top[a.ntop++];
      to.c64 = opc64[i];
      std::vector<std::pair<int, int>> tsd;
      int vs = -1;
      const auto& vars = opvars[i];
      const int r = (int)vars.size();
      for (int k = 0; k < r; ++k) {
        int dst = r - 1 - k;
        if (vars[k] == v) {
          vs = dst;
          continue;
        }
        int idx = (int)(std::find(out_vars.begin(), out_vars.end(), vars[k]) - out_vars.begin());
        int ob = R - 1 - idx;
        int tb = (int)(std::find(bits.begin(), bits.end(), ob) - bits.begin());
        tsd.push_back({tb, dst});
      }
      std::vector<uint32_t> runs;
      make_runs(tsd, runs);
      to.vshift = (uint32_t)vs;
      to.n_runs = (uint32_t)runs.size();
      std::copy(runs.begin(), runs.end(), to.runs);
      t_ops.push_back(i);
    }
  }
  a.table_entries = smem_off;
  for (int i : rest)
    if (!add_g(i)) {
      set_error("bucket has too many wide operands for one fused pass");
      return QTN_EINVAL;
    }
  return QTN_OK;
}

// Streaming descriptor of one bucket (qtn_stream.h): the same operand split
// as build_bucket_args (primary streamed, small operands tabulated, the rest
// gathered), runs stored whole (gathers are OR-linear over output bits, so
// the kernel splits tile-base and tile-local parts itself), tile size chosen
// so that a tile's primary slice is <= 32 KiB.
int encode_stream_desc(const BucketSpec& s, std::vector<uint8_t>& blob) {
  BucketArgs a;
  std::vector<int32_t> g_ops, t_ops;
  int rc = build_bucket_args(s.opvars, s.opc64, s.primary, s.v, s.out_vars, s.out_c64, true, a,
                             g_ops, t_ops);
  if (rc) return rc;
  if ((int)a.ng - 1 > kSMaxG || (int)a.nt > kSMaxT || (int)a.ntop > kSMaxTOps) {
    set_error("bucket has too many operands for the streaming kernel");
    return QTN_EINVAL;
  }
  const size_t base = blob.size();
  const int ng = (int)a.ng - 1;
  const size_t bytes = sizeof(SHdr) + ng * sizeof(SGRec) + a.nt * sizeof(STRec) +
                       a.ntop * sizeof(SORec);
  blob.resize(base + bytes, 0);
  SHdr* h = reinterpret_cast<SHdr*>(blob.data() + base);
  const int R = (int)s.out_vars.size();
  const bool pc64 = s.opc64[s.primary] != 0;
  const int tb = std::min(R, pc64 ? kTileBitsC64 : kTileBitsC128);
  h->out = s.out_tag;
  h->p = s.optag[s.primary];
  h->R = (uint8_t)R;
  h->out_c64 = s.out_c64 ? 1 : 0;
  h->p_c64 = pc64 ? 1 : 0;
  h->p_k = (uint8_t)a.p_k;
  h->p_rank = (uint8_t)s.opvars[s.primary].size();
  h->ng = (uint8_t)ng;
  h->nt = (uint8_t)a.nt;
  h->ntop = (uint8_t)a.ntop;
  // tile-local bits: ta low bits of the primary + tn of the new (high) bits,
  // so an expanding bucket (output wider than the primary) reuses each
  // primary slice from shared memory instead of re-reading it 2^(new) times
  const int rp1 = (int)s.opvars[s.primary].size() - 1;
  const int dnew = R - rp1;
  // e-bit of an output bit for a given split (ta, tn); -1: not tile-local
  auto e_bit = [&](int ob, int ta_, int tn_) -> int {
    if (ob < ta_) return ob;
    if (ob >= rp1 && ob < rp1 + tn_) return ta_ + (ob - rp1);
    return -1;
  };
  // choose tn (new-bit part of the tile) by a per-tile byte model: primary
  // slice + gathered operands (staged slice if it depends on <= kStageMaxK
  // tile-local bits, else one 32-byte sector per element and v)
  int ta = std::min(rp1, tb), tn = tb - ta;
  {
    double best = 1e300;
    const int esz = pc64 ? 8 : 16;
    const char* tmv = getenv("QTN_TN_MAX");  // experiment knob: cap the new-bit tile part
    const int tn_max = tmv ? atoi(tmv) : 64;
    const char* swv = getenv("QTN_STAGE_W");
    const double stage_w = swv ? atof(swv) : 1024.0;  // measured: a cp.async-gathered entry costs far more than a bulk byte
    for (int tn_c = std::max(0, tb - rp1); tn_c <= std::min(std::min(dnew, tb), std::max(tn_max, tb - rp1)); ++tn_c) {
      const int ta_c = tb - tn_c;
      // ta = 0 with v off bit 0 of the primary would need the two-chunk
      // (split) slice, which the tile kernel only takes for ta >= 1
      if (ta_c > rp1 || ta_c < 0 || (ta_c == 0 && a.p_k >= 1)) continue;
      double cost = (double)(2 << ta_c) * esz;
      for (int i = 1; i < (int)a.ng; ++i) {
        int k = 0;
        const GOpArg& src = a.g[i];
        for (uint32_t r = 0; r < src.n_lo + src.n_hi; ++r) {
          const uint32_t w = r < src.n_lo ? src.lo[r] : src.hi[r - src.n_lo];
          for (uint32_t q = 0; q < ((w >> 16) & 0xff); ++q)
            if (e_bit((int)(w & 0xff) + (int)q, ta_c, tn_c) >= 0) ++k;
        }
        cost += (i == 1 && k <= kStageMaxK) ? (double)(2 << k) * stage_w : (double)(2 << tb) * 32.0;
      }
      if (cost < best - 1e-9) {
        best = cost;
        ta = ta_c;
        tn = tn_c;
      }
    }
  }
  h->tb = (uint8_t)tb;
  h->ta = (uint8_t)ta;
  h->tn = (uint8_t)tn;
  auto e_of = [&](int ob) -> int { return e_bit(ob, ta, tn); };
  auto pairs_of = [](const uint32_t* runs, int n) {
    std::vector<std::pair<int, int>> pr;
    for (int r = 0; r < n; ++r)
      for (uint32_t q = 0; q < ((runs[r] >> 16) & 0xff); ++q)
        pr.push_back({(int)(runs[r] & 0xff) + (int)q, (int)((runs[r] >> 8) & 0xff) + (int)q});
    return pr;
  };
  auto eruns_of = [&](const uint32_t* runs, int n, std::vector<uint32_t>& out) {
    std::vector<std::pair<int, int>> ep;
    for (auto& pr : pairs_of(runs, n)) {
      const int e = e_of(pr.first);
      if (e >= 0) ep.push_back({e, pr.second});
    }
    make_runs(ep, out);
  };
  h->table_entries = (uint16_t)a.table_entries;
  h->desc_bytes = (uint16_t)bytes;
  h->n_tiles = 1ull << (R - ta - tn);
  SGRec* g = reinterpret_cast<SGRec*>(blob.data() + base + sizeof(SHdr));
  for (int i = 0; i < ng; ++i) {
    const GOpArg& src = a.g[i + 1];
    g[i].ptr = s.optag[g_ops[i + 1]];
    g[i].vshift = (uint8_t)src.vshift;
    g[i].c64 = (uint8_t)src.c64;
    g[i].n_runs = (uint8_t)(src.n_lo + src.n_hi);
    std::copy(src.lo, src.lo + src.n_lo, g[i].runs);
    std::copy(src.hi, src.hi + src.n_hi, g[i].runs + src.n_lo);
    std::vector<uint32_t> er;
    eruns_of(g[i].runs, g[i].n_runs, er);
    if ((int)er.size() > kERuns) {
      set_error("gathered operand needs too many tile-local runs");
      return QTN_EINVAL;
    }
    g[i].n_erun = (uint8_t)er.size();
    std::copy(er.begin(), er.end(), g[i].erun);
    // Staging: if the operand depends on only k <= 7 tile-local bits, a tile
    // touches 2^(k+1) of its entries; the producer warp gathers that slice
    // into the stage with cp.async instead of every element re-reading it
    // from L2 (the "two wide operands -> wider output" buckets).
    g[i].stage_k = 0xff;
    std::vector<std::pair<int, int>> s_sd, g_sd;
    {
      std::vector<std::pair<int, int>> ep;
      for (auto& pr : pairs_of(g[i].runs, g[i].n_runs)) {
        const int e = e_of(pr.first);
        if (e >= 0) ep.push_back({e, pr.second});
      }
      std::sort(ep.begin(), ep.end());
      for (auto& pr : ep) {
        s_sd.push_back({pr.first, (int)s_sd.size()});
        g_sd.push_back({(int)g_sd.size(), pr.second});
      }
    }
    const int k = (int)s_sd.size();
    if (i == 0 && k <= kStageMaxK && k <= tb - 2) {
      std::vector<uint32_t> sr, grr;
      make_runs(s_sd, sr);
      make_runs(g_sd, grr);
      g[i].stage_k = (uint8_t)k;
      g[i].n_srun = (uint8_t)sr.size();
      g[i].n_grun = (uint8_t)grr.size();
      std::copy(sr.begin(), sr.end(), g[i].srun);
      std::copy(grr.begin(), grr.end(), g[i].grun);
    }
  }
  if (getenv("QTN_DEBUG_DESC") && R >= atoi(getenv("QTN_DEBUG_DESC")))
    fprintf(stderr, "desc R=%d prank=%d pc64=%d oc64=%d tb=%d ta=%d tn=%d pk=%d ng=%d nt=%d stage_k=%d\n", R,
            (int)h->p_rank, (int)pc64, (int)h->out_c64, tb, ta, tn, (int)a.p_k, ng, (int)a.nt,
            ng ? (int)g[0].stage_k : -1);
  STRec* t = reinterpret_cast<STRec*>(blob.data() + base + sizeof(SHdr) + ng * sizeof(SGRec));
  for (uint32_t j = 0; j < a.nt; ++j) {
    const TableArg& src = a.t[j];
    t[j].nbits = (uint8_t)src.nbits;
    t[j].n_runs = (uint8_t)(src.n_lo + src.n_hi);
    t[j].first_op = (uint8_t)src.first_op;
    t[j].n_ops = (uint8_t)src.n_ops;
    t[j].smem_off = (uint16_t)src.smem_off;
    std::copy(src.lo, src.lo + src.n_lo, t[j].runs);
    std::copy(src.hi, src.hi + src.n_hi, t[j].runs + src.n_lo);
    std::vector<uint32_t> er;
    eruns_of(t[j].runs, t[j].n_runs, er);
    t[j].n_erun = (uint8_t)er.size();
    std::copy(er.begin(), er.end(), t[j].erun);
  }
  SORec* o = reinterpret_cast<SORec*>(blob.data() + base + sizeof(SHdr) + ng * sizeof(SGRec) +
                                      a.nt * sizeof(STRec));
  for (uint32_t k = 0; k < a.ntop; ++k) {
    const TOpArg& src = a.top[k];
    o[k].ptr = s.optag[t_ops[k]];
    o[k].vshift = (uint8_t)src.vshift;
    o[k].c64 = (uint8_t)src.c64;
    o[k].n_runs = (uint8_t)src.n_runs;
    std::copy(src.runs, src.runs + src.n_runs, o[k].runs);
  }
  return QTN_OK;
}

// Expanding-bucket descriptor (qtn_stream.h XDesc, kernel in qtn_expand.cu).
// Geometry: A bits = output bits 0-5 plus 3 more bits the B-side operands do
// not depend on where possible (so the stage stays small), B bits = the
// lowest h bits no A-side operand depends on, h as large as the stage
// (<= kXStageMax entries) and a healthy tile count allow.
bool encode_expand_desc(const BucketSpec& s, XDesc& d) {
  const char* ev = getenv("QTN_EXPAND_MIN_R");
  const int min_r = ev ? atoi(ev) : 14;  // measured: 14 beats 18 on configs 3 default and 4
  const int R = (int)s.out_vars.size();
  if (R < min_r || R > 40) return false;
  std::memset(&d, 0, sizeof(d));
  auto obit = [&](int32_t u) -> int {
    for (int i = 0; i < R; ++i)
      if (s.out_vars[i] == u) return R - 1 - i;
    return -1;
  };
  const int n = (int)s.opvars.size();
  std::vector<uint64_t> dep(n, 0);  // output bits each operand depends on
  for (int t = 0; t < n; ++t)
    for (int32_t u : s.opvars[t])
      if (u != s.v) {
        const int b = obit(u);
        if (b < 0) return false;
        dep[t] |= 1ull << b;
      }
  const uint64_t pdep = dep[s.primary];
  std::vector<int> A, Bs;
  for (int t = 0; t < n; ++t) ((dep[t] & ~pdep) == 0 ? A : Bs).push_back(t);
  if (Bs.empty() || (int)A.size() > kXMaxOps || (int)Bs.size() > kXMaxOps) return false;
  uint64_t adep = 0, bdep = 0;
  for (int t : A) adep |= dep[t];
  for (int t : Bs) bdep |= dep[t];
  // A bits: 0..5 (coalesced 512-byte warp stores) + 3 more, never a bit the
  // A side does not depend on (those are the candidates for B bits)
  std::vector<int> ta;
  for (int b = 0; b < 6; ++b) {
    if (!((adep >> b) & 1)) return false;
    ta.push_back(b);
  }
  for (int pass = 0; pass < 2 && (int)ta.size() < kXABits; ++pass)
    for (int b = 6; b < R && (int)ta.size() < kXABits; ++b) {
      if (!((adep >> b) & 1) || std::find(ta.begin(), ta.end(), b) != ta.end()) continue;
      if (pass == 0 && ((bdep >> b) & 1)) continue;  // first: bits B does not see
      ta.push_back(b);
    }
  if ((int)ta.size() < kXABits) return false;
  std::sort(ta.begin(), ta.end());
  std::vector<int> tc;  // tile-local A bits the B side depends on
  for (int b : ta)
    if ((bdep >> b) & 1) tc.push_back(b);
  const int c = (int)tc.size();
  std::vector<int> nbits;  // B-bit candidates: no A-side dependence
  for (int b = 0; b < R; ++b)
    if (!((adep >> b) & 1)) nbits.push_back(b);
  int h = std::min<int>((int)nbits.size(), 8);
  while (h > 0 && (2 << (h + c)) > kXStageMax) --h;
  // keep >= ~2 tiles per SM when the bucket allows it
  while (h > 2 && R - kXABits - h < 9) --h;
  if (h < 2) return false;
  std::vector<int> tb(nbits.begin(), nbits.begin() + h);
  std::vector<int> rest;
  for (int b = 0; b < R; ++b)
    if (std::find(ta.begin(), ta.end(), b) == ta.end() && std::find(tb.begin(), tb.end(), b) == tb.end())
      rest.push_back(b);
  auto put = [&](const std::vector<std::pair<int, int>>& pr, uint32_t* dst, uint8_t& cnt) {
    std::vector<uint32_t> runs;
    make_runs(pr, runs);
    if ((int)runs.size() > kXRuns) return false;
    std::copy(runs.begin(), runs.end(), dst);
    cnt = (uint8_t)runs.size();
    return true;
  };
  std::vector<std::pair<int, int>> pr;
  for (size_t i = 0; i < rest.size(); ++i) pr.push_back({(int)i, rest[i]});
  if (!put(pr, d.trun, d.n_trun)) return false;
  pr.clear();
  for (size_t i = 0; i < ta.size(); ++i) pr.push_back({(int)i, ta[i]});
  if (!put(pr, d.arun, d.n_arun)) return false;
  pr.clear();
  for (size_t i = 0; i < tb.size(); ++i) pr.push_back({(int)i, tb[i]});
  if (!put(pr, d.brun, d.n_brun)) return false;
  pr.clear();
  for (size_t i = 0; i < tc.size(); ++i) pr.push_back({(int)i, tc[i]});
  if (!put(pr, d.crun, d.n_crun)) return false;
  pr.clear();
  for (size_t i = 0; i < ta.size(); ++i) {
    auto it = std::find(tc.begin(), tc.end(), ta[i]);
    if (it != tc.end()) pr.push_back({(int)i, (int)(it - tc.begin())});
  }
  if (!put(pr, d.acrun, d.n_acrun)) return false;
  auto op_of = [&](int t, XOp& o) {
    const auto& vs = s.opvars[t];
    const int rk = (int)vs.size();
    if (rk > 32) return false;  // 32-bit operand offsets in the kernel
    std::vector<std::pair<int, int>> q;
    o.vshift = 0xff;
    for (int j = 0; j < rk; ++j) {
      if (vs[j] == s.v) o.vshift = (uint8_t)(rk - 1 - j);
      else q.push_back({obit(vs[j]), rk - 1 - j});
    }
    if (o.vshift == 0xff) return false;
    o.ptr = s.optag[t];
    o.c64 = s.opc64[t];
    return put(q, o.runs, o.n_runs);
  };
  int k = 0;
  for (int t : A)
    if (!op_of(t, d.ops[k++])) return false;
  for (int t : Bs)
    if (!op_of(t, d.ops[k++])) return false;
  d.out = s.out_tag;
  d.R = (uint8_t)R;
  d.out_c64 = s.out_c64 ? 1 : 0;
  d.h = (uint8_t)h;
  d.c = (uint8_t)c;
  d.nA = (uint8_t)A.size();
  d.nB = (uint8_t)Bs.size();
  d.n_tiles = 1ull << (R - kXABits - h);
  if (getenv("QTN_DEBUG_DESC") && R >= atoi(getenv("QTN_DEBUG_DESC")))
    fprintf(stderr, "xdesc R=%d h=%d c=%d nA=%d nB=%d tiles=%llu\n", R, h, c, (int)A.size(),
            (int)Bs.size(), (unsigned long long)d.n_tiles);
  return true;
}

// Expanding bucket + consumers chain (qtn_stream.h YDesc, kernel in
// qtn_xt.cu).  Extended bit space: F's bits [0, R), then the trailing summed
// variables s_j at R + j; v1 and v2 are strides of their own.
bool encode_xt_desc(const YPairSpec& s, YDesc& d) {
  const char* ev = getenv("QTN_XT_MIN_R");
  const int min_r = ev ? atoi(ev) : 14;
  const int R = (int)s.out_vars.size(), K = (int)s.trailing.size();
  if (R + K + 1 < min_r || R < 10 || R > 32 || K > kYMaxK) return false;
  // more than one trailing trace only into large results (measured: config 4
  // 0.575 -> 0.506 ms with them, config 3 default 2.209 -> 2.247 ms: its
  // small chains run slower with 4 groups per thread)
  const char* krv = getenv("QTN_XT_K_MIN_R");
  if (K > 1 && R < (krv ? atoi(krv) : 18)) return false;  // 18..21: config 4 0.508/0.511/0.520/0.520 ms
  std::memset(&d, 0, sizeof(d));
  auto ebit = [&](int32_t u) -> int {
    for (int i = 0; i < R; ++i)
      if (s.out_vars[i] == u) return R - 1 - i;
    for (int j = 0; j < K; ++j)
      if (s.trailing[j] == u) return R + j;
    return -1;
  };
  const int n = (int)s.opvars.size();
  std::vector<uint64_t> dep(n, 0);  // extended bits each operand depends on
  for (int t = 0; t < n; ++t)
    for (int32_t u : s.opvars[t])
      if (u != s.v1 && u != s.v2) {
        const int b = ebit(u);
        if (b < 0) return false;  // the consumers must not add variables
        dep[t] |= 1ull << b;
      }
  for (int t = s.n1; t < n; ++t)  // the consumers' operands never hold v1
    if (std::find(s.opvars[t].begin(), s.opvars[t].end(), s.v1) != s.opvars[t].end()) return false;
  const uint64_t pdep = dep[s.primary];
  std::vector<int> A, Bs, Ws;
  for (int t = 0; t < s.n1; ++t) ((dep[t] & ~pdep) == 0 ? A : Bs).push_back(t);
  if (Bs.empty() || (int)Bs.size() > kYMaxG) return false;
  uint64_t adep = 0, bdep = 0, wdep = 0;
  for (int t : A) adep |= dep[t];
  for (int t : Bs) bdep |= dep[t];
  // consumer operands: on A-side bits only -> A-type (per-thread loads),
  // otherwise staged with the loop bits (W group)
  for (int t = s.n1; t < n; ++t) {
    if ((dep[t] & ~adep) == 0) A.push_back(t);
    else {
      Ws.push_back(t);
      wdep |= dep[t];
    }
  }
  if ((int)A.size() > kYMaxA || (int)Ws.size() > kYMaxG) return false;
  // trailing summed variables: those the A side depends on are owned by the
  // thread (group bits), the others are loop bits (innermost)
  std::vector<int> gbits, sbits;
  for (int j = 0; j < K; ++j) (((adep >> (R + j)) & 1) ? gbits : sbits).push_back(R + j);
  const int g = (int)gbits.size(), hs = (int)sbits.size();
  if (g > kYMaxGB) return false;
  std::vector<int> ta;
  for (int b = 0; b < 6; ++b) {
    if (!((adep >> b) & 1)) return false;
    ta.push_back(b);
  }
  // 3 more A bits: first those neither staged group sees, then one, then any
  for (int pass = 0; pass < 3 && (int)ta.size() < kXABits; ++pass)
    for (int b = 6; b < R && (int)ta.size() < kXABits; ++b) {
      if (!((adep >> b) & 1) || std::find(ta.begin(), ta.end(), b) != ta.end()) continue;
      const int seen = (int)((bdep >> b) & 1) + (int)((wdep >> b) & 1);
      if (seen > pass) continue;
      ta.push_back(b);
    }
  if ((int)ta.size() < kXABits) return false;
  std::sort(ta.begin(), ta.end());
  ta.insert(ta.end(), gbits.begin(), gbits.end());  // element bits 9.. : the groups
  std::vector<int> nbits;  // kept loop-bit candidates: F bits with no A-side dependence
  for (int b = 0; b < R; ++b)
    if (!((adep >> b) & 1)) nbits.push_back(b);
  const char* hv = getenv("QTN_XT_MAX_H");
  const int hmax = std::min<int>(std::min<int>((int)nbits.size() + hs, hv ? atoi(hv) : kYMaxH), kYMaxH);
  std::vector<int> tc, tw;
  for (int b : ta) {
    if ((bdep >> b) & 1) tc.push_back(b);
    if ((wdep >> b) & 1) tw.push_back(b);
  }
  const int c = (int)tc.size(), cw = (int)tw.size();
  int h = hmax;
  while (h > 0 && ((4 << (h + c)) > kYStageB || (!Ws.empty() && (2 << (h + cw)) > kYStageW))) --h;
  const char* tlv = getenv("QTN_XT_TILES_LOG2");
  const int tiles_log2 = tlv ? atoi(tlv) : 9;  // measured 8..11: config 4 0.504 / 0.506 / 0.562 / 0.646 ms
  while (h - hs > 2 && R - kXABits - (h - hs) < tiles_log2) --h;  // >= ~512 tiles when the chain allows it
  if (h < 1 || h < hs || cw > 9 || c > 9) return false;
  std::vector<int> tb(sbits);  // x_b: summed loop bits lowest, then the kept ones
  tb.insert(tb.end(), nbits.begin(), nbits.begin() + (h - hs));
  std::vector<int> rest;
  for (int b = 0; b < R; ++b)
    if (std::find(ta.begin(), ta.end(), b) == ta.end() && std::find(tb.begin(), tb.end(), b) == tb.end())
      rest.push_back(b);
  {
    // Tile order: consecutive tiles of a CTA differ first in the bits neither
    // staged group depends on, then in the bits of the group whose stage
    // costs less to keep (the kernel refills a stage only when its operands'
    // bases change): the larger saving of staged entries per tile wins.
    std::vector<int> f_both, f_b, f_w, others;
    for (int b : rest) {
      const bool sb = (bdep >> b) & 1, sw = !Ws.empty() && ((wdep >> b) & 1);
      (!sb && !sw ? f_both : (!sb ? f_b : (!sw ? f_w : others))).push_back(b);
    }
    const double save_b = (double)(4 << (h + c)) * (1.0 - std::ldexp(1.0, -(int)f_b.size()));
    const double save_w = Ws.empty() ? 0.0 : (double)(2 << (h + cw)) * (1.0 - std::ldexp(1.0, -(int)f_w.size()));
    const char* ov = getenv("QTN_XT_ORDER");
    if (!(ov && ov[0] == '0')) {
      rest = f_both;
      const auto& first = save_b >= save_w ? f_b : f_w;
      const auto& second = save_b >= save_w ? f_w : f_b;
      rest.insert(rest.end(), first.begin(), first.end());
      rest.insert(rest.end(), second.begin(), second.end());
      rest.insert(rest.end(), others.begin(), others.end());
    }
  }
  auto put = [&](const std::vector<std::pair<int, int>>& pr, uint32_t* dst, uint8_t& cnt) {
    std::vector<uint32_t> runs;
    make_runs(pr, runs);
    if ((int)runs.size() > kXRuns) return false;
    std::copy(runs.begin(), runs.end(), dst);
    cnt = (uint8_t)runs.size();
    return true;
  };
  auto put_bits = [&](const std::vector<int>& bits, uint32_t* dst, uint8_t& cnt) {
    std::vector<std::pair<int, int>> pr;
    for (size_t i = 0; i < bits.size(); ++i) pr.push_back({(int)i, bits[i]});
    return put(pr, dst, cnt);
  };
  auto put_sub = [&](const std::vector<int>& sub, uint32_t* dst, uint8_t& cnt) {  // element bits -> compact
    std::vector<std::pair<int, int>> pr;
    for (size_t i = 0; i < ta.size(); ++i) {
      auto it = std::find(sub.begin(), sub.end(), ta[i]);
      if (it != sub.end()) pr.push_back({(int)i, (int)(it - sub.begin())});
    }
    return put(pr, dst, cnt);
  };
  if (!put_bits(rest, d.trun, d.n_trun) || !put_bits(ta, d.arun, d.n_arun) ||
      !put_bits(tb, d.brun, d.n_brun) || !put_bits(tc, d.crun, d.n_crun) ||
      !put_bits(tw, d.wrun, d.n_wrun) || !put_sub(tc, d.acrun, d.n_acrun) ||
      !put_sub(tw, d.awrun, d.n_awrun))
    return false;
  auto op_of = [&](int t, YOp& o) {
    const auto& vs = s.opvars[t];
    const int rk = (int)vs.size();
    if (rk > 32) return false;  // 32-bit operand offsets in the kernel
    std::vector<std::pair<int, int>> q;
    o.vs1 = o.vs2 = 0xff;
    for (int j = 0; j < rk; ++j) {
      if (vs[j] == s.v1) o.vs1 = (uint8_t)(rk - 1 - j);
      else if (vs[j] == s.v2) o.vs2 = (uint8_t)(rk - 1 - j);
      else q.push_back({ebit(vs[j]), rk - 1 - j});
    }
    o.ptr = s.optag[t];
    o.c64 = s.opc64[t];
    return put(q, o.runs, o.n_runs);
  };
  int k = 0;
  for (int t : A)
    if (!op_of(t, d.ops[k++])) return false;
  for (int t : Bs)
    if (!op_of(t, d.ops[k++])) return false;
  for (int t : Ws)
    if (!op_of(t, d.ops[k++])) return false;
  d.out = s.out_tag;
  d.R = (uint8_t)R;
  d.h = (uint8_t)h;
  d.hs = (uint8_t)hs;
  d.c = (uint8_t)c;
  d.cw = (uint8_t)cw;
  d.g = (uint8_t)g;
  d.nA = (uint8_t)A.size();
  d.nB = (uint8_t)Bs.size();
  d.nW = (uint8_t)Ws.size();
  d.n_tiles = 1ull << (R - kXABits - (h - hs));
  if (getenv("QTN_DEBUG_DESC") && R >= atoi(getenv("QTN_DEBUG_DESC")))
  {
    int afree = 0;
    for (int b : rest) afree += !((adep >> b) & 1);
    fprintf(stderr, "ydesc R=%d K=%d h=%d hs=%d g=%d c=%d cw=%d nA=%d nB=%d nW=%d tiles=%llu afree=%d nbits=%zu\n", R, K, h, hs, g,
            c, cw, (int)A.size(), (int)Bs.size(), (int)Ws.size(), (unsigned long long)d.n_tiles, afree, nbits.size());
  }
  return true;
}

// Fused product-chain descriptor (qtn_stream.h FDesc, kernel in
// qtn_fused.cu).  Tile choice: the output's lowest 5 bits (a warp stores 32
// consecutive outputs), the primary's lowest bits (contiguous staging), then
// greedily the U bit that grows the staged bytes least (a bit few or small
// operands depend on is reuse), summed bits first on ties; within one stage
// buffer and <= 11 (complex128: 10) tile output bits.  Sides: an operand
// joins the first side whose widest operand covers its tile bits if that
// side's entries are reused (>= 2 tile bits outside it); streamed sides stay
// raw copies.
namespace {
struct FPlan {
  uint64_t tile = 0;
  std::vector<std::vector<int>> sides;
  uint32_t bytes = 0;
};
}  // namespace

bool encode_fused_desc(const FChainSpec& s, FDesc& d) {
  const int R = (int)s.out_vars.size(), K = (int)s.summed.size(), n = (int)s.opvars.size();
  if (n < 1 || n > kFMaxOps || K < 1 || R + K > 62) return false;
  std::memset(&d, 0, sizeof(d));
  auto ubit = [&](int32_t u) -> int {
    for (int i = 0; i < R; ++i)
      if (s.out_vars[i] == u) return R - 1 - i;
    for (int j = 0; j < K; ++j)
      if (s.summed[j] == u) return R + j;
    return -1;
  };
  const int nu = R + K;
  std::vector<uint64_t> dep(n, 0);
  std::vector<std::vector<int>> opbit(n, std::vector<int>(nu, -1));  // U bit -> operand bit
  int prim = 0;
  for (int t = 0; t < n; ++t) {
    const auto& vs = s.opvars[t];
    const int rk = (int)vs.size();
    if (rk > 32) return false;
    for (int j = 0; j < rk; ++j) {
      const int b = ubit(vs[j]);
      if (b < 0) return false;
      dep[t] |= 1ull << b;
      opbit[t][b] = rk - 1 - j;
    }
    if (vs.size() > s.opvars[prim].size()) prim = t;
  }
  const uint32_t mesz = s.math_f32 ? 8u : 16u;
  const int max_out = kFThreadBits + kFMaxAcc;
  // tuning knobs (experiments): stage budget, terms per CTA, split threshold
  static const uint64_t fbuf = getenv("QTN_FBUF") ? strtoull(getenv("QTN_FBUF"), nullptr, 10) : kFBufBytes;
  static const int fupc = getenv("QTN_FUPC") ? atoi(getenv("QTN_FUPC")) : 16;
  static const int fsplit = getenv("QTN_FSPLIT") ? atoi(getenv("QTN_FSPLIT")) : 16;
  static const int fmaxq = getenv("QTN_FMAXQ") ? atoi(getenv("QTN_FMAXQ")) : kFMaxQ;
  // log2 of the CTAs an item keeps at least before units are packed per CTA
  static const int fmin_units = getenv("QTN_FMIN_UNITS") ? atoi(getenv("QTN_FMIN_UNITS")) : 9;
  auto esz = [&](int t) { return s.opc64[t] ? 8u : 16u; };
  auto make_sides = [&](uint64_t tl) {
    std::vector<int> ord(n);
    for (int t = 0; t < n; ++t) ord[t] = t;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
      const int fa = __builtin_popcountll(dep[a] & tl), fb = __builtin_popcountll(dep[b] & tl);
      return fa != fb ? fa > fb : s.opvars[a].size() > s.opvars[b].size();
    });
    std::vector<std::vector<int>> sides;
    for (int t : ord) {
      bool placed = false;
      for (auto& sd : sides) {
        const uint64_t sdep = dep[sd[0]] & tl;
        const int reuse_bits = __builtin_popcountll(tl) - __builtin_popcountll(sdep);
        if (((dep[t] & tl) & ~sdep) == 0 && reuse_bits >= 2) {
          sd.push_back(t);
          placed = true;
          break;
        }
      }
      if (!placed) sides.push_back({t});
    }
    return sides;
  };
  static int stream_env = -1;
  if (stream_env < 0) {
    // streamed sides are opt-in (QTN_FSTREAM=1): measured slower than the
    // cp.async stage (config 3 default 3.18 -> 3.50 ms, config 4 with every
    // chain fused 1.32 -> 1.60 ms)
    const char* sv = getenv("QTN_FSTREAM");
    stream_env = (sv && sv[0] == '1') ? 1 : 0;
  }
  auto side_kind = [&](const std::vector<int>& sd, uint64_t tl) -> uint8_t {
    if (stream_env && sd.size() == 1 && esz(sd[0]) == mesz && (dep[sd[0]] & tl) == tl &&
        __builtin_popcountll(tl) > kFThreadBits)
      return kFSideStream;
    if (sd.size() == 1 && esz(sd[0]) == mesz) return kFSideRaw;
    if (sd.size() == 1 && __builtin_popcountll(dep[sd[0]] & tl) <= kFThreadBits) return kFSideConv;
    return kFSideProd;
  };
  // stage buffer bytes of a tile: raw regions (raw and product sides' operands)
  // + math-type regions of the conversion and product sides
  auto buf_bytes = [&](uint64_t tl, const std::vector<std::vector<int>>& sides) {
    uint64_t b = 0;
    bool streamed = false;  // at most one streamed side (the kernel reads side 0 from global)
    for (const auto& sd : sides) {
      uint8_t kd = side_kind(sd, tl);
      if (kd == kFSideStream) {
        if (!streamed) {
          streamed = true;
          continue;
        }
        kd = kFSideRaw;
      }
      if (kd != kFSideConv)
        for (int t : sd) b += ((uint64_t)std::max(2u, 1u << __builtin_popcountll(dep[t] & tl)) * esz(t) + 15) & ~15ull;
      if (kd != kFSideRaw)
        b += ((uint64_t)std::max(2u, 1u << __builtin_popcountll(dep[sd[0]] & tl)) * mesz + 15) & ~15ull;
    }
    return b;
  };
  auto n_out = [&](uint64_t tl) { return __builtin_popcountll(tl & ((1ull << R) - 1)); };
  auto fits = [&](uint64_t tl) {
    return buf_bytes(tl, make_sides(tl)) <= std::min<uint64_t>(fbuf, kFBufBytes) && n_out(tl) <= max_out &&
           __builtin_popcountll(tl) <= std::min(fmaxq, kFMaxQ);
  };
  uint64_t tile = 0;
  {
    std::vector<int> want;
    for (int b = 0; b < std::min(R, 5); ++b) want.push_back(b);
    for (int ob = 0; ob < 10; ++ob)
      for (int b = 0; b < nu; ++b)
        if (opbit[prim][b] == ob) want.push_back(b);
    for (int b : want)
      if (!((tile >> b) & 1) && fits(tile | (1ull << b))) tile |= 1ull << b;
  }
  for (;;) {
    int best = -1;
    uint64_t best_f = ~0ull;
    for (int b = 0; b < nu; ++b) {
      if ((tile >> b) & 1) continue;
      const uint64_t tl = tile | (1ull << b);
      if (!fits(tl)) continue;
      uint64_t f = buf_bytes(tl, make_sides(tl)) * 2 + (b < R ? 1 : 0);  // summed bits first on ties
      if (f < best_f || (f == best_f && best >= 0 && opbit[prim][b] >= 0 && opbit[prim][best] >= 0 &&
                         opbit[prim][b] < opbit[prim][best])) {
        best_f = f;
        best = b;
      }
    }
    if (best < 0) break;
    tile |= 1ull << best;
  }
  std::vector<int> qb, lb, gb;  // tile bits (outputs ascending, then summed), loop, grid
  for (int b = 0; b < R; ++b) ((tile >> b) & 1 ? qb : gb).push_back(b);
  const int nto = (int)qb.size();
  for (int b = R; b < nu; ++b) ((tile >> b) & 1 ? qb : lb).push_back(b);
  const int nq = (int)qb.size();
  if (nq < 1) return false;
  auto put = [&](const std::vector<std::pair<int, int>>& pr, uint32_t* dst, uint8_t& cnt, int cap) {
    std::vector<uint32_t> runs;
    make_runs(pr, runs);
    if ((int)runs.size() > cap) return false;
    std::copy(runs.begin(), runs.end(), dst);
    cnt = (uint8_t)runs.size();
    return true;
  };
  std::vector<std::vector<int>> sides = make_sides(tile);
  const int nthr = std::min(nq, kFThreadBits);
  // sides that depend on in-thread tile bits first; the others are constant
  // per thread and stage (factored out of the term loop)
  uint64_t inthr = 0;
  for (int i = nthr; i < nq; ++i) inthr |= 1ull << qb[i];
  std::stable_partition(sides.begin(), sides.end(),
                        [&](const std::vector<int>& sd) { return (dep[sd[0]] & inthr) != 0; });
  int n_var = 0;
  for (const auto& sd : sides) n_var += (dep[sd[0]] & inthr) != 0 ? 1 : 0;
  // the streamed side (if any) goes first: the kernel reads side 0 from global
  {
    int first_stream = -1;
    for (size_t si = 0; si < sides.size() && first_stream < 0; ++si)
      if (side_kind(sides[si], tile) == kFSideStream && (dep[sides[si][0]] & inthr) != 0)
        first_stream = (int)si;
    if (first_stream > 0) std::rotate(sides.begin(), sides.begin() + first_stream, sides.begin() + first_stream + 1);
  }
  // raw regions first (16-byte aligned), then the non-raw side regions
  uint32_t off = 0;
  int k = 0;
  std::vector<int> slot(n, -1);  // op -> position in d.ops
  for (size_t si = 0; si < sides.size(); ++si)
    for (int t : sides[si]) slot[t] = k++;
  for (size_t si = 0; si < sides.size(); ++si) {
    FSide& S = d.sides[si];
    const uint64_t sdep = dep[sides[si][0]] & tile;
    std::vector<int> qa;  // q positions of the side's compact bits
    for (int i = 0; i < nq; ++i)
      if ((sdep >> qb[i]) & 1) qa.push_back(i);
    std::vector<std::pair<int, int>> qr;
    for (size_t c = 0; c < qa.size(); ++c) qr.push_back({qa[c], (int)c});
    if (!put(qr, S.qrun, S.n_qrun, kFQRuns)) return false;
    S.nst = (uint8_t)qa.size();
    S.first_op = (uint8_t)slot[sides[si][0]];
    S.n_ops = (uint8_t)sides[si].size();
    S.kind = side_kind(sides[si], tile);
    if (S.kind == kFSideStream && si != 0) S.kind = kFSideRaw;  // only side 0 streams
    S.tconst = (sdep & inthr) == 0 ? 1 : 0;
    {
      uint64_t slots = 0;  // in-thread output bits (q positions [nthr, nto))
      for (int i = nthr; i < nto; ++i) slots |= 1ull << qb[i];
      S.aind = (sdep & slots) == 0 ? 1 : 0;
    }
    for (int t : sides[si]) {
      FOp& o = d.ops[slot[t]];
      o.ptr = s.optag[t];
      o.c64 = s.opc64[t];
      o.side = (uint8_t)si;
      std::vector<int> oc;  // q positions of the op's compact bits
      for (int i = 0; i < nq; ++i)
        if ((dep[t] >> qb[i]) & 1) oc.push_back(i);
      o.nst = (uint8_t)oc.size();
      if (S.kind != kFSideConv && S.kind != kFSideStream) {  // no raw region: conversion, streamed
        o.raw_off = off;
        off += std::max(2u, 1u << oc.size()) * esz(t);
        off = (off + 15u) & ~15u;
      }
      std::vector<std::pair<int, int>> sr, ocr, gr, lr;
      for (size_t c = 0; c < oc.size(); ++c) sr.push_back({(int)c, opbit[t][qb[oc[c]]]});
      for (size_t c = 0; c < qa.size(); ++c) {
        auto it = std::find(oc.begin(), oc.end(), qa[c]);
        if (it != oc.end()) ocr.push_back({(int)c, (int)(it - oc.begin())});
      }
      for (size_t j = 0; j < gb.size(); ++j)
        if (opbit[t][gb[j]] >= 0) gr.push_back({(int)j, opbit[t][gb[j]]});
      for (size_t j = 0; j < lb.size(); ++j)
        if (opbit[t][lb[j]] >= 0) lr.push_back({(int)j, opbit[t][lb[j]]});
      if (!put(sr, o.srun, o.n_srun, kFQRuns) || !put(ocr, o.ocrun, o.n_ocrun, kFQRuns) ||
          !put(gr, o.grun, o.n_grun, kFGRuns) || !put(lr, o.lrun, o.n_lrun, kFGRuns))
        return false;
      // pairs: compact bit 0 is operand bit 0 (16-byte copies of 2 complex64)
      o.pairs = (o.c64 && !oc.empty() && opbit[t][qb[oc[0]]] == 0) ? 1 : 0;
    }
  }
  for (size_t si = 0; si < sides.size(); ++si) {
    FSide& S = d.sides[si];
    if (S.kind == kFSideStream) {
      S.st_off = 0;
    } else if (S.kind == kFSideRaw) {
      S.st_off = d.ops[S.first_op].raw_off;
    } else {
      S.st_off = off;
      off += std::max(2u, 1u << S.nst) * mesz;
      off = (off + 15u) & ~15u;
      if (S.kind == kFSideProd) d.has_finish = 1;
    }
  }
  d.math_f32 = s.math_f32 ? 1 : 0;
  d.n_var = (uint8_t)n_var;
  if (off > kFBufBytes + 512) return false;
  d.buf_bytes = off;
  d.n_sides = (uint8_t)sides.size();
  std::vector<std::pair<int, int>> og, oq;
  for (size_t j = 0; j < gb.size(); ++j) og.push_back({(int)j, gb[j]});
  for (int i = 0; i < nto; ++i) oq.push_back({i, qb[i]});
  if (!put(og, d.ogrun, d.n_ogrun, kFGRuns) || !put(oq, d.oqrun, d.n_oqrun, kFQRuns)) return false;
  d.out = s.out_tag;
  d.R = (uint8_t)R;
  d.K = (uint8_t)K;
  d.out_c64 = s.out_c64 ? 1 : 0;
  d.n_ops = (uint8_t)n;
  d.nq = (uint8_t)nq;
  d.nto = (uint8_t)nto;
  d.ng = (uint8_t)gb.size();
  d.nl = (uint8_t)lb.size();
  d.n_units = 1ull << gb.size();
  // split-K: a unit of more than 2^16 terms spreads its loop bits over
  // 2^sk CTAs (partial sums combined by fused_combine_kernel, fixed order)
  // when the item has few units; else units per CTA: ~2^16 terms per CTA
  // (amortises its table setup), keeping >= 512 CTAs per item
  const int nl = (int)lb.size(), ng = (int)gb.size();
  int sk = 0;
  if (ng < 9) sk = std::min(nl, std::max(0, nq + nl - fsplit));
  int upc = 0;
  if (!sk) {
    upc = std::max(0, fupc - (nq + nl));
    upc = std::min(upc, std::max(0, ng - fmin_units));
  }
  d.upc_log2 = (uint8_t)upc;
  d.sk = (uint8_t)sk;
  if (getenv("QTN_DEBUG_DESC") && R + K >= atoi(getenv("QTN_DEBUG_DESC"))) {
    // per side: which in-thread slot bits (q bits [nthr, nto)) / summed in-thread bits it depends on
    std::string sm;
    for (size_t si = 0; si < sides.size(); ++si) {
      const uint64_t sdep = dep[sides[si][0]] & tile;
      int ms = 0, js = 0;
      for (int i = nthr; i < nq; ++i)
        if ((sdep >> qb[i]) & 1) (i < nto ? ms : js) |= 1 << (i - nthr);
      sm += " s" + std::to_string(si) + "(n" + std::to_string(sides[si].size()) + ",a" + std::to_string(ms) +
            ",j" + std::to_string(js) + ")";
    }
    fprintf(stderr, "fdesc R=%d K=%d ops=%d sides=%d nv=%d nq=%d nto=%d ng=%d nl=%d buf=%u upc=%d sk=%d fin=%d%s\n",
            R, K, n, (int)sides.size(), n_var, nq, nto, ng, nl, off, upc, sk, (int)d.has_finish, sm.c_str());
  }
  return true;
}

// Warp-granular fused chain (qtn_stream.h WHdr, kernel in qtn_fusedw.cu):
// lanes = output bits 0..4, NI = 8 in-lane slots over 3 output bits the
// widest operand does not depend on (then the lowest others) when R >= 8,
// the remaining output bits index the chain's warps (chunks).
uint32_t encode_warp_chain(const FChainSpec& s, std::vector<uint8_t>& blob) {
  const int R = (int)s.out_vars.size(), K = (int)s.summed.size(), n = (int)s.opvars.size();
  if (n < 2 || n > kWMaxOps || R < 5 || K < 1 || K > kWMaxK) return 0;
  const int ni_log2 = R >= 7 ? 2 : 0;
  const int nc = R - 5 - ni_log2;  // chunk bits
  if (nc > 24) return 0;
  auto ubit = [&](int32_t u) -> int {
    for (int i = 0; i < R; ++i)
      if (s.out_vars[i] == u) return R - 1 - i;
    for (int j = 0; j < K; ++j)
      if (s.summed[j] == u) return R + j;
    return -1;
  };
  std::vector<std::vector<int>> opbit(n, std::vector<int>(R + K, -1));  // U bit -> operand bit
  int widest = 0;
  for (int t = 0; t < n; ++t) {
    const auto& vs = s.opvars[t];
    const int rk = (int)vs.size();
    if (rk > 32) return 0;
    for (int j = 0; j < rk; ++j) {
      const int b = ubit(vs[j]);
      if (b < 0) return 0;
      opbit[t][b] = rk - 1 - j;
    }
    if (vs.size() > s.opvars[widest].size()) widest = t;
  }
  std::vector<int> slot, chunkb;
  for (int pass = 0; pass < 2; ++pass)
    for (int b = 5; b < R && (int)slot.size() < ni_log2; ++b) {
      if (std::find(slot.begin(), slot.end(), b) != slot.end()) continue;
      if (pass == 0 && opbit[widest][b] >= 0) continue;
      slot.push_back(b);
    }
  for (int b = 5; b < R; ++b)
    if (std::find(slot.begin(), slot.end(), b) == slot.end()) chunkb.push_back(b);
  const int ni = 1 << ni_log2, nsv = 1 << K;
  WHdr h;
  std::memset(&h, 0, sizeof(h));
  h.out = s.out_tag;
  h.R = (uint8_t)R;
  h.K = (uint8_t)K;
  h.n_ops = (uint8_t)n;
  h.out_c64 = s.out_c64 ? 1 : 0;
  h.math_f32 = s.math_f32 ? 1 : 0;
  h.ni_log2 = (uint8_t)ni_log2;
  h.match = 1;
  std::vector<uint32_t> runs;
  {
    std::vector<std::pair<int, int>> pr;
    for (size_t j = 0; j < chunkb.size(); ++j) pr.push_back({(int)j, chunkb[j]});
    make_runs(pr, runs);
    if ((int)runs.size() > kWRuns) return 0;
    std::copy(runs.begin(), runs.end(), h.ocrun);
    h.n_ocrun = (uint8_t)runs.size();
  }
  for (int i = 0; i < ni; ++i) {
    uint32_t o = 0;
    for (int j = 0; j < ni_log2; ++j)
      if ((i >> j) & 1) o |= 1u << slot[j];
    h.slot_out[i] = o;
  }
  std::vector<WOpRec> recs(n);
  std::vector<uint32_t> tabs;  // words after the header and op records
  const uint32_t tab0 = (uint32_t)((sizeof(WHdr) + n * sizeof(WOpRec)) / 4);
  for (int t = 0; t < n; ++t) {
    WOpRec& o = recs[t];
    std::memset(&o, 0, sizeof(o));
    o.ptr = s.optag[t];
    o.c64 = s.opc64[t];
    if ((o.c64 != 0) != s.math_f32) h.match = 0;
    std::vector<std::pair<int, int>> pr;
    for (size_t j = 0; j < chunkb.size(); ++j)
      if (opbit[t][chunkb[j]] >= 0) pr.push_back({(int)j, opbit[t][chunkb[j]]});
    make_runs(pr, runs);
    if ((int)runs.size() > kWRuns) return 0;
    std::copy(runs.begin(), runs.end(), o.crun);
    o.n_crun = (uint8_t)runs.size();
    o.inv = 1;
    for (int b : slot)
      if (opbit[t][b] >= 0) o.inv = 0;
    auto off = [&](uint64_t bits_u) {  // operand offset of a set of U bits
      uint64_t x = 0;
      for (int b = 0; b < R + K; ++b)
        if (((bits_u >> b) & 1) && opbit[t][b] >= 0) x |= 1ull << opbit[t][b];
      return (uint32_t)x;
    };
    o.lane_off = tab0 + (uint32_t)tabs.size();
    for (uint32_t l = 0; l < 32; ++l) tabs.push_back(off(l));
    o.slot_off = tab0 + (uint32_t)tabs.size();
    for (int i = 0; i < ni; ++i) tabs.push_back(off(h.slot_out[i]));
    o.hs_off = tab0 + (uint32_t)tabs.size();
    for (int sv = 0; sv < nsv; ++sv) tabs.push_back(off((uint64_t)sv << R));
  }
  while (tabs.size() & 3u) tabs.push_back(0u);
  const size_t at = (blob.size() + 15) & ~(size_t)15;
  blob.resize(at, 0);
  const uint8_t* hb = reinterpret_cast<const uint8_t*>(&h);
  blob.insert(blob.end(), hb, hb + sizeof(h));
  for (const auto& o : recs) {
    const uint8_t* ob = reinterpret_cast<const uint8_t*>(&o);
    blob.insert(blob.end(), ob, ob + sizeof(o));
  }
  const uint8_t* tb = reinterpret_cast<const uint8_t*>(tabs.data());
  blob.insert(blob.end(), tb, tb + 4 * tabs.size());
  return 1u << nc;
}

}  // namespace qtn

using namespace qtn;

extern "C" const char* qtn_last_error(void) { return g_last_error.c_str(); }
extern "C" int qtn_version(void) { return 1; }

extern "C" int qtn_plan_create(const qtn_network_desc* net, const int32_t* order,
                               int32_t n_order, int32_t rank_cap, int32_t dtype,
                               int32_t mixed_rank, int64_t smem_budget, qtn_plan** out_plan,
                               int32_t* out_bad_rank) {
  if (!net || !out_plan || n_order < 0 || (n_order > 0 && !order) || net->n_tensors < 0 ||
      net->n_vars < 0) {
    set_error("qtn_plan_create: bad arguments");
    return QTN_EINVAL;
  }
  if (dtype != QTN_DTYPE_C128 && dtype != QTN_DTYPE_C64) {
    set_error("unknown dtype");
    return QTN_EINVAL;
  }
  *out_plan = nullptr;
  const int nvar = net->n_vars;
  // ---- validate: order is a permutation of the unfixed variables (60-62)
  std::vector<int32_t> unfixed;
  for (int v = 0; v < nvar; ++v)
    if (!net->is_fixed[v]) unfixed.push_back(v);
  {
    std::vector<int32_t> s(order, order + n_order);
    std::sort(s.begin(), s.end());
    if (s != unfixed) {
      set_error("order is not a permutation of the network's unfixed variables");
      return QTN_EINVAL;
    }
  }
  qtn_plan* P = new (std::nothrow) qtn_plan();
  if (!P) {
    set_error("out of host memory");
    return QTN_ENOMEM;
  }
  P->dtype = dtype;
  // ---- inputs (sliced tensors, network order)
  std::vector<std::vector<int32_t>> by_var(nvar);
  int64_t in_off = 0;
  for (int k = 0; k < net->n_tensors; ++k) {
    TensorRec t;
    t.input = true;
    const int r = net->ranks[k];
    if (r < 0 || r > 40) {
      delete P;
      set_error("tensor rank out of range");
      return QTN_EINVAL;
    }
    for (int j = 0; j < r; ++j) {
      int32_t u = net->vars[net->var_offsets[k] + j];
      if (u < 0 || u >= nvar || net->is_fixed[u]) {
        delete P;
        set_error("tensor references a fixed or out-of-range variable");
        return QTN_EINVAL;
      }
      if (std::find(t.vars.begin(), t.vars.end(), u) != t.vars.end()) {
        delete P;
        set_error("repeated variable in tensor");
        return QTN_EINVAL;
      }
      t.vars.push_back(u);
      by_var[u].push_back(k);
    }
    t.in_off = in_off;
    in_off += 1ll << r;
    P->tensors.push_back(std::move(t));
  }
  P->n_inputs = net->n_tensors;
  P->input_elems = in_off;
  // ---- symbolic elimination (75-106)
  std::vector<char> alive(P->tensors.size(), 1);
  for (int idx = 0; idx < n_order; ++idx) {
    const int32_t v = order[idx];
    std::vector<int32_t> ids = by_var[v];
    by_var[v].clear();
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    if (ids.empty()) {
      P->n_empty++;
      P->step_ranks.push_back(0);
      continue;
    }
    std::vector<std::vector<int32_t>> opvars;
    std::vector<int32_t> uni;
    for (int32_t id : ids) {
      opvars.push_back(P->tensors[id].vars);
      for (int32_t u : P->tensors[id].vars)
        if (std::find(uni.begin(), uni.end(), u) == uni.end()) uni.push_back(u);
    }
    const int rank = (int)uni.size() - 1;
    if (rank > rank_cap) {
      if (out_bad_rank) *out_bad_rank = rank;
      delete P;
      set_error("intermediate of rank " + std::to_string(rank) + " exceeds rank cap " +
                std::to_string(rank_cap));
      return QTN_ERANKCAP;
    }
    P->step_ranks.push_back(rank);
    P->width = std::max(P->width, rank);
    BucketRec b;
    b.v = v;
    b.ops = ids;
    b.rank = rank;
    std::vector<int32_t> out_vars;
    choose_layout(opvars, v, b.primary, out_vars);
    const int32_t bi = (int32_t)P->buckets.size();
    for (int32_t id : ids) {
      alive[id] = 0;
      P->tensors[id].last_use = bi;
      for (int32_t u : P->tensors[id].vars) {
        if (u == v) continue;
        auto& lst = by_var[u];
        lst.erase(std::remove(lst.begin(), lst.end(), id), lst.end());
      }
    }
    TensorRec res;
    res.vars = out_vars;
    res.born = bi;
    b.out = (int32_t)P->tensors.size();
    for (int32_t u : out_vars) by_var[u].push_back(b.out);
    P->tensors.push_back(std::move(res));
    alive.push_back(1);
    P->buckets.push_back(std::move(b));
  }
  const int32_t nb = (int32_t)P->buckets.size();
  for (size_t id = 0; id < P->tensors.size(); ++id) {
    if (!alive[id]) continue;
    if (P->tensors[id].rank() != 0) {  // cannot happen after a full permutation
      delete P;
      set_error("non-scalar tensor survived a full elimination");
      return QTN_EINVAL;
    }
    P->scalars.push_back((int32_t)id);
    P->tensors[id].last_use = nb;
  }
  // ---- storage types and cost figures
  for (auto& t : P->tensors)
    if (!t.input) t.c64 = (dtype == QTN_DTYPE_C64) && t.rank() >= mixed_rank;
  for (auto& b : P->buckets) P->flops_sum += std::ldexp(1.0, b.rank + 1);
  P->flops_sum += 2.0 * P->n_empty;

  // ---- SMEM executor feasibility: everything complex128 in shared memory
  bool smem_ok = smem_budget > 0 && nb < 65535;
  int64_t data_elems = 0;
  std::vector<Block> sblocks;
  // Input tensors are materialised (generated from the angles, or copied) in
  // one parallel pass before bucket 0 and their smem is reused by
  // intermediates once consumed.  QTN_SMEM_LAZY=1 instead materialises each
  // input right before the bucket that consumes it (every input is consumed
  // exactly once), which shrinks a set's region to the live intermediates +
  // one bucket's inputs; measured on B200 it is ~3% faster on config 2 and
  // ~25% slower on config 3, so it is not the default.
  std::vector<std::vector<int32_t>> bucket_inputs(nb);
  std::vector<int32_t> init_inputs;
  static int lazy = -1;
  if (lazy < 0) {
    const char* e = getenv("QTN_SMEM_LAZY");
    lazy = e ? atoi(e) : 0;
  }
  if (smem_ok) {
    for (int k = 0; k < P->n_inputs; ++k) {
      auto& t = P->tensors[k];
      if (t.rank() == 0 || !lazy) {
        init_inputs.push_back(k);
        t.sm_off = place(sblocks, 1ll << t.rank(), -1, t.rank() == 0 ? nb : t.last_use, 1);
        data_elems = std::max<int64_t>(data_elems, t.sm_off + ((int64_t)1 << t.rank()));
      } else {
        bucket_inputs[t.last_use].push_back(k);
      }
    }
    for (int bi = 0; bi < nb; ++bi) {
      for (int32_t k : bucket_inputs[bi]) {
        auto& t = P->tensors[k];
        t.sm_off = place(sblocks, 1ll << t.rank(), bi, bi, 1);
        data_elems = std::max<int64_t>(data_elems, t.sm_off + ((int64_t)1 << t.rank()));
      }
      auto& o = P->tensors[P->buckets[bi].out];
      o.sm_off = place(sblocks, 1ll << o.rank(), bi, o.last_use, 1);
      data_elems = std::max<int64_t>(data_elems, o.sm_off + ((int64_t)1 << o.rank()));
    }
    size_t n_ops = 0;
    int maxR = 0;
    for (auto& b : P->buckets) {
      n_ops += b.ops.size();
      maxR = std::max(maxR, (int)b.rank);
    }
    if (data_elems > 65535 || n_ops > 65535 || maxR > kSmemMaxR) smem_ok = false;
    // gather tables (deduplicated) and op records
    std::vector<uint16_t> tab;
    std::map<std::vector<uint16_t>, uint16_t> seen;
    auto intern = [&](const std::vector<uint16_t>& t) -> int64_t {
      auto it = seen.find(t);
      if (it != seen.end()) return it->second;
      const int64_t at = (int64_t)tab.size();
      if (at + (int64_t)t.size() > 65535) return -1;
      tab.insert(tab.end(), t.begin(), t.end());
      seen.emplace(t, (uint16_t)at);
      return at;
    };
    std::vector<SmemBucket> sbk(nb);
    std::vector<SmemOp> sop;
    std::vector<std::pair<int, int>> sd;
    std::vector<uint32_t> runs;
    size_t n_in_before = 0;
    for (int bi = 0; bi < nb && smem_ok; ++bi) {
      const auto& b = P->buckets[bi];
      const auto& out = P->tensors[b.out];
      sbk[bi].out_off = (uint16_t)out.sm_off;
      sbk[bi].R = (uint8_t)b.rank;
      sbk[bi].n_ops = (uint8_t)b.ops.size();
      sbk[bi].first_op = (uint16_t)sop.size();
      sbk[bi].first_in = (uint16_t)(init_inputs.size() + n_in_before);
      sbk[bi].n_in = (uint8_t)bucket_inputs[bi].size();
      n_in_before += bucket_inputs[bi].size();
      if (bucket_inputs[bi].size() > 255) smem_ok = false;
      // primary first: its entries seed the accumulator
      std::vector<int32_t> ord = b.ops;
      std::swap(ord[0], ord[b.primary]);
      const int R = b.rank;
      for (int32_t id : ord) {
        int vs;
        operand_map(P->tensors[id].vars, out.vars, b.v, sd, vs);
        make_runs(sd, runs);
        auto g = [&](uint32_t e) {
          uint32_t idx = 0;
          for (uint32_t w : runs) {
            const uint32_t s0 = w & 0xff, d0 = (w >> 8) & 0xff, l0 = (w >> 16) & 0xff;
            idx |= ((e >> s0) & ((1u << l0) - 1)) << d0;
          }
          return (uint16_t)idx;
        };
        std::vector<uint16_t> lo, hi;
        for (uint32_t e = 0; e < (1u << std::min(R, 5)); ++e) lo.push_back(g(e));
        for (uint32_t j = 0; R > 5 && j < (1u << (R - 5)); ++j) hi.push_back(g(j << 5));
        const int64_t l = intern(lo), h = R > 5 ? intern(hi) : 0;
        if (l < 0 || h < 0 || (1 << vs) > 65535) {
          smem_ok = false;
          break;
        }
        SmemOp o;
        o.off = (uint16_t)P->tensors[id].sm_off;
        o.vstep = (uint16_t)(1u << vs);
        o.lo = (uint16_t)l;
        o.hi = (uint16_t)h;
        sop.push_back(o);
      }
    }
    // input materialisation records: rank-0 inputs first, then per bucket
    std::vector<SmemIn> sin;
    auto add_in = [&](int32_t k) {
      const auto& t = P->tensors[k];
      SmemIn r{};
      r.input = (uint16_t)k;
      r.sm_off = (uint16_t)t.sm_off;
      r.in_off = (uint16_t)t.in_off;
      r.rank = (uint8_t)t.rank();
      sin.push_back(r);
    };
    for (int32_t k : init_inputs) add_in(k);
    for (int bi = 0; bi < nb; ++bi)
      for (int32_t k : bucket_inputs[bi]) add_in(k);
    if (P->n_inputs > 65535 || P->input_elems > 65535) smem_ok = false;
    int64_t prog = sizeof(SmemHeader) + sizeof(SmemBucket) * nb + sizeof(SmemOp) * n_ops +
                   2 * (int64_t)P->scalars.size();
    prog = (prog + 15) / 16 * 16;
    const int64_t sin_off = prog;
    prog += ((int64_t)sin.size() * (int64_t)sizeof(SmemIn) + 15) / 16 * 16;
    const int64_t tab_off = prog;
    prog += ((int64_t)tab.size() * 2 + 15) / 16 * 16;
    const int64_t smem = prog + 16 * data_elems;
    if (smem > smem_budget) smem_ok = false;
    if (smem_ok) {
      std::vector<uint8_t> blob(prog, 0);
      SmemHeader* h = reinterpret_cast<SmemHeader*>(blob.data());
      h->n_buckets = nb;
      h->n_ops = (uint32_t)n_ops;
      h->n_scalars = (uint32_t)P->scalars.size();
      h->pow2 = (uint32_t)P->n_empty;
      h->in_elems = (uint32_t)P->input_elems;
      h->data_elems = (uint32_t)data_elems;
      h->prog_bytes = (uint32_t)prog;
      h->tab_off = (uint32_t)tab_off;
      h->in_off = (uint32_t)sin_off;
      h->n_init = (uint32_t)init_inputs.size();
      std::memcpy(blob.data() + sin_off, sin.data(), sin.size() * sizeof(SmemIn));
      std::memcpy(blob.data() + sizeof(SmemHeader), sbk.data(), sizeof(SmemBucket) * nb);
      std::memcpy(blob.data() + sizeof(SmemHeader) + sizeof(SmemBucket) * nb, sop.data(),
                  sizeof(SmemOp) * n_ops);
      uint16_t* sc = reinterpret_cast<uint16_t*>(blob.data() + sizeof(SmemHeader) +
                                                 sizeof(SmemBucket) * nb + sizeof(SmemOp) * n_ops);
      for (size_t i = 0; i < P->scalars.size(); ++i)
        sc[i] = (uint16_t)P->tensors[P->scalars[i]].sm_off;
      std::memcpy(blob.data() + tab_off, tab.data(), tab.size() * 2);
      P->program = std::move(blob);
      P->smem_bytes = smem;
    }
  }
  if (smem_ok) {
    P->executor = QTN_EXEC_SMEM;
    for (auto& t : P->tensors) t.c64 = false;
    // ---- set-major form (levels, one region per intermediate)
    std::vector<int32_t> tlev(P->tensors.size(), 0);
    std::vector<uint32_t> toff(P->tensors.size(), 0);
    uint32_t next = 0;
    for (int bi = 0; bi < nb; ++bi) {
      const auto& b = P->buckets[bi];
      const auto& out = P->tensors[b.out];
      qtn_plan::SMBucketRec rb;
      int32_t lv = 0;
      for (int32_t id : b.ops) lv = std::max(lv, tlev[id]);
      rb.level = lv;
      tlev[b.out] = lv + 1;
      P->sm_levels = std::max(P->sm_levels, lv + 1);
      toff[b.out] = next;
      rb.out_off = next;
      next += 1u << b.rank;
      rb.R = b.rank;
      std::vector<int32_t> ord = b.ops;
      std::swap(ord[0], ord[b.primary]);
      std::vector<std::pair<int, int>> sd;
      std::vector<uint32_t> runs;
      for (int32_t id : ord) {
        const auto& t = P->tensors[id];
        int vs;
        operand_map(t.vars, out.vars, b.v, sd, vs);
        make_runs(sd, runs);
        qtn_plan::SMOpRec o;
        o.input = t.input ? id : -1;
        o.off = t.input ? 0u : toff[id];
        for (uint32_t e = 0; e < (1u << b.rank); ++e) {
          uint32_t j = 0;
          for (uint32_t w : runs)
            j |= ((e >> (w & 0xff)) & ((1u << ((w >> 16) & 0xff)) - 1)) << ((w >> 8) & 0xff);
          o.idx.push_back((uint16_t)j);
          o.idx.push_back((uint16_t)(j + (1u << vs)));
        }
        rb.ops.push_back(std::move(o));
      }
      P->sm_buckets.push_back(std::move(rb));
    }
    P->sm_elems = next;
    for (int32_t id : P->scalars) {
      if (P->tensors[id].input) P->sm_scalar_in.push_back(id);
      else P->sm_scalar_off.push_back(toff[id]);
    }
  } else {
    P->executor = QTN_EXEC_HBM;
    // Chains of single-operand buckets (a partial trace of one tensor, then
    // of its result, ...) are fused into one multi-variable sum: the
    // intermediates of the chain are never written.
    // chain_head[bi]: head bucket of bi's chain (bi itself for a head), -1
    // for buckets that are not single-operand.
    // On by default for chains of 2-4 buckets into outputs of rank >= 18
    // (QTN_FUSE_REDUCE=0 disables): reduce_kernel streams 16-byte loads
    // (config 4 782 -> 831 /s, config 3 default 79.4 k -> 80.7 k/s); longer
    // chains into small outputs leave it too few outputs for its 2^k sums.
    const char* fv = getenv("QTN_FUSE_REDUCE");
    const bool fuse = !(fv && fv[0] == '0');
    std::vector<int32_t> chain_head(nb, -1), chain_tail(nb, -1), chain_len(nb, 0);
    std::vector<char> is_fchain(nb, 0);
    std::map<int32_t, uint64_t> fpart_bytes;  // split fused chains: partial-sum block bytes
    // Expanding bucket + consumer pairs (qtn_xt.cu): the consumer of an
    // expanding bucket's result O1 eliminates one more variable without
    // adding any; the pair runs as one pass and O1 is never stored.  Marked
    // as a 2-bucket chain (head = the expanding bucket).  QTN_XT=0 disables.
    std::vector<char> is_xt(nb, 0);
    // members of the chain headed by bi: its consumer, then up to max_k
    // trailing traces (buckets whose other operands add no variables)
    auto xt_members = [&](int32_t bi, int max_k) {
      std::vector<int32_t> m;
      int32_t cur = bi;
      while ((int)m.size() < 1 + max_k) {
        const int32_t c = P->tensors[P->buckets[cur].out].last_use;
        if (c < 0 || c >= nb || chain_head[c] >= 0) break;
        const auto& cb = P->buckets[c];
        if (cb.rank != P->buckets[cur].rank - 1 || !P->tensors[cb.out].c64) break;
        m.push_back(c);
        cur = c;
      }
      return m;
    };
    auto xt_spec = [&](int32_t bi, const std::vector<int32_t>& mem, bool tags, YPairSpec& ys,
                       const std::function<uint64_t(int32_t)>& tag) {
      const auto& b = P->buckets[bi];
      for (int32_t id : b.ops) {
        ys.opvars.push_back(P->tensors[id].vars);
        ys.opc64.push_back(P->tensors[id].c64 ? 1 : 0);
        ys.optag.push_back(tags ? tag(id) : 0);
      }
      ys.n1 = (int32_t)b.ops.size();
      ys.primary = b.primary;
      int32_t running = b.out;
      for (size_t q = 0; q < mem.size(); ++q) {
        const auto& cb = P->buckets[mem[q]];
        for (int32_t id : cb.ops) {
          if (id == running) continue;
          ys.opvars.push_back(P->tensors[id].vars);
          ys.opc64.push_back(P->tensors[id].c64 ? 1 : 0);
          ys.optag.push_back(tags ? tag(id) : 0);
        }
        if (q == 0) ys.v2 = cb.v;
        else ys.trailing.push_back(cb.v);
        running = cb.out;
      }
      ys.v1 = b.v;
      ys.out_vars = P->tensors[running].vars;
      ys.out_tag = tags ? tag(running) : 0;
    };
    {
      const char* xv = getenv("QTN_XT");
      const bool xt_on = !(xv && xv[0] == '0');
      const char* kv = getenv("QTN_XT_MAX_K");
      const int max_k = std::min(kYMaxK, kv ? atoi(kv) : kYMaxK);
      for (int bi = 0; xt_on && bi < nb; ++bi) {
        const auto& b = P->buckets[bi];
        if (b.ops.size() < 2 || !P->tensors[b.out].c64 || chain_head[bi] >= 0) continue;
        int maxop = 0;
        for (int32_t id : b.ops) maxop = std::max(maxop, P->tensors[id].rank());
        if (maxop > b.rank) continue;  // not expanding: the primary alone holds every variable
        std::vector<int32_t> mem = xt_members(bi, max_k);
        for (; !mem.empty(); mem.pop_back()) {  // the longest chain that encodes
          YPairSpec ys;
          xt_spec(bi, mem, false, ys, nullptr);
          YDesc probe;
          if (encode_xt_desc(ys, probe)) break;
        }
        if (mem.empty()) continue;
        is_xt[bi] = 1;
        chain_head[bi] = bi;
        for (int32_t c : mem) chain_head[c] = bi;
        chain_tail[bi] = mem.back();
        chain_len[bi] = 1 + (int)mem.size();
      }
    }
    // Tail chains (qtn_wsum.cu): from a complex64 intermediate T of rank >=
    // QTN_WSUM_MIN_R (12) on, every bucket down to the scalar has the previous
    // result as its only intermediate operand and rank-1/2 gates on T's
    // variables otherwise: one weighted sum over T (head = the first bucket,
    // the others absorbed, no intermediate stored).  QTN_WSUM=0 disables.
    std::vector<char> is_ws(nb, 0);
    // main operand of a tail bucket: its latest-produced intermediate operand
    // (the previous result of the chain); every other operand a rank-1/2
    // tensor (a gate, or a small product of gates) on the main operand's
    // variables; -1 otherwise
    auto ws_main = [&](int32_t bi) -> int32_t {
      const auto& b = P->buckets[bi];
      int32_t m = -1;
      for (int32_t id : b.ops)
        if (!P->tensors[id].input && (m < 0 || P->tensors[id].born > P->tensors[m].born)) m = id;
      if (m < 0) return -1;
      const auto& mv = P->tensors[m].vars;
      if (b.rank != (int)mv.size() - 1) return -1;
      for (int32_t id : b.ops) {
        if (id == m) continue;
        const auto& t = P->tensors[id];
        if (t.rank() < 1 || t.rank() > 2) return -1;
        for (int32_t u : t.vars)
          if (std::find(mv.begin(), mv.end(), u) == mv.end()) return -1;
      }
      return m;
    };
    {
      const char* wv = getenv("QTN_WSUM");
      const bool ws_on = !(wv && wv[0] == '0');
      const char* wr = getenv("QTN_WSUM_MIN_R");
      const int ws_min_r = std::max(kWsL + 1, wr ? atoi(wr) : 12);
      for (int bi = 0; ws_on && bi < nb; ++bi) {
        // a tail ends at a bucket whose result is a scalar
        if (P->buckets[bi].rank != 0 || chain_head[bi] >= 0) continue;
        std::vector<int32_t> mem;  // from the scalar's bucket backwards
        int32_t head_main = -1;
        size_t n_gates = 0;
        for (int32_t c = bi; c >= 0 && chain_head[c] < 0;) {
          const int32_t m = ws_main(c);
          if (getenv("QTN_DEBUG_WS")) {
            fprintf(stderr, "  bucket %d rank %d main %d ops:", c, P->buckets[c].rank, m);
            for (int32_t id : P->buckets[c].ops)
              fprintf(stderr, " %d(r%d%s b%d lu%d)", id, P->tensors[id].rank(), P->tensors[id].input ? "i" : "", P->tensors[id].born, P->tensors[id].last_use);
            fprintf(stderr, "\n");
          }
          if (m < 0) break;
          n_gates += P->buckets[c].ops.size() - 1;
          if (n_gates > (size_t)kWsMaxGates) break;
          mem.push_back(c);
          head_main = m;
          if (P->tensors[m].born < 0 || P->tensors[m].last_use != c) break;
          c = P->tensors[m].born;
        }
        // the head's main operand must be a complex64 intermediate of rank >= min_r:
        // drop members from the head side until it is
        while (!mem.empty()) {
          const auto& t = P->tensors[head_main];
          if (t.c64 && t.rank() >= ws_min_r) break;
          mem.pop_back();
          if (!mem.empty()) head_main = ws_main(mem.back());
        }
        if (getenv("QTN_DEBUG_WS"))
          fprintf(stderr, "ws tail: end bucket %d, members %zu, head main rank %d c64 %d gates %zu\n", bi, mem.size(),
                  head_main >= 0 ? P->tensors[head_main].rank() : -1,
                  head_main >= 0 ? (int)P->tensors[head_main].c64 : -1, n_gates);
        if (mem.size() < 3) continue;
        std::reverse(mem.begin(), mem.end());  // head first
        // geometry check (tags do not change it)
        WsSpec wsp;
        wsp.src_vars = P->tensors[head_main].vars;
        wsp.src_tag = wsp.out_tag = 0;
        wsp.out_c64 = P->tensors[P->buckets[mem.back()].out].c64;
        for (int32_t c : mem) {
          const int32_t cm = ws_main(c);
          for (int32_t id : P->buckets[c].ops)
            if (id != cm) {
              wsp.gate_vars.push_back(P->tensors[id].vars);
              wsp.gate_tag.push_back(0);
              wsp.gate_c64.push_back(P->tensors[id].c64 ? 1 : 0);
            }
        }
        WsDesc probe;
        if (!encode_wsum_desc(wsp, probe)) continue;
        if (getenv("QTN_DEBUG_WS"))
          fprintf(stderr, "ws desc: R %d lo %d hi %d st %d ctas %u\n", probe.R, probe.n_lo, probe.n_hi, probe.n_st, probe.n_ctas);
        const int32_t hb = mem.front();
        is_ws[hb] = 1;
        for (int32_t c : mem) chain_head[c] = hb;
        chain_tail[hb] = mem.back();
        chain_len[hb] = (int)mem.size();
        fpart_bytes[hb] = 16ull * probe.n_ctas;
      }
    }
    // Product chains (qtn_fused.cu): a bucket of >= 2 operands whose result
    // is then reduced by single-operand buckets is one fused contraction; the
    // union-size product and the chain's intermediates are never written
    // (the GEMM census in DESIGN §3.7).  On for chains
    // whose head has union rank >= 10 and whose output rank is 1..17
    // (measured: config 3 default 3.69 -> 2.84 ms; dot products
    // into scalars and wide streaming chains run faster unfused);
    // QTN_FUSE_CHAIN=0 disables, QTN_FCHAIN_MIN_R / _MIN_OUT / _MAX_OUT move
    // the window.
    {
      const char* fcv = getenv("QTN_FUSE_CHAIN");
      const bool fchain = !(fcv && fcv[0] == '0');
      const char* fmr = getenv("QTN_FCHAIN_MIN_R");
      const int fmin_r = fmr ? atoi(fmr) : 10;
      const char* fmo = getenv("QTN_FCHAIN_MAX_OUT");
      const int fmax_out = fmo ? atoi(fmo) : 17;
      const char* fno = getenv("QTN_FCHAIN_MIN_OUT");
      const int fmin_out = fno ? atoi(fno) : 1;
      const char* fso = getenv("QTN_FCHAIN_STREAM_MAX_OUT");
      const int fstream_max_out = fso ? atoi(fso) : 13;
      for (int bi = 0; fchain && bi < nb; ++bi) {
        const auto& b = P->buckets[bi];
        if (b.ops.size() < 2 || chain_head[bi] >= 0 || b.rank + 1 < fmin_r) continue;
        std::vector<int32_t> members;
        std::vector<int32_t> summed{b.v};
        for (int32_t cur = bi;;) {
          const int32_t c = P->tensors[P->buckets[cur].out].last_use;
          if (c < 0 || c >= nb || P->buckets[c].ops.size() != 1 || chain_head[c] >= 0) break;
          members.push_back(c);
          summed.push_back(P->buckets[c].v);
          cur = c;
        }
        if (members.empty()) continue;
        {
          const int orank = P->tensors[P->buckets[members.back()].out].rank();
          if (orank > fmax_out || orank < fmin_out) continue;
          // streaming chains (one operand holds all but <= 1 of the union's
          // variables: each of its entries feeds one term) only up to
          // QTN_FCHAIN_STREAM_MAX_OUT (13): the trace/reduce kernels stream
          // them faster than the fused kernel's staged terms (config 4 in
          // 2^3 slices 1.127 -> 0.998 ms, config 3 default unchanged)
          int maxop = 0;
          for (int32_t id : b.ops) maxop = std::max(maxop, P->tensors[id].rank());
          if (maxop >= b.rank && orank > fstream_max_out) continue;
        }
        // geometry check with placeholder tags (tags do not change it)
        FChainSpec fs;
        for (int32_t id : b.ops) {
          fs.opvars.push_back(P->tensors[id].vars);
          fs.opc64.push_back(P->tensors[id].c64 ? 1 : 0);
          fs.optag.push_back(0);
        }
        fs.summed = summed;
        fs.out_vars = P->tensors[P->buckets[members.back()].out].vars;
        fs.out_c64 = P->tensors[P->buckets[members.back()].out].c64;
        fs.math_f32 = P->tensors[b.out].c64;  // head product stored complex64 -> float math
        fs.out_tag = 0;
        FDesc probe;
        if (!encode_fused_desc(fs, probe)) continue;
        if (probe.sk) fpart_bytes[bi] = fused_part_bytes(probe);
        is_fchain[bi] = 1;
        chain_head[bi] = bi;
        chain_len[bi] = 1 + (int)members.size();
        for (int32_t c : members) chain_head[c] = bi;
        chain_tail[bi] = members.back();
      }
    }
    constexpr int kRedMax = 8;  // the reduce kernel keeps 2^k source offsets in shared memory
    if (fuse) {
      for (int bi = 0; bi < nb; ++bi) {
        const auto& b = P->buckets[bi];
        if (b.ops.size() != 1 || chain_head[bi] >= 0) continue;
        const auto& src = P->tensors[b.ops[0]];
        const int32_t pb = src.input ? -1 : src.born;
        // extend the producer's chain (at most kRedMax eliminated variables)
        const bool extend = pb >= 0 && chain_head[pb] >= 0 && !is_fchain[chain_head[pb]] &&
                            !is_xt[chain_head[pb]] && !is_ws[chain_head[pb]] &&
                            chain_len[chain_head[pb]] < kRedMax;
        chain_head[bi] = extend ? chain_head[pb] : bi;
        chain_len[chain_head[bi]] += 1;
        chain_tail[chain_head[bi]] = bi;  // buckets in order: the last one wins
      }
    }
    // keep a chain fused only if its lowest eliminated bit leaves contiguous
    // runs of >= 2^min_pos source entries per output (coalesced streaming);
    // otherwise its buckets run on the tile kernel as usual
    if (fuse) {
      const char* mpv = getenv("QTN_FUSE_MIN_POS");
      const int min_pos = mpv ? atoi(mpv) : 0;
      const char* mrv = getenv("QTN_FUSE_MIN_R");
      const int fuse_min_r = mrv ? atoi(mrv) : 18;
      const char* mkv = getenv("QTN_FUSE_MAX_K");
      const int fuse_max_k = mkv ? atoi(mkv) : 4;
      for (int bi = 0; bi < nb; ++bi) {
        if (chain_head[bi] != bi || is_fchain[bi] || is_xt[bi] || is_ws[bi]) continue;
        const auto& src = P->tensors[P->buckets[bi].ops[0]];
        int lowest = 64;
        for (int32_t c = bi;; c = P->tensors[P->buckets[c].out].last_use) {
          const int32_t v = P->buckets[c].v;
          const auto it = std::find(src.vars.begin(), src.vars.end(), v);
          lowest = std::min(lowest, (int)(src.vars.end() - it) - 1);
          if (c == chain_tail[bi]) break;
        }
        // a chain of one bucket gains nothing from fusion (trace_kernel runs
        // it); long chains into small outputs leave reduce_kernel with too
        // few outputs for its 2^k-entry sums (measured: config 3 default)
        const int out_rank = P->tensors[P->buckets[chain_tail[bi]].out].rank();
        if (lowest < min_pos || chain_len[bi] < 2 || out_rank < fuse_min_r ||
            chain_len[bi] > fuse_max_k) {
          for (int32_t c = bi;; c = P->tensors[P->buckets[c].out].last_use) {
            chain_head[c] = -1;
            if (c == chain_tail[bi]) break;
          }
        }
      }
    }
    // Tiny subtrees (qtn_stream.h SubItem): connected sets of small buckets
    // (output rank <= QTN_SUBTREE_R, default 9, outside fused chains) run
    // as one CTA each with their internal intermediates in shared memory
    // (QTN_SUBTREE=0 disables).  Members are in elimination order, the root
    // (last member) writes its result to the workspace.  Opt-in
    // (QTN_SUBTREE=1): measured slower — config 4's head forest becomes a
    // few subtrees of ~100 members that one CTA walks serially (107 us vs
    // ~100 us of level launches): config 4 0.968 -> 0.999 ms, config 3
    // default 3.187 -> 3.26 ms.
    std::vector<int32_t> sub_of(nb, -1);  // subtree index of a member bucket
    std::vector<std::vector<int32_t>> subs;
    std::vector<int64_t> sm_off(P->tensors.size(), -1);  // internal tensors: shared byte offset
    std::vector<uint32_t> sub_smem;
    {
      const char* sv = getenv("QTN_SUBTREE");
      const bool on = sv && sv[0] == '1';
      const char* rv = getenv("QTN_SUBTREE_R");
      const int sub_r = rv ? atoi(rv) : kSmallR;
      std::vector<int32_t> grp(nb, -1);
      std::vector<std::vector<int32_t>> groups;
      for (int bi = 0; on && bi < nb; ++bi) {
        const auto& b = P->buckets[bi];
        if (chain_head[bi] >= 0 || b.rank > sub_r) continue;
        std::vector<int32_t> mem;
        for (int32_t id : b.ops) {
          const auto& t = P->tensors[id];
          if (t.input || t.born < 0 || grp[t.born] < 0) continue;
          auto& g = groups[grp[t.born]];
          mem.insert(mem.end(), g.begin(), g.end());
          g.clear();
        }
        mem.push_back(bi);
        std::sort(mem.begin(), mem.end());
        const int32_t gid = (int32_t)groups.size();
        for (int32_t m : mem) grp[m] = gid;
        groups.push_back(std::move(mem));
      }
      for (auto& g : groups) {
        if (g.size() < 2) continue;
        // shared memory of the internal intermediates: first fit over member positions
        std::vector<Block> blocks;
        int64_t top = 0;
        std::vector<std::pair<int32_t, int64_t>> offs;
        for (size_t k = 0; k + 1 < g.size(); ++k) {
          const int32_t id = P->buckets[g[k]].out;
          const auto& t = P->tensors[id];
          const int32_t cons = t.last_use;
          const int32_t end = (int32_t)(std::find(g.begin(), g.end(), cons) - g.begin());
          const int64_t bytes = std::max<int64_t>(16, elem_bytes(t.c64) << t.rank());
          const int64_t o = place(blocks, bytes, (int32_t)k, end, 16);
          offs.push_back({id, o});
          top = std::max(top, o + bytes);
        }
        if (top > 48 * 1024) continue;  // too large for one CTA: run level by level
        const int32_t si = (int32_t)subs.size();
        for (int32_t m : g) sub_of[m] = si;
        for (auto& pr : offs) sm_off[pr.first] = pr.second;
        subs.push_back(g);
        sub_smem.push_back((uint32_t)((top + 15) & ~15ll));
      }
    }
    // levels of the elimination tree: a bucket (or fused chain, at its head;
    // or tiny subtree, at its root) runs after the producers of its
    // intermediate operands
    std::vector<int32_t> tlevel(P->tensors.size(), 0);
    std::vector<char> virt(P->tensors.size(), 0);  // chain/subtree-internal: never stored
    std::vector<int32_t> sub_level(subs.size(), 0);
    int32_t nlev = 0;
    P->hbm_level.assign(nb, 0);
    for (int bi = 0; bi < nb; ++bi) {
      if (sub_of[bi] >= 0) {  // tiny subtree: runs at its root, after every external operand
        P->hbm_level[bi] = -1;
        const auto& g = subs[sub_of[bi]];
        if (g.back() != bi) {
          virt[P->buckets[bi].out] = 1;
          continue;
        }
        int32_t lv = 0;
        for (int32_t m : g)
          for (int32_t id : P->buckets[m].ops)
            if (sm_off[id] < 0) lv = std::max(lv, tlevel[id]);
        sub_level[sub_of[bi]] = lv;
        tlevel[P->buckets[bi].out] = lv + 1;
        nlev = std::max(nlev, lv + 1);
        continue;
      }
      const int32_t h = chain_head[bi];
      if (h >= 0 && h != bi) {  // absorbed into its chain
        P->hbm_level[bi] = -1;
        continue;
      }
      int32_t lv = 0;
      for (int32_t id : P->buckets[bi].ops) lv = std::max(lv, tlevel[id]);
      if (is_xt[bi] || is_ws[bi])  // the chain also waits for its consumers' other operands
        for (int32_t c = P->tensors[P->buckets[bi].out].last_use;; c = P->tensors[P->buckets[c].out].last_use) {
          for (int32_t id : P->buckets[c].ops)
            if (P->tensors[id].input || chain_head[P->tensors[id].born] != bi) lv = std::max(lv, tlevel[id]);
          if (c == chain_tail[bi]) break;
        }
      P->hbm_level[bi] = lv;  // 0-based level index
      const int32_t last = h >= 0 ? chain_tail[bi] : bi;
      tlevel[P->buckets[last].out] = lv + 1;
      nlev = std::max(nlev, lv + 1);
      for (int32_t c = bi; h >= 0 && c != last; c = P->tensors[P->buckets[c].out].last_use)
        virt[P->buckets[c].out] = 1;
    }
    P->n_levels = nlev;
    // level at which a bucket runs (its chain's head, its subtree's root)
    auto exec_level = [&](int32_t bi) {
      if (sub_of[bi] >= 0) return sub_level[sub_of[bi]];
      const int32_t h = chain_head[bi];
      return P->hbm_level[h >= 0 ? h : bi];
    };
    // level at which each intermediate is produced / last read
    auto born_level = [&](const TensorRec& t) { return exec_level(t.born); };
    // device arena: lifetimes in levels (concurrent buckets never alias)
    std::vector<Block> hblocks;
    int64_t ws = 0;
    for (size_t id = P->n_inputs; id < P->tensors.size(); ++id) {
      auto& t = P->tensors[id];
      if (virt[id]) continue;
      int64_t bytes = elem_bytes(t.c64) << t.rank();
      bytes = std::max<int64_t>(bytes, 256);
      const int32_t s0 = born_level(t);
      int32_t e = nlev + 1;
      if (t.last_use < nb) e = exec_level(t.last_use);
      t.ws_off = place(hblocks, bytes, s0, e, 256);
      ws = std::max(ws, t.ws_off + bytes);
    }
    // partial sums of split fused chains: live during their level only
    std::map<int32_t, int64_t> fpart_off;
    for (const auto& kv : fpart_bytes) {
      const int32_t lv = P->hbm_level[kv.first];
      const int64_t bytes = std::max<int64_t>((int64_t)kv.second, 256);
      fpart_off[kv.first] = place(hblocks, bytes, lv, lv, 256);
      ws = std::max(ws, fpart_off[kv.first] + bytes);
    }
    P->workspace_bytes = ws;
    // one streaming descriptor per bucket
    auto tag_of = [&](int32_t id) -> uint64_t {
      const auto& t = P->tensors[id];
      return t.input ? tag_in(16ull * (uint64_t)t.in_off) : tag_ws((uint64_t)t.ws_off);
    };
    P->hbm_xidx.assign(nb, -1);
    P->hbm_r1idx.assign(nb, -1);
    const char* fwv = getenv("QTN_FWARP");
    const bool fwarp_on = !(fwv && fwv[0] == '0');
    const char* fwt = getenv("QTN_FWARP_MAX_T");
    const int fwarp_max_t = fwt ? atoi(fwt) : 12;
    for (int bi = 0; bi < nb; ++bi) {
      const auto& b = P->buckets[bi];
      P->hbm_desc_off.push_back(P->hbm_desc.size());
      if (chain_head[bi] >= 0) {  // fused chain (head) or absorbed member: no descriptor
        P->hbm_tiles.push_back(0);
        if (chain_head[bi] != bi) continue;
        if (is_xt[bi]) {
          YPairSpec ys;
          std::vector<int32_t> mem;
          for (int32_t c = P->tensors[b.out].last_use;; c = P->tensors[P->buckets[c].out].last_use) {
            mem.push_back(c);
            if (c == chain_tail[bi]) break;
          }
          xt_spec(bi, mem, true, ys, tag_of);
          YDesc yd;
          if (!encode_xt_desc(ys, yd)) {
            delete P;
            set_error("expand + consumer pair: descriptor no longer encodable");
            return QTN_EINVAL;
          }
          P->hbm_ydesc.push_back(yd);
          P->hbm_ylevel.push_back(P->hbm_level[bi]);
          continue;
        }
        if (is_ws[bi]) {
          WsSpec wsp;
          const int32_t main_id = ws_main(bi);
          wsp.src_vars = P->tensors[main_id].vars;
          wsp.src_tag = tag_of(main_id);
          wsp.out_tag = tag_of(P->buckets[chain_tail[bi]].out);
          wsp.out_c64 = P->tensors[P->buckets[chain_tail[bi]].out].c64;
          for (int32_t c = bi;; c = P->tensors[P->buckets[c].out].last_use) {
            const int32_t cm = ws_main(c);
            for (int32_t id : P->buckets[c].ops)
              if (id != cm) {
                wsp.gate_vars.push_back(P->tensors[id].vars);
                wsp.gate_tag.push_back(tag_of(id));
                wsp.gate_c64.push_back(P->tensors[id].c64 ? 1 : 0);
              }
            if (c == chain_tail[bi]) break;
          }
          WsDesc wd;
          if (!encode_wsum_desc(wsp, wd) || !fpart_off.count(bi)) {
            delete P;
            set_error("tail chain: descriptor no longer encodable");
            return QTN_EINVAL;
          }
          wd.part = tag_ws((uint64_t)fpart_off[bi]);
          P->hbm_wsdesc.push_back(wd);
          P->hbm_wslevel.push_back(P->hbm_level[bi]);
          continue;
        }
        if (is_fchain[bi]) {
          FChainSpec fs;
          for (int32_t id : b.ops) {
            fs.opvars.push_back(P->tensors[id].vars);
            fs.opc64.push_back(P->tensors[id].c64 ? 1 : 0);
            fs.optag.push_back(tag_of(id));
          }
          fs.summed.push_back(b.v);
          for (int32_t c = P->tensors[b.out].last_use;; c = P->tensors[P->buckets[c].out].last_use) {
            fs.summed.push_back(P->buckets[c].v);
            if (c == chain_tail[bi]) break;
          }
          const auto& out = P->tensors[P->buckets[chain_tail[bi]].out];
          fs.out_vars = out.vars;
          fs.out_c64 = out.c64;
          fs.math_f32 = P->tensors[b.out].c64;
          fs.out_tag = tag_of(P->buckets[chain_tail[bi]].out);
          FDesc fd;
          if (!encode_fused_desc(fs, fd) || (fd.sk != 0) != (fpart_off.count(bi) != 0)) {
            delete P;
            set_error("fused chain: descriptor no longer encodable");
            return QTN_EINVAL;
          }
          if (fd.sk) fd.part = tag_ws((uint64_t)fpart_off[bi]);
          P->hbm_fdesc.push_back(fd);
          P->hbm_flevel.push_back(P->hbm_level[bi]);
          // warp-granular form (the executor picks one of the two at batch
          // creation): chains of up to QTN_FWARP_MAX_T log2 terms
          int64_t woff = -1;
          uint32_t nw = 0;
          if (fwarp_on && out.rank() + (int)fs.summed.size() <= fwarp_max_t) {
            while (P->hbm_wblob.size() & 15u) P->hbm_wblob.push_back(0);
            const size_t at = P->hbm_wblob.size();
            nw = encode_warp_chain(fs, P->hbm_wblob);
            if (nw) woff = (int64_t)at;
          }
          P->hbm_woff.push_back(woff);
          P->hbm_wwarps.push_back(nw);
          continue;
        }
        const auto& src = P->tensors[b.ops[0]];
        const auto& out = P->tensors[P->buckets[chain_tail[bi]].out];
        RedRec r;
        r.level = P->hbm_level[bi];
        r.src = tag_of(b.ops[0]);
        r.out = tag_of(P->buckets[chain_tail[bi]].out);
        r.src_c64 = src.c64 ? 1 : 0;
        r.out_c64 = out.c64 ? 1 : 0;
        r.R = (uint8_t)out.rank();
        std::vector<int> pos;
        for (size_t q = 0; q < src.vars.size(); ++q)
          if (std::find(out.vars.begin(), out.vars.end(), src.vars[q]) == out.vars.end())
            pos.push_back((int)(src.vars.size() - 1 - q));
        if (pos.size() > (size_t)kMaxRed || (int)pos.size() + out.rank() != src.rank()) {
          delete P;
          set_error("fused reduction: unexpected chain shape");
          return QTN_EINVAL;
        }
        std::sort(pos.begin(), pos.end());
        r.k = (uint8_t)pos.size();
        for (size_t q = 0; q < pos.size(); ++q) r.pos[q] = (uint8_t)pos[q];
        P->hbm_red.push_back(r);
        continue;
      }
      BucketSpec spec;
      auto tag_x = [&](int32_t id) { return sm_off[id] >= 0 ? tag_sm((uint64_t)sm_off[id]) : tag_of(id); };
      for (int32_t id : b.ops) {
        spec.opvars.push_back(P->tensors[id].vars);
        spec.opc64.push_back(P->tensors[id].c64 ? 1 : 0);
        spec.optag.push_back(tag_x(id));
      }
      spec.primary = b.primary;
      spec.v = b.v;
      spec.out_vars = P->tensors[b.out].vars;
      spec.out_c64 = P->tensors[b.out].c64;
      spec.out_tag = tag_x(b.out);
      int rc = encode_stream_desc(spec, P->hbm_desc);
      if (rc) {
        delete P;
        return rc;
      }
      if (sub_of[bi] >= 0) {  // subtree member: evaluated by its subtree's CTA only
        const SHdr* h = reinterpret_cast<const SHdr*>(P->hbm_desc.data() + P->hbm_desc_off.back());
        P->hbm_tiles.push_back(h->n_tiles);
        continue;
      }
      const SHdr* h = reinterpret_cast<const SHdr*>(P->hbm_desc.data() + P->hbm_desc_off.back());
      P->hbm_tiles.push_back(h->n_tiles);
      {
        // a (weighted) partial trace: the primary plus only v-only operands;
        // output = the primary's variables minus v, same order
        const int pi = b.primary;
        bool ok = true;
        int nw = 0, ns = 0;
        for (int i = 0; i < (int)spec.opvars.size() && ok; ++i)
          if (i != pi) {
            if (spec.opvars[i].size() == 1) ok = nw++ < kR1MaxW;
            else ok = ns++ < kR1MaxS;
          }
        std::vector<int32_t> rest;
        for (int32_t u : spec.opvars[pi])
          if (u != b.v) rest.push_back(u);
        const int rk = (int)spec.opvars[pi].size();
        int pk = -1;
        for (int j = 0; j < rk; ++j)
          if (spec.opvars[pi][j] == b.v) pk = rk - 1 - j;
        // the output must be the primary's variables minus v on its low
        // bits, in order; variables of staged operands may sit above
        const size_t nr = rest.size();
        const bool low_ok = spec.out_vars.size() >= nr &&
                            std::equal(rest.begin(), rest.end(), spec.out_vars.end() - nr);
        const bool expanding = spec.out_vars.size() > nr;
        // expanding or complex128: only through the staged path, which needs
        // a staged operand and a primary bit under the output pair
        if (ok && (expanding || !spec.out_c64 || !spec.opc64[pi]) && (ns == 0 || nr < 1)) ok = false;
        if (ok && low_ok && pk >= 0) {
          R1Dev r{};
          r.src = spec.optag[pi];
          r.out = spec.out_tag;
          r.R = (uint8_t)spec.out_vars.size();
          r.pk = (uint8_t)pk;
          r.src_c64 = spec.opc64[pi];
          r.out_c64 = spec.out_c64 ? 1 : 0;
          r.pr = (uint8_t)nr;
          const int R = (int)spec.out_vars.size();
          for (int i = 0; i < (int)spec.opvars.size() && ok; ++i) {
            if (i == pi) continue;
            const auto& vs = spec.opvars[i];
            if (vs.size() == 1) {
              r.w[r.nw] = spec.optag[i];
              r.w_c64[r.nw] = spec.opc64[i];
              ++r.nw;
              continue;
            }
            // staged operand: output bits < 12 it depends on, compacted
            R1Stage& g = r.st[r.ns++];
            g.ptr = spec.optag[i];
            g.c64 = spec.opc64[i];
            const int rk = (int)vs.size();
            std::vector<std::pair<int, int>> hi, lo;  // (output bit, operand bit)
            for (int j = 0; j < rk; ++j) {
              if (vs[j] == b.v) {
                g.vshift = (uint8_t)(rk - 1 - j);
                continue;
              }
              int ob = -1;
              for (int q = 0; q < R; ++q)
                if (spec.out_vars[q] == vs[j]) ob = R - 1 - q;
              if (ob < 0) ok = false;
              (ob < 12 ? lo : hi).push_back({ob, rk - 1 - j});
            }
            std::sort(lo.begin(), lo.end());
            if ((int)lo.size() > kR1StageBits) {
              ok = false;
              break;
            }
            g.kl = (uint8_t)lo.size();
            std::vector<std::pair<int, int>> lr, er;
            for (size_t q = 0; q < lo.size(); ++q) {
              lr.push_back({(int)q, lo[q].second});
              er.push_back({lo[q].first, (int)q});
            }
            std::vector<uint32_t> runs;
            make_runs(hi, runs);
            if (runs.size() > 24) ok = false;
            else {
              std::copy(runs.begin(), runs.end(), g.hrun);
              g.n_hrun = (uint8_t)runs.size();
            }
            make_runs(lr, runs);
            std::copy(runs.begin(), runs.end(), g.lrun);
            g.n_lrun = (uint8_t)runs.size();
            make_runs(er, runs);
            std::copy(runs.begin(), runs.end(), g.erun);
            g.n_erun = (uint8_t)runs.size();
          }
          if (ok) {
            P->hbm_r1idx[bi] = (int32_t)P->hbm_r1.size();
            P->hbm_r1.push_back(r);
          }
        }
      }
      XDesc xd;
      if (encode_expand_desc(spec, xd)) {
        P->hbm_xidx[bi] = (int32_t)P->hbm_xdesc.size();
        P->hbm_xdesc.push_back(xd);
      }
    }
    // subtree records: member descriptors contiguous, in elimination order
    for (size_t si = 0; si < subs.size(); ++si) {
      qtn_plan::SubRec r;
      r.level = sub_level[si];
      r.first = (uint32_t)P->hbm_sub_desc.size();
      r.count = (uint32_t)subs[si].size();
      r.smem = sub_smem[si];
      for (int32_t m : subs[si]) P->hbm_sub_desc.push_back(P->hbm_desc_off[m]);
      P->hbm_sub.push_back(r);
    }
    // bytes the executor moves: a fused chain (product or reduce) reads its
    // head's operands and writes its tail's output only
    double eb = 0.0;
    for (int bi = 0; bi < nb; ++bi) {
      const int32_t h = chain_head[bi];
      if (h >= 0 && h != bi) continue;
      const auto& b = P->buckets[bi];
      for (int32_t id : b.ops)
        if (sm_off[id] < 0)  // subtree-internal operands never leave the SM
          eb += std::ldexp((double)elem_bytes(P->tensors[id].c64), P->tensors[id].rank());
      if (h >= 0 && (is_xt[bi] || is_ws[bi]))
        for (int32_t c = P->tensors[b.out].last_use;; c = P->tensors[P->buckets[c].out].last_use) {
          for (int32_t id : P->buckets[c].ops)
            if (P->tensors[id].input || chain_head[P->tensors[id].born] != bi)
              eb += std::ldexp((double)elem_bytes(P->tensors[id].c64), P->tensors[id].rank());
          if (c == chain_tail[bi]) break;
        }
      if (sm_off[b.out] >= 0) continue;
      const auto& o = P->tensors[P->buckets[h >= 0 ? chain_tail[bi] : bi].out];
      eb += std::ldexp((double)elem_bytes(o.c64), o.rank());
    }
    P->exec_bytes = eb;
  }
  // algorithmic bytes: e * (operand entries + output entries) per bucket
  // (the reference's per-bucket traffic; exec_bytes above is what the fused
  // chains actually move)
  for (auto& b : P->buckets) {
    double bytes = 0.0;
    for (int32_t id : b.ops) {
      const auto& t = P->tensors[id];
      bytes += std::ldexp((double)elem_bytes(t.c64), t.rank());
    }
    const auto& o = P->tensors[b.out];
    bytes += std::ldexp((double)elem_bytes(o.c64), o.rank());
    P->alg_bytes += bytes;
  }
  *out_plan = P;
  return QTN_OK;
}

extern "C" int qtn_plan_info(const qtn_plan* P, qtn_plan_info_t* info) {
  if (!P || !info) {
    set_error("null argument");
    return QTN_EINVAL;
  }
  info->executor = P->executor;
  info->n_buckets = (int32_t)P->buckets.size();
  info->n_empty_buckets = P->n_empty;
  info->width = P->width;
  info->input_elems = P->input_elems;
  info->workspace_bytes = P->workspace_bytes;
  info->smem_bytes = P->smem_bytes;
  info->program_bytes = (int64_t)P->program.size();
  info->alg_bytes = P->alg_bytes;
  info->flops_sum = P->flops_sum;
  info->n_levels = P->n_levels;
  info->n_fused_chains = (int32_t)P->hbm_fdesc.size();
  info->exec_bytes = P->exec_bytes < 0.0 ? P->alg_bytes : P->exec_bytes;
  info->n_pairs = (int32_t)P->hbm_ydesc.size();
  info->n_tails = (int32_t)P->hbm_wsdesc.size();
  return QTN_OK;
}

extern "C" int qtn_plan_step_ranks(const qtn_plan* P, int32_t* out) {
  if (!P || !out) {
    set_error("null argument");
    return QTN_EINVAL;
  }
  std::copy(P->step_ranks.begin(), P->step_ranks.end(), out);
  return QTN_OK;
}

extern "C" int qtn_plan_input_offsets(const qtn_plan* P, int64_t* out) {
  if (!P || !out) {
    set_error("null argument");
    return QTN_EINVAL;
  }
  for (int k = 0; k < P->n_inputs; ++k) out[k] = P->tensors[k].in_off;
  return QTN_OK;
}

qtn_plan::~qtn_plan() {
  if (self_batch) qtn_batch_destroy(self_batch);
}

extern "C" int qtn_plan_destroy(qtn_plan* P) {
  delete P;
  return QTN_OK;
}

extern "C" int qtn_bucket_layout(int32_t n_ops, const int32_t* ranks, const int32_t* var_offsets,
                                 const int32_t* vars, int32_t elim_var, int32_t* out_rank,
                                 int32_t* out_vars) {
  if (n_ops < 1) {
    set_error("bucket needs at least one operand");
    return QTN_EINVAL;
  }
  std::vector<std::vector<int32_t>> opvars(n_ops);
  for (int i = 0; i < n_ops; ++i) opvars[i].assign(vars + var_offsets[i], vars + var_offsets[i] + ranks[i]);
  int32_t primary;
  std::vector<int32_t> ov;
  choose_layout(opvars, elim_var, primary, ov);
  *out_rank = (int32_t)ov.size();
  std::copy(ov.begin(), ov.end(), out_vars);
  return QTN_OK;
}

extern "C" int qtn_bucket_contract(int32_t n_ops, const int32_t* ranks, const int32_t* var_offsets,
                                   const int32_t* vars, const void* const* ptrs,
                                   const uint8_t* c64, int32_t elim_var, int32_t out_rank,
                                   const int32_t* out_vars, int32_t out_c64, void* out,
                                   void* stream) {
  if (n_ops < 1 || out_rank < 0 || out_rank > 34) {
    set_error("qtn_bucket_contract: bad arguments");
    return QTN_EINVAL;
  }
  std::vector<std::vector<int32_t>> opvars(n_ops);
  std::vector<uint8_t> opc64(n_ops);
  std::vector<int32_t> uni;
  for (int i = 0; i < n_ops; ++i) {
    opvars[i].assign(vars + var_offsets[i], vars + var_offsets[i] + ranks[i]);
    opc64[i] = c64[i] ? 1 : 0;
    if (std::find(opvars[i].begin(), opvars[i].end(), elim_var) == opvars[i].end()) {
      set_error("every bucket operand must contain the eliminated variable");
      return QTN_EINVAL;
    }
    for (int32_t u : opvars[i])
      if (std::find(uni.begin(), uni.end(), u) == uni.end()) uni.push_back(u);
  }
  std::vector<int32_t> ov(out_vars, out_vars + out_rank);
  {
    std::vector<int32_t> a = ov, b;
    for (int32_t u : uni)
      if (u != elim_var) b.push_back(u);
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    if (a != b) {
      set_error("out_vars must be the union of operand variables minus elim_var");
      return QTN_EINVAL;
    }
  }
  // the primary streams aligned only if the requested layout matches the rule
  int32_t primary;
  std::vector<int32_t> pref;
  choose_layout(opvars, elim_var, primary, pref);
  bool aligned = true;
  {
    const auto& pv = opvars[primary];
    std::vector<int32_t> low;
    for (int32_t u : pv)
      if (u != elim_var) low.push_back(u);
    aligned = ov.size() >= low.size() &&
              std::equal(low.begin(), low.end(), ov.end() - low.size());
  }
  if (aligned) {
    // the streaming kernel (bulk-copy pipeline, lookup tables)
    BucketSpec spec;
    spec.opvars = opvars;
    spec.opc64 = opc64;
    for (int i = 0; i < n_ops; ++i) spec.optag.push_back(tag_abs(ptrs[i]));
    spec.primary = primary;
    spec.v = elim_var;
    spec.out_vars = ov;
    spec.out_c64 = out_c64 != 0;
    spec.out_tag = tag_abs(out);
    std::vector<uint8_t> desc;
    int rc = encode_stream_desc(spec, desc);
    if (rc == QTN_OK) return launch_stream_single(desc, stream);
  }
  // any other layout: generic fused kernel, every operand gathered
  BucketArgs a;
  std::vector<int32_t> g_ops, t_ops;
  int rc = build_bucket_args(opvars, opc64, primary, elim_var, ov, out_c64 != 0, false, a,
                             g_ops, t_ops);
  if (rc) return rc;
  for (int i = 0; i < (int)a.ng; ++i) a.g[i].ptr = ptrs[g_ops[i]];
  for (int i = 0; i < (int)a.ntop; ++i) a.top[i].ptr = ptrs[t_ops[i]];
  a.out = out;
  return launch_bucket(a, stream);
}

// ------------------------------------------------------------- execution

extern "C" int qtn_plan_execute(qtn_plan* P, const void* inputs, void* workspace, void* result,
                                void* stream) {
  if (!P || !result || (P->input_elems > 0 && !inputs)) {
    set_error("qtn_plan_execute: null argument");
    return QTN_EINVAL;
  }
  int rc = device_check();
  if (rc) return rc;
  if (P->executor == QTN_EXEC_HBM && P->workspace_bytes > 0 && !workspace) {
    set_error("HBM executor needs a workspace of workspace_bytes");
    return QTN_EINVAL;
  }
  if (!P->self_batch) {
    qtn_plan* one[1] = {P};
    rc = qtn_batch_create(one, 1, &P->self_batch);
    if (rc) return rc;
  }
  return qtn_batch_execute(P->self_batch, inputs, 0, 1, workspace, result, stream);
}
