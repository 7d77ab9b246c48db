// planner.cu -- which kernel family and (G, R) instantiation fills each pair shape, and
// the slot lists of the resulting pair classes ("Planner").
#include "host_ctx.cuh"

#include <chrono>

namespace dtwgpu {
namespace host {

// ---- planner ------------------------------------------------------------------------
// Candidate instantiations with their measured throughput in computed lane-cells per
// ns on one B200 (tools/sweep.py, profiles/round1_sweep.md): the cost of a shape is
// the lane-cells a configuration computes (band waste, wavefront fill/drain, padding
// columns, masked rows all included) divided by that rate. Multi-pass Full fills with
// few lanes pay an extra per-pass boundary-column cost (measured on c4).
struct Cand {
  int G, R;
  double rate;  // computed lane-cells / ns
  int P = 1;    // band family: pairs per lane group
  int TR = 2;   // full family: rows per step
  bool ring = false;  // band family: shared-memory y ring
  int U = 1;          // ring variant: units per lane
  bool f32_only = false;  // full family: instantiated for fp32 only (fill_table.h)
  bool mp_rate = false;   // full family: rate measured on multi-pass shapes (no penalty)
  bool f64_only = false;  // full family: planned for fp64 only
  bool unmasked = false;  // full family: planned for unlimited windows only
  bool ysm = false;       // full family: y in shared memory (dtw_full1s_kernel)
  bool masked_only = false;  // full family: planned for banded shapes only
};
const Cand kFull[] = {{2, 23, 1913},         {2, 23, 2141, 1, 4},  {4, 12, 2026},
                      {4, 12, 1956, 1, 4},   {8, 8, 1804},         {8, 8, 1700, 1, 4},
                      {16, 8, 1800},         {16, 16, 1850},       {16, 16, 1850, 1, 4},
                      {32, 4, 1300},         {32, 8, 1650},        {32, 12, 1950},
                      {32, 15, 2000},        {32, 15, 2150, 1, 4}, {32, 16, 2100},
                      {32, 16, 2050, 1, 4},
                      // narrow masked strips for wide auto-widened bands (W = 32: 1.08x the
                      // in-band cells against 1.12x at W = 48), rate measured on c5's
                      // multi-pass shapes directly: c5 1795 -> 1829 GCUPS (fp32 c5 prefers
                      // 23-column lanes: 3770 against 3624 with this candidate)
                      {2, 16, 2000, 1, 4, false, 1, false, true, true},
                      // one lane per pair in 20/24/28-column passes, each lane its own
                      // boundary column (no shuffles, no fill/drain): c5 1829 -> 1925,
                      // c4 2192 -> 2248 GCUPS
                      {1, 20, 2000, 1, 4, false, 1, false, true, true},
                      {1, 24, 2050, 1, 4, false, 1, false, true, true},
                      {1, 28, 2250, 1, 4, false, 1, false, true, true},
                      // unlimited windows only: c4 2246 -> 2358 (masked c5 strips: 1813)
                      {1, 32, 2360, 1, 4, false, 1, false, true, true, true},
                      // fp32 only: c4 fp32 5340 GCUPS against 4598 for (32, 15, 4)
                      {16, 30, 2570, 1, 4, false, 1, true},
                      // fp32 only: c1 fp32 4310 GCUPS against 3800 for (32, 16, 2)
                      {16, 32, 2299, 1, 4, false, 1, true},
                      // fp32 only, one lane per pair (no shuffles, no wavefront fill/drain),
                      // single strip only (m <= 46): c3 fp32 5649 against 4403 for (2, 23, 4)
                      {1, 46, 2740, 1, 4, false, 1, true},
                      // ... and multi-pass (each lane its own boundary column): c4 fp32 5545
                      // against 5334 for (16, 30, 4)
                      {1, 46, 2587, 1, 4, false, 1, true, true},
                      // ... and wider passes for unlimited windows: c4 fp32 5516 -> 6129
                      // (masked c5 strips at R = 64: 3000 against 3867)
                      {1, 56, 2760, 1, 4, false, 1, true, true, false, true},
                      {1, 64, 2888, 1, 4, false, 1, true, true, false, true},
                      // fp64: one lane per pair, y in shared memory (dtw_lane_kernel),
                      // single strip only: c3 2041 -> 2278 GCUPS
                      {1, 46, 2270, 1, 2, false, 1, false, false, true},
                      // fp64, banded multi-pass: one lane per pair with y in shared memory
                      // (dtw_full1s_kernel, 3 CTAs/SM). Forced over all of c5: R=24 2066,
                      // R=20 2026 GCUPS against 1863 for the register-y R=28 strips (rates
                      // scaled from that ratio and the lane-cells each computes); unlimited
                      // windows keep the register kernel (c4: 2363 against 2456)
                      {1, 24, 2470, 1, 4, false, 1, false, true, true, false, true, true},
                      {1, 20, 2400, 1, 4, false, 1, false, true, true, false, true, true}};
const Cand kBand[] = {{16, 7, 1500},    {16, 9, 1600},    {16, 11, 1700},  {16, 13, 1800},
                      {32, 3, 1000},    {32, 5, 1250},    {32, 7, 1490},   {32, 9, 1500},
                      {32, 13, 1450},
                      {8, 16, 1900, 1, 2, true},  {8, 26, 2221, 1, 2, true},
                      {16, 8, 1500, 1, 2, true},  {16, 14, 2105, 1, 2, true},
                      {32, 6, 1300, 1, 2, true},
                      // ring with U units per lane (c2 sweep, round 1)
                      {8, 26, 2286, 1, 2, true, 3}, {8, 26, 2198, 1, 2, true, 5},
                      {16, 14, 2166, 1, 2, true, 3}, {16, 13, 2128, 1, 2, true, 2},
                      // wide bands (512-slot ring)
                      {16, 20, 2186, 1, 2, true, 3}, {16, 26, 2220, 1, 2, true, 3},
                      {32, 20, 2150, 1, 2, true, 3}, {32, 26, 2170, 1, 2, true, 3},
                      // fp32 only, wide lanes: c2 fp32 4603 GCUPS against 4211 for (8, 26, 3)
                      {4, 52, 2669, 1, 2, true, 3, true}};

// fp32 mode: the cell is FADD FMUL FMNMX3 FADD, so the Full family runs ~2.15x the fp64
// rate while the Band family (shuffle-heavy per step) gains ~1.45x (measured on c2 after the warp-uniform renormalisation).
constexpr double kFp32Full = 2.15, kFp32Band = 1.45;

// Masked Full fills: rows where the strip lies entirely inside the band run the plain
// cell; rows crossing a band edge ran the masked cell at 1.79x the cost (least-squares fit
// over hw = 101..400 at n = m = 1000, tools: exp/band_rates.py, profiles/round1_sweep.md).
// The kill-cell edges (dtw_kernels.cuh, FullRows) made those rows ~1.1x, but planning
// with 1.1 moved 0.7 M c5 pairs into the masked Full class at no net gain (2214 against
// 2210 ms), so the planner keeps the original weight.
#ifndef DTWG_MASKED_ROW_COST
#define DTWG_MASKED_ROW_COST 1.79
#endif
constexpr double kMaskedRowCost = DTWG_MASKED_ROW_COST;

double full_cost(const Shape& s, const Cand& c, bool mask, bool fp32) {
  const int64_t W = (int64_t)c.G * c.R;
  const int64_t npass = (s.m + W - 1) / W;
  double cells = 0;
  for (int64_t p = 0; p < npass; ++p) {
    const int64_t c0 = p * W;
    int64_t rs = 1, re = s.n;
    if (mask) {
      rs = std::max<int64_t>(1, c0 + 1 - s.hw);
      re = std::min<int64_t>(s.n, c0 + W + s.hw);
    }
    // TR rows per step, G-1 steps of wavefront fill/drain
    const int64_t rows = ((re - rs + c.TR) / c.TR) * c.TR;
    double eff_rows = double(rows);
    if (mask) {
      const int64_t fast = std::max<int64_t>(
          0, std::min<int64_t>(re, c0 + 1 + s.hw) - std::max<int64_t>(rs, c0 + W - s.hw) + 1);
      const int64_t masked = std::max<int64_t>(0, rows - fast);
      eff_rows = double(rows - masked) + kMaskedRowCost * double(masked);
    }
    cells += (eff_rows + c.TR * (c.G - 1)) * double(W);
  }
  double rate = c.rate * (fp32 ? kFp32Full : 1.0);
  // The per-group boundary columns stay in L2 up to ~n = 1500 (c5, L = 1000 sweeps);
  // the c4-measured penalties apply beyond. Rates measured on multi-pass c5 shapes
  // (mp_rate) already include the L2-resident boundary traffic.
  const bool l2_resident = s.n <= 1500;
  if (npass > 1 && !(c.mp_rate && l2_resident)) {  // boundary-column round trips per pass
    // fp32 with L2-resident boundary columns pays no G = 2 penalty: its 4-instruction cell
    // gains most from the 23-column lanes (c5 fp32 3359 -> 3773 GCUPS; fp64 1795 -> 1670).
    if (c.G == 2) rate *= (c.TR == 4 && l2_resident && fp32) ? 1.0 : (c.TR == 4 ? 0.68 : 0.59);
    else if (c.G == 4) rate *= (c.TR == 4 && l2_resident) ? 1.05 : (c.TR == 4 ? 0.92 : 0.78);
    else if (c.G == 8) rate *= c.TR == 4 ? 1.0 : 0.95;
  }
  return cells / rate;
}

double band_cost(const Shape& s, const Cand& c, bool fp32) {
  // fp32 / fp64 throughput ratios measured on c2 (G=8 R=26: 1.69 ring, 2.06 units;
  // G=16 R=14: 1.52 ring, 1.72 units; register-rotation band 1.45)
  const double f32 = c.ring ? (c.U > 1 ? 1.9 : 1.6) : kFp32Band;
  // wavefront fill/drain: one step per unit of the group
  return double(s.n + c.G * c.U - 1) * double(c.G * c.R) / (c.rate * (fp32 ? f32 : 1.0));
}

KernelCfg choose_cfg_model(const Shape& s, bool fp32, double* cost_out, int64_t count, int sms);

// Planner entry (choose_cfg, below): a forced (family, G, R) wins when it can legally run the shape.

// Fraction of the GPU a class of `count` pairs can keep busy with G lanes per pair: about
// 8 warps per SM are needed to cover the cell chain (c1: 4950 pairs fill it with G = 32,
// not with G = 4 -- 1765 against 946 GCUPS). count = 0: unknown (ragged classes).
double fill_factor(int64_t count, int G, int sms) {
  if (count <= 0) return 1.0;
  const double warps = double(count) * G / 32.0;
  return std::min(1.0, warps / (8.0 * sms));
}

KernelCfg choose_cfg_model(const Shape& s, bool fp32, double* cost_out, int64_t count = 0,
                           int sms = 148) {
  KernelCfg best{Family::Full, 32, 16, true, fp32};
  double bc = 1e300;
  const bool mask = s.hw < s.n - 1;  // a band that excludes some cell
  for (const Cand& c : kFull) {
    if ((c.f32_only && !fp32) || (c.f64_only && fp32) || (c.unmasked && mask) ||
        (c.masked_only && !mask))
      continue;
    if (c.G == 1 && s.m > c.R && !c.mp_rate) continue;  // single strip unless measured multi-pass
    const double cst = full_cost(s, c, mask, fp32) / fill_factor(count, c.G, sms);
    if (cst < bc) {
      bc = cst;
      best = KernelCfg{Family::Full, c.G, c.R, mask, fp32, -1, 1, c.TR};
      best.ysm = c.ysm;
    }
  }
  if (mask) {
    const int64_t K = 2 * s.hw + 1;
    for (const Cand& c : kBand) {
      if ((int64_t)c.G * c.R < K) continue;
      if ((c.f32_only && !fp32) || (c.f64_only && fp32)) continue;
      const double cst = band_cost(s, c, fp32) / fill_factor(count, c.G, sms);
      if (cst < bc) {
        bc = cst;
        // static kill position: fp64 everywhere, fp32 for the unit-ring variant
        const bool static_kr = !fp32 || (c.ring && c.U > 1);
        best = KernelCfg{Family::Band, c.G, c.R, false, fp32, static_kr ? (int)(K % c.R) : -1,
                         c.P, 2, c.ring, c.U};
      }
    }
  }
  if (cost_out) *cost_out = bc;
  return best;
}

const char* family_name(Family f) {
  return f == Family::Full ? "full" : (f == Family::Band ? "band" : "strip");
}

KernelCfg choose_cfg(const dtwg_ctx* ctx, const Shape& s, bool fp32, double* cost_out,
                     int64_t count) {
  const bool mask = s.hw < s.n - 1;
  if (ctx->force_family >= 0) {
    // 0: full (2 rows/step), 1: band, 3: full (4 rows/step), 4: band ring,
    // 10 + U: band ring with U units per lane
    const int ff = ctx->force_family;
    if (ff == 5) {  // strip family (long pairs spread over warps), G = 32, 4 rows per step
      KernelCfg f{Family::Strip, 32, ctx->force_R, mask, fp32, -1, 1, 4};
      if (dtwgpu::fill_cfg_supported(f)) {
        if (cost_out) *cost_out = 1.0;
        return f;
      }
    }
    if (ff == 6) {  // Full strips with y in shared memory, 4 rows per step
      KernelCfg f{Family::Full, ctx->force_G, ctx->force_R, mask, fp32, -1, 1, 4};
      f.ysm = true;
      if (dtwgpu::fill_cfg_supported(f)) {
        if (cost_out) *cost_out = 1.0;
        return f;
      }
    }
    const bool band = ff == 1 || ff == 2 || ff == 4 || ff > 10;
    KernelCfg f{band ? Family::Band : Family::Full, ctx->force_G, ctx->force_R,
                band ? false : mask, fp32,
                (band && (!fp32 || ff > 10) && ctx->force_R > 0) ? (int)((2 * s.hw + 1) % ctx->force_R)
                                                                  : -1,
                ff == 2 ? 2 : 1, ff == 3 ? 4 : 2, ff == 4 || ff > 10, ff > 10 ? ff - 10 : 1};
    KernelCfg one = f;  // single-strip-only instantiations (dtw_lane_kernel) for m <= G*R
    one.mp = false;
    const bool ok = (dtwgpu::fill_cfg_supported(f) ||
                     (f.family == Family::Full && s.m <= (int64_t)f.G * f.R &&
                      dtwgpu::fill_cfg_supported(one))) &&
                    (f.family == Family::Full ||
                     (mask && f.R >= 2 && (int64_t)f.G * f.R >= 2 * s.hw + 1));
    if (ok) {
      if (cost_out) *cost_out = 1.0;
      return f;
    }
  }
  return choose_cfg_model(s, fp32, cost_out, count, ctx->num_sms);
}

Shape shape_of(const dtwg_ctx* ctx, int64_t a, int64_t b, int64_t hw, int auto_widen) {
  int64_t la = ctx->h_len[a], lb = ctx->h_len[b];
  Shape s;
  s.n = std::max(la, lb);
  s.m = std::min(la, lb);
  if (hw < 0) {
    s.hw = s.n;
  } else {
    const int64_t gap = s.n - s.m;
    s.hw = (auto_widen && gap > hw) ? gap : hw;
  }
  if (s.hw > s.n) s.hw = s.n;  // a band at least max(n,m) wide is the unlimited window
  return s;
}

// A Full-family class of few, long pairs leaves most of the GPU idle (one lane group per
// pair, passes in sequence). Such classes become Strip classes: every column strip of
// every pair is a work item for a full warp, pipelined along the pair (dtw_strip_kernel).
// Rule: at most 4 pairs per SM with >= 2 strips per pair, or at most 16 pairs per SM with
// >= 8 strips per pair (c1's 4950 pairs of 2 strips stay Full: 1763 against 776 GCUPS).
// m_uniform < 0: ragged class (lengths per slot).
constexpr int kStripR = 15;
void maybe_strip(dtwg_ctx* ctx, PlanClass& pc, int64_t count, int64_t m_uniform) {
  if (count <= 0) return;
  const bool forced = pc.cfg.family == Family::Strip;  // dtwg_force_kernel(5, ., R)
  KernelCfg sc = pc.cfg;
  if (!forced) {
    if (pc.cfg.family != Family::Full || ctx->force_family >= 0) return;
    if (count > 16 * (int64_t)ctx->num_sms) return;  // enough pairs to fill the GPU already
    sc = KernelCfg{Family::Strip, 32, kStripR, pc.cfg.mask, pc.cfg.fp32, -1, 1, 4};
    if (!dtwgpu::fill_cfg_supported(sc)) return;
  }
  const int64_t W = 32 * (int64_t)sc.R;
  const int64_t min_strips = count <= 4 * (int64_t)ctx->num_sms ? 2 : 8;  // strips per pair
  if (m_uniform >= 0) {
    const int64_t S = (m_uniform + W - 1) / W;
    if (S < min_strips && !forced) return;
    pc.strips_per_pair = (int)S;
  } else {
    std::vector<int64_t> base(count + 1, 0);
    const int64_t p = ctx->p;
    for (int64_t q = 0; q < count; ++q) {
      const int64_t slot = pc.slots[q];
      int64_t lo = 0, hi = p - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (row_off(mid, p) <= slot) lo = mid;
        else hi = mid - 1;
      }
      const int64_t i = lo, j = i + 1 + (slot - row_off(i, p));
      const int64_t m = std::min(ctx->h_len[i], ctx->h_len[j]);
      base[q + 1] = base[q] + (m + W - 1) / W;
    }
    if (base[count] < min_strips * count && !forced) return;
    pc.strip_base = std::move(base);
  }
  pc.cfg = sc;
}

// Full classes whose every pair fits one strip (m <= G*R) use the single-strip kernels:
// no boundary column, fewer registers (c1's G=32 R=16: 126 instead of 168, 4 CTAs/SM).
void set_single_strip(PlanClass& pc) {
  if (pc.cfg.family != Family::Full || pc.max_m > (int64_t)pc.cfg.G * pc.cfg.R) return;
  KernelCfg one = pc.cfg;
  one.mp = false;
  if (dtwgpu::fill_cfg_supported(one)) pc.cfg = one;  // multi-pass-only instantiations keep mp
}

// Lane groups of `k` resident on the whole GPU (the persistent grid's item stride).
int64_t resident_groups(const dtwg_ctx* ctx, const KernelCfg& k) {
  return (int64_t)dtwgpu::fill_blocks_per_sm(k) * ctx->num_sms * (dtwgpu::kThreads / k.G);
}

// GPU-ns of a class of `count` same-shape pairs on `k` (cost: GPU-ns per pair at full
// occupancy, full_cost). Uniform pairs run in whole rounds of the resident lane groups, so
// a partial last round costs a full one; an underfilled launch (fewer than ~8 warps per SM)
// runs at the fill_factor fraction of the rate.
double class_time(const dtwg_ctx* ctx, const KernelCfg& k, double cost, int64_t count) {
  const double fill = fill_factor(count, k.G, ctx->num_sms);
  if (fill < 1.0) return double(count) * cost / fill;
  const int64_t groups = resident_groups(ctx, k);
  const int64_t rounds = (count + groups - 1) / groups;
  return double(std::max<int64_t>(rounds * groups, count)) * cost;
}

// Same-length pairs all cost the same, so a class of few lanes per pair (one lane per
// pair for c4) runs in whole rounds of its resident lane groups -- c4: 499,500 pairs over
// 37,888 groups = 13.18 rounds, the last one 18% occupied at the speed of a full one; one
// GPU's shard of c4 at 8 GPUs is 1.65 rounds. The pairs of that partial round become a
// second class with more lanes per pair, which runs on the whole GPU once the full rounds
// drain (classes run on concurrent side streams), when the cost model puts it below one
// full round: c4 13 + ~0.25 rounds instead of 14; c4 / 8 GPUs 1 + ~0.72 instead of 2.
// The tail configuration is the fastest candidate with more lanes per pair, its own round
// quantisation included (class_time).
void split_tail_round(dtwg_ctx* ctx, std::vector<PlanClass>& plan, const Shape& s, bool fp32,
                      int64_t sb, int64_t se) {
  if (ctx->force_family >= 0 || plan.size() != 1 || env_or("DTWGPU_TAIL_SPLIT", 1) == 0) return;
  PlanClass& pc = plan[0];
  if (pc.cfg.family != Family::Full || pc.cfg.G > 2) return;
  const int64_t count = se - sb;
  const int64_t groups = resident_groups(ctx, pc.cfg);
  const int64_t full_rounds = count / groups, tail = count - full_rounds * groups;
  if (full_rounds < 1 || tail == 0) return;
  const bool mask = s.hw < s.n - 1;
  // the partial round on the class's own configuration: one full round
  // (pc.cost: GPU-ns per pair at full occupancy -- count >= one round fills the GPU)
  const double keep = double(groups) * pc.cost;
  PlanClass t;
  double best = keep * 0.97;  // split only for a clear gain
  bool found = false;
  for (const Cand& c : kFull) {
    if (c.G <= pc.cfg.G || (c.f32_only && !fp32) || (c.f64_only && fp32) ||
        (c.unmasked && mask) || (c.masked_only && !mask))
      continue;
    KernelCfg k{Family::Full, c.G, c.R, mask, fp32, -1, 1, c.TR};
    k.ysm = c.ysm;
    if (s.m <= (int64_t)c.G * c.R) {
      KernelCfg one = k;
      one.mp = false;
      if (dtwgpu::fill_cfg_supported(one)) k = one;
    }
    if (!dtwgpu::fill_cfg_supported(k)) continue;
    const double tt = class_time(ctx, k, full_cost(s, c, mask, fp32), tail);
    if (tt < best) {
      best = tt;
      t.cfg = k;
      t.cost = tt / double(tail);
      found = true;
    }
  }
  if (!found) return;
  // With few full rounds the tail runs serially after them (same stream): their lanes all
  // finish together, while a concurrent launch let tail CTAs take SM slots first on some
  // runs and pushed full-round CTAs into a second wave (c4 / 8 GPUs: 217 -> 244 ms on one
  // shard of eight). With many rounds that delay is small against the run and the tail
  // fills the SMs whose lanes finish early: the whole c4 (13 rounds) averages 1571-1577 ms
  // concurrent against 1579-1587 serial over 15 fills each, slow fills included.
  // DTWGPU_TAIL_SERIAL = 0 / 1 forces either.
  const int64_t serial = env_or("DTWGPU_TAIL_SERIAL", -1);
  t.after_prev = serial < 0 ? full_rounds < 4 : serial != 0;
  t.max_n = pc.max_n;
  t.max_m = pc.max_m;
  set_single_strip(t);
  pc.range_begin = sb;
  pc.range_count = full_rounds * groups;
  t.range_begin = sb + pc.range_count;
  t.range_count = tail;
  plan.push_back(t);
}

// Ragged datasets whose lengths fit a (n, m) table (max length <= 8191): everything the
// plan needs per slot is a function of its shape, so one scan counts the pairs of every
// shape (in order of first appearance), the distinct shapes are costed on all host
// threads, classes and their statistics come from the shape counts (the underfill re-plan
// included), and a second scan writes every slot straight to its final position -- the
// same order as the general path below (per class: passes, then rows, then the shorter
// length, all descending; slots ascending inside a shape). c5: 12.5M pairs, ~1M shapes.
std::vector<PlanClass> make_plan_table(dtwg_ctx* ctx, int64_t hw, int auto_widen, bool fp32,
                                       int64_t sb, int64_t se, int64_t L1) {
  const int64_t p = ctx->p;
  const bool verbose = env_or("DTWGPU_VERBOSE", 0) != 0;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto ms_since = [&](std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(tnow() - t).count();
  };
  auto tp = tnow();
  int64_t i0;
  {
    int64_t lo = 0, hi = p - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (row_off(mid, p) <= sb) lo = mid;
      else hi = mid - 1;
    }
    i0 = lo;
  }
  const int64_t j0 = i0 + 1 + (sb - row_off(i0, p));
  const int64_t* len = ctx->h_len.data();
  // scan 1: pairs per shape, shapes in order of first appearance
  std::vector<int32_t> qidx((size_t)(L1 * L1), -1);
  std::vector<Shape> sh;
  std::vector<int64_t> cnt;
  {
    int64_t i = i0, j = j0;
    for (int64_t slot = sb; slot < se; ++slot) {
      const int64_t la = len[i], lb = len[j];
      const int64_t n = std::max(la, lb), m = std::min(la, lb);
      int32_t& q = qidx[(size_t)(n * L1 + m)];
      if (q < 0) {
        q = (int32_t)sh.size();
        Shape t;
        t.n = n;
        t.m = m;
        if (hw < 0) {
          t.hw = n;
        } else {
          const int64_t gap = n - m;
          t.hw = (auto_widen && gap > hw) ? gap : hw;
        }
        if (t.hw > t.n) t.hw = t.n;
        sh.push_back(t);
        cnt.push_back(0);
      }
      ++cnt[(size_t)q];
      if (++j == p) {
        ++i;
        j = i + 1;
      }
    }
  }
  const size_t ns = sh.size();
  if (verbose) fprintf(stderr, "dtwgpu: plan: %zu shapes counted in %.1f ms\n", ns, ms_since(tp));
  tp = tnow();
  // configurations per shape on all host threads (hint: pair count for the re-plan)
  std::vector<KernelCfg> cfg(ns);
  std::vector<int64_t> hint(ns, 0);
  std::vector<uint8_t> todo(ns, 1);
  auto cost_all = [&]() {
    const int nt = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)std::thread::hardware_concurrency(), (int64_t)(ns / 4096) + 1));
    std::vector<std::thread> th;
    for (int w = 0; w < nt; ++w)
      th.emplace_back([&, w] {
        for (size_t q = (size_t)w; q < ns; q += (size_t)nt) {
          if (!todo[q]) continue;
          double cst = 0;
          cfg[q] = choose_cfg(ctx, sh[q], fp32, &cst, hint[q]);
        }
      });
    for (auto& t : th) t.join();
  };
  std::vector<PlanClass> plan;
  std::vector<int> cls(ns);
  std::map<std::tuple<int, int, int, bool, int, int, int>, int> cls_of_cfg;
  auto assign = [&]() {  // classes in order of first appearance of their shapes
    plan.clear();
    cls_of_cfg.clear();
    for (size_t q = 0; q < ns; ++q) {
      const KernelCfg& c = cfg[q];
      const auto key = std::make_tuple((int)c.family * 2 + (int)c.ring + 4 * c.U, c.G, c.R,
                                       c.mask, c.kr, c.P, c.TR + 100 * (int)c.ysm);
      auto it = cls_of_cfg.find(key);
      if (it == cls_of_cfg.end()) {
        PlanClass pc;
        pc.cfg = c;
        plan.push_back(pc);
        it = cls_of_cfg.emplace(key, (int)plan.size() - 1).first;
      }
      cls[q] = it->second;
    }
  };
  cost_all();
  assign();
  // underfill re-plan (see make_plan): re-cost the shapes of Full classes that cannot keep
  // half the GPU's warp slots busy with their lanes per pair, with the class's pair count
  if (ctx->force_family < 0 && env_or("DTWGPU_UNDERFILL_REPLAN", 1) != 0) {
    std::vector<int64_t> ccount(plan.size(), 0);
    for (size_t q = 0; q < ns; ++q) ccount[(size_t)cls[q]] += cnt[q];
    bool any = false;
    for (size_t q = 0; q < ns; ++q) {
      const PlanClass& pc = plan[(size_t)cls[q]];
      const bool under = pc.cfg.family == Family::Full &&
                         fill_factor(ccount[(size_t)cls[q]], pc.cfg.G, ctx->num_sms) < 0.5;
      todo[q] = under;
      hint[q] = under ? ccount[(size_t)cls[q]] : 0;
      any = any || under;
    }
    if (any) {
      cost_all();
      assign();
    }
  }
  if (verbose) fprintf(stderr, "dtwgpu: plan: shapes costed in %.1f ms\n", ms_since(tp));
  tp = tnow();
  // per class: statistics, and the shapes in slot order -> start position of every shape
  std::vector<std::vector<int32_t>> members(plan.size());
  for (size_t q = 0; q < ns; ++q) {
    PlanClass& pc = plan[(size_t)cls[q]];
    members[(size_t)cls[q]].push_back((int32_t)q);
    pc.max_n = std::max(pc.max_n, sh[q].n);
    pc.max_m = std::max(pc.max_m, sh[q].m);
    pc.cost += double(cnt[q]) * double(sh[q].n) * double(sh[q].m);
    pc.cells += double(cnt[q]) * double(pair_cells(sh[q].n, sh[q].m, sh[q].hw));
  }
  std::vector<int64_t> start(ns, 0);
  for (size_t c = 0; c < plan.size(); ++c) {
    const KernelCfg& cc = plan[c].cfg;
    const int64_t W = (int64_t)cc.G * cc.R;
    auto npass = [&](int32_t q) { return cc.family == Family::Full ? (sh[q].m + W - 1) / W : 1; };
    auto& mem = members[c];
    std::sort(mem.begin(), mem.end(), [&](int32_t a, int32_t b) {
      const int64_t pa = npass(a), pb = npass(b);
      if (pa != pb) return pa > pb;
      if (sh[a].n != sh[b].n) return sh[a].n > sh[b].n;
      return sh[a].m > sh[b].m;
    });
    int64_t acc = 0;
    for (int32_t q : mem) {
      start[(size_t)q] = acc;
      acc += cnt[(size_t)q];
    }
    plan[c].slots.resize((size_t)acc);
  }
  // scan 2: every slot to its final position
  {
    int64_t i = i0, j = j0;
    for (int64_t slot = sb; slot < se; ++slot) {
      const int64_t la = len[i], lb = len[j];
      const int32_t q = qidx[(size_t)(std::max(la, lb) * L1 + std::min(la, lb))];
      plan[(size_t)cls[(size_t)q]].slots[(size_t)start[(size_t)q]++] = slot;
      if (++j == p) {
        ++i;
        j = i + 1;
      }
    }
  }
  if (verbose) fprintf(stderr, "dtwgpu: plan: slots placed in %.1f ms\n", ms_since(tp));
  for (auto& pc : plan) {
    maybe_strip(ctx, pc, (int64_t)pc.slots.size(), -1);
    set_single_strip(pc);
  }
  return plan;
}

std::vector<PlanClass> make_plan(dtwg_ctx* ctx, int64_t hw, int auto_widen, bool fp32,
                                 int64_t sb, int64_t se) {
  std::vector<PlanClass> plan;
  if (se <= sb) return plan;
  const int64_t p = ctx->p;
  if (ctx->uniform) {
    PlanClass pc;
    const Shape s = shape_of(ctx, 0, 1, hw, auto_widen);
    pc.cfg = choose_cfg(ctx, s, fp32, &pc.cost, se - sb);
    pc.max_n = s.n;
    pc.max_m = s.m;
    plan.push_back(pc);
    maybe_strip(ctx, plan[0], se - sb, s.m);
    set_single_strip(plan[0]);
    split_tail_round(ctx, plan, s, fp32, sb, se);
    return plan;
  }
  // Ragged dataset: classify every pair by shape (memoised on (n, m)), then bucket the
  // slots of each class by (passes, rows) with a counting sort -- longest first (LPT),
  // and pairs of equal pass count and row count adjacent, so the lane groups of one warp
  // run in lockstep. O(pairs); no comparison sort.
  int64_t maxlen = 0;
  for (int64_t t = 0; t < p; ++t) maxlen = std::max(maxlen, ctx->h_len[t]);
  const int64_t L1 = maxlen + 1;
  std::vector<int> cls_tab;
  const bool use_tab = L1 * L1 <= (int64_t)1 << 26;
  if (use_tab && env_or("DTWGPU_PLAN_TABLE", 1) != 0)
    return make_plan_table(ctx, hw, auto_widen, fp32, sb, se, L1);
  if (use_tab) cls_tab.assign((size_t)(L1 * L1), -1);
  std::map<Shape, int> cls_of_shape;
  std::map<std::tuple<int, int, int, bool, int, int, int>, int> cls_of_cfg;
  // Second classification round (below): shapes whose first-round class was too small to
  // fill the GPU with its lanes per pair are re-costed with that class's pair count.
  std::vector<int> old_tab;
  std::map<Shape, int> old_shape;
  std::vector<int64_t> old_hint;  // per first-round class: pair count if underfilled, else 0
  auto count_hint = [&](const Shape& s) -> int64_t {
    if (old_hint.empty()) return 0;
    int oc = -1;
    if (use_tab) {
      oc = old_tab[(size_t)(s.n * L1 + s.m)];
    } else {
      auto it = old_shape.find(s);
      if (it != old_shape.end()) oc = it->second;
    }
    return oc >= 0 ? old_hint[oc] : 0;
  };
  // precost (below): per distinct shape its configuration, computed on all host threads
  std::vector<int32_t> pre_idx;
  std::vector<KernelCfg> pre_cfgs;
  auto class_of_cfg = [&](const KernelCfg& cfg) -> int {
    const auto key = std::make_tuple((int)cfg.family * 2 + (int)cfg.ring + 4 * cfg.U, cfg.G, cfg.R, cfg.mask,
                                     cfg.kr, cfg.P, cfg.TR + 100 * (int)cfg.ysm);
    auto ic = cls_of_cfg.find(key);
    if (ic != cls_of_cfg.end()) return ic->second;
    PlanClass pc;
    pc.cfg = cfg;
    plan.push_back(pc);
    const int cls = (int)plan.size() - 1;
    cls_of_cfg[key] = cls;
    return cls;
  };
  auto class_of = [&](int64_t a, int64_t b, Shape& s) -> int {
    s = shape_of(ctx, a, b, hw, auto_widen);
    int* slotp = use_tab ? &cls_tab[(size_t)(s.n * L1 + s.m)] : nullptr;
    if (slotp && *slotp >= 0) return *slotp;
    if (!slotp) {
      auto it = cls_of_shape.find(s);
      if (it != cls_of_shape.end()) return it->second;
    }
    double cst = 0;
    const int32_t pre = slotp ? pre_idx[(size_t)(s.n * L1 + s.m)] : -1;
    const int cls = class_of_cfg(pre >= 0 ? pre_cfgs[(size_t)pre]
                                          : choose_cfg(ctx, s, fp32, &cst, count_hint(s)));
    if (slotp) *slotp = cls;
    else cls_of_shape[s] = cls;
    return cls;
  };
  auto bucket_of = [&](int cls, const Shape& s) -> int64_t {
    const KernelCfg& cc = plan[cls].cfg;
    const int64_t W = (int64_t)cc.G * cc.R;
    const int64_t npass = cc.family == Family::Full ? (s.m + W - 1) / W : 1;
    return npass * L1 + s.n;  // larger = earlier
  };
  int64_t i0;
  {
    int64_t lo = 0, hi = p - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (row_off(mid, p) <= sb) lo = mid;
      else hi = mid - 1;
    }
    i0 = lo;
  }
  const int64_t j0 = i0 + 1 + (sb - row_off(i0, p));
  // Shapes are costed in parallel before the passes (c5: ~1.1M distinct (n, m) shapes x
  // ~35 candidates, ~3.4 s serially): the distinct shapes of the slot range and their
  // configurations on all host threads; pass 1 then only looks them up.
  std::vector<std::pair<int32_t, int32_t>> shapes;  // distinct (n, m) of the slot range
  auto precost = [&]() {
    if (!use_tab) return;
    if (shapes.empty()) {
      std::vector<uint8_t> seen((size_t)(L1 * L1), 0);
      int64_t i = i0, j = j0;
      for (int64_t slot = sb; slot < se; ++slot) {
        const int64_t la = ctx->h_len[i], lb = ctx->h_len[j];
        const int64_t n = std::max(la, lb), m = std::min(la, lb);
        uint8_t& f = seen[(size_t)(n * L1 + m)];
        if (!f) {
          f = 1;
          shapes.emplace_back((int32_t)n, (int32_t)m);
        }
        if (++j == p) {
          ++i;
          j = i + 1;
        }
      }
      std::sort(shapes.begin(), shapes.end());
    }
    const size_t ns = shapes.size();
    std::vector<KernelCfg>& cfgs = pre_cfgs;
    // re-plan round: only shapes of underfilled first-round classes change (count hints)
    const bool again = cfgs.size() == ns;
    if (!again) cfgs.assign(ns, KernelCfg{});
    std::vector<Shape> sh(ns);
    for (size_t q = 0; q < ns; ++q) {
      // shape_of from the lengths alone (the pair's indices only pick the lengths)
      Shape t;
      t.n = shapes[q].first;
      t.m = shapes[q].second;
      if (hw < 0) {
        t.hw = t.n;
      } else {
        const int64_t gap = t.n - t.m;
        t.hw = (auto_widen && gap > hw) ? gap : hw;
      }
      if (t.hw > t.n) t.hw = t.n;
      sh[q] = t;
    }
    const int nt = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)std::thread::hardware_concurrency(), (int64_t)(ns / 4096) + 1));
    std::vector<std::thread> th;
    for (int w = 0; w < nt; ++w)
      th.emplace_back([&, w] {
        for (size_t q = (size_t)w; q < ns; q += (size_t)nt) {
          const int64_t hint = count_hint(sh[q]);
          if (again && hint == 0) continue;
          double cst = 0;
          cfgs[q] = choose_cfg(ctx, sh[q], fp32, &cst, hint);
        }
      });
    for (auto& t : th) t.join();
    // class ids are assigned in pass 1, in order of first appearance (as before)
    pre_idx.assign((size_t)(L1 * L1), -1);
    for (size_t q = 0; q < ns; ++q) pre_idx[(size_t)(sh[q].n * L1 + sh[q].m)] = (int32_t)q;
  };
  // pass 1: classes, bucket counts
  std::vector<std::vector<int64_t>> counts;
  auto pass1 = [&]() {
    int64_t i = i0, j = j0;
    Shape s;
    for (int64_t slot = sb; slot < se; ++slot) {
      const int cls = class_of(i, j, s);
      if ((int)counts.size() <= cls) counts.resize(cls + 1);
      const int64_t bk = bucket_of(cls, s);
      if ((int64_t)counts[cls].size() <= bk) counts[cls].resize(bk + 1, 0);
      counts[cls][bk]++;
      plan[cls].max_n = std::max(plan[cls].max_n, s.n);
      plan[cls].max_m = std::max(plan[cls].max_m, s.m);
      plan[cls].cost += double(s.n) * double(s.m);
      plan[cls].cells += double(pair_cells(s.n, s.m, s.hw));
      if (++j == p) {
        ++i;
        j = i + 1;
      }
    }
  };
  const bool verbose = env_or("DTWGPU_VERBOSE", 0) != 0;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto ms_since = [&](std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(tnow() - t).count();
  };
  auto tp = tnow();
  precost();
  if (verbose) fprintf(stderr, "dtwgpu: plan: %zu shapes costed in %.1f ms\n", shapes.size(), ms_since(tp));
  tp = tnow();
  pass1();
  if (verbose) fprintf(stderr, "dtwgpu: plan: pass 1 %.1f ms\n", ms_since(tp));
  // Shapes are first costed without a pair count (fill factor 1), which favours few lanes
  // per pair. A Full class that cannot keep ~half the GPU's warp slots busy with its
  // lanes per pair is re-costed with its real pair count (fill_factor), and the pass runs
  // again with those shapes re-classified (small ragged classes).
  if (ctx->force_family < 0 && env_or("DTWGPU_UNDERFILL_REPLAN", 1) != 0) {
    std::vector<int64_t> hint(plan.size(), 0);
    bool any = false;
    for (size_t c = 0; c < plan.size(); ++c) {
      int64_t n = 0;
      for (int64_t v : counts[c]) n += v;
      if (plan[c].cfg.family == Family::Full && fill_factor(n, plan[c].cfg.G, ctx->num_sms) < 0.5) {
        hint[c] = n;
        any = true;
      }
    }
    if (any) {
      old_hint = std::move(hint);
      if (use_tab) old_tab.swap(cls_tab), cls_tab.assign((size_t)(L1 * L1), -1);
      else old_shape.swap(cls_of_shape);
      plan.clear();
      cls_of_cfg.clear();
      counts.clear();
      tp = tnow();
      precost();
      pass1();
      if (verbose) fprintf(stderr, "dtwgpu: plan: underfill re-plan %.1f ms\n", ms_since(tp));
    }
  }
  tp = tnow();
  // descending bucket order -> start offsets
  std::vector<std::vector<int64_t>> start(plan.size());
  for (size_t c = 0; c < plan.size(); ++c) {
    auto& cn = counts[c];
    start[c].assign(cn.size(), 0);
    int64_t acc = 0;
    for (int64_t b = (int64_t)cn.size() - 1; b >= 0; --b) {
      start[c][b] = acc;
      acc += cn[b];
    }
    plan[c].slots.resize(acc);
  }
  // pass 2: place slots (and remember each one's shorter length)
  std::vector<std::vector<int32_t>> mkey(plan.size());
  for (size_t c = 0; c < plan.size(); ++c) mkey[c].resize(plan[c].slots.size());
  {
    int64_t i = i0, j = j0;
    Shape s;
    for (int64_t slot = sb; slot < se; ++slot) {
      const int cls = class_of(i, j, s);
      const int64_t at = start[cls][bucket_of(cls, s)]++;
      plan[cls].slots[at] = slot;
      mkey[cls][at] = (int32_t)s.m;
      if (++j == p) {
        ++i;
        j = i + 1;
      }
    }
  }
  // pass 3: inside each (passes, rows) bucket, order by the shorter length too, so the
  // lane groups of a warp mostly share one (n, m) -- same band geometry, same masked
  // steps, same trip counts. Counting sort per bucket (start[c][b] now marks its end).
  {
    std::vector<int64_t> cnt(L1 + 1);
    std::vector<int64_t> tmp;
    for (size_t c = 0; c < plan.size(); ++c) {
      auto& cn = counts[c];
      auto& sl = plan[c].slots;
      auto& mk = mkey[c];
      for (int64_t b = 0; b < (int64_t)cn.size(); ++b) {
        const int64_t e = start[c][b], a = e - cn[b];
        if (e - a < 2) continue;
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t t = a; t < e; ++t) cnt[mk[t]]++;
        int64_t acc = a;
        for (int64_t v = L1; v >= 0; --v) {  // descending m
          const int64_t k = cnt[v];
          cnt[v] = acc;
          acc += k;
        }
        tmp.assign(sl.begin() + a, sl.begin() + e);
        for (int64_t t = a; t < e; ++t) sl[cnt[mk[t]]++] = tmp[t - a];
      }
    }
  }
  if (verbose) fprintf(stderr, "dtwgpu: plan: passes 2-3 %.1f ms\n", ms_since(tp));
  tp = tnow();
  for (auto& pc : plan) {
    maybe_strip(ctx, pc, (int64_t)pc.slots.size(), -1);
    set_single_strip(pc);
  }
  if (verbose) fprintf(stderr, "dtwgpu: plan: strip check %.1f ms\n", ms_since(tp));
  return plan;
}

}  // namespace host
}  // namespace dtwgpu
