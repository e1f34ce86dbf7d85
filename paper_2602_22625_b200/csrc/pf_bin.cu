// K1 preprocess (+ optionally the fused Adam step) and K2 tile binning.
//
// Reference: bin_tiles (pkg/src/primfit/raster.py:227-265) walks primitives in
// ascending z, computes a conservative square bbox of half side
// r = scale*hypot(1, max(1, q)) + padding (bbox_half_side, raster.py:222-224),
// clips it to the canvas in float64 (ceil/floor, raster.py:248-253) and appends
// the primitive index to every tile the clipped pixel range touches, so every
// tile list is in ascending z.  adam_step: fit.py:195-238.
//
// B200 restatement (no host sync, no sort, no atomics on the binning path):
//   K1 k_prim<ADAM>  eight lanes per primitive (one per parameter): [Adam update
//                    of that parameter ->] record build split across the lanes
//                    (sincos / sigmoids / exact reciprocals on different lanes,
//                    fields exchanged with shuffles, each lane stores one
//                    16-byte slice) and the float64 bbox -> band-clipped tile
//                    rect per z position, with Python's rounding.
//   K2 k_bin_rows    one 1024-thread block per tile row, a two-digit stable
//                    radix bucketing of the z-ordered primitive stream:
//                    (a) stable compaction of the primitives covering the row
//                        (contiguous per-thread chunks + block scan), while a
//                        block reduction of "entries in earlier rows" gives the
//                        row's CSR base without any cross-block communication;
//                    (b) per-column counts (shared-memory atomics) -> block scan
//                        -> TileBins.offsets for the row's tiles;
//                    (c) one warp per column walks the row list with ballots and
//                        writes that tile's z-ascending primitive list (wide
//                        column blocks: one warp per column segment through a
//                        warp FIFO of the entries meeting it).
//   Many primitives x rows (c5, row bands): a two-level path builds the row lists
//   first -- per-chunk row counts, per-row chunk prefixes, a stable scatter --
//   and (a) reads them instead of re-reading every rect per (row, column block).
//   K1 stores records only for primitives that touch a tile of the band, and the
//   incremental variant (pf_preprocess_sync) only for primitives whose
//   parameters changed since the device copy.
// The CSR bins are bit-identical to the reference's offsets/indices.
//
// Slot mode (the fit step; ABI 6, see SlotBins in pf_bins.cuh): K1 also appends
// every (tile, primitive) pair of a primitive's band-clipped rect to the tile's
// slot list -- pos = atomicAdd(cnt[tile], 1), slot[tile][pos] = z rank -- and
// writes the fit step's records at the z rank; pf_fit_step's prologue sorts the
// lists, so no K2 launch sits between K1 and the fit step.  K1 runs 8 lanes per
// primitive, or 4 when 8 would not fit one wave of 3 blocks per SM (c5).
#include "../../include/primfit_b200.h"
#include "pf_bins.cuh"
#include "pf_common.cuh"

namespace pf {

struct AdamPart {
  double* grads;
  double* m;
  double* v;
  const uint8_t* frozen;
  double gains[8];
  const double* lr_table;
  const double* bc1_table;
  const double* bc2_table;
  int clamp;
  double s_min, s_max;
  const double* sums;    // loss sums of this step (after an allreduce), or NULL
  const double* part;    // per-warp loss partials of pf_fit_step to fold here, or NULL
  int n_part;
  double* hist_part;     // [iterations][gridDim.x][3] per-block loss sums (history)
  double* last_part;     // [gridDim.x][3] the same for the latest step only, or NULL
};

struct PreArgs {
  double* params;
  int n;
  double alpha_max, mu_blend, padding;
  int W, H, tile, ty_begin, ty_end;
  RecF* recf;
  RecG* recg;
  RecC* recc;
  RecS* recs;
  bool records;  // write records + rects (false: Adam only)
  double* mirror;     // Adam: updated parameters also written here (e.g. pinned host), or NULL
  const double* src;  // preprocess: parameters to take from here (e.g. pinned host), or NULL
  BinScratch s;
  AdamPart ad;
  unsigned long long* tl;  // diagnostics timeline or NULL
  // slot binning (pf_fit_step lists, see SlotBins): slots.cnt == NULL -> CSR mode
  // (records by primitive index, pf_bin builds the lists); else records RecS /
  // RecC go to the primitive's z rank and K1 scatters the pairs itself
  SlotBins slots;
  int ntx, n_tiles;   // band tiles (slot mode)
};

constexpr double kB1 = 0.9, kB2 = 0.999, kAdamEps = 1e-8;
#ifndef PF_SCAT_BATCH
#define PF_SCAT_BATCH 4
#endif
// slot-scatter atomics in flight per lane and round past the first two (A/B switch)
constexpr int kScatB = PF_SCAT_BATCH;
#ifndef PF_PRIM_THREADS
#define PF_PRIM_THREADS 256
#endif
constexpr int kPrimThreads = PF_PRIM_THREADS;
// K1 runs 3 blocks per SM (80 registers, no spills) with 8 lanes per primitive
// while that grid fits one wave (c3: 157 blocks), else with 4 lanes per
// primitive (c5: 313 blocks instead of 625 -- one wave; a 5-block, 48-register
// variant of the 8-lane kernel spilled and its record chain took twice as long)
constexpr int kPrimMinBlocks = 3 * 256 / kPrimThreads;
static int prim_lanes(int n) {
  return div_up(n > 0 ? n * 8 : 1, kPrimThreads) <= kPrimMinBlocks * dev_attrs().sms ? 8 : 4;
}

// adam_step for one scalar (fit.py:224-237), reference op order, no contraction.
// m, v, frozen are loaded by the caller before the PDL wait (k_step does not
// touch them); g is this step's gradient.
__device__ __forceinline__ double adam_scalar(const AdamPart& d, size_t idx, int col, bool live_p,
                                              double p, double g, double m0, double v0, double lr,
                                              double bc1, double bc2) {
  if (live_p) {
    const double mm = __dadd_rn(__dmul_rn(kB1, m0), __dmul_rn(1.0 - kB1, g));
    const double vv = __dadd_rn(__dmul_rn(kB2, v0), __dmul_rn(1.0 - kB2, __dmul_rn(g, g)));
    d.m[idx] = mm;
    d.v[idx] = vv;
    const double mh = __ddiv_rn(mm, bc1);
    const double vh = __ddiv_rn(vv, bc2);
    const double eff = __dmul_rn(lr, d.gains[col]);
    p = __dsub_rn(p, __ddiv_rn(__dmul_rn(eff, mh), __dadd_rn(__dsqrt_rn(vh), kAdamEps)));
  }
  if (d.clamp && col == 2) p = fmin(fmax(p, d.s_min), d.s_max);
  return p;
}

// LPP lanes per primitive: 8 (one parameter column each), or 4 (columns c and
// c + 4) when 8 lanes per primitive would not fit one wave at this occupancy
// (c5: 20k primitives) -- the same work on half the threads, no second wave.
template <bool ADAM, int LPP>
__global__ void __launch_bounds__(kPrimThreads, kPrimMinBlocks) k_prim(PreArgs a) {
  static_assert(LPP == 8 || LPP == 4, "lanes per primitive");
  constexpr int NC = 8 / LPP;  // parameter columns per lane
  tl_mark(a.tl, ADAM ? 2 : 3, 0);
  const int g = blockIdx.x * kPrimThreads + threadIdx.x;
  const int i = g / LPP, c = g % LPP;  // primitive, first parameter column
  const int lane = threadIdx.x & 31, gb = lane & ~(LPP - 1);
  const bool live = i < a.n;
  // static structure: one 48-byte record, independent of the parameter loads
  PrimInfo pi{2, 2, 0, 0, 1.0, 1.0, 0, 0, 0, 0};
  if (live && a.records) {
    const int4* src = reinterpret_cast<const int4*>(a.s.pinfo + i);
    const int4 w0 = __ldg(src), w1 = __ldg(src + 1), w2 = __ldg(src + 2);
    pi.wt = w0.x; pi.ht = w0.y; pi.base = w0.z; pi.pbase = w0.w;
    pi.q = __hiloint2double(w1.y, w1.x);
    pi.hyp = __hiloint2double(w1.w, w1.z);
    pi.zrank = w2.x; pi.tid = w2.y;
  }
  // this lane's columns: c + LPP * k, k < NC
  double pc[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) pc[k] = live ? a.params[(size_t)i * 8 + c + LPP * k] : 1.0;
  // incremental preprocess (src != NULL): the parameters come from src; only
  // primitives whose 8 values differ from the device copy are copied and get
  // new records / rects (the Adam launch before wrote the others' already)
  bool grp_changed = true;
  if (!ADAM && a.src) {
    bool ch = false;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const size_t pidx = (size_t)i * 8 + c + LPP * k;
      const double hv = live ? a.src[pidx] : 1.0;
      const bool chk = __double_as_longlong(hv) != __double_as_longlong(pc[k]);
      if (chk && live) a.params[pidx] = hv;
      ch |= chk;
      pc[k] = hv;
    }
    grp_changed = ((__ballot_sync(kFull, ch) >> gb) & ((1u << LPP) - 1u)) != 0u;
  }
  int it = 0;
  double fv0 = 0.0, fv1 = 0.0, fv2 = 0.0;  // loss-fold partial sums of this thread
  if (ADAM) {
    // everything k_step (the predecessor) does not write, before the PDL wait
    it = (int)a.s.done[1];  // advanced by the next pf_bin / slot-mode pf_fit_step
    const double lr = a.ad.lr_table[it], bc1 = a.ad.bc1_table[it], bc2 = a.ad.bc2_table[it];
    double m0[NC], v0[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const size_t pidx = (size_t)i * 8 + c + LPP * k;
      m0[k] = live ? a.ad.m[pidx] : 0.0;
      v0[k] = live ? a.ad.v[pidx] : 0.0;
    }
    const bool live_p = live && (a.ad.frozen == nullptr || a.ad.frozen[i] == 0);
    pdl_trigger();
    pdl_wait();
    tl_mark(a.tl, 2, 1);
    // this step's gradient and (first fold level) this block's chunk of k_step's
    // loss partials: both loads in flight before any math
    double gr[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) gr[k] = live ? a.ad.grads[(size_t)i * 8 + c + LPP * k] : 0.0;
    if (a.ad.part) {
      const int chunk = (a.ad.n_part + gridDim.x - 1) / gridDim.x;
      const int beg = blockIdx.x * chunk, end = min(beg + chunk, a.ad.n_part);
      for (int k = beg + threadIdx.x; k < end; k += kPrimThreads) {
        fv0 += __ldcg(a.ad.part + 3 * k + 0);
        fv1 += __ldcg(a.ad.part + 3 * k + 1);
        fv2 += __ldcg(a.ad.part + 3 * k + 2);
      }
    }
    if (live) {
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const size_t pidx = (size_t)i * 8 + c + LPP * k;
        a.ad.grads[pidx] = 0.0;  // ready for the next backward
        pc[k] = adam_scalar(a.ad, pidx, c + LPP * k, live_p, pc[k], gr[k], m0[k], v0[k], lr, bc1,
                            bc2);
        a.params[pidx] = pc[k];
        if (a.mirror) a.mirror[pidx] = pc[k];
      }
    }
    tl_mark(a.tl, 4, 1);
  }
  if (!ADAM) {
    pdl_wait();  // (records / rects may still be read by a predecessor)
    tl_mark(a.tl, 3, 1);
    pdl_trigger();
  }
  if (ADAM) tl_mark(a.tl, 5, 1);
  if (a.records) {
  // gather the primitive's 8 parameters from its lane group (column j lives in
  // lane j % LPP, slot j / LPP)
  auto col = [&](int j) { return __shfl_sync(kFull, pc[j / LPP], gb + j % LPP); };
  const double x = col(0), y = col(1), s = col(2), rot = col(3);
  const double nu = col(4), cl0 = col(5), cl1 = col(6), cl2 = col(7);
  const int t = pi.tid, wt = pi.wt, ht = pi.ht;
  const double q = pi.q, hyp = pi.hyp;
  const double sq = __dmul_rn(s, q);
  // bbox, float64 with Python's rounding: r = s*hyp + pad, ceil(x-r), floor(x+r)
  const double r = __dadd_rn(__dmul_rn(s, hyp), a.padding);
  // rect at the z rank: (tx0 | tx1 << 16, ty0, primitive, ty1); empty: ty0 > ty1
  // (every lane of the group computes it; lane 0 stores it)
  int4 rc = make_int4(0, 1, i, 0);
  {
    const double lo_x = fmax(ceil(__dsub_rn(x, r)), 0.0);
    const double hi_x = fmin(floor(__dadd_rn(x, r)), (double)(a.W - 1));
    const double lo_y = fmax(ceil(__dsub_rn(y, r)), 0.0);
    const double hi_y = fmin(floor(__dadd_rn(y, r)), (double)(a.H - 1));
    // NaN-safe: every comparison with NaN is false -> treated as empty
    if (lo_x <= hi_x && lo_y <= hi_y) {
      // (tile 16, the fit step's, as a shift: the operands are >= 0)
      const bool t16 = a.tile == 16;
      const int tx0 = t16 ? (int)lo_x >> 4 : (int)lo_x / a.tile;
      const int tx1 = t16 ? (int)hi_x >> 4 : (int)hi_x / a.tile;
      const int ty0 = max(t16 ? (int)lo_y >> 4 : (int)lo_y / a.tile, a.ty_begin);
      const int ty1 = min(t16 ? (int)hi_y >> 4 : (int)hi_y / a.tile, a.ty_end - 1);
      if (ty0 <= ty1) rc = make_int4(tx0 | (tx1 << 16), ty0, i, ty1);
    }
  }
  if (live && c == 0 && grp_changed) a.s.rect[pi.zrank] = rc;  // (lane 0 of the group)
  // records only for primitives in some tile of this band: nothing reads the
  // others' (every consumer walks the tile lists) -- on a row band of a
  // multi-GPU split most primitives skip the work below
  const bool need = live && rc.y <= rc.w && grp_changed;
  const bool slots = a.slots.cnt != nullptr;
  // K34-only records (RecS, RecC) sit at the z rank in slot mode: the sorted
  // tile lists hold z ranks
  const int ri = slots ? pi.zrank : i;
  // the pair scatter (see SlotBins): the rect's tiles split over the lane group;
  // the first two per lane go out before the record math (their atomics' round
  // trip overlaps it), the rest after
  const int sc_tx0 = rc.x & 0xffff, sc_nx = (rc.x >> 16) - sc_tx0 + 1;
  const int sc_nt = (slots && need) ? sc_nx * (rc.w - rc.y + 1) : 0;
  auto sc_tile = [&](int k) {
    const int ry = k / sc_nx;
    return (rc.y + ry - a.ty_begin) * a.ntx + sc_tx0 + (k - ry * sc_nx);
  };
  auto sc_put = [&](int t, int p) {
    if (p < a.slots.m) {
      a.slots.slot[(size_t)t * a.slots.m + p] = (uint32_t)pi.zrank;
    } else {
      const uint32_t o = atomicAdd(a.slots.ctl + kSlotOvf, 1u);
      if (o < (uint32_t)a.slots.ovf_cap) a.slots.ovf[o] = make_int2(t, pi.zrank);
      else a.slots.ctl[kSlotErr] = 1u;
    }
  };
  int sc_t0 = -1, sc_t1 = -1, sc_p0 = 0, sc_p1 = 0;
  if (c < sc_nt) {
    sc_t0 = sc_tile(c);
    sc_p0 = atomicAdd(a.slots.cnt + sc_t0, 1);
  }
  if (c + LPP < sc_nt) {
    sc_t1 = sc_tile(c + LPP);
    sc_p1 = atomicAdd(a.slots.cnt + sc_t1, 1);
  }
  if (__any_sync(kFull, need)) {
  // transcendental / division work split across the lane group
  double r0 = 0.0, r1 = 0.0;
  double ct, st, sig, sc0, sc1, sc2, inv_s, inv_sq;
  if (LPP == 8) {
    if (c == 0) {
      sincos(rot, &r1, &r0);  // r0 = cos, r1 = sin
    } else if (c <= 4) {
      r0 = sigmoid(c == 1 ? nu : c == 2 ? cl0 : c == 3 ? cl1 : cl2);
    } else if (c == 5) {
      r0 = __ddiv_rn(1.0, s);
      r1 = __ddiv_rn(1.0, sq);
    }
    ct = __shfl_sync(kFull, r0, gb + 0);
    st = __shfl_sync(kFull, r1, gb + 0);
    sig = __shfl_sync(kFull, r0, gb + 1);
    sc0 = __shfl_sync(kFull, r0, gb + 2);
    sc1 = __shfl_sync(kFull, r0, gb + 3);
    sc2 = __shfl_sync(kFull, r0, gb + 4);
    inv_s = __shfl_sync(kFull, r0, gb + 5);
    inv_sq = __shfl_sync(kFull, r1, gb + 5);
  } else {
    if (c == 0) {
      sincos(rot, &r1, &r0);
    } else if (c == 1) {
      r0 = sigmoid(nu);
      r1 = sigmoid(cl0);
    } else if (c == 2) {
      r0 = sigmoid(cl1);
      r1 = sigmoid(cl2);
    } else {
      r0 = __ddiv_rn(1.0, s);
      r1 = __ddiv_rn(1.0, sq);
    }
    ct = __shfl_sync(kFull, r0, gb + 0);
    st = __shfl_sync(kFull, r1, gb + 0);
    sig = __shfl_sync(kFull, r0, gb + 1);
    sc0 = __shfl_sync(kFull, r1, gb + 1);
    sc1 = __shfl_sync(kFull, r0, gb + 2);
    sc2 = __shfl_sync(kFull, r1, gb + 2);
    inv_s = __shfl_sync(kFull, r0, gb + 3);
    inv_sq = __shfl_sync(kFull, r1, gb + 3);
  }
  const double omm = __dsub_rn(1.0, a.mu_blend);

  if (need) {
#pragma unroll
  for (int kc = 0; kc < NC; ++kc) {
    const int c = lane % LPP + LPP * kc;  // the slice index this pass stores (0..7)
    // each lane stores one 16-byte slice of RecF (8 slices) and of RecG (5) / RecC (2)
    double2* pf = reinterpret_cast<double2*>(a.recf + i);
    switch (c) {
      case 0: pf[0] = make_double2(x, y); break;
      case 1: pf[1] = make_double2(ct, st); break;
      case 2: pf[2] = make_double2(inv_s, inv_sq); break;
      case 3: pf[3] = make_double2(s, sq); break;
      case 4: pf[4] = make_double2((double)(wt - 1), (double)(ht - 1)); break;
      case 5: pf[5] = make_double2(__dmul_rn(a.alpha_max, sig), __dmul_rn(omm, sc0)); break;
      case 6: pf[6] = make_double2(__dmul_rn(omm, sc1), __dmul_rn(omm, sc2)); break;
      default:
        reinterpret_cast<int4*>(pf)[7] = make_int4(pi.base, wt, ht, t);
        break;
    }
    float4* pg = reinterpret_cast<float4*>(a.recg + i);
    // (slot mode: RecG is K4's record only -- lanes 0-5 skip it; 6-7 write RecC)
    switch (slots && c < 6 ? -1 : c) {
      case -1:
        break;
      case 0:
        pg[0] = make_float4((float)(a.alpha_max * sig), (float)(omm * sc0), (float)(omm * sc1),
                            (float)(omm * sc2));
        break;
      case 1:
        pg[1] = make_float4((float)(a.alpha_max * sig * (1.0 - sig)), (float)(sc0 * (1.0 - sc0)),
                            (float)(sc1 * (1.0 - sc1)), (float)(sc2 * (1.0 - sc2)));
        break;
      case 2:
        pg[2] = make_float4((float)(-ct * inv_s), (float)(st * inv_sq), (float)(-st * inv_s),
                            (float)(-ct * inv_sq));
        break;
      case 3:  // 1/q = s / (s q)
        pg[3] = make_float4((float)inv_s, (float)q, (float)(s * inv_sq), 0.5f * (float)(wt - 1));
        break;
      case 4: {
        const double hw = 0.5 * (double)(wt - 1), hh = 0.5 * (double)(ht - 1);
        pg[4] = make_float4((float)hh, (float)(1.0 / hw), (float)(1.0 / hh), (float)omm);
        break;
      }
      case 5:
        reinterpret_cast<int4*>(pg)[5] = make_int4(pi.base, wt, ht, 0);
        break;
      default: {
        // cull record (see RecC): fp32 centre and axes, conservative slack
        const float fx = (float)x, fy = (float)y;
        const double hx = 0.5 * (kWarpW - 1), hy = 0.5 * (kWarpH - 1);
        const double e_px = fabs(x - (double)fx) + fabs(y - (double)fy);
        const double span = e_px + 1e-6 * (fabs(r) + 2.0 * kTile);
        const double act = fabs(ct), ast = fabs(st);
        float4* pc4 = reinterpret_cast<float4*>(a.recc + ri);
        if (c == 6) {
          pc4[0] = make_float4(fx, fy, (float)(ct * inv_s), (float)(st * inv_s));
        } else {
          const double eu = (act * hx + ast * hy) * inv_s + (act + ast) * inv_s * span + 1e-5;
          const double ev = (ast * hx + act * hy) * inv_sq + (act + ast) * inv_sq * span + 1e-5;
          pc4[1] = make_float4((float)(ct * inv_sq), (float)(st * inv_sq), (float)eu, (float)ev);
        }
      }
    }
    {
      // step record (RecS, pf_common.cuh): affine texel map + gradient coefficients
      const double hw = 0.5 * (double)(wt - 1), hh = 0.5 * (double)(ht - 1);
      const double au = hw * ct * inv_s, bu = hw * st * inv_s;
      const double cu = hw * (1.0 - (ct * x + st * y) * inv_s);
      const double av = -hh * st * inv_sq, bv = hh * ct * inv_sq;
      const double cv = hh * (1.0 + (st * x - ct * y) * inv_sq);
      double2* ps = reinterpret_cast<double2*>(a.recs + ri);
      float4* ps4 = reinterpret_cast<float4*>(a.recs + ri);
      const double sa_d = __dmul_rn(a.alpha_max, sig);
      // guard band of the affine U, V: >= 1e4 x their error bound
      const double du = 1e-11 * (fabs(au) * a.W + fabs(bu) * a.H + fabs(cu) + (wt - 1) + 1.0);
      const double dv = 1e-11 * (fabs(av) * a.W + fabs(bv) * a.H + fabs(cv) + (ht - 1) + 1.0);
      const double dl = fmax(du, dv);
      switch (c) {
        case 0: ps[0] = make_double2(au, bu); break;
        case 1: ps[1] = make_double2(cu - hw, av); break;
        case 2: ps[2] = make_double2(bv, cv - hh); break;
        case 3: ps[3] = make_double2(sa_d, __dmul_rn(omm, sc0)); break;
        case 4: ps[4] = make_double2(__dmul_rn(omm, sc1), __dmul_rn(omm, sc2)); break;
        case 5: ps[5] = make_double2(hw, hh); break;
        case 6: ps[6] = make_double2(hw - dl, hw + dl); break;
        default: ps[7] = make_double2(hh - dl, hh + dl); break;
      }
      switch (c) {
        case 0: reinterpret_cast<int4*>(ps4)[8] = make_int4(pi.pbase, wt + 1, i, 0); break;
        case 1:
          ps4[9] = make_float4((float)(a.alpha_max * sig * (1.0 - sig)), (float)(sc0 * (1.0 - sc0)),
                               (float)(sc1 * (1.0 - sc1)), (float)(sc2 * (1.0 - sc2)));
          break;
        case 2:
          ps4[10] = make_float4((float)(-ct * inv_s), (float)(st * inv_sq), (float)(-st * inv_s),
                                (float)(-ct * inv_sq));
          break;
        case 3: ps4[11] = make_float4((float)inv_s, (float)q, (float)(s * inv_sq), (float)hw); break;
        case 4:
          ps4[12] = make_float4((float)hh, (float)omm, (float)sa_d, 1.0f / (float)hw);
          break;
        case 5:
          ps4[13] = make_float4((float)(omm * sc0), (float)(omm * sc1), (float)(omm * sc2),
                                1.0f / (float)hh);
          break;
        default: break;
      }
    }
  }  // the lane's slices
  }
  }  // any record in this warp
  if (ADAM && need) tl_mark(a.tl, 8, 2);  // (diagnostics: records stored)
  if (sc_t0 >= 0) sc_put(sc_t0, sc_p0);
  if (sc_t1 >= 0) sc_put(sc_t1, sc_p1);
  for (int k0 = c + 2 * LPP; k0 < sc_nt; k0 += kScatB * LPP) {
    int t4[kScatB], p4[kScatB];
#pragma unroll
    for (int q = 0; q < kScatB; ++q) {
      const int k = k0 + LPP * q;
      t4[q] = k < sc_nt ? sc_tile(k) : -1;
      if (t4[q] >= 0) p4[q] = atomicAdd(a.slots.cnt + t4[q], 1);
    }
#pragma unroll
    for (int q = 0; q < kScatB; ++q)
      if (t4[q] >= 0) sc_put(t4[q], p4[q]);
  }
  if (ADAM && need) tl_mark(a.tl, 9, 2);  // (diagnostics: scatter done)
  // an edited primitive re-scattered next to its previous entries: the
  // producers validate and de-duplicate this step's lists
  if (!ADAM && a.src && sc_nt > 0 && c == 0) a.slots.ctl[kSlotDirty] = 1u;
  }  // a.records



  if (ADAM) {
    // this block's loss sums of the step (fixed-order fold of its chunk of
    // k_step's partials, or the allreduced sums from block 0) go to the history
    // buffer; the host folds the blocks in order (deterministic).  Block 0 marks
    // the iteration done: K2 of the next step advances the counter.
    __shared__ double fr[kPrimThreads / 32][3];
    tl_mark(a.tl, 6, 1);
    if (a.ad.part) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        fv0 += __shfl_xor_sync(kFull, fv0, o);
        fv1 += __shfl_xor_sync(kFull, fv1, o);
        fv2 += __shfl_xor_sync(kFull, fv2, o);
      }
      if (lane == 0) {
        fr[threadIdx.x >> 5][0] = fv0;
        fr[threadIdx.x >> 5][1] = fv1;
        fr[threadIdx.x >> 5][2] = fv2;
      }
      __syncthreads();
    }
    if (threadIdx.x < 3 && a.ad.hist_part) {
      double tsum = 0.0;
      if (a.ad.part) {
        for (int w = 0; w < kPrimThreads / 32; ++w) tsum += fr[w][threadIdx.x];
      } else if (a.ad.sums && blockIdx.x == 0) {
        tsum = a.ad.sums[threadIdx.x];
      }
      a.ad.hist_part[((size_t)it * gridDim.x + blockIdx.x) * 3 + threadIdx.x] = tsum;
      if (a.ad.last_part) a.ad.last_part[blockIdx.x * 3 + threadIdx.x] = tsum;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.s.done[2] = 1u;
  }
  tl_mark(a.tl, ADAM ? 2 : 3, 3);
}

struct RowArgs {
  int n, ntx, ty_begin, n_rows, cap, smem_list;
  BinScratch s;
  int32_t* bin_off;
  int32_t* bin_idx;
  int32_t* status;
  int32_t* classes;  // optional tile cost classes (see kTileClasses), or NULL
  int n_tiles;
  int prebuilt;      // row lists come from k_row_scatter (two-level path)
  unsigned long long* tl;
};

constexpr int kRowThreads = 1024;

// Two-level path, for many primitives x many rows (one-level K2 re-reads every
// rect once per (row, column block)).  Pass 1 (k_row_counts): per chunk of
// kRowChunk z positions, the (row pairs, tile entries) counts of every row.
// Pass 2 (k_row_offsets, one block): per row, the exclusive prefix over chunks
// (in place) and the row's list start / length / entries before it (rowinfo).
// Pass 3 (k_row_scatter): every chunk writes its (primitive, column span) pairs
// into the per-row lists, z order kept (chunk, then warp, then lane order).
// k_bin_rows then starts from the prebuilt row lists instead of scanning all
// rects.
__global__ void __launch_bounds__(kRowChunk) k_row_counts(RowArgs a) {
  extern __shared__ int2 sc[];  // [n_rows]
  const int tid = threadIdx.x;
  tl_mark(a.tl, 11, 0);
  for (int r = tid; r < a.n_rows; r += kRowChunk) sc[r] = make_int2(0, 0);
  pdl_wait();  // rects come from K1
  tl_mark(a.tl, 11, 1);
  pdl_trigger();
  __syncthreads();
  const int zp = blockIdx.x * kRowChunk + tid;
  if (zp < a.n) {
    const int4 rc = a.s.rect[zp];
    if (rc.y <= rc.w) {
      const int span = (rc.x >> 16) - (rc.x & 0xffff) + 1;
      for (int ty = rc.y; ty <= rc.w; ++ty) {
        atomicAdd(&sc[ty - a.ty_begin].x, 1);
        atomicAdd(&sc[ty - a.ty_begin].y, span);
      }
    }
  }
  __syncthreads();
  for (int r = tid; r < a.n_rows; r += kRowChunk)
    a.s.rowcnt[(size_t)blockIdx.x * a.n_rows + r] = sc[r];
  tl_mark(a.tl, 11, 3);
}

// One warp per row (4 per block): the exclusive prefix over chunks of the
// row's pair counts, in place, and the row's totals (pairs, tile entries) in
// rowinfo[r].  Row offsets (a scan over rows) are left to the consumers.
__global__ void __launch_bounds__(128) k_row_offsets(RowArgs a, int nch) {
  const int lane = threadIdx.x & 31, r = blockIdx.x * 4 + (threadIdx.x >> 5);
  tl_mark(a.tl, 13, 0);
  pdl_wait();  // the count matrix
  tl_mark(a.tl, 13, 1);
  pdl_trigger();
  if (r >= a.n_rows) return;
  int carry = 0, ent = 0;
  constexpr int kB = 8;  // chunks per lane per batch: all loads first
  for (int c0 = 0; c0 < nch; c0 += 32 * kB) {
    int2 v[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int c = c0 + i * 32 + lane;
      v[i] = c < nch ? a.s.rowcnt[(size_t)c * a.n_rows + r] : make_int2(0, 0);
    }
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int c = c0 + i * 32 + lane;
      int x = v[i].x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      if (c < nch) a.s.rowcnt[(size_t)c * a.n_rows + r].x = carry + x - v[i].x;
      carry += __shfl_sync(kFull, x, 31);
      ent += v[i].y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ent += __shfl_xor_sync(kFull, ent, o);
  if (lane == 0) a.s.rowinfo[r] = make_int4(carry, ent, 0, 0);
  tl_mark(a.tl, 13, 3);
}

__global__ void __launch_bounds__(kRowChunk) k_row_scatter(RowArgs a) {
  constexpr int kW = kRowChunk / 32;
  extern __shared__ int2 smem_rs[];
  int2* spans = smem_rs;                                    // [kRowChunk] (ty0, ty1)
  int* wcnt = reinterpret_cast<int*>(spans + kRowChunk);    // [kW warps][n_rows]: counts, offsets
  int* roff = wcnt + kW * a.n_rows;                         // [n_rows] row start + earlier chunks
  __shared__ int ws[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk = blockIdx.x;
  for (int k = tid; k < kW * a.n_rows; k += kRowChunk) wcnt[k] = 0;
  const int zp = chunk * kRowChunk + tid;
  tl_mark(a.tl, 12, 0);
  pdl_wait();  // offsets of k_row_offsets (and, through it, the rects of K1)
  tl_mark(a.tl, 12, 1);
  pdl_trigger();
  // every load up front (independent): rect, the rows' totals and chunk prefixes
  const int4 rc = zp < a.n ? a.s.rect[zp] : make_int4(0, 1, 0, 0);
  constexpr int kRP = 1024 / kRowChunk;  // rows per thread (n_rows <= 1024), contiguous
  int tot[kRP], pre[kRP];
#pragma unroll
  for (int q = 0; q < kRP; ++q) {
    const int r = tid * kRP + q;
    tot[q] = r < a.n_rows ? a.s.rowinfo[r].x : 0;
    pre[q] = r < a.n_rows ? a.s.rowcnt[(size_t)chunk * a.n_rows + r].x : 0;
  }
  const int y0 = rc.y - a.ty_begin, y1 = rc.w - a.ty_begin;  // empty: y0 > y1
  spans[tid] = make_int2(y0, y1);
  int local = 0;
#pragma unroll
  for (int q = 0; q < kRP; ++q) local += tot[q];
  int rows_total;
  int acc = block_excl_scan(local, ws, &rows_total);
#pragma unroll
  for (int q = 0; q < kRP; ++q) {
    const int r = tid * kRP + q;
    if (r < a.n_rows) roff[r] = acc + pre[q];
    acc += tot[q];
  }
  const bool fits = rows_total <= a.cap;  // else K > cap: k_bin_rows flags it
  __syncthreads();
  // this warp's pairs per row: lane L's rank in row r = covering lanes l < L
  const int wb = warp * 32;
  for (int ty = y0; ty <= y1; ++ty) {
    int before = 0, after = 0;
    for (int l = 0; l < 32; ++l) {
      const int2 sp = spans[wb + l];
      const int cov = sp.x <= ty && ty <= sp.y;
      before += (l < lane) & cov;
      after += (l > lane) & cov;
    }
    if (after == 0) wcnt[warp * a.n_rows + ty] = before + 1;  // the row's last lane
  }
  __syncthreads();
  // per row: offsets of the warps' pairs (row start + earlier chunks + earlier warps)
  for (int r = tid; r < a.n_rows; r += kRowChunk) {
    int o = roff[r];
#pragma unroll
    for (int w = 0; w < kW; ++w) {
      const int t = wcnt[w * a.n_rows + r];
      wcnt[w * a.n_rows + r] = o;
      o += t;
    }
  }
  __syncthreads();
  // scatter: (primitive, column span) at row start + offsets + lane rank
  if (fits) {
    for (int ty = y0; ty <= y1; ++ty) {
      int before = 0;
      for (int l = 0; l < lane; ++l) {
        const int2 sp = spans[wb + l];
        before += sp.x <= ty && ty <= sp.y;
      }
      a.s.rowlist[wcnt[warp * a.n_rows + ty] + before] = make_int2(rc.z, rc.x);
    }
  }
  tl_mark(a.tl, 12, 3);
}

constexpr int kRowCache = 8;  // rects per thread kept in registers between the passes

// K2: blocks (r, cb): tile row r, column block cb of gridDim.y.  See the file
// header.  Every column block of a row redoes (a) (cheap: the rects are in L2)
// and the column counts of (b); offsets, classes and the ballot walks of (c)
// cover only its own columns, so a row's work spreads over gridDim.y SMs.
template <bool CACHE>
__global__ void __launch_bounds__(kRowThreads) k_bin_rows(RowArgs a) {
  extern __shared__ int2 rsm[];  // [smem_list] row list, then [ntx] column counters
  __shared__ int ws[32];
  __shared__ int4 ws4[32];
  __shared__ int s_rl, s_base, s_rbase;
  __shared__ int s_ccnt[kTileClasses], s_cbase[kTileClasses];
  __shared__ int2 wfifo[32 * 64];  // (c) per-warp FIFO of wide column blocks
  int* col = reinterpret_cast<int*>(rsm + a.smem_list);
  int* ccls = col + a.ntx;  // per-column tile class | rank within the block << 8
  int* ccnt = ccls + a.ntx;  // per-column tile list length
  const int r = blockIdx.x, ty = a.ty_begin + r;
  const int cb = blockIdx.y, ncb = gridDim.y;
  const int cbeg = (int)((long long)a.ntx * cb / ncb), cend = (int)((long long)a.ntx * (cb + 1) / ncb);
  const int tid = threadIdx.x;
  tl_mark(a.tl, 0, 0);
  pdl_wait();     // rects come from K1
  tl_mark(a.tl, 0, 1);
  pdl_trigger();  // after the wait: a dependent that starts early sees K1 complete
  if (r == 0 && cb == 0 && tid == 0 && a.s.done[2]) {
    // the Adam step before this binning is complete: advance the iteration counter
    a.s.done[1] += 1u;
    a.s.done[2] = 0u;
  }

  // measured cost of this thread's column tile (first column of its chunk; read
  // early so the load overlaps the scan)
  const int cchunk = (a.ntx + kRowThreads - 1) / kRowThreads;
  const int c0 = min(a.ntx, tid * cchunk), c1 = min(a.ntx, c0 + cchunk);
  int32_t* cost_row = a.classes ? a.classes + tile_cost_offset(a.n_tiles) + r * a.ntx : nullptr;
  const int cost0 = (cost_row && c0 < c1 && c0 >= cbeg && c0 < cend) ? cost_row[c0] : 0;

  // (a) stable compaction of the primitives covering row ty, z order kept
  const int chunk = (a.n + kRowThreads - 1) / kRowThreads;
  const int j0 = min(a.n, tid * chunk), j1 = min(a.n, j0 + chunk);
  // rects: (tx0 | tx1 << 16, ty0, primitive, ty1), empty when ty0 > ty1 (k_prim)
  int4 rcache[CACHE ? kRowCache : 1];
  int cnt = 0, below = 0, below_rows = 0, all = 0;
  constexpr int4 kEmpty = {0, 1, 0, 0};
  auto tally = [&](const int4& rc) {
    if (rc.y > rc.w) return;  // empty
    const int span = (rc.x >> 16) - (rc.x & 0xffff) + 1;
    all += (rc.w - rc.y + 1) * span;
    if (rc.y <= ty && ty <= rc.w) ++cnt;
    if (rc.y < ty) {
      const int rows = min(rc.w, ty - 1) - rc.y + 1;
      below += rows * span;
      below_rows += rows;
    }
  };
  int tot, base, rbase, K, pos = 0;
  if (a.prebuilt) {
    // two-level path: the row lists come from k_row_scatter; this row's list
    // start / entries before it / K from a scan of the rows' totals
    const int4 ri = tid < a.n_rows ? a.s.rowinfo[tid] : make_int4(0, 0, 0, 0);
    int4 tot4;
    const int4 ex = block_excl_scan4(make_int4(ri.x, ri.y, 0, 0), ws4, &tot4);
    if (tid == r) {
      s_rl = ri.x;
      s_rbase = ex.x;
      s_base = ex.y;
    }
    __syncthreads();
    tot = s_rl;
    rbase = s_rbase;
    base = s_base;
    K = tot4.y;
  } else {
    if (CACHE) {
      // all loads first (independent), then the tallies
#pragma unroll
      for (int k = 0; k < kRowCache; ++k) rcache[k] = j0 + k < j1 ? a.s.rect[j0 + k] : kEmpty;
#pragma unroll
      for (int k = 0; k < kRowCache; ++k) tally(rcache[k]);
    } else {
      // long chunks: batches of kRowCache independent loads, then the tallies
      for (int jb = j0; jb < j1; jb += kRowCache) {
        int4 rb[kRowCache];
#pragma unroll
        for (int k = 0; k < kRowCache; ++k) rb[k] = jb + k < j1 ? a.s.rect[jb + k] : kEmpty;
#pragma unroll
        for (int k = 0; k < kRowCache; ++k) tally(rb[k]);
      }
    }
    int4 tot4;
    const int4 ex = block_excl_scan4(make_int4(cnt, below, below_rows, all), ws4, &tot4);
    tot = tot4.x;
    base = tot4.y;
    rbase = tot4.z;
    K = tot4.w;
    pos = ex.x;
  }
  if (r == 0 && cb == 0 && tid == 0) {
    // every block knows K; block (0, 0) publishes it (TileBins.offsets[-1], overflow flag)
    a.bin_off[a.n_rows * a.ntx] = K;
    a.status[0] = K;
    a.status[1] = K > a.cap ? 1 : 0;
  }
  tl_mark(a.tl, 8, 1);
  if (K > a.cap) {  // overflow (grid-uniform): nothing is written
    tl_mark(a.tl, 0, 3);
    return;
  }
  if (tid == 0 && !a.prebuilt) {  // (prebuilt: already published above)
    s_rl = tot;
    s_base = base;
    s_rbase = rbase;
  }
  for (int c = tid; c < a.ntx; c += kRowThreads) col[c] = 0;
  if (tid < kTileClasses) s_ccnt[tid] = 0;
  // long rows spill the list to HBM (every column block writes the same values)
  const bool spill_list = tot > a.smem_list;
  auto put = [&](const int4& rc) {
    // (primitive index, column span): the list order is the z order
    const int2 e = make_int2(rc.z, rc.x);
    if (pos < a.smem_list) rsm[pos] = e;
    if (spill_list) a.s.rowlist[rbase + pos] = e;  // rbase + pos < rows entries <= K <= cap
    ++pos;
  };
  if (a.prebuilt) {
    if (tot <= a.smem_list)
      for (int k = tid; k < tot; k += kRowThreads) rsm[k] = a.s.rowlist[rbase + k];
  } else if (CACHE) {
#pragma unroll
    for (int k = 0; k < kRowCache; ++k) {
      const int4 rc = rcache[k];
      if (rc.y <= ty && ty <= rc.w) put(rc);
    }
  } else {
    for (int jb = j0; jb < j1; jb += kRowCache) {
      int4 rb[kRowCache];
#pragma unroll
      for (int k = 0; k < kRowCache; ++k) rb[k] = jb + k < j1 ? a.s.rect[jb + k] : kEmpty;
#pragma unroll
      for (int k = 0; k < kRowCache; ++k)
        if (rb[k].y <= ty && ty <= rb[k].w) put(rb[k]);
    }
  }
  __syncthreads();
  const int RL = s_rl;
  const int2* list = RL <= a.smem_list ? rsm : a.s.rowlist + s_rbase;

  tl_mark(a.tl, 9, 1);
  // (b) per-column counts (all columns) -> offsets of this block's tiles
  for (int k = tid; k < RL; k += kRowThreads) {
    const int pk = list[k].y;
    for (int tx = pk & 0xffff; tx <= (pk >> 16); ++tx) atomicAdd(col + tx, 1);
  }
  __syncthreads();
  int local = 0;
  for (int c = c0; c < c1; ++c) local += col[c];
  int row_total;
  int run = s_base + block_excl_scan(local, ws, &row_total);
  for (int c = c0; c < c1; ++c) {
    const int v = col[c];
    col[c] = run;
    if (c >= cbeg && c < cend) {
      a.bin_off[r * a.ntx + c] = run;
      if (a.classes) {
        // longest-first schedule for pf_fit_step: tile -> class list of its cost
        // (measured by the previous fit step; its list length before that)
        const int w = c == c0 ? cost0 : cost_row[c];
        cost_row[c] = 0;
        const int cl = tile_class(w > 0 ? w : v);
        const int rank = atomicAdd(&s_ccnt[cl], 1);
        ccls[c] = cl | (rank << 8);
        ccnt[c] = v;
      }
    }
    run += v;
  }
  __syncthreads();
  // class bases: the global atomics' latency overlaps the ballot walks of (c)
  int cbase_mine = 0;
  if (a.classes && tid < kTileClasses)
    cbase_mine = s_ccnt[tid] ? atomicAdd(a.classes + tid, s_ccnt[tid]) : 0;

  tl_mark(a.tl, 10, 1);
  // (c) ordered ballot walks of the row list.  Narrow column blocks: one warp
  // per column.  Wide ones (more columns than warps): one warp per segment of
  // w consecutive columns, which first compacts the entries meeting its
  // segment (z order kept, 64-entry warp FIFO in shared memory), then writes
  // them column by column -- the list is read once per segment, not per column.
  const int lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int wseg = (cend - cbeg + 31) / 32;
  if (wseg <= 1) {
    for (int c = cbeg + warp; c < cend; c += kRowThreads / 32) {
      int out = col[c];
      for (int b = 0; b < RL; b += 32) {
        const int k = b + lane;
        bool hit = false;
        int j = 0;
        if (k < RL) {
          const int2 e = list[k];
          j = e.x;
          hit = (e.y & 0xffff) <= c && c <= (e.y >> 16);
        }
        const unsigned ball = __ballot_sync(kFull, hit);
        if (hit) a.bin_idx[out + __popc(ball & lt)] = j;
        out += __popc(ball);
      }
    }
  } else {
    int2* fifo = wfifo + warp * 64;
    const int s0 = cbeg + warp * wseg, s1 = min(s0 + wseg, cend) - 1;
    for (int q0 = s0; q0 <= s1; q0 += 32) {  // sub-segments of <= 32 columns (lane counters)
      const int q1 = min(q0 + 31, s1);
      int out = q0 + lane <= q1 ? col[q0 + lane] : 0;  // write position of column q0 + lane
      auto drain = [&](int ne) {  // the first ne FIFO entries, column by column
        int lo = 1, hi = 0, j = 0;
        if (lane < ne) {
          const int2 e = fifo[lane];
          j = e.x;
          lo = max(e.y & 0xffff, q0);
          hi = min(e.y >> 16, q1);
        }
        const bool any = lo <= hi;
        const unsigned cmin = __reduce_min_sync(kFull, any ? (unsigned)lo : 0xffffffffu);
        const unsigned cmax = __reduce_max_sync(kFull, any ? (unsigned)hi : 0u);
        for (int c = (int)cmin; c <= (int)cmax; ++c) {
          const bool cov = lo <= c && c <= hi;
          const unsigned m = __ballot_sync(kFull, cov);
          if (m == 0u) continue;
          const int at = __shfl_sync(kFull, out, c - q0);
          if (cov) a.bin_idx[at + __popc(m & lt)] = j;
          if (lane == c - q0) out += __popc(m);
        }
      };
      int nb = 0;
      for (int b = 0; b < RL; b += 32) {
        const int k = b + lane;
        int2 e = make_int2(0, 0);
        bool meet = false;
        if (k < RL) {
          e = list[k];
          meet = (e.y & 0xffff) <= q1 && (e.y >> 16) >= q0;
        }
        const unsigned m = __ballot_sync(kFull, meet);
        if (meet) fifo[nb + __popc(m & lt)] = e;
        nb += __popc(m);
        __syncwarp();
        if (nb >= 32) {
          drain(32);
          const int rem = nb - 32;
          int2 t = make_int2(0, 0);
          if (lane < rem) t = fifo[32 + lane];
          __syncwarp();
          if (lane < rem) fifo[lane] = t;
          __syncwarp();
          nb = rem;
        }
      }
      if (nb > 0) drain(nb);
      __syncwarp();
    }
  }
  if (a.classes) {
    if (tid < kTileClasses) s_cbase[tid] = cbase_mine;
    __syncthreads();
    for (int c = max(c0, cbeg); c < min(c1, cend); ++c) {
      const int cl = ccls[c] & 0xff, rank = ccls[c] >> 8;
      const int p = s_cbase[cl] + rank;
      if (p < a.n_tiles)
        reinterpret_cast<int4*>(a.classes + kTileClasses)[cl * a.n_tiles + p] =
            make_int4(r * a.ntx + c, col[c], ccnt[c], c | ((a.ty_begin + r) << 16));
    }
  }
  tl_mark(a.tl, 0, 3);
}

// Alpha quad atlas (see load_quad in pf_common.cuh): one thread per texel.
struct QuadArgs {
  const double* tex;  // planar [4][texels]
  int texels, n_tpl;
  const int32_t* base;
  const int32_t* w;
  const int32_t* h;
  float4* quad;
};

__global__ void k_atlas_quad(QuadArgs a) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.texels) return;
  int t = 0;
  while (t + 1 < a.n_tpl && a.base[t + 1] <= g) ++t;
  const int wt = a.w[t], ht = a.h[t], local = g - a.base[t];
  const int v = local / wt, u = local - v * wt;
  const double* al = a.tex + 3 * (size_t)a.texels + a.base[t];
  auto at = [&](int uu, int vv) { return (uu < wt && vv < ht) ? al[vv * wt + uu] : 0.0; };
  a.quad[g] = make_float4((float)at(u, v), (float)at(u + 1, v), (float)at(u, v + 1),
                          (float)at(u + 1, v + 1));
}

// Zero-padded fp32 alpha plane (RecS.pbase / wp): template t occupies
// (wt + 1) x (ht + 1) texels from pbase[t]; the extra column and row are the
// reference's zero padding (_kernels.py:35-40), so a bilinear sample with the
// cell inside the box needs no bounds checks.
struct PadArgs {
  const double* tex;
  int texels, n_tpl, pad_texels;
  const int32_t* base;
  const int32_t* pbase;
  const int32_t* w;
  const int32_t* h;
  float* apad;
};

__global__ void k_atlas_pad(PadArgs a) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.pad_texels) return;
  int t = 0;
  while (t + 1 < a.n_tpl && a.pbase[t + 1] <= g) ++t;
  const int wt = a.w[t], ht = a.h[t], local = g - a.pbase[t];
  const int v = local / (wt + 1), u = local - v * (wt + 1);
  const double* al = a.tex + 3 * (size_t)a.texels + a.base[t];
  a.apad[g] = (t < a.n_tpl && u < wt && v < ht) ? (float)al[v * wt + u] : 0.0f;
}

constexpr int kRowSmemList = 4096;  // row-list entries kept in shared memory (32 KB)

}  // namespace pf

using namespace pf;

extern "C" size_t pf_bin_scratch_bytes(int n, int n_tiles, int capacity) {
  if (n < 0 || n_tiles < 0 || capacity < 0) return 0;
  return carve(nullptr, n, capacity, n_tiles).total;
}

static bool band_ok(int W, int H, int tile, int ty_begin, int ty_end, int* ntx, int* n_rows) {
  if (W < 1 || H < 1 || tile < 1) return false;
  *ntx = div_up(W, tile);
  const int nty = div_up(H, tile);
  if (ty_begin < 0 || ty_end > nty || ty_begin > ty_end) return false;
  if (*ntx > 65535) return false;  // column packed in 16 bits
  *n_rows = ty_end - ty_begin;
  return true;
}

static int fill_pre_args(PreArgs& a, double* params, int n, double alpha_max, double mu_blend,
                         double padding, int W, int H, int tile, int ty_begin, int ty_end,
                         int capacity, void* rec, void* scratch, size_t scratch_bytes) {
  int ntx, n_rows;
  if (n < 0 || capacity < 0 || !band_ok(W, H, tile, ty_begin, ty_end, &ntx, &n_rows))
    return PF_ERR_ARG;
  if (!scratch || scratch_bytes < pf_bin_scratch_bytes(n, n_rows * ntx, capacity))
    return PF_ERR_SCRATCH;
  if (n > 0 && (!params || !rec)) return PF_ERR_ARG;
  a.params = params;
  a.n = n;
  a.alpha_max = alpha_max;
  a.mu_blend = mu_blend;
  a.padding = padding;
  a.W = W;
  a.H = H;
  a.tile = tile;
  a.ty_begin = ty_begin;
  a.ty_end = ty_end;
  a.recf = (RecF*)rec;
  a.recg = (RecG*)((char*)rec + sizeof(RecF) * (size_t)n);
  a.recc = (RecC*)((char*)rec + (sizeof(RecF) + sizeof(RecG)) * (size_t)n);
  a.recs = (RecS*)((char*)rec + (sizeof(RecF) + sizeof(RecG) + sizeof(RecC)) * (size_t)n);
  a.records = true;
  a.mirror = nullptr;
  a.src = nullptr;
  a.s = carve(scratch, n, capacity);
  a.ad = AdamPart{};
  a.tl = pf_timeline_ptr();
  a.slots = SlotBins{};
  a.ntx = ntx;
  a.n_tiles = n_rows * ntx;
  return PF_OK;
}

// Slot mode (slots != NULL): slot scratch of pf_slot_bytes(n_tiles, m, capacity);
// tile must be the render tile.  (tile_classes: the fit step's prologue builds
// the classes; accepted for symmetry with pf_fit_step.)
static int attach_slots(PreArgs& a, void* slots, int slot_m, int32_t* tile_classes,
                        int capacity) {
  (void)tile_classes;
  if (!slots) return PF_OK;
  if (a.tile != kTile || slot_m < 1) return PF_ERR_ARG;
  a.slots = slot_carve(slots, a.n_tiles, slot_m, capacity);
  return PF_OK;
}

extern "C" size_t pf_slot_bytes(int n_tiles, int m, int capacity) {
  if (n_tiles < 0 || m < 1 || capacity < 0) return 0;
  return slot_carve(nullptr, n_tiles, m, capacity).total;
}

// Empty slot lists and tile classes (before a full pf_preprocess in slot mode).
extern "C" int pf_slot_reset(void* slots, int n_tiles, int m, int capacity,
                             int32_t* tile_classes, void* stream) {
  if (!slots || n_tiles < 0 || m < 1 || capacity < 0) return PF_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const SlotBins s = slot_carve(slots, n_tiles, m, capacity);
  cudaError_t e = cudaMemsetAsync(s.ctl, 0, sizeof(uint32_t) * kSlotCtlWords, st);
  if (e == cudaSuccess && n_tiles > 0)
    e = cudaMemsetAsync(s.cnt, 0, sizeof(int32_t) * (size_t)n_tiles, st);
  if (e == cudaSuccess && tile_classes)
    e = cudaMemsetAsync(tile_classes, 0, sizeof(int32_t) * kTileClasses, st);
  return (int)e;
}

#ifndef PF_PRIM_LPP
#define PF_PRIM_LPP 0  // (A/B: 0 = by occupancy, 8 / 4 forced)
#endif
static int launch_prim(bool adam, const PreArgs& a, cudaStream_t st) {
  const int lpp = PF_PRIM_LPP ? PF_PRIM_LPP : prim_lanes(a.n);
  const int blocks = div_up(a.n > 0 ? a.n * lpp : 1, kPrimThreads);
  if (adam)
    return (int)launch_pdl(lpp == 8 ? k_prim<true, 8> : k_prim<true, 4>, blocks, kPrimThreads,
                           0, st, a);
  if (a.n > 0)
    return (int)launch_pdl(lpp == 8 ? k_prim<false, 8> : k_prim<false, 4>, blocks, kPrimThreads,
                           0, st, a);
  return (int)cudaGetLastError();
}

// One-time static structure: pinfo[zorder[j]] = {template geometry, z rank j}.
struct InfoArgs {
  const int32_t* tid;
  const int32_t* zorder;
  int n, n_tpl;
  const int32_t* base;
  const int32_t* pbase;
  const int32_t* w;
  const int32_t* h;
  const double* q;
  const double* hyp;
  PrimInfo* pinfo;
};

__global__ void k_pinfo(InfoArgs a) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  const int i = a.zorder[j];
  const int t = a.tid[i];
  PrimInfo p;
  const bool ok = t >= 0 && t < a.n_tpl;
  p.wt = ok ? a.w[t] : 2;
  p.ht = ok ? a.h[t] : 2;
  p.base = ok ? a.base[t] : 0;
  p.pbase = ok && a.pbase ? a.pbase[t] : 0;
  p.q = ok ? a.q[t] : 1.0;
  p.hyp = ok ? a.hyp[t] : 1.0;
  p.zrank = j;
  p.tid = t;
  p.pad0 = p.pad1 = 0;
  a.pinfo[i] = p;
}

extern "C" int pf_scratch_init(void* scratch, size_t scratch_bytes, const int32_t* template_id,
                               const int32_t* zorder, int n, const int32_t* tpl_base,
                               const int32_t* tpl_pbase, const int32_t* tpl_w,
                               const int32_t* tpl_h, const double* tpl_q, const double* tpl_hyp,
                               int n_tpl, int capacity, void* stream) {
  if (!scratch || n < 0 || capacity < 0 || n_tpl < 0 ||
      scratch_bytes < carve(nullptr, n, capacity).total)
    return PF_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(scratch, 0, scratch_bytes, st);
  if (e != cudaSuccess) return (int)e;
  BinScratch s = carve(scratch, n, capacity);
  if (n > 0) {
    if (!zorder || !template_id || !tpl_base || !tpl_w || !tpl_h || !tpl_q || !tpl_hyp)
      return PF_ERR_ARG;
    e = cudaMemcpyAsync(s.zprim, zorder, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return (int)e;
    InfoArgs ia{template_id, zorder, n, n_tpl, tpl_base, tpl_pbase, tpl_w, tpl_h, tpl_q, tpl_hyp,
                s.pinfo};
    k_pinfo<<<div_up(n, 256), 256, 0, st>>>(ia);
    e = cudaGetLastError();
  }
  return (int)e;
}

extern "C" int pf_preprocess(const double* params, int n, double alpha_max, double mu_blend,
                             double padding, int W, int H, int tile, int ty_begin, int ty_end,
                             int capacity, void* rec, void* scratch, size_t scratch_bytes,
                             void* slots, int slot_m, int32_t* tile_classes, void* stream) {
  pf::NvtxRange nvtx_range("pf_preprocess");
  PreArgs a;
  int rc = fill_pre_args(a, const_cast<double*>(params), n, alpha_max, mu_blend, padding,
                         W, H, tile, ty_begin, ty_end, capacity, rec, scratch, scratch_bytes);
  if (rc == PF_OK) rc = attach_slots(a, slots, slot_m, tile_classes, capacity);
  if (rc != PF_OK) return rc;
  return launch_prim(false, a, (cudaStream_t)stream);
}

extern "C" int pf_preprocess_sync(double* params, const double* src, int n, double alpha_max,
                                  double mu_blend, double padding, int W, int H, int tile,
                                  int ty_begin, int ty_end, int capacity, void* rec, void* scratch,
                                  size_t scratch_bytes, void* slots, int slot_m,
                                  int32_t* tile_classes, void* stream) {
  pf::NvtxRange nvtx_range("pf_preprocess_sync");
  if (n > 0 && !src) return PF_ERR_ARG;
  PreArgs a;
  int rc = fill_pre_args(a, params, n, alpha_max, mu_blend, padding, W, H, tile, ty_begin,
                         ty_end, capacity, rec, scratch, scratch_bytes);
  // (slot mode: only edited primitives are scattered again; the classes stand)
  if (rc == PF_OK) rc = attach_slots(a, slots, slot_m, tile_classes, capacity);
  if (rc != PF_OK) return rc;
  a.src = src;
  return launch_prim(false, a, (cudaStream_t)stream);
}

extern "C" int pf_adam_blocks(int n) {
  return div_up(n > 0 ? n * prim_lanes(n) : 1, kPrimThreads);
}

extern "C" int pf_adam_preprocess(double* params, double* grads, double* m, double* v,
                                  const uint8_t* frozen, const double* gains8,
                                  const double* lr_table, const double* bc1_table,
                                  const double* bc2_table, int clamp, double s_min, double s_max,
                                  const double* sums, const double* part, int n_part,
                                  double* hist_part, double* last_part, int n, double alpha_max,
                                  double mu_blend,
                                  double padding, int W, int H, int tile, int ty_begin,
                                  int ty_end, int capacity, void* rec, void* scratch,
                                  size_t scratch_bytes, double* mirror, void* slots, int slot_m,
                                  int32_t* tile_classes, void* stream) {
  pf::NvtxRange nvtx_range("pf_adam_preprocess");
  PreArgs a;
  // rec == NULL: Adam only (no records / rects; the caller runs pf_preprocess
  // before the next pf_bin, e.g. a host-driven step that re-reads the parameters)
  static char dummy_rec[16];
  const int rc = fill_pre_args(a, params, n, alpha_max, mu_blend, padding, W, H, tile, ty_begin,
                               ty_end, capacity, rec ? rec : dummy_rec, scratch, scratch_bytes);
  if (rc != PF_OK) return rc;
  a.records = rec != nullptr;
  a.mirror = mirror;
  if (const int rs = attach_slots(a, slots, slot_m, tile_classes, capacity)) return rs;
  if (!lr_table || !bc1_table || !bc2_table || (n > 0 && (!grads || !m || !v)))
    return PF_ERR_ARG;
  if (part && n_part < 0) return PF_ERR_ARG;
  AdamPart& d = a.ad;
  d.grads = grads;
  d.m = m;
  d.v = v;
  d.frozen = frozen;
  for (int c = 0; c < 8; ++c) d.gains[c] = gains8 ? gains8[c] : 1.0;
  d.lr_table = lr_table;
  d.bc1_table = bc1_table;
  d.bc2_table = bc2_table;
  d.clamp = clamp;
  d.s_min = s_min;
  d.s_max = s_max;
  d.sums = sums;
  d.part = part;
  d.n_part = part ? n_part : 0;
  d.hist_part = hist_part;
  d.last_part = last_part;
  return launch_prim(true, a, (cudaStream_t)stream);
}

static int sms_count() { return dev_attrs().sms; }

static int row_blocks(int n, int n_rows, int ntx, bool cache) {
  // column blocks per row: as many as fit in one wave (1024-thread blocks, one
  // per SM with the register cache), >= 16 columns each
  int ncb = (cache ? 1 : 2) * sms_count() / n_rows;
  if (diag().bin_ncb >= 0) ncb = diag().bin_ncb;  // diagnostics (A/B)
  return max(1, min(ncb, ntx / 16));
}

// Two-level path when re-reading every rect per (row, column block) is the
// cost: n x rows x column blocks above ~2M (c5 4K / 20k), or forced by
// PF_BIN_TWO_LEVEL=0/1 (A/B and tests).
static bool bin_two_level(int n, int n_rows, int ncb, size_t scat_smem) {
  bool two = (size_t)n * (size_t)n_rows * (size_t)ncb > 2000000u;
  if (diag().bin_two_level >= 0) two = diag().bin_two_level != 0;
  return two && n > 0 && n_rows <= kMaxRows2 && scat_smem <= 200 * 1024;
}

static size_t scatter_smem(int n_rows) {
  return sizeof(int) * (kRowChunk / 32 + 1) * (size_t)n_rows + sizeof(int2) * kRowChunk;
}

extern "C" int pf_bin_launches(int n, int W, int H, int tile, int ty_begin, int ty_end) {
  int ntx, n_rows;
  if (n < 0 || !band_ok(W, H, tile, ty_begin, ty_end, &ntx, &n_rows)) return -1;
  if (n_rows == 0) return 0;
  const bool cache = (n + kRowThreads - 1) / kRowThreads <= kRowCache;
  const int ncb = row_blocks(n, n_rows, ntx, cache);
  return bin_two_level(n, n_rows, ncb, scatter_smem(n_rows)) ? 4 : 1;
}

extern "C" int pf_bin(int n, int W, int H, int tile, int ty_begin, int ty_end, int capacity,
                      void* scratch, size_t scratch_bytes, int32_t* bin_off, int32_t* bin_idx,
                      int32_t* status, int32_t* tile_classes, void* stream) {
  pf::NvtxRange nvtx_range("pf_bin");
  int ntx, n_rows;
  if (n < 0 || capacity < 0 || !band_ok(W, H, tile, ty_begin, ty_end, &ntx, &n_rows))
    return PF_ERR_ARG;
  if (!bin_off || !status || (capacity > 0 && !bin_idx)) return PF_ERR_ARG;
  if (!scratch || scratch_bytes < pf_bin_scratch_bytes(n, n_rows * ntx, capacity))
    return PF_ERR_SCRATCH;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_rows == 0) {
    cudaError_t e = cudaMemsetAsync(bin_off, 0, sizeof(int32_t), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(status, 0, 2 * sizeof(int32_t), st);
    return (int)e;
  }
  RowArgs ra;
  ra.n = n;
  ra.ntx = ntx;
  ra.ty_begin = ty_begin;
  ra.n_rows = n_rows;
  ra.cap = capacity;
  ra.smem_list = kRowSmemList;
  ra.s = carve(scratch, n, capacity, n_rows * ntx);
  ra.bin_off = bin_off;
  ra.bin_idx = bin_idx;
  ra.status = status;
  ra.classes = tile_classes;
  ra.n_tiles = n_rows * ntx;
  ra.prebuilt = 0;
  ra.tl = pf_timeline_ptr();
  const size_t smem = sizeof(int2) * kRowSmemList + 3 * sizeof(int) * (size_t)ntx;
  const bool cache = (n + kRowThreads - 1) / kRowThreads <= kRowCache;
  void (*kern)(RowArgs) = cache ? k_bin_rows<true> : k_bin_rows<false>;
  // (always: the kernel's static shared memory plus 48 KB dynamic exceeds the
  // default per-block limit, so the opt-in attribute is needed at any size)
  if (const cudaError_t e = ensure_dyn_smem((const void*)kern, smem > 48 * 1024 ? smem : 48 * 1024))
    return (int)e;
  int ncb = row_blocks(n, n_rows, ntx, cache);
  const size_t scat_smem = scatter_smem(n_rows);
  if (bin_two_level(n, n_rows, ncb, scat_smem)) {
    if (const cudaError_t e = ensure_dyn_smem((const void*)k_row_scatter,
                                              scat_smem > 48 * 1024 ? scat_smem : 48 * 1024))
      return (int)e;
    const int chunks = div_up(n, kRowChunk);
    int e = (int)launch_pdl2(k_row_counts, dim3(chunks), kRowChunk, sizeof(int2) * n_rows, st, ra);
    if (e == 0) e = (int)launch_pdl2(k_row_offsets, dim3(div_up(n_rows, 4)), 128, 0, st, ra, chunks);
    if (e == 0) e = (int)launch_pdl2(k_row_scatter, dim3(chunks), kRowChunk, scat_smem, st, ra);
    if (e != 0) return e;
    ra.prebuilt = 1;
    // no rect re-reads left to spread: one wave of column blocks
    ncb = max(1, min(sms_count() / n_rows, ntx / 16));
  }
  return (int)launch_pdl2(kern, dim3(n_rows, ncb), kRowThreads, smem, st, ra);
}

extern "C" int pf_atlas_quad(const double* tex, int texels, const int32_t* tpl_base,
                             const int32_t* tpl_w, const int32_t* tpl_h, int n_tpl, float* quad,
                             void* stream) {
  if (texels < 0 || n_tpl < 0 || (texels > 0 && (!tex || !tpl_base || !tpl_w || !tpl_h || !quad)))
    return PF_ERR_ARG;
  if (texels == 0) return PF_OK;
  QuadArgs a{tex, texels, n_tpl, tpl_base, tpl_w, tpl_h, reinterpret_cast<float4*>(quad)};
  k_atlas_quad<<<div_up(texels, 256), 256, 0, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}

extern "C" int pf_atlas_pad(const double* tex, int texels, const int32_t* tpl_base,
                            const int32_t* tpl_pbase, const int32_t* tpl_w, const int32_t* tpl_h,
                            int n_tpl, int pad_texels, float* apad, void* stream) {
  if (texels < 0 || n_tpl < 0 || pad_texels < 0 ||
      (pad_texels > 0 && (!tex || !tpl_base || !tpl_pbase || !tpl_w || !tpl_h || !apad)))
    return PF_ERR_ARG;
  if (pad_texels == 0 || n_tpl == 0) return PF_OK;
  PadArgs a{tex, texels, n_tpl, pad_texels, tpl_base, tpl_pbase, tpl_w, tpl_h, apad};
  k_atlas_pad<<<div_up(pad_texels, 256), 256, 0, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}
