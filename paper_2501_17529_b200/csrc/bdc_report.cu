// bdc_report.cu -- the winner's sparse report and FP64 metric (k_rsel, k_rsweep,
// k_rmerge), and the flow probe used by the parity tests (k_probe).
//
// k_report re-evaluates the winning candidate only, in FP64 (metric_first's
// second pass, PAPER step "recompute p_n0/p_n1 for t_i^*", solver.py:652-713):
//   * the FP64 metric max(N-0, every feasible case, penalty)   (agg_m, solver.py:235-252)
//   * N-0 top-kg over reportable monitored rows               (_top_rows, :287-299)
//   * per case stable top-kc, merged by (-rel, case, position) (_merge_entries, :302-318)
// One CTA per task; each warp owns a strided subset of the cases and keeps
// its own top-kg list; a case entry below the warp's current kg-th loading
// cannot reach the final report, so it is skipped (the same exact pruning the
// reference's bound-stop implements, solver.py:686-695).
#include "bdc_device.cuh"

#include <algorithm>
#include <climits>
#include <cstdlib>

namespace bdc {

namespace {

constexpr int RT = 256;
constexpr int RW = RT / 32;
static_assert(RW == RSEL_WARPS, "k_rsel writes one partial list per warp");

__device__ __forceinline__ bool better(double r1, int p1, double r2, int p2) {
  return r1 > r2 || (r1 == r2 && p1 < p2);
}
__device__ __forceinline__ bool better3(double r1, int c1, int p1, double r2, int c2, int p2) {
  return r1 > r2 || (r1 == r2 && (c1 < c2 || (c1 == c2 && p1 < p2)));
}

// max of two loadings (>= 0): one compare and select, where fmax also handles NaN operands
// (the running value never is one; a NaN loading is dropped by both)
__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }

template <int KC>
struct LaneTop {
  double rel[KC], flow[KC];
  int pos[KC];
  __device__ void clear() {
#pragma unroll
    for (int i = 0; i < KC; ++i) { rel[i] = -1.0; flow[i] = 0.0; pos[i] = INT_MAX; }
  }
  __device__ void insert(double r, int p, double f) {
    if (!better(r, p, rel[KC - 1], pos[KC - 1])) return;
    // branch-free insertion (static register indices): entries the new one beats
    // move down one slot, the first one it does not beat keeps it below
    bool placed = false;
#pragma unroll
    for (int i = KC - 1; i > 0; --i) {
      const bool up = better(r, p, rel[i - 1], pos[i - 1]);
      const bool put = !up && !placed;
      rel[i] = up ? rel[i - 1] : (put ? r : rel[i]);
      pos[i] = up ? pos[i - 1] : (put ? p : pos[i]);
      flow[i] = up ? flow[i - 1] : (put ? f : flow[i]);
      placed |= put;
    }
    if (!placed) { rel[0] = r; pos[0] = p; flow[0] = f; }
  }
  __device__ void pop() {
#pragma unroll
    for (int i = 0; i < KC - 1; ++i) { rel[i] = rel[i + 1]; pos[i] = pos[i + 1]; flow[i] = flow[i + 1]; }
    rel[KC - 1] = -1.0; pos[KC - 1] = INT_MAX; flow[KC - 1] = 0.0;
  }
};

struct WarpList {
  double rel[KMAX], flow[KMAX];
  int cs[KMAX], pos[KMAX];
  int n;
};

// lane 0 only
__device__ void wl_insert(WarpList& L, int kg, double r, int c, int p, double f) {
  if (L.n == kg && !better3(r, c, p, L.rel[kg - 1], L.cs[kg - 1], L.pos[kg - 1])) return;
  int i = L.n < kg ? L.n : kg - 1;
  while (i > 0 && better3(r, c, p, L.rel[i - 1], L.cs[i - 1], L.pos[i - 1])) {
    L.rel[i] = L.rel[i - 1]; L.cs[i] = L.cs[i - 1]; L.pos[i] = L.pos[i - 1]; L.flow[i] = L.flow[i - 1];
    --i;
  }
  L.rel[i] = r; L.cs[i] = c; L.pos[i] = p; L.flow[i] = f;
  if (L.n < kg) ++L.n;
}

__device__ __forceinline__ double warp_thresh(const volatile WarpList& L, int kg) {
  return L.n == kg ? L.rel[kg - 1] : -1.0;
}

// Merge the lanes' lists into the warp list: up to kc rounds of warp argmax,
// stopping as soon as the best remaining head cannot enter the warp's top-kg.
template <int KC>
__device__ void warp_merge(LaneTop<KC>& lt, int kc, WarpList& L, int kg, int case_order) {
  const int lane = threadIdx.x & 31;
  for (int round = 0; round < kc; ++round) {
    const double th = warp_thresh(L, kg);
    if (!__any_sync(0xffffffffu, lt.rel[0] >= 0.0 && lt.rel[0] >= th)) break;
    double r = lt.rel[0];
    int p = lt.pos[0], src = lane;
    for (int o = 16; o; o >>= 1) {
      const double orr = __shfl_xor_sync(0xffffffffu, r, o);
      const int op = __shfl_xor_sync(0xffffffffu, p, o);
      const int os = __shfl_xor_sync(0xffffffffu, src, o);
      if (better(orr, op, r, p)) { r = orr; p = op; src = os; }
    }
    const double f = __shfl_sync(0xffffffffu, lt.flow[0], src);
    if (lane == src) lt.pop();
    if (lane == 0) wl_insert(L, kg, r, case_order, p, f);
    __syncwarp();
  }
}


// Top-kg of this warp's strided subset {i = wid*32 + lane + k*RT, i < n} by
// (value desc, index asc), kg rounds of warp argmax (no block barriers); value(i) < 0
// excludes i.  Lane 0 writes the picks to ov/oi; returns their number.
template <class F>
__device__ int warp_topk(int n, int kg, F value, double* ov, int* oi) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double pv = 1e300;
  int pi = -1, cnt = 0;
  for (int r = 0; r < kg; ++r) {
    double bv = -1.0;
    int bi = INT_MAX;
    for (int i = wid * 32 + lane; i < n; i += RT) {
      const double v = value(i);
      if (v < 0.0 || !(v < pv || (v == pv && i > pi))) continue;
      if (better(v, i, bv, bi)) { bv = v; bi = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov2, oi2, bv, bi)) { bv = ov2; bi = oi2; }
    }
    if (bv < 0.0) break;
    if (lane == 0) { ov[r] = bv; oi[r] = bi; }
    pv = bv; pi = bi;
    ++cnt;
  }
  return cnt;
}

// Merge RW warp lists (lv/li rows of stride KMAX, counts ln) into the top-kg by
// (value desc, index asc); one warp, kg rounds.  Lane 0 writes ov/oi; returns count.
__device__ int warp_merge_lists(const double (*lv)[KMAX], const int (*li)[KMAX], const int* ln, int kg,
                                double* ov, int* oi) {
  const int lane = threadIdx.x & 31;
  double pv = 1e300;
  int pi = -1, cnt = 0;
  for (int r = 0; r < kg; ++r) {
    double bv = -1.0;
    int bi = INT_MAX;
    for (int e = lane; e < RW * KMAX; e += 32) {
      const int wq = e / KMAX, k = e % KMAX;
      if (k >= ln[wq]) continue;
      const double v = lv[wq][k];
      const int i = li[wq][k];
      if (!(v < pv || (v == pv && i > pi))) continue;
      if (better(v, i, bv, bi)) { bv = v; bi = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov2, oi2, bv, bi)) { bv = ov2; bi = oi2; }
    }
    if (bv < 0.0) break;
    if (lane == 0) { ov[r] = bv; oi[r] = bi; }
    pv = bv; pi = bi;
    ++cnt;
  }
  return cnt;
}

// Was the (single case c, candidate t) pair evaluated by the N-1 stage, i.e. is
// cmax[c][t] its exact FP32 maximum?  TOP cases and live cases were evaluated for every
// candidate (bdc_single.cu); the others are dominated.
__device__ __forceinline__ bool pair_evaluated(const DevGrid& g, const Work& w, int b, int c, int t) {
  (void)t;
  if (!w.ranked && c < w.ptop) return true;
  return g.N1 > w.ptop && w.done[(size_t)b * g.N1 + c] != 0;
}

// The dominance bound of a skipped pair: max_b (m0_b(t) + scale_bc |s(c,t)|).
__device__ __forceinline__ float pair_bound(const DevGrid& g, const Work& w, int b, int c, int t) {
  const float as = fabsf(s_at(g, w, b, c, t));
  float ub = 0.f;
#pragma unroll
  for (int blk = 0; blk < SB; ++blk)
    ub = fmaxf(ub, w.m0b[((size_t)b * SB + blk) * w.T + t] + w.scale[((size_t)b * SB + blk) * g.N1 + c] * as);
  return ub;
}

// FP64 post-contingency flows, one expression each, shared by the winner report and the
// FP64 re-score (k_rescore) so that both see the same bits.
// Single-branch case: F = n0 + (D''(r, c) / den_c) n0(r_c), and exactly n0 - n0(r_c) = 0 on
// the outaged row itself (the LODF self factor -1, solver.py:498-503, 612-613).
__device__ __forceinline__ double single_flow(double nv, double dv, double idn, double sc, bool own) {
  return own ? fma(-1.0, sc, nv) : fma(dv * idn, sc, nv);
}
// Multi-branch case (st, m): F = n0 + sum_j MODF(row, j) n0(r_j) with MODF = D''[:, O] inner^-1
// (compute_modf / apply_modf_to_ptdf, factors.py:373-425; _case_flows, solver.py:614-618);
// the outaged rows get the -e_j row (flow exactly 0).  own = which outaged branch `row` is.
__device__ __forceinline__ double multi_flow(const DevGrid& g, const Work& w, int b, int st, int m, int row,
                                             double n0r, const double* sv, const double* minv,
                                             const double* Bm, int rt, int& own) {
  const int R = g.R, rs = w.rs;
  own = -1;
  for (int a = 0; a < m; ++a) if (g.mb_row[st + a] == row) own = a;
  double f = n0r;
  if (own >= 0) {
    for (int j = 0; j < m; ++j) f = fma(j == own ? -1.0 : 0.0, sv[j], f);
  } else {
    double Dv[MMAX];
    for (int i = 0; i < m; ++i) {
      double v = g.Dm64[(size_t)(st + i) * R + row];
      const double* Wq = w.Wm + ((size_t)b * g.NMB + st + i) * rs;
      for (int j = 0; j < rt; ++j) v = fma(Bm[(size_t)j * R + row], Wq[j], v);
      Dv[i] = v;
    }
    for (int j = 0; j < m; ++j) {
      double l = 0.0;
      for (int i = 0; i < m; ++i) l = fma(Dv[i], minv[i * m + j], l);
      f = fma(l, sv[j], f);
    }
  }
  return f;
}
// Injection case: F = n0 - setpoint * P''[:, col_t] (solver.py:619-622), the column of the
// candidate's slot bit in rank-coefficient form.
__device__ __forceinline__ double inj_flow(const DevGrid& g, int ca, const double* coef, double sp, int row,
                                           double n0r, const double* Bm, int rt) {
  double pc = g.P0T[(size_t)ca * g.R + row];
  for (int j = 0; j < rt; ++j) pc = fma(Bm[(size_t)j * g.R + row], coef[j], pc);
  return fma(-pc, sp, n0r);
}

// One multi-branch or injection case q (q < NM: multi) of the winner, FP64, one warp:
// lanes over monitored rows keep stable top-kc lists (entries >= the list floor),
// merged into the warp list L with the case's order.  Updates the lane's running max.
template <int KC>
__device__ void other_case_report(const DevGrid& g, const Work& w, int b, int q, int best, float theta, int kc,
                                  int kg, WarpList& L, const double* n0b, const int* sdead, int nd,
                                  double* sMinv, double& mymax) {
  const int lane = threadIdx.x & 31;
  const int R = g.R, M = g.M, T = w.T, rs = w.rs, rt = w.rank[b];
  const double* Bm = w.Bm + (size_t)b * rs * R;
  int order, kind = 1;
  if (q < g.NM) {
    order = g.mc_order[q];
  } else {
    kind = 2; q -= g.NM;
    order = g.ic_order[q];
  }
  LaneTop<KC> lt;
  lt.clear();
  // entries below theta cannot reach the final top-kg (it holds the kg largest case
  // maxima, all >= theta): a floor for the lane lists
  const double thresh = fmax(warp_thresh(L, kg), (double)theta);
  if (kind == 1) {
    const int st = g.mc_start[q], m = g.mc_start[q + 1] - st;
    for (int i = lane; i < m * m; i += 32) sMinv[i] = w.minv[((size_t)b * g.NM + q) * MMAX * MMAX + i];
    __syncwarp();
    double sv[MMAX];
    for (int j = 0; j < m; ++j) sv[j] = n0b[g.mb_row[st + j]];
    for (int p = lane; p < M; p += 32) {
      const int row = g.mon_row[p];
      if (is_dead(sdead, nd, row)) continue;
      int own;
      const double f = multi_flow(g, w, b, st, m, row, n0b[row], sv, sMinv, Bm, rt, own);
      const double rel = fabs(f) * g.inv_rating[p];
      mymax = dmax(mymax, rel);
      if (own < 0 && rel >= thresh) lt.insert(rel, p, f);
    }
  } else {
    const int sl = g.ic_slot[q];
    const int ca = sl >= 0 ? g.slot_col[sl] : g.ic_col[q];
    const bool bit = sl >= 0 && w.inj[((size_t)b * T + best) * g.K + sl];
    const double* coef = (bit ? w.cib : w.cia) + ((size_t)b * g.NI + q) * rs;
    const double sp = g.ic_sp[q];
    for (int p = lane; p < M; p += 32) {
      const int row = g.mon_row[p];
      if (is_dead(sdead, nd, row)) continue;
      const double f = inj_flow(g, ca, coef, sp, row, n0b[row], Bm, rt);
      const double rel = fabs(f) * g.inv_rating[p];
      mymax = dmax(mymax, rel);
      if (rel >= thresh) lt.insert(rel, p, f);
    }
  }
  warp_merge<KC>(lt, kc, L, kg, order);
  __syncwarp();
}

}  // namespace

// ---------------------------------------------------------------------------- k_rsel
// Winner report, part 1 (one CTA per task): the winner's FP64 N-0 column and N-0
// top-kg; which contingencies can reach the report; the multi-branch / injection
// cases among them (few, FP64, one warp per case) into partial list 0.
//
// Exact pruning: an entry of case c can enter the final top-kg only if c's true max
// loading is >= the kg-th largest true case max.  FP32 maxima are within SCREEN_EPS
// of FP64, so with kth = the kg-th largest exact FP32 maximum, every case whose upper
// bound (exact FP32 max, or the dominance bound m0 + scale_c |s(c,t)| of a pair the
// sweep skipped) is >= kth - 2 eps is visited; the metric's binding case is one of them.
template <int KC>
__global__ void __launch_bounds__(RT, 3) k_rsel(DevGrid g, DevCfg cfg, Work w) {
  const int b = blockIdx.x;
  if (w.status[b] != 0) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int R = g.R, M = g.M, T = w.T, rs = w.rs, rt = w.rank[b];
  const int best = (int)w.best[b];
  const int kc = cfg.kc, kg = cfg.kg;
  double* n0b = w.n0b + (size_t)b * R;
  const double* Bm = w.Bm + (size_t)b * rs * R;
  __shared__ WarpList wl[RW];
  __shared__ int sdead[RMAX];
  __shared__ double sMinv[RW][MMAX * MMAX];
  __shared__ double sY[RMAX];
  __shared__ double lv[2][RW][KMAX];  // per-warp top lists: [0] N-0 rows, [1] case maxima
  __shared__ int li[2][RW][KMAX];
  __shared__ int ln[2][RW];
  __shared__ double mv[KMAX];
  __shared__ int mi[KMAX];
  __shared__ int wcnt[RW], woff[RW];
  __shared__ float sTheta;
  const int nd = w.ndead[b];
  if (tid < nd) sdead[tid] = w.dead[(size_t)b * RMAX + tid];
  if (tid < rt) sY[tid] = w.Y[((size_t)b * rs + tid) * T + best];
  if (lane == 0) wl[wid].n = 0;
  __syncthreads();
  // the winner's N-0 column, FP64, from the factors
  for (int r = tid; r < R; r += RT) {
    double v = 0.0;
    if (!is_dead(sdead, nd, r)) {
      v = g.f0[r];
      for (int j = 0; j < rt; ++j) v = fma(Bm[(size_t)j * R + r], sY[j], v);
    }
    n0b[r] = v;
    const int p = g.row_mon_pos[r];
    if (p >= 0) w.n0m[(size_t)b * M + p] = v;
  }
  __syncthreads();

  // ---- per-warp candidates: N-0 report rows and the largest exact case maxima -------------
  const int N1 = g.N1, ncase = N1 + g.NM + g.NI;
  const float* cm = w.cmax + (size_t)b * ncase * T + best;
  auto feasible_case = [&](int ci) -> bool {
    if (ci < N1) return w.sc_ok[(size_t)b * N1 + ci] != 0;
    if (ci < N1 + g.NM) return w.mc_ok[(size_t)b * g.NM + (ci - N1)] != 0;
    return true;
  };
  // exact FP32 maximum (>= 0), or -1 with the dominance bound in `ub`
  auto case_value = [&](int ci, float& ub) -> float {
    if (ci >= N1) {  // multi/injection: exact unless k_oscreen skipped it (cmax = bound)
      ub = cm[(size_t)ci * T];
      return other_exact(g, w, b, ci - N1) ? ub : -1.f;
    }
    if (pair_evaluated(g, w, b, ci, best)) {
      ub = cm[(size_t)ci * T];
      return ub;
    }
    ub = pair_bound(g, w, b, ci, best);
    return -1.f;
  };
  double mymax = 0.0;
  for (int p = tid; p < M; p += RT) mymax = dmax(mymax, fabs(n0b[g.mon_row[p]]) * g.inv_rating[p]);
  {
    const int n = warp_topk(M, kg, [&](int p) -> double {
      const int row = g.mon_row[p];
      return is_dead(sdead, nd, row) ? -1.0 : fabs(n0b[row]) * g.inv_rating[p];
    }, lv[0][wid], li[0][wid]);
    if (lane == 0) ln[0][wid] = n;
    const int n2 = warp_topk(ncase, kg, [&](int ci) -> double {
      if (!feasible_case(ci)) return -1.0;
      float ub;
      return (double)case_value(ci, ub);
    }, lv[1][wid], li[1][wid]);
    if (lane == 0) ln[1][wid] = n2;
  }
  __syncthreads();
  if (wid == 0) {
    // N-0 report: top-kg rows by (rel desc, position asc) (_top_rows, solver.py:287-299)
    const int n = warp_merge_lists(lv[0], li[0], ln[0], kg, mv, mi);
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      const int p = mi[i];
      const double f = n0b[g.mon_row[p]];
      w.n0pos[(size_t)b * kg + i] = p;
      w.n0flow[(size_t)b * kg + i] = f;
      w.n0rel[(size_t)b * kg + i] = fabs(f) / g.rating[p];  // np.abs(flows) / ratings
    }
    if (lane == 0) w.n0cnt[b] = n;
  } else if (wid == 1) {
    // Exact pruning: an entry of case c can enter the final top-kg only if c's true max
    // loading is >= the kg-th largest true case max.  FP32 maxima are within SCREEN_EPS
    // of FP64, so with kth = the kg-th largest exact FP32 maximum, every case whose upper
    // bound (exact FP32 max, or the dominance bound m0 + scale_c |s(c,t)| of a pair the
    // sweep skipped) is >= kth - 2 eps is visited; the metric's binding case is one of them.
    __shared__ double tv[KMAX];
    __shared__ int ti[KMAX];
    const int n = warp_merge_lists(lv[1], li[1], ln[1], kg, tv, ti);
    __syncwarp();
    if (lane == 0) sTheta = n == kg ? (float)tv[kg - 1] - 2.f * SCREEN_EPS : -1.f;
  }
  __syncthreads();
  const float theta = sTheta;
  if (tid == 0) w.theta[b] = theta;
  // single cases to visit, ascending: warp-contiguous segments, ordered compaction
  {
    const int seg = (N1 + RW - 1) / RW, s0 = wid * seg, s1 = min(N1, s0 + seg);
    int cnt = 0;
    for (int c0 = s0; c0 < s1; c0 += 32) {
      const int c = c0 + lane;
      bool take = false;
      if (c < s1 && feasible_case(c)) {
        float ub;
        case_value(c, ub);
        take = ub >= theta;
      }
      cnt += __popc(__ballot_sync(0xffffffffu, take));
    }
    if (lane == 0) wcnt[wid] = cnt;
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int i = 0; i < RW; ++i) { woff[i] = acc; acc += wcnt[i]; }
      w.rcnt[b] = acc;
      atomicAdd(w.lf + 3, (unsigned long long)acc);
    }
    __syncthreads();
    int* rl = w.rlist + (size_t)b * N1;
    int off = woff[wid];
    for (int c0 = s0; c0 < s1; c0 += 32) {
      const int c = c0 + lane;
      bool take = false;
      if (c < s1 && feasible_case(c)) {
        float ub;
        case_value(c, ub);
        take = ub >= theta;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      if (take) rl[off + __popc(bal & ((1u << lane) - 1u))] = c;
      off += __popc(bal);
    }
  }

  // ---- multi-branch and injection cases of the report (FP64, warp per case) --------------
  for (int ci = N1 + wid; ci < ncase; ci += RW) {
    if (!feasible_case(ci) || !(cm[(size_t)ci * T] >= theta)) continue;
    other_case_report<KC>(g, w, b, ci - N1, best, theta, kc, kg, wl[wid], n0b, sdead, nd, sMinv[wid], mymax);
  }
  // each warp's list and max is one partial slot (merged by k_rmerge)
  for (int o = 16; o; o >>= 1) mymax = fmax(mymax, __shfl_xor_sync(0xffffffffu, mymax, o));
  const size_t o = ((size_t)b * w.nslot + wid) * KMAX;
  for (int e = lane; e < kg; e += 32) {
    const bool has = e < wl[wid].n;
    w.pcase[o + e] = has ? wl[wid].cs[e] : INT_MAX;
    w.ppos[o + e] = has ? wl[wid].pos[e] : INT_MAX;
    w.pflow[o + e] = has ? wl[wid].flow[e] : 0.0;
    w.prel[o + e] = has ? wl[wid].rel[e] : -1.0;
  }
  if (lane == 0) w.pmax[(size_t)b * w.nslot + wid] = mymax;
}

// --------------------------------------------------------------------------- k_rsel_w
// k_rsel for small grids (M, cases <= 32 NCW): a warp per task, RW tasks per CTA, no
// block barriers.  The N-0 loadings and the case values live in registers; the N-0
// top-kg and the kg-th case value are kg rounds of warp argmax (same order as k_rsel:
// value desc, index asc); the warp's list is partial slot 0 (slots 1..RW-1 empty).
template <int KC, int NCW>
__global__ void __launch_bounds__(RT, 3) k_rsel_w(DevGrid g, DevCfg cfg, Work w) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int b = blockIdx.x * RW + wid;
  __shared__ WarpList wl[RW];
  __shared__ int sdead[RW][RMAX];
  __shared__ double sMinv[RW][MMAX * MMAX];
  __shared__ double sY[RW][RMAX];
  if (b >= w.Wb || w.status[b] != 0) return;  // warp-uniform; no block barrier below
  const int R = g.R, M = g.M, T = w.T, rs = w.rs, rt = w.rank[b];
  const int best = (int)w.best[b];
  const int kc = cfg.kc, kg = cfg.kg;
  const int N1 = g.N1, ncase = N1 + g.NM + g.NI;
  double* n0b = w.n0b + (size_t)b * R;
  double* n0m = w.n0m + (size_t)b * M;
  const double* Bm = w.Bm + (size_t)b * rs * R;
  const int nd = w.ndead[b];
  if (lane < nd) sdead[wid][lane] = w.dead[(size_t)b * RMAX + lane];
  if (lane < rt) sY[wid][lane] = w.Y[((size_t)b * rs + lane) * T + best];
  if (lane == 0) wl[wid].n = 0;
  __syncwarp();
  // the winner's N-0 column, FP64, from the factors
  for (int r = lane; r < R; r += 32) {
    double v = 0.0;
    if (!is_dead(sdead[wid], nd, r)) {
      v = g.f0[r];
      for (int j = 0; j < rt; ++j) v = fma(Bm[(size_t)j * R + r], sY[wid][j], v);
    }
    n0b[r] = v;
    const int p = g.row_mon_pos[r];
    if (p >= 0) n0m[p] = v;
  }
  __syncwarp();
  // N-0 loadings (dead rows excluded from the report, 0 in the metric)
  double nv[NCW];
  double mymax = 0.0;
#pragma unroll
  for (int k = 0; k < NCW; ++k) {
    const int p = lane + 32 * k;
    nv[k] = -1.0;
    if (p < M) {
      const double v = fabs(n0m[p]) * g.inv_rating[p];
      mymax = dmax(mymax, v);
      if (!is_dead(sdead[wid], nd, g.mon_row[p])) nv[k] = v;
    }
  }
  // N-0 report: top-kg by (rel desc, position asc) (_top_rows, solver.py:287-299)
  int cnt = 0;
  for (int e = 0; e < kg; ++e) {
    double bv = -1.0;
    int bi = INT_MAX;
#pragma unroll
    for (int k = 0; k < NCW; ++k)
      if (nv[k] >= 0.0 && better(nv[k], lane + 32 * k, bv, bi)) { bv = nv[k]; bi = lane + 32 * k; }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    if (bv < 0.0) break;
    if (lane == 0) {
      const double f = n0m[bi];
      w.n0pos[(size_t)b * kg + e] = bi;
      w.n0flow[(size_t)b * kg + e] = f;
      w.n0rel[(size_t)b * kg + e] = fabs(f) / g.rating[bi];
    }
#pragma unroll
    for (int k = 0; k < NCW; ++k)
      if (lane + 32 * k == bi) nv[k] = -1.0;
    ++cnt;
  }
  if (lane == 0) w.n0cnt[b] = cnt;
  // case values: exact FP32 maximum (or -1) and upper bound (exact, or the dominance bound)
  const float* cm = w.cmax + (size_t)b * ncase * T + best;
  float cv[NCW], cub[NCW];
#pragma unroll
  for (int k = 0; k < NCW; ++k) {
    const int ci = lane + 32 * k;
    cv[k] = -1.f;
    cub[k] = -1.f;
    if (ci >= ncase) continue;
    bool feas;
    if (ci < N1) feas = w.sc_ok[(size_t)b * N1 + ci] != 0;
    else if (ci < N1 + g.NM) feas = w.mc_ok[(size_t)b * g.NM + (ci - N1)] != 0;
    else feas = true;
    if (!feas) continue;
    if (ci >= N1) {  // multi/injection: exact unless k_oscreen skipped it (cmax = bound)
      cub[k] = cm[(size_t)ci * T];
      cv[k] = other_exact(g, w, b, ci - N1) ? cub[k] : -1.f;
    } else if (pair_evaluated(g, w, b, ci, best)) {
      cv[k] = cm[(size_t)ci * T];
      cub[k] = cv[k];
    } else {
      cub[k] = pair_bound(g, w, b, ci, best);
    }
  }
  // kg-th largest exact case value -> theta (k_rsel's exact pruning rule)
  float kth = -1.f;
  int nfound = 0;
  {
    float sel[NCW];
#pragma unroll
    for (int k = 0; k < NCW; ++k) sel[k] = cv[k];
    for (int e = 0; e < kg; ++e) {
      float bv = -1.f;
      int bi = INT_MAX;
#pragma unroll
      for (int k = 0; k < NCW; ++k)
        if (sel[k] >= 0.f && (sel[k] > bv || (sel[k] == bv && lane + 32 * k < bi))) { bv = sel[k]; bi = lane + 32 * k; }
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (bv < 0.f) break;
#pragma unroll
      for (int k = 0; k < NCW; ++k)
        if (lane + 32 * k == bi) sel[k] = -1.f;
      kth = bv;
      ++nfound;
    }
  }
  const float theta = nfound == kg ? kth - 2.f * SCREEN_EPS : -1.f;
  if (lane == 0) w.theta[b] = theta;
  // single cases to visit, ascending (cases lane + 32 k: k-major order is ascending)
  int off = 0;
#pragma unroll
  for (int k = 0; k < NCW; ++k) {
    const int ci = lane + 32 * k;
    const bool take = ci < N1 && cub[k] >= theta && cub[k] >= 0.f;
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (take) w.rlist[(size_t)b * N1 + off + __popc(bal & ((1u << lane) - 1u))] = ci;
    off += __popc(bal);
  }
  if (lane == 0) {
    w.rcnt[b] = off;
    atomicAdd(w.lf + 3, (unsigned long long)off);
  }
  // multi-branch and injection cases (FP64)
  for (int ci = N1; ci < ncase; ++ci) {
    bool feas = ci < N1 + g.NM ? w.mc_ok[(size_t)b * g.NM + (ci - N1)] != 0 : true;
    if (!feas || !(cm[(size_t)ci * T] >= theta)) continue;
    other_case_report<KC>(g, w, b, ci - N1, best, theta, kc, kg, wl[wid], n0b, sdead[wid], nd, sMinv[wid], mymax);
  }
  for (int o = 16; o; o >>= 1) mymax = fmax(mymax, __shfl_xor_sync(0xffffffffu, mymax, o));
  // slot 0: this warp's list and max; slots 1..RW-1 empty
  for (int sl = 0; sl < RSEL_WARPS; ++sl) {
    const size_t o = ((size_t)b * w.nslot + sl) * KMAX;
    for (int e = lane; e < kg; e += 32) {
      const bool has = sl == 0 && e < wl[wid].n;
      w.pcase[o + e] = has ? wl[wid].cs[e] : INT_MAX;
      w.ppos[o + e] = has ? wl[wid].pos[e] : INT_MAX;
      w.pflow[o + e] = has ? wl[wid].flow[e] : 0.0;
      w.prel[o + e] = has ? wl[wid].rel[e] : -1.0;
    }
    if (lane == 0) w.pmax[(size_t)b * w.nslot + sl] = sl == 0 ? mymax : 0.0;
  }
}

// --------------------------------------------------------------------------- k_rsweep
// Winner report, part 2: the listed single cases in FP64 for the winning candidate, RCW
// cases per CTA in groups of RW (a warp per case, lanes over monitored rows).  The rows
// stream in chunks of SRC through a cp.async double buffer holding the task's B'' rows,
// N-0 column and 1/rating for the chunk -- shared by the group's RW cases -- while each
// warp reads its case's D_base column (coalesced).  Each lane keeps its rows' stable
// top-kc (rel desc, position asc; solver.py:287-299), merged per case into the warp's
// top-kg by (rel desc, case order, position) (_merge_entries, solver.py:302-318); the
// CTA merges its warps' lists into one partial slot.
// NTH threads per CTA: 256, or 128 on one-chunk grids (smaller footprint, twice the tasks
// in flight per SM: the one-chunk sweep is latency-bound per task).
template <int KC, int CQ, int RPL, int NTH>  // CQ: cases per warp evaluated together; RPL: rows per lane
__global__ void __launch_bounds__(NTH, NTH == 128 ? 8 : (CQ == 1 ? 4 : 3)) k_rsweep(DevGrid g, DevCfg cfg, Work w) {
  constexpr int RT = NTH, RW = NTH / 32;
  constexpr int SRC = 32 * RPL;  // monitored rows per chunk
  const int b = blockIdx.y, tile = blockIdx.x;
  if (w.status[b] != 0) return;
  const int n = w.rcnt[b];
  const int RC = w.rcw;
  if (tile * RC >= n) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int M = g.M, N1 = g.N1, rs = w.rs, rt = w.rank[b], kc = cfg.kc, kg = cfg.kg;
  const int base = tile * RC, ncs = min(n, base + RC) - base;
  // one chunk (small grids): a single staging buffer and no per-case lists (each case
  // merges straight into its warp's list) -- see rsweep_dyn_bytes
  const bool one1 = M <= SRC;
  const int nbf = one1 ? 1 : 2, kcl = one1 ? 0 : KC;
  extern __shared__ __align__(16) double rsm[];
  double* sB = rsm;                    // [nbf][rt][SRC] B'' on the chunk's monitored rows
  double* sN = sB + nbf * rs * SRC;    // [nbf][SRC] N-0 column
  double* sI = sN + nbf * SRC;         // [nbf][SRC] 1 / rating
  double* sWc = sI + nbf * SRC;        // [RC][rs] the cases' W rows
  double* cRel = sWc + RC * rs;        // [RC][KC] each case's running top-kc (multi-chunk)
  double* cFlow = cRel + RC * kcl;
  double* sIdn = cFlow + RC * kcl;     // [RC] 1 / den
  double* sSc = sIdn + RC;             // [RC] N-0 flow of the outaged row
  int* cPos = (int*)(sSc + RC);        // [RC][KC] (multi-chunk)
  int* sC = cPos + RC * kcl;           // [RC] case index
  int* sOwn = sC + RC;                 // [RC] monitored position of the outaged row
  int* cN = sOwn + RC;                 // [RC] entries in the case's list
  __shared__ WarpList wl[RW];
  __shared__ double wmax[RW];
  __shared__ int sdeadp[RMAX];  // monitored positions of the disconnected rows (-1: unmonitored)
  const int nd = w.ndead[b];
  if (tid < nd) sdeadp[tid] = g.row_mon_pos[w.dead[(size_t)b * RMAX + tid]];
  if (lane == 0) wl[wid].n = 0;
  for (int i = tid; i < RC; i += RT) {
    const int c = i < ncs ? w.rlist[(size_t)b * N1 + base + i] : -1;
    sC[i] = c;
    cN[i] = 0;
    if (c >= 0) {
      const int rowc = g.sc_row[c];
      sOwn[i] = g.row_mon_pos[rowc];
      sIdn[i] = 1.0 / w.den[(size_t)b * N1 + c];
      sSc[i] = w.n0b[(size_t)b * g.R + rowc];
    } else {
      sOwn[i] = -1; sIdn[i] = 0.0; sSc[i] = 0.0;
    }
  }
  for (int idx = tid; idx < ncs * rt; idx += RT) {
    const int i = idx / rt, j = idx - i * rt;
    const int c = w.rlist[(size_t)b * N1 + base + i];
    sWc[i * rs + j] = w.Wsc[((size_t)b * N1 + c) * rs + j];
  }
  const double* n0m = w.n0m + (size_t)b * M;
  const double* Bmon = w.Bmon + (size_t)b * rs * M;
  const double floor_rel = (double)w.theta[b];  // entries below theta are never reported
  double mymax = 0.0;
  LaneTop<KC> lt;
  auto issue = [&](int m0, int bf) {
    for (int idx = tid; idx < rt * SRC; idx += RT) {
      const int j = idx / SRC, r = idx % SRC, m = m0 + r;
      cp8(&sB[(bf * rs + j) * SRC + r], m < M ? &Bmon[(size_t)j * M + m] : Bmon, m < M);
    }
    for (int r = tid; r < SRC; r += RT) {
      const int m = m0 + r;
      cp8(&sN[bf * SRC + r], m < M ? &n0m[m] : n0m, m < M);
      cp8(&sI[bf * SRC + r], m < M ? &g.inv_rating[m] : g.inv_rating, m < M);
    }
    cp_commit();
  };
  // chunk-outer, case-inner: the staged B'' chunk serves all RC cases of the tile; each
  // warp evaluates CQ of its cases at once (the B'' loads shared by the CQ columns) and
  // folds each case's chunk top-kc into the case's running list
  const int nchunks = (M + SRC - 1) / SRC;
  // one chunk (small grids): every case completes in one pass, so its lanes' lists merge
  // straight into the warp's top-kg (and the warp's kg-th entry prunes the next cases)
  const bool one = nchunks == 1;
  issue(0, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int bf = ch & 1, m0 = ch * SRC;
    if (ch + 1 < nchunks) {
      issue(m0 + SRC, bf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    unsigned skip = 0;  // rows past M or disconnected (flow exactly 0)
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int p = m0 + lane + 32 * u;
      if (p >= M || is_dead(sdeadp, nd, p)) skip |= 1u << u;
    }
    const double* cB = sB + bf * rs * SRC + lane;
    const double* cNv = sN + bf * SRC + lane;  // this lane's rows: N-0 flow, 1 / rating
    const double* cIv = sI + bf * SRC + lane;
    for (int i0 = wid * CQ; i0 < ncs; i0 += RW * CQ) {
      double dv[CQ][RPL];
#pragma unroll
      for (int q = 0; q < CQ; ++q) {
        const int c = sC[i0 + q];
        const double* Dc = g.DM64 + (size_t)(c >= 0 ? c : 0) * M;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int p = m0 + lane + 32 * u;
          dv[q][u] = p < M ? __ldg(&Dc[p]) : 0.0;
        }
      }
      const double* W0 = sWc + i0 * rs;
      for (int j = 0; j < rt; ++j) {
        double bv[RPL];
#pragma unroll
        for (int u = 0; u < RPL; ++u) bv[u] = cB[j * SRC + 32 * u];
#pragma unroll
        for (int q = 0; q < CQ; ++q) {
          const double wj = W0[q * rs + j];
#pragma unroll
          for (int u = 0; u < RPL; ++u) dv[q][u] = fma(bv[u], wj, dv[q][u]);
        }
      }
#pragma unroll
      for (int q = 0; q < CQ; ++q) {
        const int i = i0 + q;
        if (sC[i] < 0) continue;
        const int ownp = sOwn[i];
        const double idn = sIdn[i], sc = sSc[i];
        const double thresh = one ? fmax(floor_rel, warp_thresh(wl[wid], kg))
                                  : fmax(floor_rel, cN[i] == kc ? cRel[i * KC + kc - 1] : -1.0);
        lt.clear();
        // the outaged row (flow exactly 0: never reported, 0 in the metric) joins the
        // skipped rows, so the row loop is single_flow's regular branch only
        unsigned skq = skip;
        {
          const int ou = ownp - m0 - lane;
          if (ownp >= 0 && ou >= 0 && (ou & 31) == 0 && (ou >> 5) < RPL) skq |= 1u << (ou >> 5);
        }
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          if (skq & (1u << u)) continue;
          const double f = fma(dv[q][u] * idn, sc, cNv[32 * u]);  // single_flow, not the own row
          const double rel = fabs(f) * cIv[32 * u];
          mymax = dmax(mymax, rel);
          if (rel >= thresh) lt.insert(rel, m0 + lane + 32 * u, f);
        }
        if (!__any_sync(0xffffffffu, lt.rel[0] >= 0.0)) continue;
        if (one) {
          warp_merge<KC>(lt, kc, wl[wid], kg, g.sc_order[sC[i]]);
          __syncwarp();
          continue;
        }
        // fold: the case's list joins lane 0's, then kc rounds of warp argmax rewrite it
        if (lane == 0)
          for (int e = 0; e < cN[i]; ++e) lt.insert(cRel[i * KC + e], cPos[i * KC + e], cFlow[i * KC + e]);
        __syncwarp();
        int cnt = 0;
        for (; cnt < kc; ++cnt) {
          double r = lt.rel[0];
          int p = lt.pos[0], src = lane;
          for (int o = 16; o; o >>= 1) {
            const double orr = __shfl_xor_sync(0xffffffffu, r, o);
            const int op = __shfl_xor_sync(0xffffffffu, p, o);
            const int os = __shfl_xor_sync(0xffffffffu, src, o);
            if (better(orr, op, r, p)) { r = orr; p = op; src = os; }
          }
          if (r < 0.0) break;
          const double f = __shfl_sync(0xffffffffu, lt.flow[0], src);
          if (lane == src) lt.pop();
          if (lane == 0) { cRel[i * KC + cnt] = r; cPos[i * KC + cnt] = p; cFlow[i * KC + cnt] = f; }
        }
        if (lane == 0) cN[i] = cnt;
        __syncwarp();
      }
    }
    __syncthreads();
  }
  // each warp merges its cases' lists into its top-kg by (rel desc, case order, position)
  for (int i0 = wid * CQ; i0 < ncs; i0 += RW * CQ) {
    for (int q = 0; q < CQ; ++q) {
      const int i = i0 + q, c = sC[i];
      if (c < 0 || cN[i] == 0) continue;
      lt.clear();
      if (lane == 0)
        for (int e = 0; e < cN[i]; ++e) lt.insert(cRel[i * KC + e], cPos[i * KC + e], cFlow[i * KC + e]);
      warp_merge<KC>(lt, kc, wl[wid], kg, g.sc_order[c]);
    }
  }
  __syncwarp();
  for (int o = 16; o; o >>= 1) mymax = fmax(mymax, __shfl_xor_sync(0xffffffffu, mymax, o));
  if (lane == 0) wmax[wid] = mymax;
  __syncthreads();
  if (wid != 0) return;
  // warp 0: the CTA's partial top-kg, kg rounds of argmax over the RW sorted warp lists
  const int slot = RSEL_WARPS + tile;
  const size_t o = ((size_t)b * w.nslot + slot) * KMAX;
  double mx = lane < RW ? wmax[lane] : 0.0;
  for (int k = 16; k; k >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, k));
  if (lane == 0) w.pmax[(size_t)b * w.nslot + slot] = mx;
  int hd = 0;  // lane l < RW: next entry of warp list l
  for (int e = 0; e < kg; ++e) {
    double r = -1.0;
    int ord = INT_MAX, p = INT_MAX, src = lane;
    if (lane < RW && hd < wl[lane].n) { r = wl[lane].rel[hd]; ord = wl[lane].cs[hd]; p = wl[lane].pos[hd]; }
    for (int k = 16; k; k >>= 1) {
      const double orr = __shfl_xor_sync(0xffffffffu, r, k);
      const int oo = __shfl_xor_sync(0xffffffffu, ord, k);
      const int op = __shfl_xor_sync(0xffffffffu, p, k);
      const int os = __shfl_xor_sync(0xffffffffu, src, k);
      if (better3(orr, oo, op, r, ord, p) || (orr == r && oo == ord && op == p && os < src)) {
        r = orr; ord = oo; p = op; src = os;
      }
    }
    if (lane == src && r >= 0.0) {
      w.prel[o + e] = r; w.pcase[o + e] = ord; w.ppos[o + e] = p; w.pflow[o + e] = wl[lane].flow[hd];
      ++hd;
    }
    if (r < 0.0) {
      for (int e2 = e + lane; e2 < kg; e2 += 32) {
        w.prel[o + e2] = -1.0; w.pcase[o + e2] = INT_MAX; w.ppos[o + e2] = INT_MAX;
      }
      break;
    }
    __syncwarp();
  }
}

// --------------------------------------------------------------------------- k_rmerge
// Winner report, part 3 (one warp per task): the final top-kg over the partial lists
// and the FP64 metric max(N-0, every feasible case, penalty) (agg_m, solver.py:235-252).
__global__ void k_rmerge(DevGrid g, DevCfg cfg, Work w) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = gt >> 5, lane = gt & 31;
  if (b >= w.Wb || w.status[b] != 0) return;
  const int kg = cfg.kg;
  const int nsl = RSEL_WARPS + (w.rcnt[b] + w.rcw - 1) / w.rcw;
  double mx = 0.0;
  for (int s = lane; s < nsl; s += 32) mx = fmax(mx, w.pmax[(size_t)b * w.nslot + s]);
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const size_t base = (size_t)b * w.nslot * KMAX;
  const int ne = nsl * KMAX;
  double pr = 1e300;
  int pc = -1, pp = -1, cnt = 0;
  for (int e = 0; e < kg; ++e) {
    double br = -1.0;
    int bc = INT_MAX, bp = INT_MAX, bi = -1;
    for (int i = lane; i < ne; i += 32) {
      if ((i % KMAX) >= kg) continue;
      const double r = w.prel[base + i];
      if (r < 0.0) continue;
      const int c = w.pcase[base + i], p = w.ppos[base + i];
      // strictly after the previous pick in (rel desc, case, pos) order
      if (!better3(pr, pc, pp, r, c, p)) continue;
      if (better3(r, c, p, br, bc, bp)) { br = r; bc = c; bp = p; bi = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const double orr = __shfl_xor_sync(0xffffffffu, br, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better3(orr, oc, op, br, bc, bp)) { br = orr; bc = oc; bp = op; bi = oi; }
    }
    if (br < 0.0) break;
    if (lane == 0) {
      w.n1case[(size_t)b * kg + e] = bc;
      w.n1pos[(size_t)b * kg + e] = bp;
      w.n1flow[(size_t)b * kg + e] = w.pflow[base + bi];
      w.n1rel[(size_t)b * kg + e] = fabs(w.pflow[base + bi]) / g.rating[bp];  // true division, as agg_i
    }
    pr = br; pc = bc; pp = bp;
    ++cnt;
  }
  if (lane == 0) {
    if (w.nisl[b] > 0) mx = fmax(mx, cfg.penalty);
    w.metric[b] = mx;
    w.n1cnt[b] = cnt;
  }
}

// -------------------------------------------------------------------------- k_rescore
// FP64 re-score of the winner's near-tie band (solver.py:804-823: best = the first argmin
// of the FP64 metrics).  k_select took the first FP32 argmin (value vmin) and queued the
// tasks with more than one candidate within 2E of it, E = RESCORE_EPS max(1, vmin) bounding
// |m32 - m64|: the FP64 argmin is one of them.  A CTA per queued task walks the band in
// ascending candidate order, up to RCH members per pass, with the running FP64 minimum
// best64 of the earlier passes:
//   * a candidate with v(t) - E >= best64 cannot beat it (m64 >= v - E);
//   * with islanded cases, one with m32 + E < penalty has m64 = penalty exactly, the
//     smallest possible metric, so no later candidate can win and the walk ends with it;
//   * every other member is re-evaluated in FP64 through the winner report's flow
//     expressions (the same bits as k_rsel / k_rsweep), so the metric reported for the
//     chosen candidate is the very value it was chosen by.
// The flows of N-0, single- and multi-branch cases depend on the candidate only through
// its rank coefficients y_t (n0 = f0 + B'' y_t, solver.py:575-595), an injection case's
// additionally through its own slot bit (solver.py:619-622, 642-649).  Members are grouped
// by bitwise-equal y_t (classes).  Every element that can reach th = vmin - 2E for some
// class is found by ONE pass at the first class's y0: an N-0 or single-case flow moves by
// at most |B''(r,:)| dy (+ |L(r,c)| |B''(r_c,:)| dy) between classes, dy_j = max over the
// pass's classes |y_j - y0_j|, so elements with |F(y0)|/rating + that bound below th - E
// can never be a class maximum that matters (m64 >= vmin - E).  Each class is then
// evaluated on that short "hot" list only (a warp per class), with the same per-element
// expression, so its maximum is the exact FP64 value whenever it is >= th.  Multi-branch
// cases and injection cases (per slot-bit value) are evaluated in full when their FP32
// maximum reaches th.  Single cases are pre-filtered per task by their screening key
// (bkey_c >= every pair bound of case c).  A hot list that overflows falls back to the
// full per-class evaluation (warp_class_max).
namespace {
constexpr int RREL = 512;   // single cases listed per task (more: full per-class evaluation)
constexpr int RHOT = 256;   // hot (case, row) elements per pass

// N-0 flow of `row` for rank coefficients y (the k_rsel expression; 0 on disconnected rows)
__device__ __forceinline__ double n0_at(const DevGrid& g, const double* Bm, const double* y, int rt,
                                        const int* sdead, int nd, int row) {
  if (is_dead(sdead, nd, row)) return 0.0;
  double v = g.f0[row];
  for (int j = 0; j < rt; ++j) v = fma(Bm[(size_t)j * g.R + row], y[j], v);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long h, unsigned long long v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  return h * 0xff51afd7ed558ccdull;
}

__device__ __forceinline__ unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }

// Per-task inputs of a class evaluation
struct RsTask {
  int b, rt, nd, T;
  float th;
  const double *Bm, *Bmon;
  const float* cm;
  const uint32_t* key;
  const int *sdead, *sdeadp;
};

// FP64 |F|/rating of one element for coefficients y: c < 0 the N-0 flow at monitored
// position p, else single case c at p (the expressions of warp_class_max, element by element)
__device__ __forceinline__ double elem_value(const DevGrid& g, const Work& w, const RsTask& k, const double* y,
                                             int c, int p) {
  const int M = g.M, rt = k.rt;
  double nv = g.f0[g.mon_row[p]];
  if (c < 0) {
    for (int j = 0; j < rt; ++j) nv = fma(k.Bmon[(size_t)j * M + p], y[j], nv);
    return fabs(nv) * g.inv_rating[p];
  }
  const int rowc = g.sc_row[c], ownp = g.row_mon_pos[rowc];
  const double idn = 1.0 / w.den[(size_t)k.b * g.N1 + c];
  const double sc = n0_at(g, k.Bm, y, rt, k.sdead, k.nd, rowc);
  const double* Wc = w.Wsc + ((size_t)k.b * g.N1 + c) * w.rs;
  double dv = g.DM64[(size_t)c * M + p];
  for (int j = 0; j < rt; ++j) {
    const double bj = k.Bmon[(size_t)j * M + p];
    nv = fma(bj, y[j], nv);
    dv = fma(bj, Wc[j], dv);
  }
  return fabs(single_flow(nv, dv, idn, sc, p == ownp)) * g.inv_rating[p];
}

// FP64 max over the multi-branch cases whose FP32 maximum for candidate t reaches th (one
// warp); `mask` (q < 32) lists them when the caller has tested them already
__device__ double warp_multi_max(const DevGrid& g, const Work& w, const RsTask& k, int t, const double* y,
                                 double* sMinv, unsigned mask = 0xffffffffu) {
  const int lane = threadIdx.x & 31;
  const int M = g.M, N1 = g.N1, NM = g.NM, rt = k.rt, nd = k.nd, b = k.b;
  double mx = 0.0;
  for (int q = 0; q < NM; ++q) {
    if (q < 32 && !((mask >> q) & 1u)) continue;
    if (!w.mc_ok[(size_t)b * NM + q] || !(k.cm[(size_t)(N1 + q) * k.T + t] >= k.th)) continue;
    const int st = g.mc_start[q], m = g.mc_start[q + 1] - st;
    for (int e = lane; e < m * m; e += 32) sMinv[e] = w.minv[((size_t)b * NM + q) * MMAX * MMAX + e];
    __syncwarp();
    double sv[MMAX];
    for (int j = 0; j < m; ++j) sv[j] = n0_at(g, k.Bm, y, rt, k.sdead, nd, g.mb_row[st + j]);
    for (int p = lane; p < M; p += 32) {
      const int row = g.mon_row[p];
      if (is_dead(k.sdead, nd, row)) continue;
      int own;
      const double f = multi_flow(g, w, b, st, m, row, n0_at(g, k.Bm, y, rt, k.sdead, nd, row), sv, sMinv, k.Bm, rt, own);
      mx = dmax(mx, fabs(f) * g.inv_rating[p]);
    }
    __syncwarp();
  }
  return warp_max(mx);
}

// FP64 max over N-0 and the relevant single / multi-branch cases for coefficients y (one
// warp, every monitored row; candidate t is any member of the class).  Single cases come
// from rel[0..nrel) or, with rel_all, from every case with a screening key >= th.
__device__ double warp_class_max(const DevGrid& g, const Work& w, const RsTask& k, int t, const double* y,
                                 const int* rel, int nrel, bool rel_all, double* sMinv) {
  const int lane = threadIdx.x & 31;
  const int M = g.M, N1 = g.N1, nd = k.nd, b = k.b, T = k.T;
  double mx = 0.0;
  for (int p = lane; p < M; p += 32)
    if (!is_dead(k.sdeadp, nd, p)) mx = dmax(mx, elem_value(g, w, k, y, -1, p));
  const int ncand = rel_all ? N1 : nrel;
  for (int k0 = 0; k0 < ncand; k0 += 32) {
    const int kk = k0 + lane;
    bool take = false;
    int c = 0;
    if (kk < ncand) {
      c = rel_all ? kk : rel[kk];
      if (!rel_all || (w.sc_ok[(size_t)b * N1 + c] && (!w.ranked || __uint_as_float(k.key[c]) >= k.th))) {
        const float ub = pair_evaluated(g, w, b, c, t) ? k.cm[(size_t)c * T + t] : pair_bound(g, w, b, c, t);
        take = ub >= k.th;
      }
    }
    unsigned todo = __ballot_sync(0xffffffffu, take);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const int cc = __shfl_sync(0xffffffffu, c, src);
      for (int p = lane; p < M; p += 32)
        if (!is_dead(k.sdeadp, nd, p)) mx = dmax(mx, elem_value(g, w, k, y, cc, p));
    }
  }
  return fmax(warp_max(mx), warp_multi_max(g, w, k, t, y, sMinv));
}

// FP64 max |F|/rating of injection case q with slot bit `bit` for coefficients y (one warp)
__device__ double warp_inj_max(const DevGrid& g, const Work& w, const RsTask& k, int q, bool bit, const double* y) {
  const int lane = threadIdx.x & 31;
  const int sl = g.ic_slot[q];
  const int ca = sl >= 0 ? g.slot_col[sl] : g.ic_col[q];
  const double* coef = (bit ? w.cib : w.cia) + ((size_t)k.b * g.NI + q) * w.rs;
  const double sp = g.ic_sp[q];
  double iv = 0.0;
  for (int p = lane; p < g.M; p += 32) {
    const int row = g.mon_row[p];
    if (is_dead(k.sdead, k.nd, row)) continue;
    const double f = inj_flow(g, ca, coef, sp, row, n0_at(g, k.Bm, y, k.rt, k.sdead, k.nd, row), k.Bm, k.rt);
    iv = dmax(iv, fabs(f) * g.inv_rating[p]);
  }
  return warp_max(iv);
}
}  // namespace

template <int NT>
__global__ void __launch_bounds__(NT, NT == 64 ? 12 : 3) k_rescore(DevGrid g, DevCfg cfg, Work w) {
  constexpr int NW = NT / 32;
  constexpr int RCH = NT == 64 ? 128 : 256;  // band members per pass
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __shared__ int sdead[RMAX], sdeadp[RMAX];
  __shared__ double sYw[NW][RMAX];            // the warp's class coefficients y_t
  __shared__ double sMinv[NW][MMAX * MMAX];
  __shared__ int sRel[RREL];                  // single cases with bkey >= th
  __shared__ int sRel2[RREL];                 // ... that reach th for some class of the pass
  __shared__ int sMem[RCH];                   // this pass's members (candidates, ascending)
  __shared__ int sCls[RCH];                   // index of the member's class representative
  __shared__ int sReps[RCH];                  // class representatives
  __shared__ unsigned char sKnown[RCH];       // m64 known without evaluation (= penalty)
  __shared__ unsigned long long sHash[RCH];   // hash of the member's y_t bits
  __shared__ unsigned long long sM64[RCH];    // FP64 metric bits (non-negative: ordered as integers)
  __shared__ unsigned sNeedI[RCH], sBitI[RCH];  // injection cases a member needs / its slot bits
  __shared__ unsigned sNeedM[RCH];              // multi-branch cases a member needs
  __shared__ double sY0[RMAX];                // y of the pass's reference class
  __shared__ unsigned long long sDy[RMAX];    // max over the pass's classes |y_j - y0_j|
  __shared__ int sHotC[RHOT], sHotP[RHOT];    // hot elements (case or -1 for N-0, monitored pos)
  __shared__ int sCnt[NW];
  __shared__ double sRed[NW];
  __shared__ int sRi[NW];
  __shared__ int sN, sEnd, sNext, sNRel, sNRel2, sNCls, sNHot, sI0;
  const int M = g.M, N1 = g.N1, NM = g.NM, NI = g.NI, T = w.T, rs = w.rs;
  const unsigned nq = *w.rsq_n;
  const bool full_env = w.rescore_full != 0;
  for (unsigned qi = blockIdx.x; qi < nq; qi += gridDim.x) {
    const int b = w.rsq[qi];
    const int rt = w.rank[b], nd = w.ndead[b];
    const int tn = w.tcount ? w.tcount[b] : T;
    const bool pen = w.nisl[b] > 0;
    const float penf = (float)cfg.penalty;
    const float* m32 = reinterpret_cast<const float*>(w.m32) + (size_t)b * T;
    const int t32 = (int)w.best[b];
    auto vof = [&](int t) -> float {
      const float v = m32[t];
      return pen ? fmaxf(v, penf) : v;
    };
    const float vmin = vof(t32);
    const float E = RESCORE_EPS * fmaxf(1.f, vmin);
    const float hi = vmin + 2.f * E;
    const float th = vmin - 2.f * E;  // case relevance: m64(t) >= v(t) - E >= vmin - E
    const double hot_th = (double)th - (double)E;
    const double* Bm = w.Bm + (size_t)b * rs * g.R;
    const double* Bmon = w.Bmon + (size_t)b * rs * M;
    const double* Y = w.Y + (size_t)b * rs * T;
    const uint8_t* inj = w.inj + (size_t)b * T * g.K;
    const float* cm = w.cmax + (size_t)b * (N1 + NM + NI) * T;
    const uint32_t* key = w.bkey + (size_t)b * N1;
    __syncthreads();  // the previous task's shared state is consumed
    if (tid < nd) {
      const int row = w.dead[(size_t)b * RMAX + tid];
      sdead[tid] = row;
      sdeadp[tid] = g.row_mon_pos[row];
    }
    if (tid == 0) sNRel = 0;
    __syncthreads();
    // single cases that can reach th for some candidate (bkey_c bounds every pair of c)
    for (int c0 = 0; w.ranked && c0 < N1; c0 += NT) {
      const int c = c0 + tid;
      const bool take = c < N1 && w.sc_ok[(size_t)b * N1 + c] && __uint_as_float(key[c]) >= th;
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      if (bal && lane == 0) sCnt[wid] = atomicAdd(&sNRel, __popc(bal));
      __syncwarp();
      const int base = __shfl_sync(0xffffffffu, sCnt[wid], 0);
      const int k = base + __popc(bal & ((1u << lane) - 1u));
      if (take && k < RREL) sRel[k] = c;
      __syncwarp();
    }
    __syncthreads();
    // too many, or no screening keys (screen off / every case in the TOP tile): full
    // per-class evaluation over every case
    const bool rel_all = !w.ranked || sNRel > RREL;
    const int nrel = rel_all ? N1 : sNRel;
    const RsTask tk{b, rt, nd, T, th, Bm, Bmon, cm, key, sdead, sdeadp};
    double best64 = __longlong_as_double(0x7ff0000000000000ll);
    int bestt = t32;
    unsigned long long nres = 0;
    int t0 = 0;
    bool stop = false;
    while (t0 < tn && !stop) {
      // ---- gather this pass's members, ascending (ballot compaction per NT candidates)
      if (tid == 0) { sN = 0; sEnd = 0; sNext = tn; }
      __syncthreads();
      for (int tb = t0; tb < tn; tb += NT) {
        const int n = sN;
        if (sEnd || n > RCH - NT) {
          if (tid == 0 && !sEnd) sNext = tb;
          break;
        }
        const int tt = tb + tid;
        bool inb = false, known = false;
        if (tt < tn) {
          const float v = vof(tt);
          inb = v <= hi && (double)v - (double)E < best64;
          known = inb && pen && (double)m32[tt] + (double)E < cfg.penalty;
        }
        // members past the first candidate with m64 = penalty cannot win
        const unsigned kb = __ballot_sync(0xffffffffu, known);
        if (lane == 0) sCnt[wid] = kb ? wid * 32 + __ffs(kb) - 1 : INT_MAX;
        __syncthreads();
        int firstk = INT_MAX;
        for (int i = 0; i < NW; ++i) firstk = min(firstk, sCnt[i]);
        __syncthreads();
        if (tid > firstk) inb = false;
        const unsigned bal = __ballot_sync(0xffffffffu, inb);
        if (lane == 0) sCnt[wid] = __popc(bal);
        __syncthreads();
        int off = n, cnt = 0;
        for (int i = 0; i < NW; ++i) {
          off += i < wid ? sCnt[i] : 0;
          cnt += sCnt[i];
        }
        if (inb) {
          const int k = off + __popc(bal & ((1u << lane) - 1u));
          sMem[k] = tt;
          sKnown[k] = known;
        }
        __syncthreads();
        if (tid == 0) {
          sN = n + cnt;
          if (firstk != INT_MAX) { sEnd = 1; sNext = tn; }
        }
        __syncthreads();
      }
      __syncthreads();
      const int n = sN;
      t0 = sNext;
      stop = sEnd;
      __syncthreads();  // sN / sNext / sEnd are read before the next pass resets them
      if (n == 0) continue;
      // ---- classes of bitwise-equal y_t
      for (int i = tid; i < n; i += NT) {
        unsigned long long h = 0x243f6a8885a308d3ull;
        const int t = sMem[i];
        for (int j = 0; j < rt; ++j) h = mix64(h, dbits(Y[(size_t)j * T + t]));
        sHash[i] = sKnown[i] ? 0ull : (h | 1ull);
        sM64[i] = sKnown[i] ? dbits(cfg.penalty) : 0ull;
        // injection cases whose FP32 maximum for t reaches th, and t's slot bit of each
        unsigned need = 0u, bits = 0u;
        for (int q = 0; q < NI && !sKnown[i]; ++q) {
          const int sl = g.ic_slot[q];
          const bool bit = sl >= 0 && inj[(size_t)t * g.K + sl];
          if (cm[(size_t)(N1 + NM + q) * T + t] >= th) need |= q < 32 ? 1u << q : 0u;
          bits |= (bit && q < 32) ? 1u << q : 0u;
        }
        sNeedI[i] = NI > 32 ? 0xffffffffu : need;
        sBitI[i] = bits;
        unsigned mneed = NM > 32 ? 0xffffffffu : 0u;  // multi-branch cases reaching th (y only)
        for (int q = 0; q < NM && q < 32 && !sKnown[i]; ++q)
          if (w.mc_ok[(size_t)b * NM + q] && cm[(size_t)(N1 + q) * T + t] >= th) mneed |= 1u << q;
        sNeedM[i] = mneed;
      }
      if (tid == 0) { sNCls = 0; sNHot = 0; sNRel2 = 0; sI0 = INT_MAX; }
      if (tid < RMAX) sDy[tid] = 0ull;
      __syncthreads();
      for (int i = tid; i < n; i += NT) {
        int rep = i;
        if (!sKnown[i]) {
          const int t = sMem[i];
          for (int k = 0; k < i; ++k) {
            if (sHash[k] != sHash[i]) continue;
            const int u = sMem[k];
            bool same = true;
            for (int j = 0; j < rt && same; ++j) same = dbits(Y[(size_t)j * T + t]) == dbits(Y[(size_t)j * T + u]);
            if (same) { rep = k; break; }
          }
          if (rep == i) {
            sReps[atomicAdd(&sNCls, 1)] = i;
            atomicMin(&sI0, i);
          }
        }
        sCls[i] = sKnown[i] ? -1 : rep;
      }
      __syncthreads();
      const int ncls = sNCls;
      nres += ncls;
      bool hot_ok = false;
      if (ncls > 0 && !rel_all && !full_env) {
        // ---- the hot elements, from one pass at the first class's y0
        const int tr = sMem[sI0];
        if (tid < rt) sY0[tid] = Y[(size_t)tid * T + tr];
        __syncthreads();
        for (int e = tid; e < ncls * rt; e += NT) {
          const int j = e % rt, t = sMem[sReps[e / rt]];
          atomicMax(&sDy[j], dbits(fabs(Y[(size_t)j * T + t] - sY0[j])));
        }
        for (int kk = tid; kk < nrel; kk += NT) sRel2[kk] = 0;
        __syncthreads();
        // single cases some class of the pass can take to th
        for (int e = tid; e < nrel * ncls; e += NT) {
          const int kk = e / ncls, c = sRel[kk], t = sMem[sReps[e % ncls]];
          const float ub = pair_evaluated(g, w, b, c, t) ? cm[(size_t)c * T + t] : pair_bound(g, w, b, c, t);
          if (ub >= th) sRel2[kk] = -1 - c;  // marked (any writer)
        }
        __syncthreads();
        if (tid == 0) {
          int m = 0;
          for (int kk = 0; kk < nrel; ++kk)
            if (sRel2[kk] < 0 && sRel2[kk] == -1 - sRel[kk]) sRel2[m++] = sRel[kk];
          sNRel2 = m;
        }
        __syncthreads();
        const double* dy = reinterpret_cast<const double*>(sDy);
        // N-0 rows
        for (int p = tid; p < M; p += NT) {
          if (is_dead(sdeadp, nd, p)) continue;
          double mv = 0.0;
          for (int j = 0; j < rt; ++j) mv = fma(fabs(Bmon[(size_t)j * M + p]), dy[j], mv);
          const double v = elem_value(g, w, tk, sY0, -1, p);
          if (v + (mv * g.inv_rating[p]) * (1.0 + 1e-9) >= hot_th) {
            const int h = atomicAdd(&sNHot, 1);
            if (h < RHOT) { sHotC[h] = -1; sHotP[h] = p; }
          }
        }
        // single cases: (case, row) pairs over the whole CTA (few cases, long rows on
        // large grids; many cases, short rows on small ones)
        const int nr2 = sNRel2;
        for (int e = tid; e < nr2 * M; e += NT) {
          const int kk = e / M, p = e - kk * M;
          const int c = sRel2[kk];
          const int rowc = g.sc_row[c], ownp = g.row_mon_pos[rowc];
          const double idn = 1.0 / w.den[(size_t)b * N1 + c];
          double ms = 0.0;  // bound of the move of n0(r_c)
          if (!is_dead(sdead, nd, rowc))
            for (int j = 0; j < rt; ++j) ms = fma(fabs(Bm[(size_t)j * g.R + rowc]), dy[j], ms);
          const double* Wc = w.Wsc + ((size_t)b * N1 + c) * rs;
          {
            if (is_dead(sdeadp, nd, p) || p == ownp) continue;  // the own row's flow is exactly 0
            double mv = 0.0, dv = g.DM64[(size_t)c * M + p];
            for (int j = 0; j < rt; ++j) {
              const double bj = Bmon[(size_t)j * M + p];
              mv = fma(fabs(bj), dy[j], mv);
              dv = fma(bj, Wc[j], dv);
            }
            mv = fma(fabs(dv * idn), ms, mv);
            const double v = elem_value(g, w, tk, sY0, c, p);
            if (v + (mv * g.inv_rating[p]) * (1.0 + 1e-9) >= hot_th) {
              const int h = atomicAdd(&sNHot, 1);
              if (h < RHOT) { sHotC[h] = c; sHotP[h] = p; }
            }
          }
        }
        __syncthreads();
        hot_ok = sNHot <= RHOT;
      }
      // ---- evaluate each class once, a warp per class
      const int nhot = sNHot;
      for (int ci = wid; ci < ncls; ci += NW) {
        const int i = sReps[ci], t = sMem[i];
        double* y = sYw[wid];
        if (lane < rt) y[lane] = Y[(size_t)lane * T + t];
        __syncwarp();
        double mx;
        if (hot_ok) {
          mx = 0.0;
          for (int h = lane; h < nhot; h += 32) mx = dmax(mx, elem_value(g, w, tk, y, sHotC[h], sHotP[h]));
          mx = warp_max(mx);
          if (sNeedM[i]) mx = fmax(mx, warp_multi_max(g, w, tk, t, y, sMinv[wid], sNeedM[i]));
        } else {
          mx = warp_class_max(g, w, tk, t, y, sRel, nrel, rel_all, sMinv[wid]);
        }
        const unsigned long long ab = dbits(mx);
        for (int k = lane; k < n; k += 32)
          if (sCls[k] == i) atomicMax(&sM64[k], ab);
        // injection cases, once per slot-bit value some member of the class needs
        unsigned need1 = 0u, need0 = 0u;  // (q, bit) pairs the class's members need
        for (int k = lane; k < n; k += 32) {
          if (sCls[k] != i) continue;
          need1 |= sNeedI[k] & sBitI[k];
          need0 |= sNeedI[k] & ~sBitI[k];
        }
        for (int o = 16; o; o >>= 1) {
          need1 |= __shfl_xor_sync(0xffffffffu, need1, o);
          need0 |= __shfl_xor_sync(0xffffffffu, need0, o);
        }
        for (int pr = 0; (need0 | need1) && pr < 2 * NI; ++pr) {
          const int q = pr >> 1;
          const bool bit = pr & 1;
          if (q < 32 && !(((bit ? need1 : need0) >> q) & 1u)) continue;
          const int sl = g.ic_slot[q];
          if (sl < 0 && bit) continue;  // a fixed column: no bit dependence
          bool need = false;
          for (int k = lane; k < n; k += 32) {
            if (sCls[k] != i) continue;
            const int u = sMem[k];
            const bool ub = sl >= 0 && inj[(size_t)u * g.K + sl];
            need |= ub == bit && cm[(size_t)(N1 + NM + q) * T + u] >= th;
          }
          if (!__any_sync(0xffffffffu, need)) continue;
          const unsigned long long vb = dbits(warp_inj_max(g, w, tk, q, bit, y));
          for (int k = lane; k < n; k += 32) {
            if (sCls[k] != i) continue;
            const bool ub = sl >= 0 && inj[(size_t)sMem[k] * g.K + sl];
            if (ub == bit) atomicMax(&sM64[k], vb);
          }
        }
        __syncwarp();
      }
      __syncthreads();
      // ---- the pass's first FP64 argmin (penalty floor), then the running minimum
      double bv = __longlong_as_double(0x7ff0000000000000ll);
      int bi = INT_MAX;
      for (int k = tid; k < n; k += NT) {
        double v = __longlong_as_double((long long)sM64[k]);
        if (pen) v = fmax(v, cfg.penalty);
        if (v < bv) { bv = v; bi = k; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { sRed[wid] = bv; sRi[wid] = bi; }
      __syncthreads();
      bv = sRed[0];
      bi = sRi[0];
      for (int k = 1; k < NW; ++k)
        if (sRed[k] < bv || (sRed[k] == bv && sRi[k] < bi)) { bv = sRed[k]; bi = sRi[k]; }
      if (bv < best64) {
        best64 = bv;
        bestt = sMem[bi];
      }
      if (pen && best64 == cfg.penalty) stop = true;
      __syncthreads();  // sMem / sCls / sM64 are rewritten by the next pass
    }
    if (tid == 0) {
      w.best[b] = bestt;
      atomicAdd(w.lf + 4, nres);
      if (bestt != t32) atomicAdd(w.lf + 5, 1ull);
    }
  }
}

// ------------------------------------------------------------------------------ probe
// Every flow of one task (b = 0) in FP64: n0 (R,T) and n1 (NC,R,T) in contingency
// order, NaN for islanded cases (candidate_case_flows, solver.py:919-958).
__global__ void k_probe(DevGrid g, Work w, double* n0o, double* n1o, uint8_t* ok) {
  const int ci = blockIdx.y;  // local case index over N1, NM, NI; ci == ncase -> N-0
  const int ncase = g.N1 + g.NM + g.NI;
  const int R = g.R, T = w.T, rs = w.rs, rt = w.rank[0];
  const double* Bm = w.Bm;
  const int nd = w.ndead[0];
  const int* dead = w.dead;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < (long long)R * T;
       idx += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(idx / T), t = (int)(idx % T);
    const double n0v = n0_at(g, w, 0, row, t, rt, dead, nd);
    if (ci == ncase) { n0o[idx] = n0v; continue; }
    const bool drow = is_dead(dead, nd, row);
    int order;
    double f = nan;
    if (ci < g.N1) {
      order = g.sc_order[ci];
      if (w.sc_ok[ci]) {
        const int rowc = g.sc_row[ci];
        const double sc = n0_at(g, w, 0, rowc, t, rt, dead, nd);
        if (drow) f = 0.0;
        else if (row == rowc) f = n0v - sc;
        else {
          double dv = g.D64[(size_t)ci * R + row];
          for (int j = 0; j < rt; ++j) dv = fma(Bm[(size_t)j * R + row], w.Wsc[(size_t)ci * rs + j], dv);
          f = n0v + (dv / w.den[ci]) * sc;
        }
      }
    } else if (ci < g.N1 + g.NM) {
      const int q = ci - g.N1;
      order = g.mc_order[q];
      if (w.mc_ok[q]) {
        const int st = g.mc_start[q], m = g.mc_start[q + 1] - st;
        if (drow) f = 0.0;
        else {
          int own = -1;
          for (int a = 0; a < m; ++a) if (g.mb_row[st + a] == row) own = a;
          f = n0v;
          for (int j = 0; j < m; ++j) {
            double l = 0.0;
            if (own >= 0) l = (j == own) ? -1.0 : 0.0;
            else
              for (int i = 0; i < m; ++i) {
                double v = g.Dm64[(size_t)(st + i) * R + row];
                for (int jj = 0; jj < rt; ++jj) v = fma(Bm[(size_t)jj * R + row], w.Wm[(size_t)(st + i) * rs + jj], v);
                l += v * w.minv[(size_t)q * MMAX * MMAX + i * m + j];
              }
            f += l * n0_at(g, w, 0, g.mb_row[st + j], t, rt, dead, nd);
          }
        }
      }
    } else {
      const int q = ci - g.N1 - g.NM;
      order = g.ic_order[q];
      const int sl = g.ic_slot[q];
      const int ca = sl >= 0 ? g.slot_col[sl] : g.ic_col[q];
      const bool bit = sl >= 0 && w.inj[(size_t)t * g.K + sl];
      const double* coef = (bit ? w.cib : w.cia) + (size_t)q * rs;
      double pc = g.P0T[(size_t)ca * R + row];
      for (int j = 0; j < rt; ++j) pc = fma(Bm[(size_t)j * R + row], coef[j], pc);
      f = drow ? 0.0 : n0v - pc * g.ic_sp[q];
    }
    n1o[((size_t)order * R + row) * T + t] = f;
    if (idx == 0) ok[order] = (f == f);
  }
}

namespace {
size_t rsweep_dyn_bytes(int rs, int kc, int src, int rcw, int M) {
  const size_t nbf = M <= src ? 1 : 2, kcl = M <= src ? 0 : kc;
  return (nbf * rs * src + 2 * nbf * src + (size_t)rcw * rs + 2 * (size_t)rcw * kcl + 2 * rcw) * sizeof(double) +
         ((size_t)rcw * kcl + 3 * rcw) * sizeof(int);
}
template <int KC>
void launch_report_t(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  const int nc = g.N1 + g.NM + g.NI;
  launch_oexact(g, w, s);  // exact winner maxima of the screened-out multi/injection cases
  if (!w.rsel_cta && g.M <= 32 * 8 && nc <= 32 * 8)
    k_rsel_w<KC, 8><<<(w.Wb + RW - 1) / RW, RT, 0, s>>>(g, c, w);
  else if (!w.rsel_cta && g.M <= 32 * 16 && nc <= 32 * 16)
    k_rsel_w<KC, 16><<<(w.Wb + RW - 1) / RW, RT, 0, s>>>(g, c, w);
  else
    k_rsel<KC><<<w.Wb, RT, 0, s>>>(g, c, w);
  if (g.N1 > 0 && g.M > 0) {
    // one case per warp at a time, a single row chunk where M <= 192; on large grids four
    // cases per warp (their B'' loads shared) -- the test hook BDC_RSWEEP_CQ forces either
    const char* cq_env = getenv("BDC_RSWEEP_CQ");
    const int cq = cq_env ? atoi(cq_env) : (g.M <= 2048 ? 1 : 4);
    const int rpl = cq == 1 && g.M <= 64 ? 2 : cq == 1 && g.M > 128 && g.M <= 192 ? 6 : 4;
    const size_t dyn = rsweep_dyn_bytes(w.rs, KC, 32 * rpl, w.rcw, g.M);
    const dim3 grid((g.N1 + w.rcw - 1) / w.rcw, w.Wb);
    // one-chunk grids: 128-thread CTAs (test hook BDC_RSWEEP_NT=256 keeps 256)
    const char* nt_env = getenv("BDC_RSWEEP_NT");
    const bool small = g.M <= 32 * rpl && cq == 1 && !(nt_env && atoi(nt_env) == 256);
    auto go = [&](auto kern, int nth) {
      smem_opt_in((const void*)kern, (int)dyn);
      kern<<<grid, nth, dyn, s>>>(g, c, w);
    };
    if (cq != 1) go(k_rsweep<KC, 4, 4, 256>, 256);
    else if (rpl == 2) small ? go(k_rsweep<KC, 1, 2, 128>, 128) : go(k_rsweep<KC, 1, 2, 256>, 256);
    else if (rpl == 6) small ? go(k_rsweep<KC, 1, 6, 128>, 128) : go(k_rsweep<KC, 1, 6, 256>, 256);
    else small ? go(k_rsweep<KC, 1, 4, 128>, 128) : go(k_rsweep<KC, 1, 4, 256>, 256);
  }
  const long long threads = (long long)w.Wb * 32;
  k_rmerge<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(g, c, w);
}
}  // namespace

void launch_report(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  if (c.kc <= 5) launch_report_t<5>(g, c, w, s);
  else if (c.kc <= 8) launch_report_t<8>(g, c, w, s);
  else if (c.kc <= 16) launch_report_t<16>(g, c, w, s);
  else launch_report_t<32>(g, c, w, s);
}

void launch_rescore(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  // persistent CTAs over the device-side queue k_select filled: two warps per task on small
  // grids (a few classes, short rows), eight on large ones
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // tests: force a CTA size (BDC_RESCORE_NT) or the full per-class evaluation instead of
  // the hot elements (BDC_RESCORE_FULL=1); both must give bit-identical winners
  const char* nt_env = getenv("BDC_RESCORE_NT");
  const char* full_env = getenv("BDC_RESCORE_FULL");
  Work wr = w;
  wr.rescore_full = full_env && full_env[0] == '1';
  const int nt = nt_env ? atoi(nt_env) : (g.M <= 512 ? 64 : 256);
  if (nt == 64) {
    k_rescore<64><<<std::max(1, std::min(w.Wb, 16 * nsm)), 64, 0, s>>>(g, c, wr);
  } else {
    k_rescore<256><<<std::max(1, std::min(w.Wb, 4 * nsm)), 256, 0, s>>>(g, c, wr);
  }
}

void launch_probe(const DevGrid& g, const Work& w, double* n0, double* n1, uint8_t* ok,
                  cudaStream_t s) {
  const int ncase = g.N1 + g.NM + g.NI;
  dim3 grid(64, ncase + 1);
  k_probe<<<grid, 256, 0, s>>>(g, w, n0, n1, ok);
}

int kernels_per_wave(const DevGrid& g, const Work& w) {
  const bool single = g.N1 > 0 && g.M > 0;
  // update, N-0, select + FP64 re-score, report select + merge (+ single: the N-1 stage's
  // launches and the report sweep) (+ multi/injection: the correction terms and k_other)
  return 6 + (single ? single_launches(g, w) + 1 : 0) + (2 + 2 * w.oscr) * (g.NM + g.NI > 0 && g.M > 0);
}

}  // namespace bdc
