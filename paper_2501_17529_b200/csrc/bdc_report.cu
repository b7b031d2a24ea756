// bdc_report.cu -- Kernel 5: the winner's sparse report and FP64 metric, and the
// flow probe used by the parity tests.
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

#include <climits>

namespace bdc {

namespace {

constexpr int RT = 256;
constexpr int RW = RT / 32;
constexpr int CAND_CAP = 1024;

__device__ __forceinline__ bool better(double r1, int p1, double r2, int p2) {
  return r1 > r2 || (r1 == r2 && p1 < p2);
}
__device__ __forceinline__ bool better3(double r1, int c1, int p1, double r2, int c2, int p2) {
  return r1 > r2 || (r1 == r2 && (c1 < c2 || (c1 == c2 && p1 < p2)));
}

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
#pragma unroll
    for (int i = KC - 1; i > 0; --i) {
      if (better(r, p, rel[i - 1], pos[i - 1])) {
        rel[i] = rel[i - 1]; pos[i] = pos[i - 1]; flow[i] = flow[i - 1];
      } else {
        rel[i] = r; pos[i] = p; flow[i] = f;
        return;
      }
    }
    rel[0] = r; pos[0] = p; flow[0] = f;
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

}  // namespace

template <int KC>
__global__ void __launch_bounds__(RT, 3) k_report(DevGrid g, DevCfg cfg, Work w) {
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
  __shared__ double sred[RW];
  __shared__ double sbr[2][RW];
  __shared__ int sbp[2][RW];
  __shared__ double sWc[RW][RMAX];
  __shared__ double sMinv[RW][MMAX * MMAX];
  __shared__ double sY[RMAX];
  __shared__ int sN0pos[KMAX];
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
  }
  __syncthreads();

  double mymax = 0.0;
  // ---- N-0 report: kg rounds of block argmax (one barrier per round) ----------------
  {
    double pr = 1e300;
    int pp = -1;
    int n0n = 0;
    for (int round = 0; round < kg; ++round) {
      double br = -1.0;
      int bp = INT_MAX;
      for (int p = tid; p < M; p += RT) {
        const int row = g.mon_row[p];
        const double rel = fabs(n0b[row]) * g.inv_rating[p];
        if (round == 0) mymax = fmax(mymax, rel);
        if (is_dead(sdead, nd, row)) continue;
        // next entry in (rel desc, pos asc) order after the previous pick
        if (!(rel < pr || (rel == pr && p > pp))) continue;
        if (better(rel, p, br, bp)) { br = rel; bp = p; }
      }
      for (int o = 16; o; o >>= 1) {
        const double orr = __shfl_xor_sync(0xffffffffu, br, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (better(orr, op, br, bp)) { br = orr; bp = op; }
      }
      const int sl = round & 1;
      if (lane == 0) { sbr[sl][wid] = br; sbp[sl][wid] = bp; }
      __syncthreads();
      br = sbr[sl][0]; bp = sbp[sl][0];
      for (int i = 1; i < RW; ++i)
        if (better(sbr[sl][i], sbp[sl][i], br, bp)) { br = sbr[sl][i]; bp = sbp[sl][i]; }
      if (br < 0.0) break;
      if (tid == 0) sN0pos[round] = bp;
      pr = br; pp = bp;
      ++n0n;
    }
    if (tid == 0) {
      w.n0cnt[b] = n0n;
      for (int i = 0; i < n0n; ++i) {
        const int p = sN0pos[i];
        const double f = n0b[g.mon_row[p]];
        w.n0pos[(size_t)b * kg + i] = p;
        w.n0flow[(size_t)b * kg + i] = f;
        w.n0rel[(size_t)b * kg + i] = fabs(f) * g.inv_rating[p];
      }
    }
  }

  // ---- which contingencies can matter: exact pruning on the FP32 screening maxima --------
  // A case can place an entry in the final top-kg only if its true max loading is at
  // least the kg-th largest true case max; with |FP32 - FP64| <= SCREEN_EPS that means
  // cmax >= kth(cmax) - 2 eps.  The metric's binding case satisfies the same bound.
  const int ncase = g.N1 + g.NM + g.NI;
  const float* cm = w.cmax + (size_t)b * ncase * T + best;
  auto feasible_case = [&](int ci) -> bool {
    if (ci < g.N1) return w.sc_ok[(size_t)b * g.N1 + ci] != 0;
    if (ci < g.N1 + g.NM) return w.mc_ok[(size_t)b * g.NM + (ci - g.N1)] != 0;
    return true;
  };
  float theta = -1.f;
  {
    float pv = 3.4e38f;
    int pi = -1, found = 0;
    float kth = -1.f;
    for (int round = 0; round < kg; ++round) {
      double br = -1.0;
      int bp = INT_MAX;
      for (int ci = tid; ci < ncase; ci += RT) {
        if (!feasible_case(ci)) continue;
        const float v = cm[(size_t)ci * T];
        if (v < 0.f) continue;  // screened-out pair: only an upper bound is known
        if (!(v < pv || (v == pv && ci > pi))) continue;
        if (better(v, ci, br, bp)) { br = v; bp = ci; }
      }
      for (int o = 16; o; o >>= 1) {
        const double orr = __shfl_xor_sync(0xffffffffu, br, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (better(orr, op, br, bp)) { br = orr; bp = op; }
      }
      const int sl = round & 1;
      if (lane == 0) { sbr[sl][wid] = br; sbp[sl][wid] = bp; }
      __syncthreads();
      br = sbr[sl][0]; bp = sbp[sl][0];
      for (int i = 1; i < RW; ++i)
        if (better(sbr[sl][i], sbp[sl][i], br, bp)) { br = sbr[sl][i]; bp = sbp[sl][i]; }
      if (br < 0.0) break;
      pv = (float)br; pi = bp; kth = (float)br;
      ++found;
    }
    theta = found == kg ? kth - 2.f * SCREEN_EPS : -1.f;
  }
  __shared__ int sCand[CAND_CAP];
  __shared__ int sNCand;
  if (tid == 0) sNCand = 0;
  __syncthreads();
  for (int ci = tid; ci < ncase; ci += RT) {
    if (feasible_case(ci) && fabsf(cm[(size_t)ci * T]) >= theta) {
      const int p = atomicAdd(&sNCand, 1);
      if (p < CAND_CAP) sCand[p] = ci;
    }
  }
  __syncthreads();
  const int ncand = sNCand;
  const bool listed = ncand <= CAND_CAP;  // else scan every case with the same predicate
  const int nloop = listed ? ncand : ncase;

  // ---- FP64 re-evaluation of the candidate cases for the winner ----------------------------
  LaneTop<KC> lt;
  for (int li = wid; li < nloop; li += RW) {
    const int ci = listed ? sCand[li] : li;
    if (!listed && !(feasible_case(ci) && fabsf(cm[(size_t)ci * T]) >= theta)) continue;
    int order, kind = 0, q = ci;
    if (ci < g.N1) {
      order = g.sc_order[ci];
    } else if (ci < g.N1 + g.NM) {
      kind = 1; q = ci - g.N1;
      order = g.mc_order[q];
    } else {
      kind = 2; q = ci - g.N1 - g.NM;
      order = g.ic_order[q];
    }
    lt.clear();
    const double thresh = warp_thresh(wl[wid], kg);
    if (kind == 0) {
      const int rowc = g.sc_row[q];
      const double sc = n0b[rowc];
      const double idn = 1.0 / w.den[(size_t)b * g.N1 + q];
      for (int j = lane; j < rt; j += 32) sWc[wid][j] = w.Wsc[((size_t)b * g.N1 + q) * rs + j];
      __syncwarp();
      const double* Dc = g.D64 + (size_t)q * R;
      for (int p = lane; p < M; p += 32) {
        const int row = g.mon_row[p];
        if (is_dead(sdead, nd, row)) continue;  // flow exactly 0: neither metric nor report
        double f;
        if (row == rowc) {
          f = n0b[row] + (-1.0) * sc;
        } else {
          double dv = Dc[row];
          for (int j = 0; j < rt; ++j) dv = fma(Bm[(size_t)j * R + row], sWc[wid][j], dv);
          f = n0b[row] + (dv * idn) * sc;
        }
        const double rel = fabs(f) * g.inv_rating[p];
        mymax = fmax(mymax, rel);
        if (row != rowc && rel >= thresh) lt.insert(rel, p, f);
      }
    } else if (kind == 1) {
      const int st = g.mc_start[q], m = g.mc_start[q + 1] - st;
      for (int i = lane; i < m * m; i += 32) sMinv[wid][i] = w.minv[((size_t)b * g.NM + q) * MMAX * MMAX + i];
      __syncwarp();
      double sv[MMAX];
      for (int j = 0; j < m; ++j) sv[j] = n0b[g.mb_row[st + j]];
      for (int p = lane; p < M; p += 32) {
        const int row = g.mon_row[p];
        if (is_dead(sdead, nd, row)) continue;
        int own = -1;
        for (int a = 0; a < m; ++a) if (g.mb_row[st + a] == row) own = a;
        double f = n0b[row];
        if (own >= 0) {
          for (int j = 0; j < m; ++j) f += (j == own ? -1.0 : 0.0) * sv[j];
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
            for (int i = 0; i < m; ++i) l += Dv[i] * sMinv[wid][i * m + j];
            f += l * sv[j];
          }
        }
        const double rel = fabs(f) * g.inv_rating[p];
        mymax = fmax(mymax, rel);
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
        double pc = g.P0T[(size_t)ca * R + row];
        for (int j = 0; j < rt; ++j) pc = fma(Bm[(size_t)j * R + row], coef[j], pc);
        const double f = n0b[row] - pc * sp;
        const double rel = fabs(f) * g.inv_rating[p];
        mymax = fmax(mymax, rel);
        if (rel >= thresh) lt.insert(rel, p, f);
      }
    }
    warp_merge<KC>(lt, kc, wl[wid], kg, order);
    __syncwarp();
  }

  // ---- FP64 metric and final merge --------------------------------------------------------
  for (int o = 16; o; o >>= 1) mymax = fmax(mymax, __shfl_xor_sync(0xffffffffu, mymax, o));
  if (lane == 0) sred[wid] = mymax;
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int i = 0; i < RW; ++i) mx = fmax(mx, sred[i]);
    if (w.nisl[b] > 0) mx = fmax(mx, cfg.penalty);
    w.metric[b] = mx;
    WarpList& F = wl[0];
    for (int i = 1; i < RW; ++i)
      for (int e = 0; e < wl[i].n; ++e)
        wl_insert(F, kg, wl[i].rel[e], wl[i].cs[e], wl[i].pos[e], wl[i].flow[e]);
    w.n1cnt[b] = F.n;
    for (int e = 0; e < F.n; ++e) {
      w.n1case[(size_t)b * kg + e] = F.cs[e];
      w.n1pos[(size_t)b * kg + e] = F.pos[e];
      w.n1flow[(size_t)b * kg + e] = F.flow[e];
      w.n1rel[(size_t)b * kg + e] = F.rel[e];
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

void launch_report(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  if (c.kc <= 5) k_report<5><<<w.Wb, RT, 0, s>>>(g, c, w);
  else if (c.kc <= 8) k_report<8><<<w.Wb, RT, 0, s>>>(g, c, w);
  else if (c.kc <= 16) k_report<16><<<w.Wb, RT, 0, s>>>(g, c, w);
  else k_report<32><<<w.Wb, RT, 0, s>>>(g, c, w);
}

void launch_probe(const DevGrid& g, const Work& w, double* n0, double* n1, uint8_t* ok,
                  cudaStream_t s) {
  const int ncase = g.N1 + g.NM + g.NI;
  dim3 grid(64, ncase + 1);
  k_probe<<<grid, 256, 0, s>>>(g, w, n0, n1, ok);
}

int kernels_per_wave(const DevGrid& g, const Work& w) {
  const bool single = g.N1 > 0 && g.M > 0;
  // update, select, report (+ single: [scale, top-k,] top tile, screened sweep) (+ other)
  return 3 + (single ? 1 + (g.N1 > w.ptop ? 1 : 0) + (w.ranked ? 2 : 0) : 0) +
         (g.NM + g.NI > 0 && g.M > 0);
}

}  // namespace bdc
