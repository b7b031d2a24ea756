// bdc_flows.cu -- Kernels 2-4: N-0 contraction, fused N-1 screening, winner selection.
//
//   k_n0      N-0 flows of every candidate: n0 = f0 + B'' y_t (FP64), the
//             rank-r form of `_candidate_base_flows` (solver.py:575-595);
//             writes n0 (FP64) and the rating-scaled FP32 copy n0s that the
//             N-1 stage streams, and folds max|n0|/rating into the metric.
//   k_single  THE hot kernel.  Single-branch N-1 for every (case, candidate)
//             pair of a task, fused: forms LODF columns on the fly from the
//             shared base D_base and the task's rank-r factors
//             (L = (D_base + B'' W^T) / den, solver.py:474-485), applies the
//             outage update F = n0 + L n0[r_c] (solver.py:612-613), takes
//             |F|/rating and max-reduces over monitored rows and cases into
//             the per-candidate metric (solver.py:625-631, agg_m :235-252).
//             The (case x candidate x branch) tensor never leaves registers.
//   k_other   multi-branch (MODF, solver.py:614-618) and injection
//             (solver.py:619-622) contingencies, same fusion, FP64.
//   k_select  islanding penalty floor and first-index argmin (solver.py:804-823).
#include "bdc_device.cuh"

namespace bdc {

// ------------------------------------------------------------------------------- k_n0
namespace {
constexpr int N0_TB = 128;
constexpr int N0_RB = 32;
}  // namespace

__global__ void __launch_bounds__(N0_TB) k_n0(DevGrid g, Work w) {
  const int b = blockIdx.z, r0 = blockIdx.y * N0_RB, tid = threadIdx.x;
  const int t = blockIdx.x * N0_TB + tid;
  if (w.status[b] != 0) return;
  const int rs = w.rs, rt = w.rank[b], T = w.T, R = g.R;
  __shared__ double sB[RMAX][N0_RB];
  __shared__ int sdead[RMAX];
  const int nd = w.ndead[b];
  for (int idx = tid; idx < rt * N0_RB; idx += N0_TB) {
    int j = idx / N0_RB, rr = idx % N0_RB, r = r0 + rr;
    sB[j][rr] = r < R ? w.Bm[((size_t)b * rs + j) * R + r] : 0.0;
  }
  if (tid < nd) sdead[tid] = w.dead[(size_t)b * RMAX + tid];
  __syncthreads();
  if (t >= T) return;
  double y[RMAX];
#pragma unroll
  for (int j = 0; j < RMAX; ++j) y[j] = (j < rt) ? w.Y[((size_t)b * rs + j) * T + t] : 0.0;
  float mx = 0.f;
  const int rend = min(R, r0 + N0_RB);
  for (int r = r0; r < rend; ++r) {
    const int rr = r - r0;
    double v = g.f0[r];
#pragma unroll
    for (int j = 0; j < RMAX; ++j)
      if (j < rt) v = fma(sB[j][rr], y[j], v);
    if (is_dead(sdead, nd, r)) v = 0.0;
    w.n0[((size_t)b * R + r) * T + t] = v;
    const int p = g.row_mon_pos[r];
    if (p >= 0) {
      const float sc = (float)(v * g.inv_rating[p]);
      w.n0s[((size_t)b * g.M + p) * T + t] = sc;
      mx = fmaxf(mx, fabsf(sc));
    }
  }
  atomic_max_pos(&w.m32[(size_t)b * T + t], mx);
}

// --------------------------------------------------------------------------- k_single
// Thread tile: CPT cases x TPT candidates; CTA tile NC = CPT*TX cases x TT = TPT*TY
// candidates; monitored rows streamed through shared memory RC at a time.
template <int CPT, int TPT, int TX, int TY>
__global__ void __launch_bounds__(TX* TY) k_single(DevGrid g, Work w) {
  constexpr int NTH = TX * TY, NC = CPT * TX, TT = TPT * TY, RC = 32;
  const int b = blockIdx.z;
  if (w.status[b] != 0) return;
  const int c0 = blockIdx.x * NC, t0 = blockIdx.y * TT;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int rs = w.rs, rt = w.rank[b], T = w.T, M = g.M, N1 = g.N1, R = g.R;
  extern __shared__ double sW[];  // [NC][rt]
  __shared__ double sInvDen[NC];
  __shared__ int sRowC[NC];
  __shared__ double sB[RMAX][RC];
  __shared__ double sInv[RC];
  __shared__ int sRow[RC];
  __shared__ __align__(16) float sL[RC][NC];
  __shared__ __align__(16) float sN[RC][TT];
  __shared__ int sdead[RMAX];
  const int nd = w.ndead[b];

  for (int idx = tid; idx < NC * rt; idx += NTH) {
    const int cc = idx / rt, j = idx % rt, c = c0 + cc;
    sW[idx] = c < N1 ? w.Wsc[((size_t)b * N1 + c) * rs + j] : 0.0;
  }
  for (int cc = tid; cc < NC; cc += NTH) {
    const int c = c0 + cc;
    const bool ok = c < N1 && w.sc_ok[(size_t)b * N1 + c];
    sInvDen[cc] = ok ? 1.0 / w.den[(size_t)b * N1 + c] : 0.0;
    sRowC[cc] = c < N1 ? g.sc_row[c] : -1;
  }
  if (tid < nd) sdead[tid] = w.dead[(size_t)b * RMAX + tid];
  __syncthreads();

  float acc[CPT][TPT], sv[CPT][TPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int row = sRowC[tx * CPT + i];
#pragma unroll
    for (int jj = 0; jj < TPT; ++jj) {
      const int t = t0 + ty * TPT + jj;
      sv[i][jj] = (row >= 0 && t < T) ? (float)w.n0[((size_t)b * R + row) * T + t] : 0.f;
      acc[i][jj] = 0.f;
    }
  }
  const bool vecN = (T % 4) == 0;

  for (int m0 = 0; m0 < M; m0 += RC) {
    __syncthreads();
    for (int rr = tid; rr < RC; rr += NTH) {
      const int m = m0 + rr;
      int row = -1;
      double inv = 0.0;
      if (m < M) {
        row = g.mon_row[m];
        inv = g.inv_rating[m];
        if (is_dead(sdead, nd, row)) row = -1;
      }
      sRow[rr] = row;
      sInv[rr] = inv;
    }
    for (int idx = tid; idx < rt * RC; idx += NTH) {
      const int j = idx / RC, rr = idx % RC, m = m0 + rr;
      sB[j][rr] = m < M ? w.Bm[((size_t)b * rs + j) * R + g.mon_row[m]] : 0.0;
    }
    if (vecN) {
      for (int idx = tid; idx < RC * (TT / 4); idx += NTH) {
        const int rr = idx / (TT / 4), q = idx % (TT / 4), m = m0 + rr, t = t0 + 4 * q;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < M && t < T) v = *reinterpret_cast<const float4*>(&w.n0s[((size_t)b * M + m) * T + t]);
        *reinterpret_cast<float4*>(&sN[rr][4 * q]) = v;
      }
    } else {
      for (int idx = tid; idx < RC * TT; idx += NTH) {
        const int rr = idx / TT, tt = idx % TT, m = m0 + rr, t = t0 + tt;
        sN[rr][tt] = (m < M && t < T) ? w.n0s[((size_t)b * M + m) * T + t] : 0.f;
      }
    }
    __syncthreads();
    // LODF columns of this row chunk, formed on the fly in FP64, stored scaled by 1/rating
    for (int idx = tid; idx < RC * NC; idx += NTH) {
      const int rr = idx / NC, cc = idx % NC, m = m0 + rr, c = c0 + cc;
      const int row = sRow[rr];
      float lv = 0.f;
      if (row >= 0 && c < N1 && sInvDen[cc] != 0.0) {
        if (row == sRowC[cc]) {
          lv = (float)(-sInv[rr]);
        } else {
          double v = (double)g.D32[(size_t)m * N1 + c];
          for (int j = 0; j < rt; ++j) v = fma(sB[j][rr], sW[cc * rt + j], v);
          lv = (float)(v * sInvDen[cc] * sInv[rr]);
        }
      }
      sL[rr][cc] = lv;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < RC; ++rr) {
      float l[CPT], n[TPT];
#pragma unroll
      for (int i = 0; i < CPT; ++i) l[i] = sL[rr][tx * CPT + i];
#pragma unroll
      for (int jj = 0; jj < TPT; ++jj) n[jj] = sN[rr][ty * TPT + jj];
#pragma unroll
      for (int i = 0; i < CPT; ++i)
#pragma unroll
        for (int jj = 0; jj < TPT; ++jj)
          acc[i][jj] = fmaxf(acc[i][jj], fabsf(fmaf(l[i], sv[i][jj], n[jj])));
    }
  }
  constexpr int GW = TX < 32 ? TX : 32;  // lanes of a warp sharing one candidate group
#pragma unroll
  for (int jj = 0; jj < TPT; ++jj) {
    float v = acc[0][jj];
#pragma unroll
    for (int i = 1; i < CPT; ++i) v = fmaxf(v, acc[i][jj]);
#pragma unroll
    for (int o = GW / 2; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int t = t0 + ty * TPT + jj;
    if ((tx % GW) == 0 && t < T) atomic_max_pos(&w.m32[(size_t)b * T + t], v);
  }
}

// ---------------------------------------------------------------------------- k_other
namespace {
constexpr int OT = 256;   // threads; one candidate per thread per t-chunk
constexpr int ORC = 128;  // monitored rows per chunk
}  // namespace

__global__ void __launch_bounds__(OT) k_other(DevGrid g, Work w) {
  const int q = blockIdx.x, b = blockIdx.z, tid = threadIdx.x;
  const int t = blockIdx.y * OT + tid;
  if (w.status[b] != 0) return;
  const bool multi = q < g.NM;
  if (multi && !w.mc_ok[(size_t)b * g.NM + q]) return;  // islanded: penalty, not flows
  const int rs = w.rs, rt = w.rank[b], T = w.T, R = g.R, M = g.M;
  __shared__ double sL[ORC][MMAX];
  __shared__ double sInv[ORC];
  __shared__ int sRow[ORC];
  __shared__ int sdead[RMAX];
  __shared__ double sMinv[MMAX * MMAX];
  __shared__ double sW[MMAX][RMAX];
  __shared__ double sCa[RMAX], sCb[RMAX];
  const int nd = w.ndead[b];
  if (tid < nd) sdead[tid] = w.dead[(size_t)b * RMAX + tid];
  int m, st = 0, qi = 0, ca = 0;
  double sp = 0.0;
  if (multi) {
    st = g.mc_start[q];
    m = g.mc_start[q + 1] - st;
    for (int i = tid; i < m * m; i += OT) sMinv[i] = w.minv[((size_t)b * g.NM + q) * MMAX * MMAX + i];
    for (int i = tid; i < m * rt; i += OT) sW[i / rt][i % rt] = w.Wm[((size_t)b * g.NMB + st + i / rt) * rs + i % rt];
  } else {
    qi = q - g.NM;
    m = 2;
    const int sl = g.ic_slot[qi];
    ca = sl >= 0 ? g.slot_col[sl] : g.ic_col[qi];
    sp = g.ic_sp[qi];
    for (int j = tid; j < rt; j += OT) {
      sCa[j] = w.cia[((size_t)b * g.NI + qi) * rs + j];
      sCb[j] = w.cib[((size_t)b * g.NI + qi) * rs + j];
    }
  }
  // per-candidate multipliers of the correction columns
  double sv[MMAX];
  for (int j = 0; j < MMAX; ++j) sv[j] = 0.0;
  if (t < T) {
    if (multi) {
      for (int j = 0; j < m; ++j) sv[j] = w.n0[((size_t)b * R + g.mb_row[st + j]) * T + t];
    } else {
      const int sl = g.ic_slot[qi];
      sv[0] = 1.0;
      sv[1] = (sl >= 0 && w.inj[((size_t)b * T + t) * g.K + sl]) ? 1.0 : 0.0;
    }
  }
  float mx = 0.f;
  for (int m0 = 0; m0 < M; m0 += ORC) {
    __syncthreads();
    for (int rr = tid; rr < ORC; rr += OT) {
      const int mm = m0 + rr;
      int row = -1;
      if (mm < M) {
        row = g.mon_row[mm];
        sInv[rr] = g.inv_rating[mm];
        if (is_dead(sdead, nd, row)) row = -1;
      } else {
        sInv[rr] = 0.0;
      }
      sRow[rr] = row;
      double L[MMAX];
      for (int j = 0; j < MMAX; ++j) L[j] = 0.0;
      if (row >= 0) {
        if (multi) {
          int own = -1;
          for (int a = 0; a < m; ++a) if (g.mb_row[st + a] == row) own = a;
          if (own >= 0) {
            L[own] = -1.0;
          } else {
            double Dv[MMAX];
            for (int i = 0; i < m; ++i) {
              double v = g.Dm64[(size_t)(st + i) * R + row];
              for (int j = 0; j < rt; ++j) v = fma(w.Bm[((size_t)b * rs + j) * R + row], sW[i][j], v);
              Dv[i] = v;
            }
            for (int j = 0; j < m; ++j) {
              double v = 0.0;
              for (int i = 0; i < m; ++i) v += Dv[i] * sMinv[i * m + j];
              L[j] = v;
            }
          }
        } else {
          double pa = g.P0T[(size_t)ca * R + row], pb = pa;
          for (int j = 0; j < rt; ++j) {
            const double bv = w.Bm[((size_t)b * rs + j) * R + row];
            pa = fma(bv, sCa[j], pa);
            pb = fma(bv, sCb[j], pb);
          }
          L[0] = -sp * pa;
          L[1] = -sp * (pb - pa);
        }
      }
      for (int j = 0; j < MMAX; ++j) sL[rr][j] = L[j];
    }
    __syncthreads();
    if (t < T) {
      const int rend = min(ORC, M - m0);
      for (int rr = 0; rr < rend; ++rr) {
        const int row = sRow[rr];
        if (row < 0) continue;
        double f = w.n0[((size_t)b * R + row) * T + t];
        for (int j = 0; j < m; ++j) f = fma(sL[rr][j], sv[j], f);
        mx = fmaxf(mx, (float)(fabs(f) * sInv[rr]));
      }
    }
  }
  if (t < T) atomic_max_pos(&w.m32[(size_t)b * T + t], mx);
}

// --------------------------------------------------------------------------- k_select
__global__ void k_select(DevGrid g, DevCfg cfg, Work w) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = gt >> 5, lane = gt & 31;
  if (b >= w.Wb) return;
  if (w.status[b] != 0) {
    if (lane == 0) { w.best[b] = -1; w.feasible[b] = 0; w.metric[b] = __longlong_as_double(0x7ff8000000000000ll); }
    return;
  }
  const int T = w.T;
  const int tn = w.tcount ? w.tcount[b] : T;
  const bool pen = w.nisl[b] > 0;
  const float penalty = (float)cfg.penalty;
  float bv = __int_as_float(0x7f800000);
  int bi = 0x7fffffff;
  for (int t = lane; t < tn; t += 32) {
    float v = __uint_as_float(w.m32[(size_t)b * T + t]);
    if (pen) v = fmaxf(v, penalty);
    if (v < bv) { bv = v; bi = t; }
  }
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) {
    w.best[b] = bi;
    w.feasible[b] = 1;
    const int nf = g.NC - w.nisl[b];
    atomicAdd(w.lf, (unsigned long long)tn * (unsigned long long)(1 + nf));
  }
}

// ---------------------------------------------------------------------------- launches
void launch_n0(const DevGrid& g, const Work& w, cudaStream_t s) {
  dim3 grid((w.T + N0_TB - 1) / N0_TB, (g.R + N0_RB - 1) / N0_RB, w.Wb);
  k_n0<<<grid, N0_TB, 0, s>>>(g, w);
}

template <int CPT, int TPT, int TX, int TY>
static void launch_single_t(const DevGrid& g, const Work& w, cudaStream_t s) {
  constexpr int NC = CPT * TX, TT = TPT * TY;
  const size_t dyn = (size_t)NC * w.rs * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_single<CPT, TPT, TX, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         64 * 1024);
    attr = true;
  }
  dim3 grid((g.N1 + NC - 1) / NC, (w.T + TT - 1) / TT, w.Wb);
  k_single<CPT, TPT, TX, TY><<<grid, TX * TY, dyn, s>>>(g, w);
}

void launch_single(const DevGrid& g, const Work& w, cudaStream_t s) {
  if (g.N1 == 0) return;
  if (w.T >= 96) launch_single_t<2, 16, 32, 8>(g, w, s);       // 64 cases x 128 candidates
  else if (w.T >= 48) launch_single_t<2, 8, 32, 8>(g, w, s);   // 64 x 64
  else if (w.T >= 24) launch_single_t<4, 4, 32, 8>(g, w, s);   // 128 x 32
  else if (w.T >= 12) launch_single_t<4, 4, 64, 4>(g, w, s);   // 256 x 16
  else launch_single_t<4, 2, 64, 4>(g, w, s);                  // 256 x 8
}

void launch_other(const DevGrid& g, const Work& w, cudaStream_t s) {
  const int nq = g.NM + g.NI;
  if (nq == 0) return;
  dim3 grid(nq, (w.T + OT - 1) / OT, w.Wb);
  k_other<<<grid, OT, 0, s>>>(g, w);
}

void launch_select(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  const int threads = 256;
  const long long total = (long long)w.Wb * 32;
  k_select<<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(g, c, w);
}

}  // namespace bdc
