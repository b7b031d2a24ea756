// bdc_single.cu -- the single-branch N-1 stage (the hot path).
//
// Forms LODF columns on the fly from the shared base D_base and the task's
// rank-r factors, L = (D_base + B'' W^T) / den (solver.py:474-485), in FP64,
// rounded once to FP32 and scaled by 1/rating; monitored rows stream through
// shared memory in chunks (cp.async double buffer of D_base, B'' rows and
// n0/rating); every (case, candidate) pair of a tile is evaluated as
// F = n0 + L n0[r_c] (solver.py:612-613), |F|/rating, max over rows, and the
// per-candidate max is folded into the metric (solver.py:625-631).  The
// (case x candidate x branch) tensor never leaves registers.
//
// Exact dominance screen (the reference's metric_first, solver.py:798-822):
//   k_scale      an upper bound scale_c of max_r |L'(r,c)| per case and the ranking
//                key max_t(m0(t) + scale_c |s(c,t)|);
//   pass TOP     the ptop cases with the largest key (k_topk) are evaluated first,
//                for every candidate -- the reference likewise visits likely-binding
//                cases first;
//   pass SCREEN  every other tile; a pair whose bound cannot exceed the running
//                metric of its candidate cannot change it and is skipped, per CTA
//                tile and per warp.  Evaluated pairs store their exact FP32 max in
//                cmax; the alive map records which warps evaluated, so the winner
//                report re-derives the bound of skipped pairs.
#include "bdc_device.cuh"

namespace bdc {

enum { PASS_SCREEN = 0, PASS_TOP = 1 };

template <int CPT, int TPT, int TX, int TY, int RC, int MINB, int PASS>
__global__ void __launch_bounds__(TX* TY, MINB) k_single(DevGrid g, DevCfg cfg, Work w) {
  constexpr int NTH = TX * TY, NC = CPT * TX, TT = TPT * TY;
  const int b = blockIdx.z;
  if (w.status[b] != 0) return;
  const int c0 = blockIdx.x * NC, t0 = blockIdx.y * TT;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int rs = w.rs, rt = w.rank[b], T = w.T, M = g.M, N1 = g.N1, R = g.R;
  // dynamic: [sW rs*NC f64][sBb 2*rs*RC f64][sN 2*RC*TT f32][sD 2*RC*NC f32]
  extern __shared__ __align__(16) unsigned char dsm[];
  double* sW = reinterpret_cast<double*>(dsm);   // [rt][NC]
  double* sBb = sW + NC * rs;                    // [2][rt][RC] B'' rows of the chunk
  float* sNp = reinterpret_cast<float*>(sBb + 2 * rs * RC);
  float* sDp = sNp + 2 * RC * TT;
#define SN(bf, r_, t_) sNp[((bf) * RC + (r_)) * TT + (t_)]
#define SD(bf, r_, c_) sDp[((bf) * RC + (r_)) * NC + (c_)]
  __shared__ int sCase[NC];        // case index of each tile column, -1 = none / skip
  __shared__ double sInvDen[NC];
  __shared__ int sRowC[NC];
  __shared__ double sInv[2][RC];
  __shared__ int sRow[2][RC];
  __shared__ __align__(16) float sL[RC][NC];
  __shared__ int sdead[RMAX];
  const int nd = w.ndead[b];
  const double* Bm = w.Bm + (size_t)b * rs * R;
  const float* n0s = w.n0s + (size_t)b * M * T;
  const float* s32 = w.s32 + (size_t)b * N1 * T;
  float* cm = w.cmax + (size_t)b * (N1 + g.NM + g.NI) * T;
  const bool vecN = TT % 4 == 0 && (T % 4) == 0 && (t0 % 4) == 0;
  // contiguous tile columns allow 16-byte D_base copies; the TOP tile gathers
  const bool vecD = PASS != PASS_TOP;

  // cases of the TOP tile: ranked by screening key, or simply the first ptop cases
  auto done_c = [&](int c) -> bool { return w.ranked ? w.done[(size_t)b * N1 + c] != 0 : c < w.ptop; };
  if (tid < nd) sdead[tid] = w.dead[(size_t)b * RMAX + tid];
  for (int cc = tid; cc < NC; cc += NTH) {
    int c = -1;
    if constexpr (PASS == PASS_TOP)
      c = w.ranked ? (cc < w.ptop ? w.top[(size_t)b * w.ptop + cc] : -1) : (cc < min(w.ptop, N1) ? cc : -1);
    else c = c0 + cc < N1 ? c0 + cc : -1;
    sCase[cc] = c;
    const bool ok = c >= 0 && w.sc_ok[(size_t)b * N1 + c];
    sInvDen[cc] = ok ? 1.0 / w.den[(size_t)b * N1 + c] : 0.0;
    sRowC[cc] = c >= 0 ? g.sc_row[c] : -1;
  }
  __syncthreads();
  for (int idx = tid; idx < NC * rt; idx += NTH) {
    const int cc = idx / rt, j = idx % rt, c = sCase[cc];
    sW[j * NC + cc] = c >= 0 ? w.Wsc[((size_t)b * N1 + c) * rs + j] : 0.0;
  }

  // s(c,t) = n0[r_c][t] (FP32, from the update kernel) and the accumulators
  float acc[CPT][TPT], sv[CPT][TPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = sCase[tx * CPT + i];
#pragma unroll
    for (int jj = 0; jj < TPT; ++jj) {
      const int t = t0 + ty * TPT + jj;
      sv[i][jj] = (c >= 0 && t < T) ? s32[(size_t)c * T + t] : 0.f;
      acc[i][jj] = 0.f;
    }
  }
  bool warp_alive = true;
  if constexpr (PASS == PASS_SCREEN) {
    // |F| <= m0(t) + scale_c |s(c,t)| (update kernel): a pair whose bound cannot
    // exceed a lower bound of its candidate's final metric -- the running metric
    // (N-0, multi/injection cases, the TOP pass) and, for tasks with islanded cases,
    // the penalty floor -- cannot change the metric.  Cases already evaluated by the
    // TOP pass are skipped outright.
    bool live[CPT];
    float scl[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int cc = tx * CPT + i, c = sCase[cc];
      live[i] = c >= 0 && !done_c(c);
      scl[i] = (w.screen && live[i]) ? w.scale[(size_t)b * N1 + c] : 0.f;
      if (w.screen) live[i] = live[i] && sInvDen[cc] != 0.0;
    }
    bool need = false;
    if (w.screen) {
      const float pen = w.nisl[b] > 0 ? (float)cfg.penalty : 0.f;
#pragma unroll
      for (int jj = 0; jj < TPT; ++jj) {
        const int t = t0 + ty * TPT + jj;
        if (t >= T) continue;
        const float lb = fmaxf(__uint_as_float(w.m32[(size_t)b * T + t]), pen);
        const float m0 = w.m0[(size_t)b * T + t];
#pragma unroll
        for (int i = 0; i < CPT; ++i) need |= live[i] && (m0 + scl[i] * fabsf(sv[i][jj])) > lb;
      }
    } else {
#pragma unroll
      for (int i = 0; i < CPT; ++i) need |= live[i];
    }
    warp_alive = __any_sync(0xffffffffu, need);
    // which warps evaluated their pairs: the winner report takes exact maxima from
    // alive warps and re-derives the dominance bound for the others
    if ((tid & 31) == 0)
      w.alive[(((size_t)b * w.nct + blockIdx.x) * w.ntt + blockIdx.y) * SWEEP_WARPS + (tid >> 5)] = warp_alive;
    const bool block_alive = __syncthreads_or(need);
    if (!block_alive) return;  // no cp.async in flight yet
  }
  if (warp_alive) {
    // evaluated (case, candidate) pairs, for the roofline accounting
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int c = sCase[tx * CPT + i];
      if (c < 0 || (PASS == PASS_SCREEN && done_c(c))) continue;
#pragma unroll
      for (int jj = 0; jj < TPT; ++jj) cnt += (t0 + ty * TPT + jj) < T;
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((tid & 31) == 0 && cnt) atomicAdd(w.pairs, (unsigned long long)cnt);
  }

  // ---- stage one row chunk (async): row ids + 1/rating, B'' rows, n0/rating, D_base
  auto issue = [&](int m0, int buf) {
    for (int rr = tid; rr < RC; rr += NTH) {
      const int m = m0 + rr;
      int row = -1;
      double inv = 0.0;
      if (m < M) {
        row = g.mon_row[m];
        inv = g.inv_rating[m];
        if (is_dead(sdead, nd, row)) row = -1;
      }
      sRow[buf][rr] = row;
      sInv[buf][rr] = inv;
    }
    for (int idx = tid; idx < rt * RC; idx += NTH) {
      const int j = idx / RC, rr = idx % RC, m = m0 + rr;
      const bool ok = m < M;
      cp8(&sBb[(buf * rs + j) * RC + rr], ok ? &Bm[(size_t)j * R + g.mon_row[m]] : Bm, ok);
    }
    if constexpr (TT % 4 == 0) {
      if (vecN) {
        constexpr int TQ = TT / 4;
        for (int idx = tid; idx < RC * TQ; idx += NTH) {
          const int rr = idx / TQ, q = idx % TQ, m = m0 + rr, t = t0 + 4 * q;
          const bool ok = m < M && t < T;
          cp16(&SN(buf, rr, 4 * q), ok ? &n0s[(size_t)m * T + t] : n0s, ok);
        }
      }
    }
    if (!vecN) {
      for (int idx = tid; idx < RC * TT; idx += NTH) {
        const int rr = idx / TT, tt = idx % TT, m = m0 + rr, t = t0 + tt;
        const bool ok = m < M && t < T;
        cp4(&SN(buf, rr, tt), ok ? &n0s[(size_t)m * T + t] : n0s, ok);
      }
    }
    if (vecD) {
      for (int idx = tid; idx < RC * (NC / 4); idx += NTH) {
        const int rr = idx / (NC / 4), q = idx % (NC / 4), m = m0 + rr, c = c0 + 4 * q;
        const bool ok = m < M && c < g.N1p;  // rows are zero-padded to N1p
        cp16(&SD(buf, rr, 4 * q), ok ? &g.D32[(size_t)m * g.N1p + c] : g.D32, ok);
      }
    } else {
      for (int idx = tid; idx < RC * NC; idx += NTH) {
        const int rr = idx / NC, cc = idx % NC, m = m0 + rr, c = sCase[cc];
        const bool ok = m < M && c >= 0;
        cp4(&SD(buf, rr, cc), ok ? &g.D32[(size_t)m * g.N1p + c] : g.D32, ok);
      }
    }
    cp_commit();
  };

  issue(0, 0);
  const int nchunks = (M + RC - 1) / RC;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) {
      issue((ch + 1) * RC, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    // LODF columns of this chunk, formed on the fly in FP64, stored scaled by 1/rating.
    // Thread owns one case column cc and RPT rows; the rank-r correction runs as
    // j-outer register accumulation (W[j][cc] once, B rows broadcast from smem).
    {
      constexpr int RG = NTH / NC;   // row groups
      constexpr int RPT = RC / RG;   // rows per thread (multiple of 8)
      static_assert(RPT % 8 == 0, "row tile");
      const int cc = tid % NC, rg = tid / NC;
      const double idn = sInvDen[cc];
      const int rowc = sRowC[cc];
#pragma unroll
      for (int kb = 0; kb < RPT; kb += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (double)SD(buf, rg + (kb + k) * RG, cc);
        for (int j = 0; j < rt; ++j) {
          const double wj = sW[j * NC + cc];
          const double* Bj = &sBb[(buf * rs + j) * RC + rg];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = fma(Bj[(kb + k) * RG], wj, v[k]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int rr = rg + (kb + k) * RG;
          const int row = sRow[buf][rr];
          const double sc = idn * sInv[buf][rr];
          float lv = 0.f;
          if (row >= 0 && idn != 0.0) lv = (row == rowc) ? (float)(-sInv[buf][rr]) : (float)(v[k] * sc);
          sL[rr][cc] = lv;
        }
      }
    }
    __syncthreads();
    if (warp_alive) {
      const int rend = min(RC, M - ch * RC);
      if (rend == RC) {
        // two rows x two candidates per step: FFMA2 (packed FP32 FMA, same rounding as
        // fmaf) and one FMNMX3 (|.| on every input) per accumulator
        static_assert(TPT % 2 == 0, "candidate pairs");
#pragma unroll 2
        for (int rr = 0; rr < RC; rr += 2) {
          float2 l2[2][CPT], n2[2][TPT / 2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int i = 0; i < CPT; ++i) {
              const float lv = sL[rr + h][tx * CPT + i];
              l2[h][i] = make_float2(lv, lv);
            }
#pragma unroll
            for (int p = 0; p < TPT / 2; ++p)
              n2[h][p] = *reinterpret_cast<const float2*>(&SN(buf, rr + h, ty * TPT + 2 * p));
          }
#pragma unroll
          for (int i = 0; i < CPT; ++i)
#pragma unroll
            for (int p = 0; p < TPT / 2; ++p) {
              const float2 sp = make_float2(sv[i][2 * p], sv[i][2 * p + 1]);
              const float2 f0 = __ffma2_rn(l2[0][i], sp, n2[0][p]);
              const float2 f1 = __ffma2_rn(l2[1][i], sp, n2[1][p]);
              acc[i][2 * p] = max3abs(acc[i][2 * p], f0.x, f1.x);
              acc[i][2 * p + 1] = max3abs(acc[i][2 * p + 1], f0.y, f1.y);
            }
        }
      } else {
        for (int rr = 0; rr < rend; ++rr) {
          float l[CPT], n[TPT];
#pragma unroll
          for (int i = 0; i < CPT; ++i) l[i] = sL[rr][tx * CPT + i];
#pragma unroll
          for (int jj = 0; jj < TPT; ++jj) n[jj] = SN(buf, rr, ty * TPT + jj);
#pragma unroll
          for (int i = 0; i < CPT; ++i)
#pragma unroll
            for (int jj = 0; jj < TPT; ++jj)
              acc[i][jj] = fmaxf(acc[i][jj], fabsf(fmaf(l[i], sv[i][jj], n[jj])));
        }
      }
    }
    __syncthreads();
  }

  if (!warp_alive) return;
  // exact per-(case, candidate) maxima for the winner report; the per-candidate max
  // over the tile's cases goes into the running metric
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = sCase[tx * CPT + i];
    if (c < 0 || (PASS == PASS_SCREEN && done_c(c))) continue;
#pragma unroll
    for (int jj = 0; jj < TPT; ++jj) {
      const int t = t0 + ty * TPT + jj;
      if (t < T) cm[(size_t)c * T + t] = acc[i][jj];
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
#undef SN
#undef SD
}

// ---------------------------------------------------------------------------- k_scale
// Per-case screening scale: an upper bound of max_r |L'(r,c)| over the monitored rows
// (L' = the FP32 LODF/rating values the sweep multiplies), from an FP32 evaluation
// L~ = D_base + sum_j B''_j W_j with a rigorous rounding term:
//     |L - L~| <= gamma (|D| + sum_j |B''_j| |W_j|),  gamma = (rt + 8) 2^-23,
// bounded per case by sc_dscale_c + sum_j |W_cj| max_r |B''(r,j)|/rating_r.  The own
// row contributes 1/rating (L' = -1/rating there), disconnected rows nothing.  Then the
// ranking key bkey_c = max_t (m0(t) + scale_c |s(c,t)|) (solver.py:634-639, 815).
// One thread per case, monitored-row chunks of D_base and B'' through a cp.async
// double buffer; 4 rows of B'' per 16-byte shared load.
namespace {
constexpr int SC_NC = 256, SC_RC = 16;  // static shared memory stays under 48 KB
}

// RS = rank bucket >= every task's rank in the wave: W in registers, B'' terms past a
// task's own rank are zero-filled, so the inner loop is straight-line FFMAs.  TB tasks
// share a CTA: the D_base chunk (the shared operand) is staged and read once for all.
template <int RS, int TB>
__global__ void __launch_bounds__(SC_NC, 2) k_scale(DevGrid g, Work w) {
  const int tb0 = blockIdx.y * TB;
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * SC_NC, c = c0 + tid < g.N1 ? c0 + tid : -1;
  const int rs = w.rs, M = g.M, N1 = g.N1, T = w.T;
  __shared__ __align__(16) float sD[2][SC_RC][SC_NC];
  __shared__ __align__(16) float sB[2][TB][RS][SC_RC];
  __shared__ __align__(16) float sInv[2][TB][SC_RC];
  __shared__ int sdead[TB][RMAX];
  __shared__ int snd[TB], srt[TB];
  __shared__ float sm0[TB];
  if (tid < TB) {
    const int b = tb0 + tid;
    const bool on = b < w.Wb && w.status[b] == 0;
    snd[tid] = on ? w.ndead[b] : 0;
    srt[tid] = on ? w.rank[b] : -1;  // -1: slot idle
    sm0[tid] = 0.f;
  }
  __syncthreads();
  for (int i = tid; i < TB * RMAX; i += SC_NC) {
    const int k = i / RMAX, d = i % RMAX;
    if (d < snd[k]) sdead[k][d] = w.dead[(size_t)(tb0 + k) * RMAX + d];
  }
  // max_t m0(t) of each task (ranking key)
  {
    const int lane = tid & 31, wid = tid >> 5;
    for (int k = wid; k < TB; k += SC_NC / 32) {
      if (srt[k] < 0) continue;
      float v = 0.f;
      for (int t = lane; t < T; t += 32) v = fmaxf(v, w.m0[(size_t)(tb0 + k) * T + t]);
      for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) sm0[k] = v;
    }
  }
  __syncthreads();
  bool any = false;
#pragma unroll
  for (int k = 0; k < TB; ++k) any |= srt[k] >= 0;
  if (!any) return;
  float wr[TB][RS];
#pragma unroll
  for (int k = 0; k < TB; ++k)
#pragma unroll
    for (int j = 0; j < RS; ++j) wr[k][j] = 0.f;
  if (c >= 0) {
#pragma unroll
    for (int k = 0; k < TB; ++k) {
      const int b = tb0 + k;
#pragma unroll
      for (int j = 0; j < RS; ++j)
        if (j < srt[k]) wr[k][j] = (float)w.Wsc[((size_t)b * N1 + c) * rs + j];
    }
  }
  auto issue = [&](int m0, int buf) {
    for (int idx = tid; idx < SC_RC * (SC_NC / 4); idx += SC_NC) {
      const int rr = idx / (SC_NC / 4), q = 4 * (idx % (SC_NC / 4)), m = m0 + rr;
      const bool okd = m < M && c0 + q < g.N1p;  // rows are zero-padded to N1p
      cp16(&sD[buf][rr][q], okd ? &g.D32[(size_t)m * g.N1p + c0 + q] : g.D32, okd);
    }
    for (int idx = tid; idx < TB * RS * SC_RC; idx += SC_NC) {
      const int k = idx / (RS * SC_RC), j = (idx / SC_RC) % RS, rr = idx % SC_RC, m = m0 + rr;
      const bool okb = m < M && j < srt[k];  // zero-fill terms past the task's rank
      const float* src = w.B32 + ((size_t)(tb0 + k) * rs + j) * M + m;
      cp4(&sB[buf][k][j][rr], okb ? src : w.B32, okb);
    }
    for (int idx = tid; idx < TB * SC_RC; idx += SC_NC) {
      const int k = idx / SC_RC, rr = idx % SC_RC, m = m0 + rr;
      sInv[buf][k][rr] = (m < M && srt[k] >= 0 && !is_dead(sdead[k], snd[k], g.mon_row[m]))
                             ? (float)g.inv_rating[m] : 0.f;
    }
    cp_commit();
  };
  float mx[TB];
#pragma unroll
  for (int k = 0; k < TB; ++k) mx[k] = 0.f;
  const int ownp = c >= 0 ? g.row_mon_pos[g.sc_row[c]] : -1;
  issue(0, 0);
  const int nchunks = (M + SC_RC - 1) / SC_RC;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1, m0 = ch * SC_RC;
    if (ch + 1 < nchunks) {
      issue(m0 + SC_RC, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int ownrr = ownp - m0;
#pragma unroll 2
    for (int r4 = 0; r4 < SC_RC; r4 += 4) {
      float d[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) d[q] = sD[buf][r4 + q][tid];
#pragma unroll
      for (int k = 0; k < TB; ++k) {
        float l0 = d[0], l1 = d[1], l2 = d[2], l3 = d[3];
#pragma unroll
        for (int j = 0; j < RS; ++j) {
          const float4 bq = *reinterpret_cast<const float4*>(&sB[buf][k][j][r4]);
          l0 = fmaf(bq.x, wr[k][j], l0);
          l1 = fmaf(bq.y, wr[k][j], l1);
          l2 = fmaf(bq.z, wr[k][j], l2);
          l3 = fmaf(bq.w, wr[k][j], l3);
        }
        const float4 iq = *reinterpret_cast<const float4*>(&sInv[buf][k][r4]);
        mx[k] = fmaxf(mx[k], (r4 + 0 == ownrr) ? 0.f : fabsf(l0) * iq.x);
        mx[k] = fmaxf(mx[k], (r4 + 1 == ownrr) ? 0.f : fabsf(l1) * iq.y);
        mx[k] = fmaxf(mx[k], (r4 + 2 == ownrr) ? 0.f : fabsf(l2) * iq.z);
        mx[k] = fmaxf(mx[k], (r4 + 3 == ownrr) ? 0.f : fabsf(l3) * iq.w);
      }
    }
    __syncthreads();
  }
  if (c < 0) return;
#pragma unroll
  for (int k = 0; k < TB; ++k) {
    const int b = tb0 + k, rt = srt[k];
    if (rt < 0) continue;
    const bool ok = w.sc_ok[(size_t)b * N1 + c] != 0;
    float U = 0.f;
    if (ok) {
      const double idn = 1.0 / w.den[(size_t)b * N1 + c];
      float wsum = 0.f;
      for (int j = 0; j < rt; ++j)
        wsum += (float)fabs(w.Wsc[((size_t)b * N1 + c) * rs + j]) * w.bmax[(size_t)b * rs + j];
      const float gam = (float)(rt + 8) * 1.1920929e-7f;
      U = (float)fabs(idn) * (mx[k] + gam * ((float)g.sc_dscale[c] + wsum));
      const int rowc = g.sc_row[c];
      if (ownp >= 0 && !is_dead(sdead[k], snd[k], rowc)) U = fmaxf(U, (float)g.inv_rating[ownp]);
      U *= 1.f + 4e-6f;
    }
    w.scale[(size_t)b * N1 + c] = U;
    // ranking key for the TOP tile (ordering only; exactness rests on the per-pair bound)
    w.bkey[(size_t)b * N1 + c] = ok ? __float_as_uint(sm0[k] + U * w.smax[(size_t)b * N1 + c]) : 0u;
  }
}

namespace {
template <int RS, int TB>
void launch_scale_t(const DevGrid& g, const Work& w, cudaStream_t s) {
  const dim3 grid((g.N1 + SC_NC - 1) / SC_NC, (w.Wb + TB - 1) / TB);
  k_scale<RS, TB><<<grid, SC_NC, 0, s>>>(g, w);
}
void launch_scale(const DevGrid& g, const Work& w, cudaStream_t s) {
  const int r = w.rs;
  if (r <= 1) launch_scale_t<1, 4>(g, w, s);
  else if (r <= 2) launch_scale_t<2, 4>(g, w, s);
  else if (r <= 3) launch_scale_t<3, 4>(g, w, s);
  else if (r <= 4) launch_scale_t<4, 4>(g, w, s);
  else if (r <= 6) launch_scale_t<6, 4>(g, w, s);
  else if (r <= 8) launch_scale_t<8, 2>(g, w, s);
  else if (r <= 16) launch_scale_t<16, 1>(g, w, s);
  else launch_scale_t<32, 1>(g, w, s);
}
}  // namespace

namespace {

template <int CPT, int TPT, int TX, int TY, int RC, int MINB, int PASS>
void launch_single_t(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  constexpr int NC = CPT * TX, TT = TPT * TY;
  const size_t dyn = ((size_t)NC * w.rs + 2 * (size_t)w.rs * RC) * sizeof(double) +
                     (2 * (size_t)RC * TT + 2 * (size_t)RC * NC) * sizeof(float);
  static int max_dyn = -1;
  if (max_dyn < 0) {
    // opt in to every byte of shared memory the kernel's static part leaves free
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_single<CPT, TPT, TX, TY, RC, MINB, PASS>);
    max_dyn = optin - (int)fa.sharedSizeBytes;
    cudaFuncSetAttribute(k_single<CPT, TPT, TX, TY, RC, MINB, PASS>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
  }
  const int ctiles = PASS == PASS_TOP ? 1 : (g.N1 + NC - 1) / NC;
  dim3 grid(ctiles, (w.T + TT - 1) / TT, w.Wb);
  k_single<CPT, TPT, TX, TY, RC, MINB, PASS><<<grid, TX * TY, dyn, s>>>(g, c, w);
}

template <int PASS>
void launch_pass(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  // must match sweep_shape(T) (bdc_device.cuh): the report decodes the alive map with it
  const SweepShape sh = sweep_shape(w.T);
  if (sh.TPT == 16) launch_single_t<2, 16, 32, 8, 32, 2, PASS>(g, c, w, s);      // 64 cases x 128 candidates
  else if (sh.TPT == 8) launch_single_t<2, 8, 32, 8, 32, 3, PASS>(g, c, w, s);   // 64 x 64
  else if (sh.TX == 32) launch_single_t<4, 4, 32, 8, 32, 3, PASS>(g, c, w, s);   // 128 x 32
  else if (sh.TPT == 4) launch_single_t<4, 4, 64, 4, 32, 3, PASS>(g, c, w, s);   // 256 x 16
  else launch_single_t<4, 2, 64, 4, 32, 3, PASS>(g, c, w, s);                    // 256 x 8
}

}  // namespace

void launch_single(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  if (g.N1 == 0 || g.M == 0) return;
  if (w.ranked) {
    // per-case scale bound and ranking key, then the top tile by key
    launch_scale(g, w, s);
    launch_topk(g, w, s);
  }
  launch_pass<PASS_TOP>(g, c, w, s);
  if (g.N1 > w.ptop) launch_pass<PASS_SCREEN>(g, c, w, s);
}

}  // namespace bdc
