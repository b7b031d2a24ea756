// bdc_single.cu -- the single-branch N-1 stage (the hot path).
//
// Every (case, candidate) pair needs max_r |n0(r,t) + L(r,c) s(c,t)| / rating_r with
// L = (D_base + B'' W^T) / den the LODF column of case c on the updated topology
// (solver.py:474-485, 612-613, 625-631).  LODF columns are formed on the fly in FP64
// from the shared base D_base and the task's rank-r factors, rounded once to FP32 and
// scaled by 1/rating; the (case x candidate x branch) tensor never leaves registers.
//
// Exact dominance screen (the reference's metric_first, solver.py:798-822):
//   k_scale  per case and screening row block b an upper bound scale_bc of
//            max_{r in b} |L'(r,c)|, and the ranking key of the case (tcgen05,
//            bdc_scale.cu);
//   k_topk   the TOPC cases with the largest key (bdc_update.cu);
//   k_top    those cases for every candidate (dense tile, FFMA2 + FMNMX3): they fix a
//            good lower bound lb(t) of every candidate's metric, as the reference's
//            visit order (descending bound) does;
//   k_live   every other pair is bounded by |F| <= max_b (m0_b(t) + scale_bc |s(c,t)|);
//            a pair whose bound cannot exceed lb(t) cannot change the metric; a case
//            with any pair above its bound is live and queued in groups of TOPC;
//   k_pairs  the live groups, as TOP tiles (every candidate of a live case).
// Every evaluated pair uses the same FP32 expression fabsf(fmaf(L', s, n0')) in every
// kernel, so a metric never depends on which kernel evaluated the binding pair.
#include "bdc_device.cuh"

namespace bdc {

// ---------------------------------------------------------------------------- k_top
// The TOP tile: NC = CPT*TX cases (the task's ranked list, or the first cases when the
// screen is off / N1 <= TOPC) x TT = TPT*TY candidates per CTA, thread (tx, ty) owns
// CPT cases x TPT candidates.  Monitored rows stream through shared memory in chunks of
// RC (cp.async double buffer of D_base columns, B'' rows and n0/rating).
// One tile: task b, cases list[0..nlist) (entries < 0 are empty; list == nullptr means
// cases 0..nlist-1), candidates t0..t0+TT.  Ends with the block synchronised.
template <int CPT, int TPT, int TX, int TY, int RC, int RGS>
__device__ __forceinline__ void top_tile(const DevGrid& g, const Work& w, int b, const int* list, int nlist, int t0) {
  constexpr int TG = TX * TY, NTH = TG * RGS, NC = CPT * TX, TT = TPT * TY;
  static_assert(TG % 32 == 0, "row groups are whole warps");
  // RGS row groups of TG threads split each chunk's rows (maxima combined at the end)
  const int tid = threadIdx.x, gi = tid / TG, tl = tid % TG, tx = tl % TX, ty = tl / TX;
  const int rs = w.rs, rt = w.rank[b], T = w.T, M = g.M, N1 = g.N1, R = g.R;
  // dynamic: [sW rs*NC f64][sBb 2*rs*RC f64][sN 2*RC*TT f32][sD 2*RC*NC f32]
  extern __shared__ __align__(16) unsigned char dsm[];
  double* sW = reinterpret_cast<double*>(dsm);   // [rt][NC]
  double* sBb = sW + NC * rs;                    // [2][rt][RC] B'' rows of the chunk
  float* sNp = reinterpret_cast<float*>(sBb + 2 * rs * RC);
  float* sDp = sNp + 2 * RC * TT;
#define SN(bf, r_, t_) sNp[((bf) * RC + (r_)) * TT + (t_)]
#define SD(bf, r_, c_) sDp[((bf) * RC + (r_)) * NC + (c_)]
  __shared__ int sCase[NC];        // case index of each tile column, -1 = none
  __shared__ double sInvDen[NC];
  __shared__ int sRowC[NC];
  __shared__ double sInv[2][RC];
  __shared__ int sRow[2][RC];
  __shared__ __align__(16) float sL[RC][NC];
  __shared__ int sdead[RMAX];
  __shared__ unsigned sAcc[RGS > 1 ? NC : 1][RGS > 1 ? TT : 1];  // row groups' maxima
  const int nd = w.ndead[b];
  const double* Bm = w.Bm + (size_t)b * rs * R;
  const float* n0s = w.n0s + (size_t)b * M * T;
  float* cm = w.cmax + (size_t)b * (N1 + g.NM + g.NI) * T;
  const bool vecN = TT % 4 == 0 && (T % 4) == 0 && (t0 % 4) == 0;

  if (tid < nd) sdead[tid] = w.dead[(size_t)b * RMAX + tid];
  for (int cc = tid; cc < NC; cc += NTH) {
    const int c = cc < nlist ? (list ? list[cc] : cc) : -1;
    sCase[cc] = c;
    const bool ok = c >= 0 && w.sc_ok[(size_t)b * N1 + c];
    sInvDen[cc] = ok ? 1.0 / w.den[(size_t)b * N1 + c] : 0.0;
    sRowC[cc] = c >= 0 ? g.sc_row[c] : -1;
  }
  if constexpr (RGS > 1)
    for (int i = tid; i < NC * TT; i += NTH) (&sAcc[0][0])[i] = 0u;
  __syncthreads();
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
    for (int idx = tid; idx < RC * NC; idx += NTH) {
      const int rr = idx / NC, cc = idx % NC, m = m0 + rr, c = sCase[cc];
      const bool ok = m < M && c >= 0;
      cp4(&SD(buf, rr, cc), ok ? &g.D32[(size_t)m * g.N1p + c] : g.D32, ok);
    }
    cp_commit();
  };

  issue(0, 0);  // the first chunk is in flight while the tile's factors load
  for (int idx = tid; idx < NC * rt; idx += NTH) {
    const int cc = idx / rt, j = idx % rt, c = sCase[cc];
    sW[j * NC + cc] = c >= 0 ? w.Wsc[((size_t)b * N1 + c) * rs + j] : 0.0;
  }

  // s(c,t) = n0[r_c][t] (FP32, from k_n0) and the accumulators
  float acc[CPT][TPT], sv[CPT][TPT];
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = sCase[tx * CPT + i];
#pragma unroll
    for (int jj = 0; jj < TPT; ++jj) {
      const int t = t0 + ty * TPT + jj;
      sv[i][jj] = (c >= 0 && t < T) ? s_at(g, w, b, c, t) : 0.f;
      acc[i][jj] = 0.f;
      cnt += gi == 0 && c >= 0 && t < T;
    }
  }
  // evaluated (case, candidate) pairs, for the roofline accounting
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((tid & 31) == 0 && cnt) atomicAdd(w.pairs, (unsigned long long)cnt);

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
      constexpr int RPT = RC / RG;   // rows per thread
      constexpr int KB = RPT < 8 ? RPT : 8;
      static_assert(RPT % KB == 0, "row tile");
      const int cc = tid % NC, rg = tid / NC;
      const double idn = sInvDen[cc];
      const int rowc = sRowC[cc];
#pragma unroll
      for (int kb = 0; kb < RPT; kb += KB) {
        double v[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) v[k] = (double)SD(buf, rg + (kb + k) * RG, cc);
        for (int j = 0; j < rt; ++j) {
          const double wj = sW[j * NC + cc];
          const double* Bj = &sBb[(buf * rs + j) * RC + rg];
#pragma unroll
          for (int k = 0; k < KB; ++k) v[k] = fma(Bj[(kb + k) * RG], wj, v[k]);
        }
#pragma unroll
        for (int k = 0; k < KB; ++k) {
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
    // rows past M were staged as zero rows (n0' = 0, L' = 0): they add |0| to the maxima,
    // so the last chunk runs the same paired loop over an even row count
    const int rend = min(RC, (M - ch * RC + 1) & ~1);
    {
      // two rows x two candidates per step: FFMA2 (packed FP32 FMA, same rounding as
      // fmaf) and one FMNMX3 (|.| on every input) per accumulator
      static_assert(TPT % 2 == 0, "candidate pairs");
#pragma unroll 2
      for (int rr = 2 * gi; rr < rend; rr += 2 * RGS) {
        float2 l2[2][CPT], n2[2][TPT / 2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if constexpr (CPT % 2 == 0) {
#pragma unroll
            for (int i = 0; i < CPT; i += 2) {
              const float2 lv = *reinterpret_cast<const float2*>(&sL[rr + h][tx * CPT + i]);
              l2[h][i] = make_float2(lv.x, lv.x);
              l2[h][i + 1] = make_float2(lv.y, lv.y);
            }
          } else {
#pragma unroll
            for (int i = 0; i < CPT; ++i) {
              const float lv = sL[rr + h][tx * CPT + i];
              l2[h][i] = make_float2(lv, lv);
            }
          }
          if constexpr (TPT % 4 == 0) {
#pragma unroll
            for (int p = 0; p < TPT / 2; p += 2) {
              const float4 q4 = *reinterpret_cast<const float4*>(&SN(buf, rr + h, ty * TPT + 2 * p));
              n2[h][p] = make_float2(q4.x, q4.y);
              n2[h][p + 1] = make_float2(q4.z, q4.w);
            }
          } else {
#pragma unroll
            for (int p = 0; p < TPT / 2; ++p)
              n2[h][p] = *reinterpret_cast<const float2*>(&SN(buf, rr + h, ty * TPT + 2 * p));
          }
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
    }
    __syncthreads();
  }

  // exact per-(case, candidate) maxima for the winner report; the per-candidate max
  // over the tile's cases goes into the running metric
  if constexpr (RGS > 1) {  // combine the row groups' maxima (all >= 0: ordered as uint)
#pragma unroll
    for (int i = 0; i < CPT; ++i)
#pragma unroll
      for (int jj = 0; jj < TPT; ++jj)
        if (gi > 0) atomicMax(&sAcc[tx * CPT + i][ty * TPT + jj], __float_as_uint(acc[i][jj]));
    __syncthreads();
#pragma unroll
    for (int i = 0; i < CPT; ++i)
#pragma unroll
      for (int jj = 0; jj < TPT; ++jj) acc[i][jj] = fmaxf(acc[i][jj], __uint_as_float(sAcc[tx * CPT + i][ty * TPT + jj]));
  }
  if (gi == 0) {
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = sCase[tx * CPT + i];
    if (c < 0) continue;
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
  }
  __syncthreads();  // the caller may reuse the shared buffers for the next tile
#undef SN
#undef SD
}

template <int CPT, int TPT, int TX, int TY, int RC, int RGS, int MINB>
__global__ void __launch_bounds__(TX* TY* RGS, MINB) k_top(DevGrid g, DevCfg cfg, Work w) {
  const int b = blockIdx.z;
  if (w.status[b] != 0) return;
  const int* list = w.ranked ? w.top + (size_t)b * w.ptop : nullptr;
  const int nlist = w.ranked ? w.ptop : min(w.ptop, g.N1);
  top_tile<CPT, TPT, TX, TY, RC, RGS>(g, w, b, list, nlist, blockIdx.y * (TPT * TY));
}

// Live cases, TOPC per item, every candidate tile: persistent over the queue.
template <int CPT, int TPT, int TX, int TY, int RC, int RGS, int MINB>
__global__ void __launch_bounds__(TX* TY* RGS, MINB) k_pairs(DevGrid g, DevCfg cfg, Work w) {
  const unsigned nq = *w.qcount;
  for (unsigned it = blockIdx.x; it < nq; it += gridDim.x) {
    const int2 q = w.queue[it];
    const int b = q.x, grp = q.y >> 16, tt = q.y & 0xffff;
    const int n = min(TOPC, w.lcnt[b] - grp * TOPC);
    top_tile<CPT, TPT, TX, TY, RC, RGS>(g, w, b, w.llist + (size_t)b * g.N1 + grp * TOPC, n, tt * (TPT * TY));
  }
}

// k_scale (the per-case, per-block screening scales) runs on the tensor cores: bdc_scale.cu.

// ---------------------------------------------------------------------------- k_live
// The screen proper, pair by pair: for a case outside the TOP tile, candidate t is live
// iff max_b (m0_b(t) + scale_bc |s(c,t)|) > lb(t) = max(running metric, penalty floor)
// (every TOP case, multi/injection case and the N-0 flows are already in m32).  A
// skipped pair is provably dominated: it cannot change the metric (solver.py:809-812).
// A case with any live candidate is evaluated for all of them (k_pairs): done[c] = 2 and
// listed in llist (k_queue then queues the lists in groups of TOPC x candidate tiles).
// With the screen off every feasible case is live.  CTA = (task, LC cases), a warp per
// 32 cases: lanes load the cases' flags and block scales (coalesced), then the warp walks
// its cases with lanes over candidates; lb and the block N-0 maxima are staged per CTA.
namespace {
constexpr int LC = 128;        // cases per k_live CTA (4 warps x 32)
constexpr int LV_TMAX = 1024;  // candidates staged in shared memory (larger T: global reads)
}
__global__ void __launch_bounds__(LC) k_live(DevGrid g, DevCfg cfg, Work w) {
  const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (w.status[b] != 0) return;
  const int T = w.T, N1 = g.N1;
  __shared__ float sLb[LV_TMAX];
  __shared__ float sM0[SB][LV_TMAX];
  const bool staged = T <= LV_TMAX;
  const float pen = w.nisl[b] > 0 ? (float)cfg.penalty : 0.f;
  const float* m32 = reinterpret_cast<const float*>(w.m32) + (size_t)b * T;
  const float* m0b = w.m0b + (size_t)b * SB * T;
  // case-level reject: max_b (max_t m0_b + scale_bc max_t |s(c,t)|) <= min_t lb(t)
  // bounds every pair of the case, so it is dominated without reading s(c, .)
  __shared__ unsigned sLbMin, sM0Max[SB];
  if (tid == 0) sLbMin = 0x7f800000u;
  if (tid < SB) sM0Max[tid] = 0u;
  __syncthreads();
  if (w.screen) {
    float lmin = __int_as_float(0x7f800000), mm[SB];
#pragma unroll
    for (int blk = 0; blk < SB; ++blk) mm[blk] = 0.f;
    for (int t = tid; t < T; t += LC) {
      const float lbt = fmaxf(m32[t], pen);
      lmin = fminf(lmin, lbt);
      if (staged) sLb[t] = lbt;
#pragma unroll
      for (int blk = 0; blk < SB; ++blk) {
        const float v = m0b[(size_t)blk * T + t];
        mm[blk] = fmaxf(mm[blk], v);
        if (staged) sM0[blk][t] = v;
      }
    }
    atomicMin(&sLbMin, __float_as_uint(lmin));
#pragma unroll
    for (int blk = 0; blk < SB; ++blk) atomicMax(&sM0Max[blk], __float_as_uint(mm[blk]));
  }
  __syncthreads();
  uint8_t* done = w.done + (size_t)b * N1;
  const int cl = blockIdx.x * LC + wid * 32 + lane;  // this lane's case
  bool cand = false;
  float scl[SB];
#pragma unroll
  for (int blk = 0; blk < SB; ++blk) scl[blk] = 0.f;
  if (cl < N1) {
    const bool top = w.ranked ? done[cl] != 0 : cl < w.ptop;
    cand = !top && w.sc_ok[(size_t)b * N1 + cl] != 0;
    if (cand && w.screen) {
      const float smx = smax_at(g, w, b, cl);
      float coarse = 0.f;
#pragma unroll
      for (int blk = 0; blk < SB; ++blk) {
        scl[blk] = w.scale[((size_t)b * SB + blk) * N1 + cl];
        coarse = fmaxf(coarse, __uint_as_float(sM0Max[blk]) + scl[blk] * smx);
      }
      if (coarse <= __uint_as_float(sLbMin)) cand = false;
    }
  }
  bool mylive = cand && !w.screen;
  unsigned todo = __ballot_sync(0xffffffffu, cand && w.screen);
  // two cases per pass: their s rows are loaded together, so each pass waits on one memory
  // latency for two cases (the loop is latency-bound); a case's verdict is the same --
  // "live" once any candidate's bound exceeds the lower bound, extra chunks cannot undo it
  while (todo) {
    const int k1 = __ffs(todo) - 1;
    todo &= todo - 1;
    int k2 = -1;
    if (todo) {
      k2 = __ffs(todo) - 1;
      todo &= todo - 1;
    }
    const int c1 = blockIdx.x * LC + wid * 32 + k1;
    const int c2 = k2 >= 0 ? blockIdx.x * LC + wid * 32 + k2 : c1;
    float sk1[SB], sk2[SB];
#pragma unroll
    for (int blk = 0; blk < SB; ++blk) {
      sk1[blk] = __shfl_sync(0xffffffffu, scl[blk], k1);
      sk2[blk] = __shfl_sync(0xffffffffu, scl[blk], k2 >= 0 ? k2 : k1);
    }
    // s(c, .): a row of s32, or the N-0 row of the outaged branch times its rating
    const float* sc1 = g.s_mon ? w.n0s + ((size_t)b * g.M + g.sc_pos[c1]) * T : w.s32 + ((size_t)b * N1 + c1) * T;
    const float* sc2 = g.s_mon ? w.n0s + ((size_t)b * g.M + g.sc_pos[c2]) * T : w.s32 + ((size_t)b * N1 + c2) * T;
    const float srat1 = g.s_mon ? g.sc_rat[c1] : 1.f;
    const float srat2 = g.s_mon ? g.sc_rat[c2] : 1.f;
    bool live1 = false, live2 = k2 < 0;
    for (int t0 = 0; t0 < T && !(live1 && live2); t0 += 32) {
      const int t = t0 + lane;
      bool lt1 = false, lt2 = false;
      if (t < T) {
        const float v1 = sc1[t], v2 = sc2[t];
        const float as1 = g.s_mon ? fabsf(v1 * srat1) : fabsf(v1);
        const float as2 = g.s_mon ? fabsf(v2 * srat2) : fabsf(v2);
        float b1 = 0.f, b2 = 0.f;
#pragma unroll
        for (int blk = 0; blk < SB; ++blk) {
          const float m0v = staged ? sM0[blk][t] : m0b[(size_t)blk * T + t];
          b1 = fmaxf(b1, m0v + sk1[blk] * as1);
          b2 = fmaxf(b2, m0v + sk2[blk] * as2);
        }
        const float lbt = staged ? sLb[t] : fmaxf(m32[t], pen);
        lt1 = b1 > lbt;
        lt2 = k2 >= 0 && b2 > lbt;
      }
      live1 = live1 || __any_sync(0xffffffffu, lt1);
      live2 = live2 || __any_sync(0xffffffffu, lt2);
    }
    if (lane == k1) mylive = live1;
    if (k2 >= 0 && lane == k2) mylive = live2;
  }
  if (cl < N1 && (cand || !w.ranked)) {
    // TOP cases keep done = 1 (k_topk); unranked tasks have no k_topk pass
    if (!(w.ranked ? false : cl < w.ptop)) done[cl] = mylive ? 2 : 0;
  }
  const unsigned lb = __ballot_sync(0xffffffffu, mylive);
  if (lb) {
    int base = 0;
    if (lane == 0) base = atomicAdd(&w.lcnt[b], __popc(lb));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (mylive) w.llist[(size_t)b * N1 + base + __popc(lb & ((1u << lane) - 1u))] = cl;
  }
}

// Queue the live lists: per task, groups of TOPC cases x candidate tiles (k_pairs counts
// the evaluated pairs as it goes).
__global__ void k_queue(DevGrid g, Work w) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= w.Wb || w.status[b] != 0) return;
  const int n = w.lcnt[b];
  if (n == 0) return;
  const int TT = top_tile_cands(w.T), ntt = (w.T + TT - 1) / TT, ng = (n + TOPC - 1) / TOPC;
  const unsigned q0 = atomicAdd(w.qcount, (unsigned)(ng * ntt));
  for (int i = 0; i < ng * ntt; ++i) w.queue[q0 + i] = make_int2(b, ((i / ntt) << 16) | (i % ntt));
}

namespace {
template <int CPT, int TPT, int TX, int TY, int RC, int RGS, int MINB>
void launch_top_t(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  constexpr int NC = CPT * TX, TT = TPT * TY;
  static_assert(NC == TOPC, "TOP tile = TOPC cases");
  const size_t dyn = ((size_t)NC * w.rs + 2 * (size_t)w.rs * RC) * sizeof(double) +
                     (2 * (size_t)RC * TT + 2 * (size_t)RC * NC) * sizeof(float);
  smem_opt_in((const void*)k_top<CPT, TPT, TX, TY, RC, RGS, MINB>, (int)dyn);
  dim3 grid(1, (w.T + TT - 1) / TT, w.Wb);
  k_top<CPT, TPT, TX, TY, RC, RGS, MINB><<<grid, TX * TY * RGS, dyn, s>>>(g, c, w);
}

template <int CPT, int TPT, int TX, int TY, int RC, int RGS, int MINB>
void launch_pairs_t(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  constexpr int NC = CPT * TX, TT = TPT * TY;
  const size_t dyn = ((size_t)NC * w.rs + 2 * (size_t)w.rs * RC) * sizeof(double) +
                     (2 * (size_t)RC * TT + 2 * (size_t)RC * NC) * sizeof(float);
  int per_sm = 1, nsm = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  smem_opt_in((const void*)k_pairs<CPT, TPT, TX, TY, RC, RGS, MINB>, (int)dyn);
  // persistent: as many CTAs as fit at once for this rank stride's shared memory
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pairs<CPT, TPT, TX, TY, RC, RGS, MINB>, TX * TY * RGS, dyn);
  k_pairs<CPT, TPT, TX, TY, RC, RGS, MINB><<<nsm * (per_sm > 0 ? per_sm : 1), TX * TY * RGS, dyn, s>>>(g, c, w);
}

// tile shapes: 16 cases x top_tile_cands(T) candidates (bdc_device.cuh)
void launch_top(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  // thread tile 2 cases x 8 or 4 candidates; 2 or 4 row groups split each chunk's rows
  if (w.T >= 96) launch_top_t<2, 8, 8, 16, 64, 2, 3>(g, c, w, s);       // 16 cases x 128 candidates
  else if (w.T >= 48) launch_top_t<2, 4, 8, 16, 64, 2, 3>(g, c, w, s);  // 16 x 64
  else launch_top_t<2, 4, 8, 8, 64, 4, 3>(g, c, w, s);                 // 16 x 32
}
void launch_pairs(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  if (w.T >= 96) launch_pairs_t<2, 8, 8, 16, 64, 2, 3>(g, c, w, s);
  else if (w.T >= 48) launch_pairs_t<2, 4, 8, 16, 64, 2, 3>(g, c, w, s);
  else launch_pairs_t<2, 4, 8, 8, 64, 4, 3>(g, c, w, s);
}
}  // namespace

// ev (optional): ev[1], ev[2], ev[3] are recorded after the scales, the top-k and the
// TOP tile (stage boundaries of bdc_solve's timing).
void launch_single_top(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s, cudaEvent_t* ev) {
  auto mark = [&](int i) { if (ev) cudaEventRecord(ev[i], s); };
  if (g.N1 == 0 || g.M == 0) {
    mark(0); mark(1); mark(2);
    return;
  }
  // per-case block scales and ranking key, then the TOP tile by key
  if (w.ranked) launch_scale(g, w, s);
  mark(0);
  if (w.ranked) launch_topk(g, w, s);
  mark(1);
  launch_top(g, c, w, s);
  mark(2);
}

void launch_single_screen(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  if (g.N1 == 0 || g.M == 0) return;
  if (g.N1 > w.ptop) {
    k_live<<<dim3((g.N1 + LC - 1) / LC, w.Wb), LC, 0, s>>>(g, c, w);
    k_queue<<<(w.Wb + 255) / 256, 256, 0, s>>>(g, w);
    launch_pairs(g, c, w, s);
  }
}

int single_launches(const DevGrid& g, const Work& w) {
  if (g.N1 == 0 || g.M == 0) return 0;
  return (w.ranked ? 2 : 0) + 1 + (g.N1 > w.ptop ? 3 : 0);
}

}  // namespace bdc
