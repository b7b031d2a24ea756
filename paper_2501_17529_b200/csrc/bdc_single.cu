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
//   pass TOP     the ptop cases with the largest bound max_t(m0(t) + scale_c |s(c,t)|)
//                (selected by the update kernel) are evaluated first, for every
//                candidate -- the reference likewise visits likely-binding cases first;
//   pass SCREEN  every other tile; a pair whose bound cannot exceed the running
//                metric of its candidate cannot change it and is skipped, per CTA
//                tile and per warp.  Skipped pairs store -bound in cmax (an upper
//                bound the winner report prunes with); evaluated pairs store the
//                exact FP32 max.
#include "bdc_device.cuh"

namespace bdc {

enum { PASS_SCREEN = 0, PASS_TOP = 1, PASS_SCALE = 2 };

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
  constexpr int LR = PASS == PASS_SCALE ? 1 : RC;  // the scale pass keeps no LODF tile
  __shared__ __align__(16) float sL[LR][NC];
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
      sv[i][jj] = (PASS != PASS_SCALE && c >= 0 && t < T) ? s32[(size_t)c * T + t] : 0.f;
      acc[i][jj] = 0.f;
    }
  }
  bool warp_alive = PASS != PASS_SCALE;
  float colmax = 0.f;  // PASS_SCALE: running max |L|/rating of this thread's column
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
    if constexpr (PASS != PASS_SCALE && TT % 4 == 0) {
      if (vecN) {
        constexpr int TQ = TT / 4;
        for (int idx = tid; idx < RC * TQ; idx += NTH) {
          const int rr = idx / TQ, q = idx % TQ, m = m0 + rr, t = t0 + 4 * q;
          const bool ok = m < M && t < T;
          cp16(&SN(buf, rr, 4 * q), ok ? &n0s[(size_t)m * T + t] : n0s, ok);
        }
      }
    }
    if (PASS != PASS_SCALE && !vecN) {
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
          if constexpr (PASS == PASS_SCALE) colmax = fmaxf(colmax, fabsf(lv));
          else sL[rr][cc] = lv;
        }
      }
    }
    __syncthreads();
    if (PASS != PASS_SCALE && warp_alive) {
      const int rend = min(RC, M - ch * RC);
      if (rend == RC) {
#pragma unroll 4
        for (int rr = 0; rr < RC; ++rr) {
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

  if constexpr (PASS == PASS_SCALE) {
    // scale_c = max over the rows of |L(r,c)|/rating_r (exact FP32 of the values the
    // sweep multiplies), then the ranking key bkey_c = max_t(m0(t) + scale_c |s(c,t)|)
    float* sMax = sDp;  // reuse the (idle) D_base buffer
    for (int cc = tid; cc < NC; cc += NTH) sMax[cc] = 0.f;
    __syncthreads();
    atomicMax(reinterpret_cast<unsigned*>(&sMax[tid % NC]), __float_as_uint(colmax));
    __syncthreads();
    const int lane = tid & 31, wid = tid >> 5;
    const float* m0 = w.m0 + (size_t)b * T;
    for (int cc = wid; cc < NC; cc += NTH / 32) {
      const int c = sCase[cc];
      if (c < 0) continue;
      const float sc = sMax[cc] * (1.f + 1e-6f);
      float bm = 0.f;
      for (int t = lane; t < T; t += 32) bm = fmaxf(bm, m0[t] + sc * fabsf(s32[(size_t)c * T + t]));
      for (int o = 16; o; o >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
      if (lane == 0) {
        w.scale[(size_t)b * N1 + c] = sc;
        w.bkey[(size_t)b * N1 + c] = sInvDen[cc] != 0.0 ? __float_as_uint(bm) : 0u;
      }
    }
    return;
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
  dim3 grid(ctiles, PASS == PASS_SCALE ? 1 : (w.T + TT - 1) / TT, w.Wb);
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
    // exact per-case scale and ranking key, then the top tile by key
    launch_single_t<1, 1, 256, 1, 32, 3, PASS_SCALE>(g, c, w, s);
    launch_topk(g, w, s);
  }
  launch_pass<PASS_TOP>(g, c, w, s);
  if (g.N1 > w.ptop) launch_pass<PASS_SCREEN>(g, c, w, s);
}

}  // namespace bdc
