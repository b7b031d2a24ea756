// bdc_flows.cu -- Kernels 2-4: N-0 contraction, fused N-1 screening, winner selection.
//
//   k_n0      N-0 flows of every candidate on the monitored rows,
//             n0 = f0 + B'' y_t (FP64, the rank-r form of `_candidate_base_flows`,
//             solver.py:575-595), written once as FP32 n0/rating (the only
//             per-task tensor the N-1 stage streams) and folded into the metric.
//   k_single  THE hot kernel.  Single-branch N-1 for every (case, candidate)
//             pair of a task, fused: forms LODF columns on the fly from the
//             shared base D_base and the task's rank-r factors
//             (L = (D_base + B'' W^T) / den, solver.py:474-485), applies the
//             outage update F = n0 + L n0[r_c] (solver.py:612-613), takes
//             |F|/rating and max-reduces over monitored rows and cases into
//             the per-candidate metric (solver.py:625-631, agg_m :235-252).
//             The (case x candidate x branch) tensor never leaves registers;
//             row chunks of n0/rating and D_base stream through shared memory
//             with cp.async double buffering.
//   k_other   multi-branch (MODF, solver.py:614-618) and injection
//             (solver.py:619-622) contingencies of one task, same fusion.
//   k_select  islanding penalty floor and first-index argmin (solver.py:804-823).
#include "bdc_device.cuh"

namespace bdc {

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// 4-byte async copy global->shared; src_bytes = 0 zero-fills.
__device__ __forceinline__ void cp4(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(ok ? 4 : 0));
}
__device__ __forceinline__ void cp8(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

constexpr int N0_TB = 128;
constexpr int N0_RB = 32;

}  // namespace

// ------------------------------------------------------------------------------- k_n0
__global__ void __launch_bounds__(N0_TB) k_n0(DevGrid g, Work w) {
  const int b = blockIdx.z, p0 = blockIdx.y * N0_RB, tid = threadIdx.x;
  const int t = blockIdx.x * N0_TB + tid;
  if (w.status[b] != 0) return;
  const int rs = w.rs, rt = w.rank[b], T = w.T, R = g.R, M = g.M;
  __shared__ double sB[RMAX][N0_RB];
  __shared__ double sF[N0_RB], sI[N0_RB];
  __shared__ int sdead[RMAX];
  const int nd = w.ndead[b];
  if (tid < nd) sdead[tid] = w.dead[(size_t)b * RMAX + tid];
  __syncthreads();
  for (int idx = tid; idx < rt * N0_RB; idx += N0_TB) {
    const int j = idx / N0_RB, pp = idx % N0_RB, p = p0 + pp;
    sB[j][pp] = p < M ? w.Bm[((size_t)b * rs + j) * R + g.mon_row[p]] : 0.0;
  }
  for (int pp = tid; pp < N0_RB; pp += N0_TB) {
    const int p = p0 + pp;
    const int row = p < M ? g.mon_row[p] : -1;
    const bool live = row >= 0 && !is_dead(sdead, nd, row);
    sF[pp] = live ? g.f0[row] : 0.0;
    sI[pp] = live ? g.inv_rating[p] : 0.0;  // dead rows: flow exactly 0
  }
  __syncthreads();
  if (t >= T) return;
  double y[RMAX];
#pragma unroll
  for (int j = 0; j < RMAX; ++j) y[j] = (j < rt) ? w.Y[((size_t)b * rs + j) * T + t] : 0.0;
  float mx = 0.f;
  const int pend = min(M, p0 + N0_RB);
  for (int p = p0; p < pend; ++p) {
    const int pp = p - p0;
    double v = sF[pp];
#pragma unroll
    for (int j = 0; j < RMAX; ++j)
      if (j < rt) v = fma(sB[j][pp], y[j], v);
    const float sc = (float)(v * sI[pp]);
    w.n0s[((size_t)b * M + p) * T + t] = sc;
    mx = fmaxf(mx, fabsf(sc));
  }
  atomic_max_pos(&w.m32[(size_t)b * T + t], mx);
}

// --------------------------------------------------------------------------- k_single
// Thread tile: CPT cases x TPT candidates; CTA tile NC = CPT*TX cases x
// TT = TPT*TY candidates; monitored rows streamed RC at a time through a
// cp.async double buffer (n0/rating chunk [RC][TT], D_base chunk [RC][NC],
// B'' rows [rt][RC]).
template <int CPT, int TPT, int TX, int TY, int RC, int MINB>
__global__ void __launch_bounds__(TX* TY, MINB) k_single(DevGrid g, Work w) {
  constexpr int NTH = TX * TY, NC = CPT * TX, TT = TPT * TY;
  const int b = blockIdx.z;
  if (w.status[b] != 0) return;
  const int c0 = blockIdx.x * NC, t0 = blockIdx.y * TT;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int rs = w.rs, rt = w.rank[b], T = w.T, M = g.M, N1 = g.N1, R = g.R;
  // dynamic: [sW NC*rs f64][sBb 2*rs*RC f64][sN 2*RC*TT f32][sD 2*RC*NC f32]
  extern __shared__ __align__(16) unsigned char dsm[];
  double* sW = reinterpret_cast<double*>(dsm);   // [NC][rt]
  double* sBb = sW + NC * rs;                    // [2][rt][RC] B'' rows of the chunk
  float* sNp = reinterpret_cast<float*>(sBb + 2 * rs * RC);
  float* sDp = sNp + 2 * RC * TT;
#define SN(bf, r_, t_) sNp[((bf) * RC + (r_)) * TT + (t_)]
#define SD(bf, r_, c_) sDp[((bf) * RC + (r_)) * NC + (c_)]
  __shared__ double sInvDen[NC];
  __shared__ int sRowC[NC];
  __shared__ double sInv[2][RC];
  __shared__ int sRow[2][RC];
  __shared__ __align__(16) float sL[RC][NC];
  __shared__ int sdead[RMAX];
  const int nd = w.ndead[b];
  const double* Bm = w.Bm + (size_t)b * rs * R;
  const float* n0s = w.n0s + (size_t)b * M * T;
  const bool vecN = (T % 4) == 0 && (t0 % 4) == 0;
  const bool vecD = (N1 % 4) == 0;

  if (tid < nd) sdead[tid] = w.dead[(size_t)b * RMAX + tid];
  for (int idx = tid; idx < NC * rt; idx += NTH) {
    const int cc = idx / rt, j = idx % rt, c = c0 + cc;
    sW[j * NC + cc] = c < N1 ? w.Wsc[((size_t)b * N1 + c) * rs + j] : 0.0;
  }
  for (int cc = tid; cc < NC; cc += NTH) {
    const int c = c0 + cc;
    const bool ok = c < N1 && w.sc_ok[(size_t)b * N1 + c];
    sInvDen[cc] = ok ? 1.0 / w.den[(size_t)b * N1 + c] : 0.0;
    sRowC[cc] = c < N1 ? g.sc_row[c] : -1;
  }
  __syncthreads();

  // stage one row chunk (async): row ids + 1/rating, B'' rows, n0/rating, D_base
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
    if (vecN) {
      for (int idx = tid; idx < RC * (TT / 4); idx += NTH) {
        const int rr = idx / (TT / 4), q = idx % (TT / 4), m = m0 + rr, t = t0 + 4 * q;
        const bool ok = m < M && t < T;
        cp16(&SN(buf, rr, 4 * q), ok ? &n0s[(size_t)m * T + t] : n0s, ok);
      }
    } else {
      for (int idx = tid; idx < RC * TT; idx += NTH) {
        const int rr = idx / TT, tt = idx % TT, m = m0 + rr, t = t0 + tt;
        const bool ok = m < M && t < T;
        cp4(&SN(buf, rr, tt), ok ? &n0s[(size_t)m * T + t] : n0s, ok);
      }
    }
    if (vecD) {
      for (int idx = tid; idx < RC * (NC / 4); idx += NTH) {
        const int rr = idx / (NC / 4), q = idx % (NC / 4), m = m0 + rr, c = c0 + 4 * q;
        const bool ok = m < M && c < N1;
        cp16(&SD(buf, rr, 4 * q), ok ? &g.D32[(size_t)m * N1 + c] : g.D32, ok);
      }
    } else {
      for (int idx = tid; idx < RC * NC; idx += NTH) {
        const int rr = idx / NC, cc = idx % NC, m = m0 + rr, c = c0 + cc;
        const bool ok = m < M && c < N1;
        cp4(&SD(buf, rr, cc), ok ? &g.D32[(size_t)m * N1 + c] : g.D32, ok);
      }
    }
    cp_commit();
  };

  issue(0, 0);

  // s(c,t) = n0[r_c][t] from the factors (FP64 -> FP32), computed cooperatively
  // RC cases at a time into the (still idle) second n0 buffer while chunk 0 is in flight
  float acc[CPT][TPT], sv[CPT][TPT];
  {
    const double* Y = w.Y + (size_t)b * rs * T;
    for (int cb = 0; cb < NC; cb += RC) {
      for (int idx = tid; idx < RC * TT; idx += NTH) {
        const int cc = cb + idx / TT, tt = idx % TT, t = t0 + tt;
        const int row = sRowC[cc];
        float sval = 0.f;
        if (row >= 0 && t < T && !is_dead(sdead, nd, row)) {
          double v = g.f0[row];
          for (int j = 0; j < rt; ++j) v = fma(Bm[(size_t)j * R + row], Y[(size_t)j * T + t], v);
          sval = (float)v;
        }
        SN(1, idx / TT, tt) = sval;
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const int cc = tx * CPT + i;
        if (cc >= cb && cc < cb + RC) {
#pragma unroll
          for (int jj = 0; jj < TPT; ++jj) sv[i][jj] = SN(1, cc - cb, ty * TPT + jj);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < CPT; ++i)
#pragma unroll
      for (int jj = 0; jj < TPT; ++jj) acc[i][jj] = 0.f;
  }

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
    __syncthreads();
  }
  // per-(case, candidate) maxima: the winner report's exact pruning bound
  {
    float* cm = w.cmax + (size_t)b * (N1 + g.NM + g.NI) * T;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int c = c0 + tx * CPT + i;
      if (c >= N1) continue;
#pragma unroll
      for (int jj = 0; jj < TPT; ++jj) {
        const int t = t0 + ty * TPT + jj;
        if (t < T) cm[(size_t)c * T + t] = acc[i][jj];
      }
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

// ---------------------------------------------------------------------------- k_other
// One CTA per (task, candidate tile): every multi-branch and injection case of
// the task, FP32 like k_single.  The update kernel already laid the cases out
// as correction terms, F = n0 + sum_j Lo[r][j] So[j][t] (MODF columns with the
// pre-outage flows of the outaged rows, or the injection column with 1 and the
// candidate's slot bit), so this is a pure stream over monitored-row chunks.
namespace {
constexpr int OT = 256;   // threads
constexpr int OTT = 64;   // candidates per CTA
constexpr int ORC = 32;   // monitored rows per chunk
constexpr int OQG = OT / OTT;  // case groups
}  // namespace

__global__ void __launch_bounds__(OT) k_other(DevGrid g, Work w) {
  const int b = blockIdx.y, tid = threadIdx.x, t0 = blockIdx.x * OTT;
  if (w.status[b] != 0) return;
  const int T = w.T, M = g.M, NTM = w.NTERM, nq = g.NM + g.NI;
  extern __shared__ __align__(16) float osm[];
  float* sS = osm;                        // [NTM][OTT]
  float* sLo = sS + NTM * OTT;            // [2][ORC][NTM]
  float* sN = sLo + 2 * ORC * NTM;        // [2][ORC][OTT]
  const float* Lo = w.Lo + (size_t)b * M * NTM;
  const float* n0s = w.n0s + (size_t)b * M * T;
  const int tt = tid % OTT, qg = tid / OTT, t = t0 + tt;
  for (int idx = tid; idx < NTM * OTT; idx += OT) {
    const int j = idx / OTT, u = t0 + idx % OTT;
    sS[idx] = u < T ? w.So[((size_t)b * NTM + j) * T + u] : 0.f;
  }
  auto issue = [&](int m0, int buf) {
    for (int idx = tid; idx < ORC * NTM; idx += OT) {
      const int rr = idx / NTM, j = idx % NTM, m = m0 + rr;
      const bool ok = m < M;
      cp4(&sLo[(buf * ORC + rr) * NTM + j], ok ? &Lo[(size_t)m * NTM + j] : Lo, ok);
    }
    for (int idx = tid; idx < ORC * OTT; idx += OT) {
      const int rr = idx / OTT, u = idx % OTT, m = m0 + rr;
      const bool ok = m < M && t0 + u < T;
      cp4(&sN[(buf * ORC + rr) * OTT + u], ok ? &n0s[(size_t)m * T + t0 + u] : n0s, ok);
    }
    cp_commit();
  };
  // this thread's cases: q = qg, qg + OQG, ...; islanded multi cases are skipped
  constexpr int QMAX = 16;
  float acc[QMAX];
#pragma unroll
  for (int k = 0; k < QMAX; ++k) acc[k] = 0.f;
  issue(0, 0);
  const int nchunks = (M + ORC - 1) / ORC;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) {
      issue((ch + 1) * ORC, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const float* L = &sLo[buf * ORC * NTM];
    const float* N = &sN[buf * ORC * OTT];
    int k = 0;
    for (int q = qg; q < nq && k < QMAX; q += OQG, ++k) {
      int st, m;
      if (q < g.NM) { st = g.mc_start[q]; m = g.mc_start[q + 1] - st; }
      else { st = g.NMB + 2 * (q - g.NM); m = 2; }
      float a = acc[k];
      for (int rr = 0; rr < ORC; ++rr) {
        float f = N[rr * OTT + tt];
        for (int j = 0; j < m; ++j) f = fmaf(L[rr * NTM + st + j], sS[(st + j) * OTT + tt], f);
        a = fmaxf(a, fabsf(f));
      }
      acc[k] = a;
    }
    __syncthreads();
  }
  // per-(case, candidate) maxima, then the per-candidate max over cases
  float* cm = w.cmax + (size_t)b * (g.N1 + nq) * T;
  float mx = 0.f;
  int k = 0;
  for (int q = qg; q < nq && k < QMAX; q += OQG, ++k) {
    const bool ok = q >= g.NM || w.mc_ok[(size_t)b * g.NM + q];
    const float v = ok ? acc[k] : 0.f;
    if (t < T) cm[(size_t)(g.N1 + q) * T + t] = v;
    mx = fmaxf(mx, v);
  }
  float* sMax = sN;  // reuse
  if (tid < OTT) sMax[tid] = 0.f;
  __syncthreads();
  atomicMax(reinterpret_cast<unsigned*>(&sMax[tt]), __float_as_uint(mx));
  __syncthreads();
  if (tid < OTT && t0 + tid < T) atomic_max_pos(&w.m32[(size_t)b * T + t0 + tid], sMax[tid]);
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
  if (g.M == 0) return;
  dim3 grid((w.T + N0_TB - 1) / N0_TB, (g.M + N0_RB - 1) / N0_RB, w.Wb);
  k_n0<<<grid, N0_TB, 0, s>>>(g, w);
}

template <int CPT, int TPT, int TX, int TY, int RC, int MINB>
static void launch_single_t(const DevGrid& g, const Work& w, cudaStream_t s) {
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
    cudaFuncGetAttributes(&fa, k_single<CPT, TPT, TX, TY, RC, MINB>);
    max_dyn = optin - (int)fa.sharedSizeBytes;
    cudaFuncSetAttribute(k_single<CPT, TPT, TX, TY, RC, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
  }
  dim3 grid((g.N1 + NC - 1) / NC, (w.T + TT - 1) / TT, w.Wb);
  k_single<CPT, TPT, TX, TY, RC, MINB><<<grid, TX * TY, dyn, s>>>(g, w);
}

void launch_single(const DevGrid& g, const Work& w, cudaStream_t s) {
  if (g.N1 == 0 || g.M == 0) return;
  if (w.T >= 96) launch_single_t<2, 16, 32, 8, 32, 2>(g, w, s);      // 64 cases x 128 candidates
  else if (w.T >= 48) launch_single_t<2, 8, 32, 8, 32, 3>(g, w, s);  // 64 x 64
  else if (w.T >= 24) launch_single_t<4, 4, 32, 8, 32, 3>(g, w, s);  // 128 x 32
  else if (w.T >= 12) launch_single_t<4, 4, 64, 4, 32, 3>(g, w, s);  // 256 x 16
  else launch_single_t<4, 2, 64, 4, 32, 3>(g, w, s);                 // 256 x 8
}

void launch_other(const DevGrid& g, const Work& w, cudaStream_t s) {
  const int nq = g.NM + g.NI;
  if (nq == 0 || g.M == 0) return;
  const size_t dyn = ((size_t)w.NTERM * OTT + 2 * (size_t)ORC * w.NTERM + 2 * (size_t)ORC * OTT) * 4;
  static int max_dyn = -1;
  if (max_dyn < 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    max_dyn = optin;
    cudaFuncSetAttribute(k_other, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
  }
  dim3 grid((w.T + OTT - 1) / OTT, w.Wb);
  k_other<<<grid, OT, dyn, s>>>(g, w);
}

void launch_select(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  const int threads = 256;
  const long long total = (long long)w.Wb * 32;
  k_select<<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(g, c, w);
}

}  // namespace bdc
