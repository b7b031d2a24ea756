// bdc_flows.cu -- the multi-branch / injection N-1 stage and winner selection.
//
//   k_other   multi-branch (MODF, solver.py:614-618) and injection (solver.py:619-622)
//             contingencies of every candidate, fused: F = n0 + sum_j Lo So,
//             |F|/rating, max over monitored rows, per-(case, candidate) maxima for the
//             report and the per-candidate max folded into the metric (agg_m,
//             solver.py:235-252).  Nothing of size (case x candidate x branch) is written.
//   k_select  islanding penalty floor and first-index argmin (solver.py:804-823).
//
// The single-branch N-1 stage (the hot path) is bdc_single.cu; the N-0 contraction
// is fused into the update kernel (bdc_update.cu).
#include "bdc_device.cuh"

#include <cstdlib>

namespace bdc {

// ---------------------------------------------------------------------------- k_other
// Multi-branch (MODF, solver.py:614-618) and injection (solver.py:619-622)
// contingencies of one task, FP32 like k_single.  The update kernel laid every
// case out as MT zero-padded correction terms, F = n0 + sum_j Lo[r][q][j] So[q][j][t]
// (MODF columns with the pre-outage flows of the outaged rows, or the injection
// column with 1 and the candidate's slot bit), so this is a pure stream over
// monitored-row chunks.  CTA = (task, tile of 32*TPT candidates); lane = TPT
// consecutive candidates for a batch of QC cases (the multipliers So in registers, the
// n0 loads shared by the batch's cases); the 8 warps split each chunk's row pairs and
// their maxima are combined in shared memory at the end of the batch.
namespace {
constexpr int OT = 256;        // threads
constexpr int OW = OT / 32;    // warps (row groups)
constexpr int ORC = 64;        // monitored rows per chunk
}  // namespace

template <int MT, int QC, int TPT, bool LIST>  // LIST: the cases k_oscreen left, else all
__global__ void __launch_bounds__(OT) k_other(DevGrid g, Work w) {
  constexpr int TT = 32 * TPT, LQ = QC * MT;  // candidates per CTA, Lo floats per row
  const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int t0 = blockIdx.x * TT;
  if (w.status[b] != 0) return;
  const int T = w.T, M = g.M, NQ = g.NM + g.NI;
  extern __shared__ __align__(16) float osm[];
  float* sN = osm;                   // [2][ORC][TT]  n0 / rating
  float* sL = sN + 2 * ORC * TT;     // [2][ORC][LQ]  correction columns of the batch
  __shared__ unsigned sAcc[QC][TT];  // the row groups' maxima (>= 0: ordered as uint)
  __shared__ float sMax[TT];
  const float* Lo = w.Lo + (size_t)b * M * NQ * MT;
  const float* n0s = w.n0s + (size_t)b * M * T;
  const float* So = w.So + (size_t)b * NQ * MT * T;
  float* cm = w.cmax + (size_t)b * (g.N1 + NQ) * T;
  // the cases k_oscreen left (ascending), or all of them
  const int* ol = w.olist + (size_t)b * NQ;
  const int nq = LIST ? w.ocnt[b] : NQ;
  const bool vecN = (T % 4) == 0;
  for (int i = tid; i < TT; i += OT) sMax[i] = 0.f;

  for (int qb = 0; qb < nq; qb += QC) {
    const int nqb = min(QC, nq - qb), LW = nqb * MT;  // cases / Lo floats of this batch
    float sv[QC][MT][TPT], acc[QC][TPT];
#pragma unroll
    for (int k = 0; k < QC; ++k) {
#pragma unroll
      for (int j = 0; j < MT; ++j)
#pragma unroll
        for (int i = 0; i < TPT; ++i) {
          const int t = t0 + lane * TPT + i;
          sv[k][j][i] = (k < nqb && t < T) ? So[((size_t)(LIST ? ol[qb + k] : qb + k) * MT + j) * T + t] : 0.f;
        }
#pragma unroll
      for (int i = 0; i < TPT; ++i) acc[k][i] = 0.f;
    }
    for (int i = tid; i < QC * TT; i += OT) (&sAcc[0][0])[i] = 0u;
    auto issue = [&](int m0, int buf) {
      if (vecN) {
        for (int idx = tid; idx < ORC * (TT / 4); idx += OT) {
          const int rr = idx / (TT / 4), u = 4 * (idx % (TT / 4)), m = m0 + rr;
          const bool ok = m < M && t0 + u < T;
          cp16(&sN[(buf * ORC + rr) * TT + u], ok ? &n0s[(size_t)m * T + t0 + u] : n0s, ok);
        }
      } else {
        for (int idx = tid; idx < ORC * TT; idx += OT) {
          const int rr = idx / TT, u = idx % TT, m = m0 + rr;
          const bool ok = m < M && t0 + u < T;
          cp4(&sN[(buf * ORC + rr) * TT + u], ok ? &n0s[(size_t)m * T + t0 + u] : n0s, ok);
        }
      }
      // LW = nqb * MT is a multiple of 2; rows of Lo are NQ*MT floats (8-byte aligned)
      for (int idx = tid; idx < ORC * (LW / 2); idx += OT) {
        const int rr = idx / (LW / 2), u = 2 * (idx % (LW / 2)), m = m0 + rr;
        const bool ok = m < M;
        const int q = LIST ? ol[qb + u / MT] : qb + u / MT;
        cp8(&sL[(buf * ORC + rr) * LQ + u], ok ? &Lo[((size_t)m * NQ + q) * MT + (u % MT)] : Lo, ok);
      }
      cp_commit();
    };
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
      // rows past M were staged as zeros (n0 = 0, Lo = 0): |F| = 0 there, so the paired
      // loop runs over whole chunks; two rows per step: FFMA2 over the row pair (same
      // rounding as fmaf), one FMNMX3 per accumulator
      const int rend = min(ORC, (M - ch * ORC + 1) & ~1);
      for (int rr = 2 * wid; rr < rend; rr += 2 * OW) {
        const float* n0r = &sN[(buf * ORC + rr) * TT + lane * TPT];
        float2 n[TPT];
        if constexpr (TPT == 2) {
          const float2 a = *reinterpret_cast<const float2*>(n0r);
          const float2 c = *reinterpret_cast<const float2*>(n0r + TT);
          n[0] = make_float2(a.x, c.x);
          n[1] = make_float2(a.y, c.y);
        } else {
#pragma unroll
          for (int i = 0; i < TPT; ++i) n[i] = make_float2(n0r[i], n0r[TT + i]);
        }
        const float* lrow0 = &sL[(buf * ORC + rr) * LQ];
#pragma unroll
        for (int k = 0; k < QC; ++k) {
          if (k >= nqb) break;  // uniform
          float2 l[MT];
#pragma unroll
          for (int j = 0; j < MT; j += 2) {
            const float2 a = *reinterpret_cast<const float2*>(&lrow0[k * MT + j]);
            const float2 c = *reinterpret_cast<const float2*>(&lrow0[LQ + k * MT + j]);
            l[j] = make_float2(a.x, c.x);
            l[j + 1] = make_float2(a.y, c.y);
          }
#pragma unroll
          for (int i = 0; i < TPT; ++i) {
            float2 f = n[i];
#pragma unroll
            for (int j = 0; j < MT; ++j) f = __ffma2_rn(l[j], make_float2(sv[k][j][i], sv[k][j][i]), f);
            acc[k][i] = max3abs(acc[k][i], f.x, f.y);
          }
        }
      }
      __syncthreads();
    }
    // combine the row groups, then per-(case, candidate) maxima (islanded multi cases
    // contribute 0) and the candidate max
#pragma unroll
    for (int k = 0; k < QC; ++k) {
      if (k >= nqb) break;
#pragma unroll
      for (int i = 0; i < TPT; ++i) atomicMax(&sAcc[k][lane * TPT + i], __float_as_uint(acc[k][i]));
    }
    __syncthreads();
    for (int idx = tid; idx < nqb * TT; idx += OT) {
      const int k = idx / TT, u = idx % TT, q = LIST ? ol[qb + k] : qb + k, t = t0 + u;
      const bool ok = q >= g.NM || w.mc_ok[(size_t)b * g.NM + q];
      const float v = ok ? __uint_as_float(sAcc[k][u]) : 0.f;
      if (t < T) {
        cm[(size_t)(g.N1 + q) * T + t] = v;
        atomicMax(reinterpret_cast<unsigned*>(&sMax[u]), __float_as_uint(v));
      }
    }
    __syncthreads();  // sAcc is cleared by the next batch
  }
  for (int u = tid; u < TT; u += OT)
    if (t0 + u < T) atomic_max_pos(&w.m32[(size_t)b * T + t0 + u], sMax[u]);
}

// k_other_w: the same stream for many cases (NQ > 8 with more than 64 candidates): a
// warp per case (up to QW per warp, the Lo reads shared-memory broadcasts), lanes over
// TPT candidates each, one pass over the task's n0 for up to 32 cases.
namespace {
constexpr int ORC_W = 32;      // monitored rows per chunk (k_other_w)
}  // namespace

template <int MT, int QW, int TPT, bool LIST>
__global__ void __launch_bounds__(OT) k_other_w(DevGrid g, Work w) {
  constexpr int TT = 32 * TPT, QB = OW * QW;  // candidates per CTA, cases per batch
  const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int t0 = blockIdx.x * TT;
  if (w.status[b] != 0) return;
  const int T = w.T, M = g.M, NQ = g.NM + g.NI;
  extern __shared__ __align__(16) float osm[];
  float* sN = osm;                   // [2][ORC_W][TT]   n0 / rating
  float* sL = sN + 2 * ORC_W * TT;     // [2][ORC_W][QB*MT] correction columns of the batch
  __shared__ float sMax[TT];
  const float* Lo = w.Lo + (size_t)b * M * NQ * MT;
  const float* n0s = w.n0s + (size_t)b * M * T;
  const float* So = w.So + (size_t)b * NQ * MT * T;
  float* cm = w.cmax + (size_t)b * (g.N1 + NQ) * T;
  // the cases k_oscreen left (ascending), or all of them
  const int* ol = w.olist + (size_t)b * NQ;
  const int nq = LIST ? w.ocnt[b] : NQ;
  const bool vecN = (T % 4) == 0;
  for (int i = tid; i < TT; i += OT) sMax[i] = 0.f;

  for (int qb = 0; qb < nq; qb += QB) {
    const int nqb = min(QB, nq - qb), LW = nqb * MT;  // cases / Lo floats of this batch
    float sv[QW][MT][TPT], acc[QW][TPT];
#pragma unroll
    for (int k = 0; k < QW; ++k) {
      const int qi = qb + wid + OW * k;
#pragma unroll
      for (int j = 0; j < MT; ++j)
#pragma unroll
        for (int i = 0; i < TPT; ++i) {
          const int t = t0 + lane * TPT + i;
          sv[k][j][i] = (qi < nq && t < T) ? So[((size_t)(LIST ? ol[qi] : qi) * MT + j) * T + t] : 0.f;
        }
#pragma unroll
      for (int i = 0; i < TPT; ++i) acc[k][i] = 0.f;
    }
    auto issue = [&](int m0, int buf) {
      if (vecN) {
        for (int idx = tid; idx < ORC_W * (TT / 4); idx += OT) {
          const int rr = idx / (TT / 4), u = 4 * (idx % (TT / 4)), m = m0 + rr;
          const bool ok = m < M && t0 + u < T;
          cp16(&sN[(buf * ORC_W + rr) * TT + u], ok ? &n0s[(size_t)m * T + t0 + u] : n0s, ok);
        }
      } else {
        for (int idx = tid; idx < ORC_W * TT; idx += OT) {
          const int rr = idx / TT, u = idx % TT, m = m0 + rr;
          const bool ok = m < M && t0 + u < T;
          cp4(&sN[(buf * ORC_W + rr) * TT + u], ok ? &n0s[(size_t)m * T + t0 + u] : n0s, ok);
        }
      }
      // LW = nqb * MT is a multiple of 2; rows of Lo are NQ*MT floats (8-byte aligned)
      for (int idx = tid; idx < ORC_W * (LW / 2); idx += OT) {
        const int rr = idx / (LW / 2), u = 2 * (idx % (LW / 2)), m = m0 + rr;
        const bool ok = m < M;
        const int q = LIST ? ol[qb + u / MT] : qb + u / MT;
        cp8(&sL[(buf * ORC_W + rr) * QB * MT + u], ok ? &Lo[((size_t)m * NQ + q) * MT + (u % MT)] : Lo, ok);
      }
      cp_commit();
    };
    issue(0, 0);
    const int nchunks = (M + ORC_W - 1) / ORC_W;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int buf = ch & 1;
      if (ch + 1 < nchunks) {
        issue((ch + 1) * ORC_W, buf ^ 1);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      const int rend = min(ORC_W, M - ch * ORC_W);  // zero-filled rows past M are harmless
      (void)rend;
      // two rows per step: FFMA2 over the row pair (same rounding as fmaf), one FMNMX3
#pragma unroll 2
      for (int rr = 0; rr < ORC_W; rr += 2) {
        float2 n[TPT];
#pragma unroll
        for (int i = 0; i < TPT; ++i)
          n[i] = make_float2(sN[(buf * ORC_W + rr) * TT + lane * TPT + i], sN[(buf * ORC_W + rr + 1) * TT + lane * TPT + i]);
#pragma unroll
        for (int k = 0; k < QW; ++k) {
          if (wid + OW * k >= nqb) break;  // warp-uniform
          const float* lrow0 = &sL[(buf * ORC_W + rr) * QB * MT + (wid + OW * k) * MT];
          const float* lrow1 = lrow0 + QB * MT;
          float2 l[MT];
#pragma unroll
          for (int j = 0; j < MT; ++j) l[j] = make_float2(lrow0[j], lrow1[j]);
#pragma unroll
          for (int i = 0; i < TPT; ++i) {
            float2 f = n[i];
#pragma unroll
            for (int j = 0; j < MT; ++j) f = __ffma2_rn(l[j], make_float2(sv[k][j][i], sv[k][j][i]), f);
            acc[k][i] = max3abs(acc[k][i], f.x, f.y);
          }
        }
      }
      __syncthreads();
    }
    // per-(case, candidate) maxima (islanded multi cases contribute 0), candidate max
#pragma unroll
    for (int k = 0; k < QW; ++k) {
      const int qi = qb + wid + OW * k;
      if (qi >= nq) break;
      const int q = LIST ? ol[qi] : qi;
      const bool ok = q >= g.NM || w.mc_ok[(size_t)b * g.NM + q];
#pragma unroll
      for (int i = 0; i < TPT; ++i) {
        const int u = lane * TPT + i, t = t0 + u;
        const float v = ok ? acc[k][i] : 0.f;
        if (t < T) {
          cm[(size_t)(g.N1 + q) * T + t] = v;
          atomicMax(reinterpret_cast<unsigned*>(&sMax[u]), __float_as_uint(v));
        }
      }
    }
  }
  __syncthreads();
  for (int u = tid; u < TT; u += OT)
    if (t0 + u < T) atomic_max_pos(&w.m32[(size_t)b * T + t0 + u], sMax[u]);
}

// -------------------------------------------------------------------------- k_oscreen
// The exact dominance screen for the multi-branch and injection cases (the reference
// evaluates every one, solver.py:608-622; skipping a dominated one leaves every metric
// bit-identical).  Runs after the TOP tile, so lb(t) = m32(t) already holds the N-0 and
// TOP-case maxima (and the islanding penalty floors it).  Per case q (a warp each):
//   |F'(r, t)| = |n0'(r, t) + sum_j Lo(r, q, j) So(q, j, t)|
//              <= m0(t) + sum_j max_r |Lo(r, q, j)| |So(q, j, t)|   (FFMA chain: x (1 + 1e-5))
// and a case whose bound stays <= lb(t) for every candidate cannot raise a metric: it is
// skipped (its bound goes to cmax as the report's / re-score's upper bound, oskip marks
// it inexact).  Islanded multi cases (mc_ok = 0) contribute 0 and are skipped too.  The
// remaining cases are listed, ascending, for k_other.
__global__ void __launch_bounds__(256) k_oscreen(DevGrid g, DevCfg cfg, Work w) {
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int NQ = g.NM + g.NI, M = g.M, T = w.T, MT = g.MT;
  if (w.status[b] != 0) {
    if (tid == 0) w.ocnt[b] = 0;
    return;
  }
  const float* Lo = w.Lo + (size_t)b * M * NQ * MT;
  const float* So = w.So + (size_t)b * NQ * MT * T;
  const float* m0 = w.m0 + (size_t)b * T;
  const float* m32 = reinterpret_cast<const float*>(w.m32) + (size_t)b * T;
  float* cm = w.cmax + (size_t)b * (g.N1 + NQ) * T;
  const bool pen = w.nisl[b] > 0;
  const float penf = (float)cfg.penalty;
  for (int q = wid; q < NQ; q += 8) {
    const bool dead = q < g.NM && !w.mc_ok[(size_t)b * g.NM + q];
    bool skip = dead;
    float lm[8];
    if (!dead && w.screen) {
      for (int j = 0; j < MT; ++j) {
        float v = 0.f;
        for (int r = lane; r < M; r += 32) v = fmaxf(v, fabsf(Lo[((size_t)r * NQ + q) * MT + j]));
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        lm[j] = v;
      }
      bool dom = true;
      for (int t = lane; t < T; t += 32) {
        float ub = m0[t];
        for (int j = 0; j < MT; ++j) ub = fmaf(lm[j], fabsf(So[((size_t)q * MT + j) * T + t]), ub);
        const float lb = pen ? fmaxf(m32[t], penf) : m32[t];
        dom &= ub * (1.f + 1e-5f) <= lb;
      }
      skip = __all_sync(0xffffffffu, dom);
      if (skip)  // the report's and the re-score's upper bound of the skipped pairs
        for (int t = lane; t < T; t += 32) {
          float ub = m0[t];
          for (int j = 0; j < MT; ++j) ub = fmaf(lm[j], fabsf(So[((size_t)q * MT + j) * T + t]), ub);
          cm[(size_t)(g.N1 + q) * T + t] = ub * (1.f + 1e-5f);
        }
    }
    if (dead)
      for (int t = lane; t < T; t += 32) cm[(size_t)(g.N1 + q) * T + t] = 0.f;
    if (lane == 0) w.oskip[(size_t)b * NQ + q] = skip;
  }
  __syncthreads();  // the block's oskip writes are visible to warp 0
  if (wid == 0) {  // the kept cases, ascending
    int off = 0;
    for (int q0 = 0; q0 < NQ; q0 += 32) {
      const bool keep = q0 + lane < NQ && !w.oskip[(size_t)b * NQ + q0 + lane];
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) w.olist[(size_t)b * NQ + off + __popc(bal & ((1u << lane) - 1u))] = q0 + lane;
      off += __popc(bal);
    }
    if (lane == 0) w.ocnt[b] = off;
  }
}

// --------------------------------------------------------------------------- k_oexact
// The winner's exact FP32 maximum of every feasible multi/injection case k_oscreen skipped:
// the report's kg-th case value (k_rsel) is taken over exact maxima, so the skipped cases
// get k_other's expression (n0' + sum_j Lo_j So_j by fmaf in j order, the scalar form of
// its FFMA2) at the winning candidate and are marked exact again.
__global__ void __launch_bounds__(256) k_oexact(DevGrid g, Work w) {
  constexpr int QP = 64;  // skipped cases per pass
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  if (w.status[b] != 0) return;
  const int NQ = g.NM + g.NI, M = g.M, T = w.T, MT = g.MT, t = (int)w.best[b];
  const float* Lo = w.Lo + (size_t)b * M * NQ * MT;
  const float* So = w.So + (size_t)b * NQ * MT * T;
  const float* n0s = w.n0s + (size_t)b * M * T;
  __shared__ int sq[QP];
  __shared__ float ss[QP][8];
  __shared__ unsigned smx[QP];
  __shared__ int nsq;
  for (int q0 = 0; q0 < NQ; q0 += QP) {
    if (tid == 0) nsq = 0;
    __syncthreads();
    if (tid < QP && q0 + tid < NQ) {
      const int q = q0 + tid;
      if (w.oskip[(size_t)b * NQ + q] && (q >= g.NM || w.mc_ok[(size_t)b * g.NM + q])) {
        const int k = atomicAdd(&nsq, 1);
        sq[k] = q;
        smx[k] = 0u;
      }
    }
    __syncthreads();
    const int n = nsq;
    if (n == 0) continue;
    for (int i = tid; i < n * MT; i += 256) ss[i / MT][i % MT] = So[((size_t)sq[i / MT] * MT + i % MT) * T + t];
    __syncthreads();
    // rows over the block: each row's n0 once for every skipped case; per-case maxima by
    // warp reduction, one shared-memory atomic per warp and case
    for (int r0 = 0; r0 < M; r0 += 256) {
      const int r = r0 + tid;
      const float nv = r < M ? n0s[(size_t)r * T + t] : 0.f;
      for (int k = 0; k < n; ++k) {
        float f = nv;
        if (r < M)
          for (int j = 0; j < MT; ++j) f = fmaf(Lo[((size_t)r * NQ + sq[k]) * MT + j], ss[k][j], f);
        unsigned v = __float_as_uint(fabsf(f));
        v = __reduce_max_sync(0xffffffffu, v);
        if (lane == 0) atomicMax(&smx[k], v);
      }
    }
    __syncthreads();
    if (tid < n) {
      w.cmax[((size_t)b * (g.N1 + NQ) + g.N1 + sq[tid]) * T + t] = __uint_as_float(smx[tid]);
      w.oskip[(size_t)b * NQ + sq[tid]] = 0;
    }
    __syncthreads();
  }
}

void launch_oexact(const DevGrid& g, const Work& w, cudaStream_t s) {
  if (w.oscr && g.NM + g.NI > 0 && g.M > 0) k_oexact<<<w.Wb, 256, 0, s>>>(g, w);
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
  // near-tie band: candidates whose FP32 metric lies within 2 E of the minimum may be the
  // FP64 argmin (|m32 - m64| <= E); more than one -> queue the task for k_rescore
  // With islanded cases, a winner whose m32 + E lies below the penalty has m64 = penalty
  // exactly, the smallest metric possible: only an earlier band member could tie it.
  const float E = RESCORE_EPS * fmaxf(1.f, bv);
  const float hi = bv + 2.f * E;
  const bool exact = pen && (double)__uint_as_float(w.m32[(size_t)b * T + bi]) + (double)E < cfg.penalty;
  int nband = 0;
  for (int t = lane; t < tn; t += 32) {
    float v = __uint_as_float(w.m32[(size_t)b * T + t]);
    if (pen) v = fmaxf(v, penalty);
    nband += v <= hi && (!exact || t < bi);
  }
  for (int o = 16; o; o >>= 1) nband += __shfl_xor_sync(0xffffffffu, nband, o);
  if (exact && nband > 0) ++nband;  // the winner itself
  if (lane == 0) {
    w.best[b] = bi;
    w.feasible[b] = 1;
    const int nf = g.NC - w.nisl[b];
    atomicAdd(w.lf, (unsigned long long)tn * (unsigned long long)(1 + nf));
    if (nband > 1) {
      w.rsq[atomicAdd(w.rsq_n, 1u)] = b;
      atomicAdd(w.lf + 6, 1ull);
    }
  }
}

// ---------------------------------------------------------------------------- launches
namespace {
template <int MT, int QC, int TPT>
void launch_other_t(const DevGrid& g, const Work& w, cudaStream_t s) {
  constexpr int TT = 32 * TPT;
  const size_t dyn = (2 * (size_t)ORC * TT + 2 * (size_t)ORC * QC * MT) * sizeof(float);
  dim3 grid((w.T + TT - 1) / TT, w.Wb);
  auto go = [&](auto kern) {
    smem_opt_in((const void*)kern, (int)dyn);
    kern<<<grid, OT, dyn, s>>>(g, w);
  };
  if (w.oscr) go(k_other<MT, QC, TPT, true>);
  else go(k_other<MT, QC, TPT, false>);
}
template <int MT, int QC>
void launch_other_m(const DevGrid& g, const Work& w, cudaStream_t s) {
  if (w.T > 32) launch_other_t<MT, QC, 2>(g, w, s);
  else launch_other_t<MT, QC, 1>(g, w, s);
}
template <int MT, int QW, int TPT>
void launch_other_w(const DevGrid& g, const Work& w, cudaStream_t s) {
  constexpr int TT = 32 * TPT;
  const size_t dyn = (2 * (size_t)ORC_W * TT + 2 * (size_t)ORC_W * OW * QW * MT) * sizeof(float);
  dim3 grid((w.T + TT - 1) / TT, w.Wb);
  auto go = [&](auto kern) {
    smem_opt_in((const void*)kern, (int)dyn);
    kern<<<grid, OT, dyn, s>>>(g, w);
  };
  if (w.oscr) go(k_other_w<MT, QW, TPT, true>);
  else go(k_other_w<MT, QW, TPT, false>);
}
template <int MT, int QW>
void launch_other_wm(const DevGrid& g, const Work& w, cudaStream_t s) {
  launch_other_w<MT, QW, 4>(g, w, s);
}
}  // namespace

// The multi/injection screen pays where the stream is long (many cases over many
// candidates: G1k 4.98 -> 1.46 ms per step); on small grids its per-task pass costs more than
// it skips (G118 +0.7 ms).  Tests force it either way (BDC_OSCREEN=0/1).
bool other_screened(const DevGrid& g, const Work& w) {
  const int nq = g.NM + g.NI;
  const char* e = getenv("BDC_OSCREEN");
  if (e) return w.screen && e[0] == '1';
  return w.screen && nq > 8 && w.T > 64;
}
void launch_other(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  const int nq = g.NM + g.NI;
  if (nq == 0 || g.M == 0) return;
  if (w.oscr) k_oscreen<<<w.Wb, 256, 0, s>>>(g, c, w);
  // every lane carries a batch of cases and the warps split the rows; many cases over
  // more than 64 candidates: a warp per case, one pass over n0 (measured faster there)
  if (nq > 8 && w.T > 64) {
    if (g.MT <= 2) launch_other_wm<2, 4>(g, w, s);
    else if (g.MT <= 4) launch_other_wm<4, 2>(g, w, s);
    else launch_other_wm<8, 1>(g, w, s);
  } else if (g.MT <= 2) {
    launch_other_m<2, 8>(g, w, s);
  } else if (g.MT <= 4) {
    launch_other_m<4, 4>(g, w, s);
  } else {
    launch_other_m<8, 2>(g, w, s);
  }
}

void launch_select(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s) {
  const int threads = 256;
  const long long total = (long long)w.Wb * 32;
  k_select<<<(unsigned)((total + threads - 1) / threads), threads, 0, s>>>(g, c, w);
  launch_rescore(g, c, w, s);
}

}  // namespace bdc
