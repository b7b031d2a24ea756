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


}  // namespace

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
