// bdc_gen.cu -- device-side random task generation.
//
// Replaces the reference's host generator batchdc.bench.random_tasks
// (src/batchdc/bench.py:33-91) for batches of 10^5..10^6 topologies: the same
// distribution, drawn on the GPU straight into the session's array layout
// (session.py:9-19) so the engine is fed at rate:
//   * k distinct substations chosen uniformly among those with >= 2 branch
//     elements (rng.choice(len(eligible), k, replace=False), bench.py:54-58);
//   * per chosen substation, uniform assignment bits over its elements,
//     redrawn while all False (bench.py:62-65);
//   * d distinct disconnected branches, uniform over the branches (bench.py:67-73;
//     folded branches, which the reference rejects, are never drawn);
//   * T injection bit-rows, uniform over the K slots (bench.py:76-79).
// The reference rejects and redraws a task whose splits are singular or
// degenerate or whose disconnections island the grid (_feasible_at_n0,
// bench.py:96-110).  Here the engine itself is the acceptance test: the
// caller solves the drawn batch, and the tasks whose status is one of those
// failures are redrawn with the next attempt number (redraw mask), which
// changes their topology draw only -- the injection rows are independent of
// acceptance, so drawing them once gives the same distribution.
//
// Random numbers: Philox4x32-10 (counter-based: key = seed, counter = task,
// attempt, purpose, word), so any task's draw is reproducible on its own and
// the result does not depend on the launch configuration.  The random stream
// is not numpy's PCG64: the draws match the reference's distribution, not its
// exact samples (parity is checked on the drawn tasks themselves).
#include "bdc_device.cuh"

namespace bdc {

namespace {

struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Random words for one (task, attempt, purpose) stream, four per Philox call.
struct Stream {
  uint32_t k0, k1, task, att, purpose, ctr = 0, n = 0;
  U4 buf{};
  __device__ uint32_t next() {
    if (n == 0) {
      buf = philox(U4{task, att, purpose, ctr++}, k0, k1);
      n = 4;
    }
    const uint32_t v = n == 4 ? buf.x : n == 3 ? buf.y : n == 2 ? buf.z : buf.w;
    --n;
    return v;
  }
  // uniform integer in [0, m) (multiply-shift; bias <= m / 2^32)
  __device__ uint32_t below(uint32_t m) { return (uint32_t)(((uint64_t)next() * m) >> 32); }
};

constexpr uint32_t P_SUBS = 1, P_BITS = 2, P_DISC = 3, P_INJ = 4;

// a branch the reference can disconnect: a retained PTDF row with both endpoint columns
// (folded ones raise ValidationError, which random_tasks rejects, bench.py:108-109)
__device__ __forceinline__ bool outageable(const DevGrid& g, int k) {
  const int r = g.branch_row[k];
  return r >= 0 && g.row_from[r] >= 0 && g.row_to[r] >= 0;
}
constexpr int GEN_SMAX = 4096;  // eligible substations staged in shared memory

// Topology draw of the masked tasks: one warp per task.  Clears the task's (S, E) split
// block and (D) disconnection row, then lane 0 draws the substations, bits and branches.
__global__ void k_gen_topo(DevGrid g, GenArgs a) {
  __shared__ int elig[GEN_SMAX];
  __shared__ int nel, nret;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { nel = 0; nret = 0; }
  __syncthreads();
  // branches that can be disconnected (a disconnection of a folded branch is a
  // ValidationError the reference rejects, bench.py:108-109: drawing among the others
  // directly gives the same conditional distribution)
  {
    int c = 0;
    for (int k = threadIdx.x; k < g.NBR; k += blockDim.x) c += outageable(g, k);
    atomicAdd(&nret, c);
  }
  // eligible substations (>= 2 branch elements), ascending: the reference's `eligible`
  if (g.S <= GEN_SMAX) {
    for (int s0 = 0; s0 < g.S; s0 += blockDim.x) {
      const int s = s0 + threadIdx.x;
      const bool ok = s < g.S && g.sub_count[s] >= 2;
      // ordered compaction: count of eligible substations before s
      __syncthreads();
      if (ok) {
        int before = 0;
        for (int u = s0; u < s; ++u) before += g.sub_count[u] >= 2;
        elig[nel + before] = s;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int c = 0;
        for (int u = s0; u < min(g.S, s0 + (int)blockDim.x); ++u) c += g.sub_count[u] >= 2;
        nel += c;
      }
      __syncthreads();
    }
  }
  const int ne = nel, nr = nret;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= a.B) return;
  if (a.redraw && !a.redraw[b]) return;
  const uint32_t att = a.attempt ? (uint32_t)a.attempt[b] : 0u;
  uint8_t* sp = a.splits + b * (int64_t)g.S * a.E;
  for (int i = lane; i < g.S * a.E; i += 32) sp[i] = 0;
  int64_t* dc = a.discos ? a.discos + b * a.D : nullptr;
  for (int i = lane; dc && i < a.D; i += 32) dc[i] = -1;
  __syncwarp();
  if (lane != 0) return;
  // k distinct eligible substations (Floyd's sampling), uniform over k-subsets
  const int k = min(a.n_splits, ne);
  int chosen[RMAX];
  Stream rs{a.k0, a.k1, (uint32_t)b, att, P_SUBS};
  int nc = 0;
  for (int j = ne - k; j < ne; ++j) {
    const int r = (int)rs.below((uint32_t)j + 1u);
    bool dup = false;
    for (int i = 0; i < nc; ++i) dup |= chosen[i] == r;
    chosen[nc++] = dup ? j : r;
  }
  Stream bs{a.k0, a.k1, (uint32_t)b, att, P_BITS};
  for (int i = 0; i < nc; ++i) {
    int s = -1;
    if (g.S <= GEN_SMAX) {
      s = elig[chosen[i]];
    } else {  // scan for the chosen[i]-th eligible substation
      int c = -1;
      for (int u = 0; u < g.S; ++u)
        if (g.sub_count[u] >= 2 && ++c == chosen[i]) { s = u; break; }
    }
    const int n_el = g.sub_count[s];
    const uint32_t mask = n_el >= 32 ? 0xffffffffu : ((1u << n_el) - 1u);
    uint32_t bits = 0u;
    while (bits == 0u) bits = bs.next() & mask;  // not all False (bench.py:63-65)
    for (int e = 0; e < n_el && e < a.E; ++e) sp[(int64_t)s * a.E + e] = (bits >> e) & 1u;
  }
  // d distinct branches, uniform over the retained branches (Floyd's sampling)
  if (dc && a.n_disc > 0) {
    Stream ds{a.k0, a.k1, (uint32_t)b, att, P_DISC};
    int pick[RMAX];
    int np = 0;
    const int d = min(a.n_disc, min(nr, a.D));
    for (int j = nr - d; j < nr; ++j) {
      const int r = (int)ds.below((uint32_t)j + 1u);
      bool dup = false;
      for (int i = 0; i < np; ++i) dup |= pick[i] == r;
      pick[np++] = dup ? j : r;
    }
    for (int i = 0; i < np; ++i) {
      int64_t br = pick[i];
      if (nr != g.NBR) {  // the pick[i]-th retained branch
        int c = -1;
        for (int k = 0; k < g.NBR; ++k)
          if (outageable(g, k) && ++c == pick[i]) { br = k; break; }
      }
      dc[i] = br;
    }
  }
}

// Injection rows: one thread per (task, candidate, 128-slot chunk) -- HBM-bound writes.
__global__ void k_gen_inj(DevGrid g, GenArgs a) {
  const int nch = (g.K + 127) / 128;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = a.B * (int64_t)a.T * nch;
  if (i >= total) return;
  const int ch = (int)(i % nch);
  const int64_t bt = i / nch;
  const uint32_t b = (uint32_t)(bt / a.T), t = (uint32_t)(bt % a.T);
  const U4 r = philox(U4{b, t, P_INJ, (uint32_t)ch}, a.k0, a.k1);
  const uint32_t wds[4] = {r.x, r.y, r.z, r.w};
  uint8_t* dst = a.inj + bt * g.K + ch * 128;
  const int n = min(128, g.K - ch * 128);
  for (int e = 0; e < n; ++e) dst[e] = (wds[e >> 5] >> (e & 31)) & 1u;
}

}  // namespace

cudaError_t launch_draw(const DevGrid& g, const GenArgs& a, cudaStream_t s) {
  if (a.B <= 0) return cudaSuccess;
  const int64_t warps = a.B;
  k_gen_topo<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(g, a);
  if (a.inj && a.T > 0 && g.K > 0) {
    const int64_t n = a.B * (int64_t)a.T * ((g.K + 127) / 128);
    k_gen_inj<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, a);
  }
  return cudaGetLastError();
}

}  // namespace bdc
