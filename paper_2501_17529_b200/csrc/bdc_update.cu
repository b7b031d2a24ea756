// bdc_update.cu -- Kernel 1: the per-topology low-rank PTDF update.
//
// One CTA per task, FP64 throughout.  The updated PTDF of a task is never
// materialised; it is carried as a rank-r correction of the shared base
//     P''[row, col] = P0[row, base(col)] + sum_j B[j][row] * C[j][col]
// (rows of disconnected branches forced to exactly 0), where the first k
// terms are the sequential busbar-split chain and the next d terms the
// disconnections.  Logical column ids: 0..C0-1 are the base columns, C0+j is
// the new busbar column of split j (base(C0+j) = column of its substation).
//
// Follows, step for step:
//   decode + canonical order      session.py:207-225, solver.py:148-197
//   compute_bsdf / apply_bsdf     factors.py:428-585  (split chain, _apply_splits solver.py:363-378)
//   compute_modf / apply_modf     factors.py:373-425  (disconnections, solver.py:389-406)
//   lodf_column / apply_outage    factors.py:333-370  (multi_outage_method="sequential")
//   single-outage LODF block      solver.py:474-503   (den, islanding, W factors)
//   multi-branch cases            solver.py:448-454   (m x m inner system per case)
//   injection cases / slots       solver.py:455-467, 555-572
//   candidate injection vectors   solver.py:575-595   (y_t = C''^T p_t, so n0 = f0 + B'' y_t)
#include "bdc_device.cuh"

#include <algorithm>
#include <cstdlib>

namespace bdc {

namespace {

constexpr int NT = 256;  // k_n0, k_topk
constexpr int NW = NT / 32;
constexpr int UWMAX = 16;  // k_update: one task per CTA of 128..512 threads (by grid size)

struct UpdShared {
  int sub[RMAX];
  unsigned bits[RMAX];
  int k, d, nd, fail, farg, nrh, nact;
  int pmode, pslot;    // prefix memo of the current split (PFX_*) and its table slot
  int wcnt[UWMAX];
  int dead[RMAX];
  int orow[RMAX];      // outage rows in task order
  int ofc[RMAX], otc[RMAX];  // current endpoint columns of the outaged rows
  // split step scratch
  int a, nm, nst;
  int mrow[EMAX], mend[EMAX];
  double msign[EMAX];
  int srow[EMAX], sfar[EMAX];
  double ssign[EMAX], sw[EMAX];
  double den;
  double sCa[RMAX];          // C[i][a]
  double coefC[RMAX];        // sum_m sign_m B_i[row_m]            (coupler row of split j)
  double coefB[RMAX];        // sum_st w_st (C_i[far_st] - C_i[a]) (numerator of split j)
  double inner[MMAX * MMAX];
  double inv[MMAX * MMAX];   // MODF inverse (d <= MMAX outages)
  double ybase[RMAX];
  int act_slot[ACTMAX], act_ca[ACTMAX], act_cb[ACTMAX];
  double act_sp[ACTMAX];
  int nisl;
};

__device__ __forceinline__ int base_col(const DevGrid& g, const UpdShared& s, int col) {
  return col < g.C0 ? col : g.sub_col[s.sub[col - g.C0]];
}

__device__ __forceinline__ int curcol(const UpdShared& s, const int* rh_key, const int* rh_col, int row,
                                      int end, int dflt) {
  int key = row * 2 + end, c = dflt;
  for (int i = 0; i < s.nrh; ++i)
    if (rh_key[i] == key) c = rh_col[i];
  return c;
}

// Dynamic shared memory of k_update (bytes), sized by the wave's rank stride rs and
// the widest substation E: moved-row B values, far-end coupler values, outage-row B
// values and the re-homed branch ends.
__host__ __device__ inline size_t update_dyn_bytes(int rs, int E) {
  const int e2 = E > 2 ? E : 2;
  return ((size_t)E * rs + (size_t)e2 * rs + (size_t)rs * rs) * sizeof(double) + 2 * (size_t)rs * E * sizeof(int);
}

// Ordered block-wide compaction helper: returns this thread's slot among the
// flagged threads of the current chunk and the chunk total (all threads).
__device__ __forceinline__ int block_rank(bool flag, int* wcnt, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned bal = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) wcnt[wid] = __popc(bal);
  __syncthreads();
  int off = 0;
  total = 0;
  for (int i = 0; i < nw; ++i) {
    if (i < wid) off += wcnt[i];
    total += wcnt[i];
  }
  __syncthreads();
  return off + __popc(bal & ((1u << lane) - 1u));
}

__device__ void set_island(const Work& w, int b, int order) {
  atomicOr(&w.isl[(size_t)b * w.NCw + (order >> 5)], 1u << (order & 31));
}

}  // namespace

// ---- prefix-shared split chains (tree.py:50-113 on the device).  Split j's factors
// (B_j over the rows, the coupler row C_j over columns 0..C0+j, and whether it is singular)
// depend only on the canonical prefix (sub_0, bits_0, ..., sub_j, bits_j).  The first task
// of a wave to reach a prefix claims its slot in a hash table, computes the split and
// publishes it; every other task with the same prefix waits for it and copies, so each
// shared tree edge is computed once per wave (levels < PFX_LEVELS, not the last split of a
// task).  Copies are the producer's bits, so results do not depend on who computed.
constexpr int PFX_OFF = 0, PFX_PUBLISH = 1, PFX_WAIT = 2;

__device__ __forceinline__ unsigned long long pfx_hash(const UpdShared& s, int j) {
  unsigned long long h = 0x9e3779b97f4a7c15ull ^ (unsigned long long)(j + 1);
  for (int i = 0; i <= j; ++i) {
    h ^= (unsigned long long)s.sub[i] * 0xbf58476d1ce4e5b9ull + s.bits[i];
    h = (h ^ (h >> 31)) * 0x94d049bb133111ebull;
  }
  return h | 1ull;  // 0 marks an empty slot
}

// thread 0: find or claim the slot of prefix j (PFX_PUBLISH: ours to compute, PFX_WAIT:
// someone else's, PFX_OFF: table full around the home slot -- compute locally)
__device__ int pfx_lookup(const Work& w, const UpdShared& s, int j, int& slot) {
  const unsigned long long h = pfx_hash(s, j);
  const unsigned cap = (unsigned)w.pfx_cap;
  unsigned sl = (unsigned)(h ^ (h >> 32)) & (cap - 1u);
  for (int probe = 0; probe < 32; ++probe, sl = (sl + 1u) & (cap - 1u)) {
    const unsigned long long key = atomicCAS(&w.pfx_key[sl], 0ull, h);
    int* id = w.pfx_id + (size_t)sl * 2 * PFX_LEVELS;
    if (key == 0ull) {  // claimed: record the prefix, then announce it
      for (int i = 0; i <= j; ++i) { id[2 * i] = s.sub[i]; id[2 * i + 1] = (int)s.bits[i]; }
      for (int i = j + 1; i < PFX_LEVELS; ++i) { id[2 * i] = -1; id[2 * i + 1] = 0; }
      __threadfence();
      atomicExch(&w.pfx_state[sl], 1);
      slot = (int)sl;
      return PFX_PUBLISH;
    }
    if (key != h) continue;
    while (atomicAdd(&w.pfx_state[sl], 0) == 0) __nanosleep(64);  // the claimer writes id first
    bool same = true;
    for (int i = 0; i < PFX_LEVELS && same; ++i) {
      const int vs = __ldcg(&id[2 * i]), vb = __ldcg(&id[2 * i + 1]);
      same = i <= j ? (vs == s.sub[i] && vb == (int)s.bits[i]) : vs == -1;
    }
    if (same) {
      slot = (int)sl;
      return PFX_WAIT;
    }
  }
  return PFX_OFF;
}

// UT threads per task: 128 for small grids (many tasks in flight), more for large grids,
// whose row and column loops need the memory parallelism (few tasks per SM).
template <int UT, int MINB>
__global__ void __launch_bounds__(UT, MINB) k_update(DevGrid g, DevCfg cfg, Work w) {
  constexpr int UW = UT / 32;
  __shared__ UpdShared s;
  __shared__ double mA[UW][MMAX * MMAX];  // per-warp m x m inner system of a multi-branch case
  const int b = blockIdx.x, tid = threadIdx.x;
  const int R = g.R, C0 = g.C0, rs = w.rs, Cs = w.Cs;
  const int E = g.E > 0 ? g.E : 1, E2 = E > 2 ? E : 2;
  extern __shared__ double udyn[];
  double* mB = udyn;                 // [E][rs]   B[i][moved row m]
  double* sCfar = mB + E * rs;       // [E2][rs]  C[i][far end of stay element st]
  double* oB = sCfar + E2 * rs;      // [rs][rs]  B[i'][outage row i]
  int* rh_key = reinterpret_cast<int*>(oB + rs * rs);  // [rs*E] row*2 + end
  int* rh_col = rh_key + rs * E;
#define MB(m, i) mB[(m) * rs + (i)]
#define SCF(st, i) sCfar[(st) * rs + (i)]
#define OB(i, ip) oB[(i) * rs + (ip)]
  double* Bm = w.Bm + (size_t)b * rs * R;
  double* Cm = w.Cm + (size_t)b * rs * Cs;

  if (tid == 0) {
    s.k = 0; s.d = 0; s.nd = 0; s.fail = 0; s.farg = 0; s.nrh = 0; s.nact = 0; s.nisl = 0;
    s.pmode = PFX_OFF;
  }
  for (int i = tid; i < w.NCw; i += UT) w.isl[(size_t)b * w.NCw + i] = 0u;
  __syncthreads();

  // ---- decode splits in canonical (ascending substation) order ----------------
  const uint8_t* sp = w.splits + (size_t)b * g.S * w.Ein;
  for (int c0 = 0; c0 < g.S; c0 += UT) {
    int si = c0 + tid;
    unsigned bits = 0;
    if (si < g.S) {
      int cnt = g.sub_count[si];
      for (int e = 0; e < cnt; ++e)
        if (sp[(size_t)si * w.Ein + e]) bits |= 1u << e;
    }
    int total;
    int pos = block_rank(bits != 0, s.wcnt, total);
    if (bits != 0) {
      int p = s.k + pos;
      if (p < RMAX) { s.sub[p] = si; s.bits[p] = bits; }
    }
    __syncthreads();
    if (tid == 0) s.k += total;
    __syncthreads();
  }
  if (tid == 0) {
    const int64_t* dr = w.discos + (size_t)b * w.D;
    int d = 0;
    for (int i = 0; i < w.D; ++i) {
      int64_t k = dr[i];
      if (k >= 0) {
        if (d < RMAX) s.orow[d] = g.branch_row[k];
        ++d;
      }
    }
    s.d = d;
    if (s.k + d > rs) { s.fail = BDC_TASK_DETACHED; s.farg = -2; }
  }
  __syncthreads();
  const int k = s.k;
  if (s.fail) goto done;

  // ---- split chain (factors.py:428-585) -----------------------------------------
  for (int j = 0; j < k; ++j) {
    // split setup, warp 0: a lane per branch element of the substation (the element
    // loads and end lookups in parallel), lists compacted in element order
    if (tid < 32) {
      const int lane = tid;
      const int si = s.sub[j], a = g.sub_col[si], cnt = g.sub_count[si];
      const unsigned bits = s.bits[j];
      const bool in = lane < cnt, mv = in && ((bits >> lane) & 1u);
      const double be = in ? g.sub_elem_b[si * g.E + lane] : 0.0;
      // sum of the stay susceptances in element order (as the reference sums them)
      double stay_b = 0.0;
      for (int e = 0; e < cnt; ++e) {
        const double v = __shfl_sync(0xffffffffu, be, e);
        if (!((bits >> e) & 1u)) stay_b += v;
      }
      int row = -1, fc = -1, tc = -1;
      if (in) {
        row = g.sub_elem_row[si * g.E + lane];
        fc = curcol(s, rh_key, rh_col, row, 0, g.row_from[row]);
        tc = curcol(s, rh_key, rh_col, row, 1, g.row_to[row]);
      }
      const bool detached = in && fc != a && tc != a;
      const unsigned dmask = __ballot_sync(0xffffffffu, detached);
      const unsigned mmask = __ballot_sync(0xffffffffu, mv), smask = __ballot_sync(0xffffffffu, in && !mv);
      const unsigned lt = (1u << lane) - 1u;
      if (!(stay_b > 0.0)) {
        if (lane == 0) { s.fail = BDC_TASK_DEGENERATE_SPLIT; s.farg = j; }
      } else if (dmask) {
        if (lane == 0) { s.fail = BDC_TASK_DETACHED; s.farg = j; }
      } else if (in) {
        const bool atf = fc == a;
        const double sign = atf ? 1.0 : -1.0;
        if (mv) {
          const int q = __popc(mmask & lt);
          s.mrow[q] = row; s.msign[q] = sign; s.mend[q] = atf ? 0 : 1;
        } else {
          const int q = __popc(smask & lt);
          s.srow[q] = row; s.ssign[q] = sign; s.sfar[q] = atf ? tc : fc;
          s.sw[q] = be / stay_b;
        }
      }
      if (lane == 0) { s.a = a; s.nm = __popc(mmask); s.nst = __popc(smask); }
    }
    __syncthreads();
    if (s.fail) goto done;
    const int a = s.a, nm = s.nm, nst = s.nst;
    if (w.pfx_cap > 0) {  // uniform: no extra barrier on the default (flat) chain
      if (tid == 0) {
        s.pmode = PFX_OFF;
        if (j < PFX_LEVELS && j + 1 < k) s.pmode = pfx_lookup(w, s, j, s.pslot);
      }
      __syncthreads();
    }
    if (s.pmode == PFX_WAIT) {
      // another task computed this prefix: copy its split (B_j, C_j[0..C0+j]) or failure
      const int sl = s.pslot;
      if (tid == 0) {
        while (atomicAdd(&w.pfx_state[sl], 0) != 2) __nanosleep(128);
        __threadfence();
        const int f = __ldcg(&w.pfx_fail[sl]);
        if (f) { s.fail = f; s.farg = j; }
      }
      __syncthreads();
      if (s.fail) goto done;
      for (int r = tid; r < R; r += UT) Bm[(size_t)j * R + r] = __ldcg(&w.pfx_B[(size_t)sl * R + r]);
      for (int col = tid; col <= C0 + j; col += UT) Cm[(size_t)j * Cs + col] = __ldcg(&w.pfx_C[(size_t)sl * Cs + col]);
      for (int i = tid; i < j; i += UT) Cm[(size_t)i * Cs + C0 + j] = Cm[(size_t)i * Cs + a];
      if (tid == 0) {
        for (int m = 0; m < nm; ++m) {
          rh_key[s.nrh] = s.mrow[m] * 2 + s.mend[m];
          rh_col[s.nrh] = C0 + j;
          ++s.nrh;
        }
        atomicAdd(w.lf + 7, 1ull);  // split applications shared (copied)
      }
      __syncthreads();
      continue;
    }
    for (int idx = tid; idx < nm * j; idx += UT) {
      int m = idx / j, i = idx % j;
      MB(m, i) = Bm[(size_t)i * R + s.mrow[m]];
    }
    __syncthreads();
    // coupler row over every current column: c[col] = sum_moved sign * P_{j-1}[row, col]
    //   = sum_m sign_m P0[row_m, base(col)] + sum_i (sum_m sign_m B_i[row_m]) C_i[col]:
    // the rank-i coefficients once per split, then j (not nm * j) loads of C per column
    for (int i = tid; i < j; i += UT) {
      double cf = 0.0;
      for (int m = 0; m < nm; ++m) cf += s.msign[m] * MB(m, i);
      s.coefC[i] = cf;
    }
    __syncthreads();
    const int ncols = C0 + j;
    for (int col = tid; col < ncols; col += UT) {
      const int bc = base_col(g, s, col);
      double c = 0.0;
      for (int m = 0; m < nm; ++m) c += s.msign[m] * g.P0[(size_t)s.mrow[m] * C0 + bc];
      for (int i = 0; i < j; ++i) c = fma(s.coefC[i], Cm[(size_t)i * Cs + col], c);
      Cm[(size_t)j * Cs + col] = c;
    }
    // the new busbar column starts as a copy of column a for every earlier term
    for (int i = tid; i < j; i += UT) Cm[(size_t)i * Cs + C0 + j] = Cm[(size_t)i * Cs + a];
    __syncthreads();
    if (tid == 0) {
      const double ca = Cm[(size_t)j * Cs + a];
      Cm[(size_t)j * Cs + C0 + j] = ca - 1.0;
      double den = ca;
      for (int st = 0; st < nst; ++st) den -= s.sw[st] * Cm[(size_t)j * Cs + s.sfar[st]];
      if (fabs(den) < ISL_TOL) { s.fail = BDC_TASK_SINGULAR_SPLIT; s.farg = j; }
      s.den = den;
      if (s.pmode == PFX_PUBLISH && s.fail) {  // waiters learn the failure
        w.pfx_fail[s.pslot] = s.fail;
        __threadfence();
        atomicExch(&w.pfx_state[s.pslot], 2);
      }
    }
    for (int idx = tid; idx < (nst + 1) * j; idx += UT) {
      int st = idx / j, i = idx % j;
      if (st < nst) SCF(st, i) = Cm[(size_t)i * Cs + s.sfar[st]];
      else s.sCa[i] = Cm[(size_t)i * Cs + a];
    }
    __syncthreads();
    if (s.fail) goto done;
    // numerator num[r] = sum_st w_st (P_{j-1}[r, far_st] - P_{j-1}[r, a]) (+ own rows)
    //   = sum_st w_st (P0[r, base(far_st)] - P0[r, a]) + sum_i B_i[r] coefB_i,
    //   coefB_i = sum_st w_st (C_i[far_st] - C_i[a]): j loads of B per row, not (nst+1) j
    for (int i = tid; i < j; i += UT) {
      double cf = 0.0;
      for (int st = 0; st < nst; ++st) cf += s.sw[st] * (SCF(st, i) - s.sCa[i]);
      s.coefB[i] = cf;
    }
    __syncthreads();
    {
      const double den = s.den;
      for (int r = tid; r < R; r += UT) {
        const double p0a = g.P0T[(size_t)a * R + r];
        double num = 0.0;
        for (int st = 0; st < nst; ++st) {
          const int bf = base_col(g, s, s.sfar[st]);
          num += s.sw[st] * (g.P0T[(size_t)bf * R + r] - p0a);
          if (r == s.srow[st]) num += s.ssign[st] * s.sw[st];
        }
        for (int i = 0; i < j; ++i) num = fma(Bm[(size_t)i * R + r], s.coefB[i], num);
        Bm[(size_t)j * R + r] = num / den;
      }
    }
    if (s.pmode == PFX_PUBLISH) {  // the split for every task sharing this prefix
      const int sl = s.pslot;
      for (int r = tid; r < R; r += UT) w.pfx_B[(size_t)sl * R + r] = Bm[(size_t)j * R + r];
      for (int col = tid; col <= C0 + j; col += UT) w.pfx_C[(size_t)sl * Cs + col] = Cm[(size_t)j * Cs + col];
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        w.pfx_fail[sl] = 0;
        __threadfence();
        atomicExch(&w.pfx_state[sl], 2);
      }
    }
    if (tid == 0) {
      for (int m = 0; m < nm; ++m) {
        rh_key[s.nrh] = s.mrow[m] * 2 + s.mend[m];
        rh_col[s.nrh] = C0 + j;
        ++s.nrh;
      }
    }
    __syncthreads();
  }

  // ---- disconnections (solver.py:389-406) ------------------------------------------
  if (s.d > 0) {
    const int d = s.d;
    if (d > cfg.maxout) {
      if (tid == 0) { s.fail = BDC_TASK_TOO_MANY_OUTAGES; s.farg = d; }
      __syncthreads();
      goto done;
    }
    if (tid == 0)
      for (int i = 0; i < d; ++i) {
        int row = s.orow[i];
        if (row < 0) { s.fail = BDC_TASK_DETACHED; s.farg = -4; break; }
        s.ofc[i] = curcol(s, rh_key, rh_col, row, 0, g.row_from[row]);
        s.otc[i] = curcol(s, rh_key, rh_col, row, 1, g.row_to[row]);
        // a folded endpoint column cannot be outaged (the host raises the reference's
        // ValidationError first, Engine._check_outage_columns); never read column -1
        if (s.ofc[i] < 0 || s.otc[i] < 0) { s.fail = BDC_TASK_DETACHED; s.farg = -4; }
      }
    __syncthreads();
    if (s.fail) goto done;
    if (cfg.method == 0) {
      // MODF: one d x d inner system against the post-split matrix (factors.py:373-425)
      // rhs[i][r] = P'[r, f'_i] - P'[r, t'_i] into B slots k+i
      for (int r = tid; r < R; r += UT) {
        for (int i = 0; i < d; ++i) {
          const int fc = s.ofc[i], tc = s.otc[i];
          double pf = g.P0T[(size_t)base_col(g, s, fc) * R + r];
          double pt = g.P0T[(size_t)base_col(g, s, tc) * R + r];
          for (int ip = 0; ip < k; ++ip) {
            const double bv = Bm[(size_t)ip * R + r];
            pf = fma(bv, Cm[(size_t)ip * Cs + fc], pf);
            pt = fma(bv, Cm[(size_t)ip * Cs + tc], pt);
          }
          Bm[(size_t)(k + i) * R + r] = pf - pt;
        }
      }
      __syncthreads();
      if (tid == 0) {
        double A[MMAX * MMAX];
        bool big = d > MMAX;
        if (!big) {
          for (int aa = 0; aa < d; ++aa)
            for (int bb = 0; bb < d; ++bb)
              A[aa * d + bb] = (aa == bb ? 1.0 : 0.0) - Bm[(size_t)(k + bb) * R + s.orow[aa]];
          double smax, smin;
          svd_minmax(A, d, smax, smin);
          if (smin < ISL_TOL * fmax(1.0, smax)) { s.fail = BDC_TASK_DISCONNECT_ISLAND; s.farg = -1; }
          else invert_small(A, d, s.inv);
        } else {
          s.fail = BDC_TASK_DETACHED; s.farg = -3;
        }
      }
      for (int idx = tid; idx < d * k; idx += UT) {
        int i = idx / k, ip = idx % k;
        OB(i, ip) = Bm[(size_t)ip * R + s.orow[i]];
      }
      __syncthreads();
      if (s.fail) goto done;
      // MODF values in place: modf[r][i] = sum_bb rhs[bb][r] inv[bb][i]; rows O -> -e_i
      for (int r = tid; r < R; r += UT) {
        double rhs[MMAX];
        for (int bb = 0; bb < d; ++bb) rhs[bb] = Bm[(size_t)(k + bb) * R + r];
        int own = -1;
        for (int aa = 0; aa < d; ++aa) if (s.orow[aa] == r) own = aa;
        for (int i = 0; i < d; ++i) {
          double v;
          if (own >= 0) v = (own == i) ? -1.0 : 0.0;
          else {
            v = 0.0;
            for (int bb = 0; bb < d; ++bb) v += rhs[bb] * s.inv[bb * d + i];
          }
          Bm[(size_t)(k + i) * R + r] = v;
        }
      }
      // outage rows of the post-split matrix become the new coupler rows
      const int ncols = C0 + k;
      for (int idx = tid; idx < d * ncols; idx += UT) {
        int i = idx / ncols, col = idx % ncols;
        double v = g.P0[(size_t)s.orow[i] * C0 + base_col(g, s, col)];
        for (int ip = 0; ip < k; ++ip) v = fma(OB(i, ip), Cm[(size_t)ip * Cs + col], v);
        Cm[(size_t)(k + i) * Cs + col] = v;
      }
      if (tid == 0) {
        for (int i = 0; i < d; ++i) s.dead[i] = s.orow[i];
        s.nd = d;
      }
      __syncthreads();
    } else {
      // sequential single outages (factors.py:333-370), each one rank-1 term
      for (int i = 0; i < d; ++i) {
        const int kk = k + i, row = s.orow[i], fc = s.ofc[i], tc = s.otc[i];
        const int bf = base_col(g, s, fc), bt = base_col(g, s, tc);
        for (int ip = tid; ip < kk; ip += UT) {
          SCF(0, ip) = Cm[(size_t)ip * Cs + fc];
          SCF(1, ip) = Cm[(size_t)ip * Cs + tc];
          OB(0, ip) = Bm[(size_t)ip * R + row];
        }
        __syncthreads();
        for (int r = tid; r < R; r += UT) {
          double v = 0.0;
          if (!is_dead(s.dead, s.nd, r)) {
            double pf = g.P0T[(size_t)bf * R + r], pt = g.P0T[(size_t)bt * R + r];
            for (int ip = 0; ip < kk; ++ip) {
              double bv = Bm[(size_t)ip * R + r];
              pf = fma(bv, SCF(0, ip), pf);
              pt = fma(bv, SCF(1, ip), pt);
            }
            v = pf - pt;
          }
          Bm[(size_t)kk * R + r] = v;
        }
        __syncthreads();
        if (tid == 0) {
          double den = 1.0 - Bm[(size_t)kk * R + row];
          if (fabs(den) < ISL_TOL) { s.fail = BDC_TASK_DISCONNECT_ISLAND; s.farg = i; }
          s.den = den;
        }
        __syncthreads();
        if (s.fail) goto done;
        for (int r = tid; r < R; r += UT)
          Bm[(size_t)kk * R + r] = (r == row) ? -1.0 : Bm[(size_t)kk * R + r] / s.den;
        const int ncols = C0 + k;
        for (int col = tid; col < ncols; col += UT) {
          double v = g.P0[(size_t)row * C0 + base_col(g, s, col)];
          for (int ip = 0; ip < kk; ++ip) v = fma(OB(0, ip), Cm[(size_t)ip * Cs + col], v);
          Cm[(size_t)kk * Cs + col] = v;
        }
        __syncthreads();
        if (tid == 0) { s.dead[s.nd] = row; ++s.nd; }
        __syncthreads();
      }
    }
  }

  {
    // ---- contingency factors (solver.py:438-503) -----------------------------------
    const int rt = k + s.d;
    const int nd = s.nd;
    // single-branch cases: W(c,:), den_c, feasibility
    for (int c = tid; c < g.N1; c += UT) {
      const int row = g.sc_row[c];
      const int fc = curcol(s, rh_key, rh_col, row, 0, g.row_from[row]), tc = curcol(s, rh_key, rh_col, row, 1, g.row_to[row]);
      double* Wc = w.Wsc + ((size_t)b * g.N1 + c) * rs;
      double diag = g.sc_delta[c];
      const bool dead = is_dead(s.dead, nd, row);
      for (int j = 0; j < rt; ++j) {
        double wv = Cm[(size_t)j * Cs + fc] - Cm[(size_t)j * Cs + tc];
        Wc[j] = wv;
        diag = fma(Bm[(size_t)j * R + row], wv, diag);
      }
      if (dead) diag = 0.0;
      const double den = 1.0 - diag;
      const bool ok = fabs(den) >= ISL_TOL;
      w.den[(size_t)b * g.N1 + c] = den;
      w.sc_ok[(size_t)b * g.N1 + c] = ok;
      if (!ok) { set_island(w, b, g.sc_order[c]); atomicAdd(&s.nisl, 1); }
    }
    // multi-branch cases: m x m inner system, SVD islanding test, inverse; a warp per case
    // (lanes form the member W rows and the m x m entries, lane 0 factorises)
    for (int q = tid >> 5; q < g.NM; q += UW) {
      const int lane = tid & 31, wid = tid >> 5;
      const int st = g.mc_start[q], m = g.mc_start[q + 1] - st;
      for (int idx = lane; idx < m * rt; idx += 32) {
        const int i = idx / rt, j = idx % rt;
        const int row = g.mb_row[st + i];
        const int fc = curcol(s, rh_key, rh_col, row, 0, g.row_from[row]), tc = curcol(s, rh_key, rh_col, row, 1, g.row_to[row]);
        w.Wm[((size_t)b * g.NMB + st + i) * rs + j] = Cm[(size_t)j * Cs + fc] - Cm[(size_t)j * Cs + tc];
      }
      __syncwarp();
      double* A = mA[wid];
      for (int idx = lane; idx < m * m; idx += 32) {
        const int aa = idx / m, bb = idx % m;
        const int ra = g.mb_row[st + aa];
        double v = g.Dm64[(size_t)(st + bb) * R + ra];
        const double* Wq = w.Wm + ((size_t)b * g.NMB + st + bb) * rs;
        for (int j = 0; j < rt; ++j) v = fma(Bm[(size_t)j * R + ra], Wq[j], v);
        if (is_dead(s.dead, nd, ra)) v = 0.0;
        A[aa * m + bb] = (aa == bb ? 1.0 : 0.0) - v;
      }
      __syncwarp();
      if (lane == 0) {
        double smax, smin;
        double* inv = w.minv + ((size_t)b * g.NM + q) * MMAX * MMAX;
        bool ok;
        if (m == 2) {
          // closed form: sigma_max from the Frobenius norm and |det|, sigma_min = |det| / sigma_max
          const double a = A[0], bq = A[1], c = A[2], d = A[3];
          const double S = a * a + bq * bq + c * c + d * d, det = a * d - bq * c;
          smax = sqrt(0.5 * (S + sqrt(fmax(S * S - 4.0 * det * det, 0.0))));
          smin = smax > 0.0 ? fabs(det) / smax : 0.0;
          ok = !(smin < ISL_TOL * fmax(1.0, smax));
          if (ok) {
            const double id = 1.0 / det;
            inv[0] = d * id; inv[1] = -bq * id; inv[2] = -c * id; inv[3] = a * id;
          }
        } else {
          svd_minmax(A, m, smax, smin);
          ok = !(smin < ISL_TOL * fmax(1.0, smax));
          if (ok) invert_small(A, m, inv);
        }
        w.mc_ok[(size_t)b * g.NM + q] = ok;
        if (!ok) { set_island(w, b, g.mc_order[q]); atomicAdd(&s.nisl, 1); }
      }
      __syncwarp();
    }
    // injection cases: coupler coefficients of the outaged injection's columns
    for (int q = tid; q < g.NI; q += UT) {
      int ca, cb;
      const int sl = g.ic_slot[q];
      if (sl >= 0) {
        ca = g.slot_col[sl]; cb = ca;
        for (int j = 0; j < k; ++j) if (s.sub[j] == g.slot_sub[sl]) cb = C0 + j;
      } else {
        ca = cb = g.ic_col[q];
      }
      double* pa = w.cia + ((size_t)b * g.NI + q) * rs;
      double* pb = w.cib + ((size_t)b * g.NI + q) * rs;
      for (int j = 0; j < rt; ++j) { pa[j] = Cm[(size_t)j * Cs + ca]; pb[j] = Cm[(size_t)j * Cs + cb]; }
    }
    // active slots (slot at a split substation, nonzero setpoint), in slot order
    for (int c0 = 0; c0 < g.K; c0 += UT) {
      const int sl = c0 + tid;
      int cb = -1;
      if (sl < g.K && g.slot_sp[sl] != 0.0)
        for (int j = 0; j < k; ++j) if (s.sub[j] == g.slot_sub[sl]) cb = C0 + j;
      int total;
      int pos = block_rank(cb >= 0, s.wcnt, total);
      if (cb >= 0) {
        int p = s.nact + pos;
        if (p < ACTMAX) {
          s.act_slot[p] = sl; s.act_ca[p] = g.slot_col[sl]; s.act_cb[p] = cb;
          s.act_sp[p] = g.slot_sp[sl];
        }
      }
      __syncthreads();
      if (tid == 0) s.nact += total;
      __syncthreads();
    }
    if (s.nact > ACTMAX) {
      if (tid == 0) { s.fail = BDC_TASK_DETACHED; s.farg = -4; }
      __syncthreads();
      goto done;
    }
    // y_base[j] = sum_col p_base[col] C[j][col]  (every slot at home)
    {
      const int lane = tid & 31, wid = tid >> 5;
      for (int j = wid; j < rt; j += UW) {
        double acc = 0.0;
        for (int col = lane; col < C0; col += 32) acc = fma(g.p_base[col], Cm[(size_t)j * Cs + col], acc);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) s.ybase[j] = acc;
      }
    }
    __syncthreads();
    // Y[j][t] = y_base[j] + sum_active bit(t, s) * sp_s (C[j][col_b] - C[j][col_a])
    const uint8_t* ib = w.inj + (size_t)b * w.T * g.K;
    double* Y = w.Y + (size_t)b * rs * w.T;
    for (int idx = tid; idx < rt * w.T; idx += UT) {
      const int j = idx / w.T, t = idx % w.T;
      double y = s.ybase[j];
      for (int a2 = 0; a2 < s.nact; ++a2)
        if (ib[(size_t)t * g.K + s.act_slot[a2]])
          y += s.act_sp[a2] * (Cm[(size_t)j * Cs + s.act_cb[a2]] - Cm[(size_t)j * Cs + s.act_ca[a2]]);
      Y[idx] = y;
    }
    __syncthreads();
    if (tid == 0) {
      if (s.nisl > 0 && cfg.policy == 1) { s.fail = BDC_TASK_ISLAND_ERROR; s.farg = s.nisl; }
      w.rank[b] = rt;
    }
    __syncthreads();
  }
  __syncthreads();

done:
  if (tid == 0) {
    w.status[b] = s.fail;
    w.sarg[b] = s.farg;
    w.nsplit[b] = s.k;
    w.ndead[b] = s.nd;
    w.nisl[b] = s.nisl;
    for (int i = 0; i < s.nd; ++i) w.dead[(size_t)b * RMAX + i] = s.dead[i];
    for (int j = 0; j < s.k && j < RMAX; ++j) w.splitsub[(size_t)b * RMAX + j] = s.sub[j];
    // splits applied until the first failure (Instrumentation.count_bsdf, solver.py:375)
    int applied = s.k;
    if (s.fail == BDC_TASK_DEGENERATE_SPLIT || s.fail == BDC_TASK_SINGULAR_SPLIT) applied = s.farg;
    atomicAdd(w.bsdf, (unsigned long long)applied);
  }
#undef MB
#undef SCF
#undef OB
}

// ---- multi-branch and injection cases as correction terms (solver.py:614-622):
// F = n0 + sum_j Lo[r][j] So[j][t], columns formed once per task in FP64 and rounded
// to FP32 (scaled by 1/rating) for k_other.  grid (blocks, task): a thread per monitored
// row forms that row's terms of every case (its B'' values loaded once), the remaining
// threads the (term, candidate) multipliers.
__global__ void __launch_bounds__(NT) k_terms(DevGrid g, Work w) {
  const int b = blockIdx.y;
  if (w.status[b] != 0) return;
  const int R = g.R, rs = w.rs, rt = w.rank[b], T = w.T, M = g.M;
  const int NTM = w.NTERM, MT = g.MT, NQ = g.NM + g.NI;
  const int nd = w.ndead[b];
  const int* dead = w.dead + (size_t)b * RMAX;
  const double* Bm = w.Bm + (size_t)b * rs * R;
  float* Lo = w.Lo + (size_t)b * M * NTM;
  float* So = w.So + (size_t)b * NTM * T;
  const uint8_t* ib = w.inj + (size_t)b * T * g.K;
  const double* Wm = w.Wm + (size_t)b * g.NMB * rs;
  const double* Mi = w.minv + (size_t)b * g.NM * MMAX * MMAX;
  const uint8_t* mok = w.mc_ok + (size_t)b * g.NM;
  const int nlo = M, nso = NTM * T;
  for (int idx = blockIdx.x * NT + threadIdx.x; idx < nlo + nso; idx += gridDim.x * NT) {
    if (idx < nlo) {
      const int p = idx;
      const int row = g.mon_row[p];
      const double inv = g.inv_rating[p];
      float* out = Lo + (size_t)p * NQ * MT;
      if (is_dead(dead, nd, row)) {
        for (int i = 0; i < NQ * MT; ++i) out[i] = 0.f;
        continue;
      }
      double bv[RMAX];
#pragma unroll 8
      for (int j = 0; j < rt; ++j) bv[j] = Bm[(size_t)j * R + row];
      for (int q = 0; q < g.NM; ++q) {
        float* o = out + q * MT;
        for (int j = 0; j < MT; ++j) o[j] = 0.f;
        if (!mok[q]) continue;
        const int st = g.mc_start[q], m = g.mc_start[q + 1] - st;
        int own = -1;
        for (int a2 = 0; a2 < m; ++a2) if (g.mb_row[st + a2] == row) own = a2;
        if (own >= 0) {
          o[own] = (float)(-inv);
          continue;
        }
        double Dv[MMAX];
        for (int i = 0; i < m; ++i) {
          double v = g.Dm64[(size_t)(st + i) * R + row];
          const double* Wq = Wm + (size_t)(st + i) * rs;
          for (int j = 0; j < rt; ++j) v = fma(bv[j], Wq[j], v);
          Dv[i] = v;
        }
        const double* Mq = Mi + (size_t)q * MMAX * MMAX;
        for (int j = 0; j < m; ++j) {
          double v = 0.0;
          for (int i = 0; i < m; ++i) v += Dv[i] * Mq[i * m + j];
          o[j] = (float)(v * inv);
        }
      }
      for (int qi = 0; qi < g.NI; ++qi) {
        float* o = out + (g.NM + qi) * MT;
        const int sl = g.ic_slot[qi];
        const int ca = sl >= 0 ? g.slot_col[sl] : g.ic_col[qi];
        const double* pa_ = w.cia + ((size_t)b * g.NI + qi) * rs;
        const double* pb_ = w.cib + ((size_t)b * g.NI + qi) * rs;
        double pa = g.P0T[(size_t)ca * R + row], pb = pa;
        for (int j = 0; j < rt; ++j) {
          pa = fma(bv[j], pa_[j], pa);
          pb = fma(bv[j], pb_[j], pb);
        }
        const double sp = g.ic_sp[qi];
        o[0] = (float)(-sp * pa * inv);
        o[1] = (float)(-sp * (pb - pa) * inv);
        for (int j = 2; j < MT; ++j) o[j] = 0.f;
      }
    } else {
      const int i2 = idx - nlo;
      const int qj = i2 / T, t = i2 % T, q = qj / MT, j = qj % MT;
      float v = 0.f;
      if (q < g.NM) {
        const int st = g.mc_start[q], m = g.mc_start[q + 1] - st;
        if (j < m) v = (float)n0_at(g, w, b, g.mb_row[st + j], t, rt, dead, nd);
      } else if (j < 2) {
        const int sl = g.ic_slot[q - g.NM];
        v = j == 0 ? 1.f : ((sl >= 0 && ib[(size_t)t * g.K + sl]) ? 1.f : 0.f);
      }
      So[i2] = v;
    }
  }
}

// ---- N-0 contraction (solver.py:575-595): n0 = f0 + B'' y_t, emitted for
//   * every monitored row as FP32 n0/rating (the only per-task tensor the N-1 stage
//     streams); its max over rows is the N-0 part of the metric (m0, m32), and
//   * the outaged row of every single case as FP32 n0, s(c,t) = n0[r_c][t]
//     (solver.py:612-613, 815), 0 for islanded cases.
// CTA = (task, N0_ROWS emitted rows); a warp takes 4 rows x 128 candidates (4 per
// lane), so every B'' / Y value it loads feeds 4 DFMAs.  Same FP64 expression as
// the reference's dgemm column (f0 + sum_j B''_j y_j), rounded once.
constexpr int N0_ROWS = 128;

// ROWS emitted rows per CTA: 192 when every row fits one CTA (small grids: one CTA per
// task instead of a full and a thin one), else 128.
template <int TPL, int ROWS>
__global__ void __launch_bounds__(NT) k_n0(DevGrid g, Work w) {
  const int b = blockIdx.y;
  if (w.status[b] != 0) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // rows emitted: monitored positions, then (unless s is read from n0s) single cases
  const int R = g.R, T = w.T, M = g.M, N1 = g.N1, NL = g.s_mon ? M : M + N1, rs = w.rs, rt = w.rank[b];
  const int r0 = blockIdx.x * ROWS, nr = min(NL - r0, ROWS);
  const double* Bm = w.Bm + (size_t)b * rs * R;
  const double* Y = w.Y + (size_t)b * rs * T;
  float* n0s = w.n0s + (size_t)b * M * T;
  float* s32 = w.s32 + (size_t)b * N1 * T;
  constexpr int TCH = 32 * TPL, RG = 4;
  extern __shared__ __align__(16) double n0sm[];
  double* sB = n0sm;                       // [rt][ROWS]  B'' on the CTA's rows
  double* sY = sB + (size_t)rs * ROWS;  // [rt][TCH]      y_t of the candidate chunk
  __shared__ double sF0[ROWS], sScl[ROWS];
  __shared__ int sLive[ROWS];
  __shared__ float sSmax[ROWS];  // max_t |s(c,t)| of the CTA's single-case rows
  __shared__ int sdead[RMAX];
  __shared__ unsigned tmax[TCH];
  __shared__ unsigned tmaxb[SB][TCH];  // per screening row block
  const int MB = screen_block_rows(M);
  const int nd = w.ndead[b];
  if (tid < nd) sdead[tid] = w.dead[(size_t)b * RMAX + tid];
  __syncthreads();
  // the CTA's emitted rows: monitored positions (n0 / rating) then single cases (n0[r_c]);
  // a thread per row (ROWS <= NT)
  static_assert(ROWS <= NT, "one emitted row per thread");
  {
    const int i = tid, li = r0 + i;
    int row = 0, live = 0;
    double scl = 1.0;
    if (i < ROWS) {
      if (li < M) {
        row = g.mon_row[li];
        scl = g.inv_rating[li];
        live = !is_dead(sdead, nd, row);
      } else if (li < NL) {
        const int c = li - M;
        row = g.sc_row[c];
        live = w.sc_ok[(size_t)b * N1 + c] && !is_dead(sdead, nd, row);
      }
      sF0[i] = live ? g.f0[row] : 0.0;
      sScl[i] = scl;
      sSmax[i] = 0.f;
      sLive[i] = live;
    }
    for (int j = 0; j < rt; ++j) {
      const double bv = i < nr ? Bm[(size_t)j * R + row] : 0.0;
      if (i < ROWS) sB[j * ROWS + i] = bv;
      unsigned bm = 0u;
      if (i < ROWS && li < M) {
        // FP32 B'' on monitored rows and max_r |B''(r,j)|/rating_r for the scale bound
        w.B32[(size_t)b * b32_task_floats(rs, M) + b32_off(rs, li, j)] = live ? (float)(bv * scl) : 0.f;
        w.Bmon[((size_t)b * rs + j) * M + li] = bv;
        if (live) bm = __float_as_uint((float)(fabs(bv) * scl) * (1.f + 1e-6f));
      }
      // one atomic per warp and rank term (same-address atomics from every row are slow)
      bm = __reduce_max_sync(0xffffffffu, bm);
      if (lane == 0 && bm) atomicMax(reinterpret_cast<unsigned*>(&w.bmax[(size_t)b * rs + j]), bm);
    }
  }
  for (int tc = 0; tc < T; tc += TCH) {
    for (int i = tid; i < TCH; i += NT) tmax[i] = 0u;
    for (int i = tid; i < SB * TCH; i += NT) (&tmaxb[0][0])[i] = 0u;
    for (int idx = tid; idx < rt * TCH; idx += NT) {
      const int j = idx / TCH, t = tc + idx % TCH;
      sY[idx] = t < T ? Y[(size_t)j * T + t] : 0.0;
    }
    __syncthreads();
    float mx[TPL];
#pragma unroll
    for (int k = 0; k < TPL; ++k) mx[k] = 0.f;
    for (int i0 = wid * RG; i0 < nr; i0 += NW * RG) {
      double acc[RG][TPL];
#pragma unroll
      for (int i = 0; i < RG; ++i)
#pragma unroll
        for (int k = 0; k < TPL; ++k) acc[i][k] = sF0[i0 + i];
      for (int j = 0; j < rt; ++j) {
        double bv[RG], yv[TPL];
#pragma unroll
        for (int i = 0; i < RG; ++i) bv[i] = sB[j * ROWS + i0 + i];
#pragma unroll
        for (int k = 0; k < TPL; ++k) yv[k] = sY[j * TCH + lane + 32 * k];
#pragma unroll
        for (int i = 0; i < RG; ++i)
#pragma unroll
          for (int k = 0; k < TPL; ++k) acc[i][k] = fma(bv[i], yv[k], acc[i][k]);
      }
      float gm[TPL];  // this row group's max per candidate (one screening block: MB % RG == 0)
#pragma unroll
      for (int k = 0; k < TPL; ++k) gm[k] = 0.f;
      // (TPL <= 2 only: with four candidates per lane the second copy of the loop cost
      // registers -- G1k N-0 stage 2.25 -> 2.83 ms)
      if (TPL <= 2 && i0 + RG <= nr && r0 + i0 + RG <= M && tc + TCH <= T) {
        // the common case -- RG monitored rows, a full candidate chunk: the same values
        // without the per-element guards
#pragma unroll
        for (int i = 0; i < RG; ++i) {
          float* dst = n0s + (size_t)(r0 + i0 + i) * T + tc + lane;
          const bool live = sLive[i0 + i] != 0;
          const double scl = sScl[i0 + i];
          float rmax = 0.f;
#pragma unroll
          for (int k = 0; k < TPL; ++k) {
            const float v = live ? (float)(acc[i][k] * scl) : 0.f;
            dst[32 * k] = v;
            const float a = fabsf(v);
            mx[k] = fmaxf(mx[k], a);
            gm[k] = fmaxf(gm[k], a);
            rmax = fmaxf(rmax, a);
          }
          rmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(rmax)));
          if (lane == 0) sSmax[i0 + i] = fmaxf(sSmax[i0 + i], rmax);
        }
      } else
#pragma unroll
      for (int i = 0; i < RG; ++i) {
        const int li = r0 + i0 + i;
        if (i0 + i >= nr) break;
        float* dst = li < M ? n0s + (size_t)li * T : s32 + (size_t)(li - M) * T;
        const bool live = sLive[i0 + i] != 0;
        const double scl = sScl[i0 + i];
        float rmax = 0.f;
#pragma unroll
        for (int k = 0; k < TPL; ++k) {
          const int t = tc + lane + 32 * k;
          if (t >= T) continue;
          const float v = live ? (float)(acc[i][k] * scl) : 0.f;
          dst[t] = v;
          if (li < M) {
            mx[k] = fmaxf(mx[k], fabsf(v));
            gm[k] = fmaxf(gm[k], fabsf(v));
          }
          rmax = fmaxf(rmax, fabsf(v));
        }
        {  // warp-uniform: the row's max over this candidate chunk (non-negative floats
           // order as their bit patterns: one redux instead of five shuffle + max steps)
          rmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(rmax)));
          if (lane == 0) sSmax[i0 + i] = fmaxf(sSmax[i0 + i], rmax);
        }
      }
      if (r0 + i0 < M) {
        const int blk = (r0 + i0) / MB;
#pragma unroll
        for (int k = 0; k < TPL; ++k) atomicMax(&tmaxb[blk][lane + 32 * k], __float_as_uint(gm[k]));
      }
    }
#pragma unroll
    for (int k = 0; k < TPL; ++k) atomicMax(&tmax[lane + 32 * k], __float_as_uint(mx[k]));
    __syncthreads();
    if (r0 < M) {  // CTAs with monitored rows fold their per-candidate max into m0 / m32
      for (int i = tid; i < min(TCH, T - tc); i += NT) {
        atomicMax(&w.m32[(size_t)b * T + tc + i], tmax[i]);
        atomicMax(reinterpret_cast<unsigned*>(&w.m0[(size_t)b * T + tc + i]), tmax[i]);
      }
      const int blo = r0 / MB, bhi = (min(r0 + nr, M) - 1) / MB;
      for (int blk = blo; blk <= bhi; ++blk)
        for (int i = tid; i < min(TCH, T - tc); i += NT)
          atomicMax(reinterpret_cast<unsigned*>(&w.m0b[((size_t)b * SB + blk) * T + tc + i]), tmaxb[blk][i]);
      // and max_t m0_b(t), the screening key's N-0 term (k_scale_tc): one atomic per block
      if (wid == 0)
        for (int blk = blo; blk <= bhi; ++blk) {
          unsigned v = 0u;
          for (int i = lane; i < min(TCH, T - tc); i += 32) v = max(v, tmaxb[blk][i]);
          v = __reduce_max_sync(0xffffffffu, v);
          if (lane == 0 && v) atomicMax(reinterpret_cast<unsigned*>(&w.m0bx[(size_t)b * SB + blk]), v);
        }
    }
    __syncthreads();
  }
  for (int i = tid; i < nr; i += NT) {
    if (r0 + i >= M) w.smax[(size_t)b * N1 + (r0 + i - M)] = sSmax[i];
    else w.rmax[(size_t)b * M + r0 + i] = sSmax[i];
  }
}

// The ptop single cases with the largest screening bound bkey_c (the cases the
// reference's metric_first visits first, solver.py:818): one CTA per task, radix
// select on the key bits, ties resolved toward the lower case index.
__global__ void __launch_bounds__(NT) k_topk(DevGrid g, Work w) {
  const int b = blockIdx.x, tid = threadIdx.x;
  if (w.status[b] != 0) return;
  __shared__ int hist[256];
  __shared__ int wcnt[NW];
  __shared__ int sel_digit, sel_above, ntop, ntie;
  const int N1 = g.N1;
  const uint32_t* key = w.bkey + (size_t)b * N1;
  const int P = min(w.ptop, N1);
  uint32_t prefix = 0, mask = 0;
  int need = P;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += NT) hist[i] = 0;
    __syncthreads();
    for (int c = tid; c < N1; c += NT) {
      const uint32_t k = key[c];
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int acc = 0, d = 255;
      for (; d > 0; --d) {
        if (acc + hist[d] >= need) break;
        acc += hist[d];
      }
      sel_digit = d;
      sel_above = acc;
    }
    __syncthreads();
    need -= sel_above;
    prefix |= (uint32_t)sel_digit << shift;
    mask |= 255u << shift;
    __syncthreads();
  }
  // prefix = the P-th largest key: every key above it is taken, then `need` ties in index order
  uint8_t* done = w.done + (size_t)b * N1;
  int* top = w.top + (size_t)b * w.ptop;
  if (tid == 0) { ntop = 0; ntie = 0; }
  __syncthreads();
  for (int c0 = 0; c0 < N1; c0 += NT) {
    const int c = c0 + tid;
    const uint32_t k = c < N1 ? key[c] : 0u;
    const bool tie = c < N1 && k == prefix;
    int total;
    const int pos = block_rank(tie, wcnt, total);
    const bool take = c < N1 && (k > prefix || (tie && ntie + pos < need));
    if (c < N1) done[c] = take ? 1 : 0;
    __syncthreads();
    if (tid == 0) ntie += total;
    __syncthreads();
  }
  for (int c0 = 0; c0 < N1; c0 += NT) {
    const int c = c0 + tid;
    const bool take = c < N1 && done[c];
    int total;
    const int pos = block_rank(take, wcnt, total);
    if (take) top[ntop + pos] = c;
    __syncthreads();
    if (tid == 0) ntop += total;
    __syncthreads();
  }
  for (int i = ntop + tid; i < w.ptop; i += NT) top[i] = -1;
}

void launch_update(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t st) {
  const size_t dyn = update_dyn_bytes(w.rs, g.E > 0 ? g.E : 1);
  if (g.R > 2048) {
    smem_opt_in((const void*)k_update<512, 2>, (int)dyn);
    k_update<512, 2><<<w.Wb, 512, dyn, st>>>(g, c, w);
  } else if (g.R > 512) {
    smem_opt_in((const void*)k_update<256, 4>, (int)dyn);
    k_update<256, 4><<<w.Wb, 256, dyn, st>>>(g, c, w);
  } else if (g.R > 256 || (getenv("BDC_UPDATE_NT") && atoi(getenv("BDC_UPDATE_NT")) == 128)) {
    smem_opt_in((const void*)k_update<128, 8>, (int)dyn);
    k_update<128, 8><<<w.Wb, 128, dyn, st>>>(g, c, w);
  } else {
    // small grids: a warp per task -- no cross-warp barrier waits on the serial split setup
    smem_opt_in((const void*)k_update<32, 32>, (int)dyn);
    k_update<32, 32><<<w.Wb, 32, dyn, st>>>(g, c, w);
  }
}

// The multi/injection correction terms (after k_update; independent of k_n0, so bdc_solve
// runs them on a side stream next to it).
void launch_terms(const DevGrid& g, const Work& w, cudaStream_t st) {
  if (w.NTERM > 0 && g.M > 0) {
    // >= 8 items per thread: small grids take one CTA per task (the per-CTA cost, not
    // the items, dominated with several thin CTAs per task), large grids up to eight
    const int work = g.M + w.NTERM * w.T;
    const dim3 grid((unsigned)std::max(1, std::min(8, work / (8 * NT))), w.Wb);
    k_terms<<<grid, NT, 0, st>>>(g, w);
  }
}

void launch_n0(const DevGrid& g, const Work& w, cudaStream_t st) {
  const int NL = g.s_mon ? g.M : g.M + g.N1;
  if (NL == 0) return;
  const int rows = NL <= 192 ? 192 : N0_ROWS;
  const dim3 grid((NL + rows - 1) / rows, w.Wb);
  const int tpl = w.T > 64 ? 4 : (w.T > 32 ? 2 : 1);
  const size_t dyn = (size_t)w.rs * (rows + 32 * tpl) * sizeof(double);
  auto go = [&](auto kern) {
    smem_opt_in((const void*)kern, (int)dyn);
    kern<<<grid, NT, dyn, st>>>(g, w);
  };
  if (rows == 192) {
    if (tpl == 4) go(k_n0<4, 192>);
    else if (tpl == 2) go(k_n0<2, 192>);
    else go(k_n0<1, 192>);
  } else {
    if (tpl == 4) go(k_n0<4, N0_ROWS>);
    else if (tpl == 2) go(k_n0<2, N0_ROWS>);
    else go(k_n0<1, N0_ROWS>);
  }
}

// k_topk for small grids (N1 <= 32 KW): a warp per task, keys in registers, ptop rounds
// of warp argmax by (key desc, index asc) -- the same set as k_topk's radix select.
template <int KW>
__global__ void __launch_bounds__(NT) k_topk_w(DevGrid g, Work w) {
  const int lane = threadIdx.x & 31, b = blockIdx.x * NW + (threadIdx.x >> 5);
  if (b >= w.Wb || w.status[b] != 0) return;
  const int N1 = g.N1, P = min(w.ptop, N1);
  const uint32_t* key = w.bkey + (size_t)b * N1;
  uint32_t kv[KW];
  bool take[KW];
#pragma unroll
  for (int k = 0; k < KW; ++k) {
    const int c = lane + 32 * k;
    kv[k] = c < N1 ? key[c] : 0u;
    take[k] = false;
  }
  for (int e = 0; e < P; ++e) {
    uint32_t bv = 0u;
    int bi = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      const int c = lane + 32 * k;
      if (c < N1 && !take[k] && (kv[k] > bv || (kv[k] == bv && c < bi))) { bv = kv[k]; bi = c; }
    }
    for (int o = 16; o; o >>= 1) {
      const uint32_t ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
#pragma unroll
    for (int k = 0; k < KW; ++k)
      if (lane + 32 * k == bi) take[k] = true;
  }
  uint8_t* done = w.done + (size_t)b * N1;
  int* top = w.top + (size_t)b * w.ptop;
  int off = 0;
#pragma unroll
  for (int k = 0; k < KW; ++k) {  // ascending case index (k-major)
    const int c = lane + 32 * k;
    if (c < N1) done[c] = take[k] ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, take[k]);
    if (take[k]) top[off + __popc(bal & ((1u << lane) - 1u))] = c;
    off += __popc(bal);
  }
  for (int i = off + lane; i < w.ptop; i += 32) top[i] = -1;
}

void launch_topk(const DevGrid& g, const Work& w, cudaStream_t st) {
  if (g.N1 == 0 || g.M == 0) return;
  if (g.N1 <= 32 * 16) k_topk_w<16><<<(w.Wb + NW - 1) / NW, NT, 0, st>>>(g, w);
  else k_topk<<<w.Wb, NT, 0, st>>>(g, w);
}

}  // namespace bdc
