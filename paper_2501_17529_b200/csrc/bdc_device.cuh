// bdc_device.cuh -- device-side data structures and small helpers shared by
// the engine's kernels.  See DESIGN.md for the data layout in HBM.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/bdc.h"

namespace bdc {

constexpr int RMAX = BDC_MAX_RANK;        // rank k+d per task
constexpr int EMAX = BDC_MAX_ELEMENTS;    // branch elements per substation
constexpr int MMAX = BDC_MAX_MULTI;       // branches per multi-branch case
constexpr int KMAX = BDC_MAX_TOPK;        // top-k limits
constexpr int ACTMAX = 64;                // active slots (slots at split substations) per task
constexpr int RHMAX = RMAX * EMAX;        // re-homed branch ends per task
constexpr int PFX_LEVELS = 2;             // split-prefix levels shared through k_update's memo
constexpr double ISL_TOL = 1e-8;          // ISLANDING_TOL == SPLIT_TOL (factors.py:48-49)
// Absolute margin (in units of relative loading) on the FP32 screening values
// used to decide which cases the FP64 winner report must revisit.  The FP32
// path's observed error is ~1e-6 (tests: <= 1e-5 enforced), so 1e-3 is a
// >= 100x safety factor; a wider margin only costs report time.
constexpr float SCREEN_EPS = 1e-3f;
// Half-width of the winner's near-tie band, relative to max(1, metric): a bound on
// |m32(t) - m64(t)| between a candidate's FP32 screening metric and its FP64 metric.  The
// FP32 flows are FP64 values rounded once and combined by one FFMA (observed error
// ~1.3e-6, tests enforce <= 1e-5); 2^-14 = 6.1e-5 keeps a > 40x margin.  Every candidate
// with m32 within 2 RESCORE_EPS of the FP32 minimum is re-scored in FP64 (k_rescore), so
// best_injection is the first argmin of the FP64 metrics, as the reference's
// (solver.py:804-823).
constexpr float RESCORE_EPS = 6.103515625e-05f;
// Single-branch N-1 stage with the exact dominance screen (bdc_single.cu):
//   TOPC  cases evaluated first for every candidate (the top of the screening ranking);
//   SB    row blocks of the screening bound |F(r,c,t)| <= max_b (m0_b(t) + scale_bc |s(c,t)|):
//         per-block maxima over monitored rows pair large N-0 rows and large LODF rows
//         only when they fall in the same block, which is much tighter than one block.
constexpr int TOPC = 16;
constexpr int SB = 4;
// Candidates per TOP-tile CTA (bdc_single.cu launch_top).
__host__ __device__ inline int top_tile_cands(int T) { return T >= 96 ? 128 : (T >= 48 ? 64 : 32); }
// B32 (k_n0 writes, k_scale_tc reads): per task, 64-row chunks of the monitored rows; each
// chunk holds KB blocks of the UMMA K-major no-swizzle core-matrix layout (64 rows x 8 TF32
// values = 2 KB: 8-row x 16-byte core matrices, K halves at +128 B, row groups at +256 B),
// so the tensor-core kernel stages a chunk with contiguous 16-byte copies.
__host__ __device__ inline int b32_kb(int rs) { return rs <= 8 ? 1 : (rs <= 16 ? 2 : 4); }
__host__ __device__ inline size_t b32_task_floats(int rs, int M) {
  return (size_t)((M + 63) / 64) * b32_kb(rs) * 512;
}
__host__ __device__ inline size_t b32_off(int rs, int m, int j) {  // in floats
  const int ch = m >> 6, r = m & 63, kb = j >> 3, jj = j & 7;
  return ((size_t)ch * b32_kb(rs) + kb) * 512 + (size_t)((r >> 3) * 64 + (jj >> 2) * 32 + (r & 7) * 4 + (jj & 3));
}
// Rows per screening block: a multiple of 32 (the k_scale epilogue's row half, also a
// multiple of the k_n0 row group), so neither straddles two blocks; block of m = m / MB.
__host__ __device__ inline int screen_block_rows(int M) {
  const int per = (M + SB - 1) / SB;
  return ((per + 31) / 32) * 32 > 0 ? ((per + 31) / 32) * 32 : 32;
}
// single cases per CTA of the winner report sweep: RCW on batches of many tasks (one CTA
// per task covers most listings), RCW_MIN where few tasks must fill the GPU (Work::rcw)
constexpr int RCW = 160;
constexpr int RCW_MIN = 64;
constexpr int RSEL_WARPS = 8;   // partial report lists written by the report-select kernel

// Grid tables, device-resident for the session lifetime.
struct DevGrid {
  int R, C0, M, S, E, K, N1, NM, NMB, NI, NC, NBR, static_col;
  int N1p;  // row stride of D32 (N1 rounded up to a multiple of 4)
  int MT;   // correction-term slots per multi/injection case (max branches, pow2 >= 2)
  const double *P0, *P0T, *f0, *p_base, *rating, *inv_rating, *sub_elem_b, *slot_sp;
  const double *sc_delta, *sc_dscale, *D64, *Dm64, *ic_sp;
  const double* DM64;  // (N1, M) D_base on monitored rows, case-major (winner report)
  const float* DsT;    // (N1, Mp) D_base / rating on monitored rows, case-major, FP32 (k_scale)
  const CUtensorMap* tm_ds;  // host pointer: TMA descriptor of DsT (box 32 rows x 128 cases, 128B swizzle)
  // pre-outage flow of single case c: when every outaged row is monitored (s_mon), it is
  // read from the N-0 table, s(c,t) = n0s[sc_pos[c]][t] * sc_rat[c]; otherwise from s32
  const int* sc_pos;   // (N1) monitored position of the outaged row (-1: unmonitored)
  const float* sc_rat; // (N1) its rating (FP32)
  int s_mon;           // 1: every single case's outaged row is monitored
  int Mp;              // M rounded up to a multiple of 4
  const float* D32;
  const int *row_from, *row_to, *branch_row, *mon_row, *row_mon_pos, *sub_col, *sub_count;
  const int *sub_elem_row, *slot_sub, *slot_col, *sc_row, *sc_order, *mc_start, *mc_order;
  const int *mb_row, *ic_slot, *ic_col, *ic_order;
};

struct DevCfg {
  int kc, kg, policy, method, maxout;
  double penalty;
};

// One wave of tasks: inputs, per-task factor workspace, outputs.
struct Work {
  int Wb;         // tasks in the wave
  int T, D, Ein;  // candidates, disconnection columns, split-array width
  int rs;         // rank stride (max k+d in the batch, >= 1)
  int Cs;         // column stride of the coupler rows = C0 + rs
  int NCw;        // 32-bit words of the islanded bitmap
  // inputs (device)
  const uint8_t* splits;   // (Wb, S, Ein)
  const int64_t* discos;   // (Wb, D)
  const uint8_t* inj;      // (Wb, T, K)
  const int* tcount;       // (Wb) or null
  const uint8_t* in2_splits; const int64_t* in2_discos; const uint8_t* in2_inj; const int* in2_tcount;  // 2nd input buffer
  // per-task scalars
  int* status; int* sarg; int* rank; int* nsplit; int* ndead; int* dead;  // dead: (Wb, RMAX)
  int* splitsub;  // (Wb, RMAX) substation of split j
  int* nisl;      // (Wb)
  uint32_t* isl;  // (Wb, NCw)
  // factors (FP64)
  double* Bm;     // (Wb, rs, R)   column j of B'' contiguous over rows
  double* Cm;     // (Wb, rs, Cs)  coupler / outage row j over logical columns
  double* Wsc;    // (Wb, N1, rs)  W(c, j) = C[j][f'_c] - C[j][t'_c]
  double* den;    // (Wb, N1)      1 - D''(r_c, c)
  uint8_t* sc_ok; // (Wb, N1)
  double* Wm;     // (Wb, NMB, rs)
  double* minv;   // (Wb, NM, MMAX*MMAX) inverse of the m x m inner system
  uint8_t* mc_ok; // (Wb, NM)
  double* cia; double* cib;  // (Wb, NI, rs) coupler coefficients of the injection column
  double* Y;      // (Wb, rs, T)   y_t = C''^T p_t
  float* n0s;     // (Wb, M, T)    N-0 flows / rating on monitored rows, FP32
  uint32_t* m32;  // (Wb, T)       FP32 screening metric (float bits, >= 0)
  float* cmax;    // (Wb, N1+NM+NI, T) FP32 max |F|/rating per (case, candidate); for single
                  //                   cases valid where evaluated (done[c] != 0, or c < ptop
                  //                   when the cases are not ranked)
  int* llist;     // (Wb, N1)      live single cases of each task (screen failed), any order
  int* lcnt;      // (Wb)          their number
  int2* queue;    // (Wb * ceil(N1/TOPC) * candidate tiles)  k_pairs items (task, group<<16 | tile)
  unsigned* qcount;  // items in the queue (device counter, reset per wave)
  float* m0b;     // (Wb, SB, T)   FP32 max |n0|/rating per screening row block
  float* m0bx;    // (Wb, SB)      max_t m0b (k_n0; the screening key's N-0 term)
  // prefix-shared split chains (k_update): hash table of split prefixes, per wave
  int pfx_cap;                    // slots (power of two), 0 = off
  unsigned long long* pfx_key;    // (cap) prefix hash, 0 = empty
  int* pfx_state;                 // (cap) 0 free, 1 claimed, 2 published
  int* pfx_fail;                  // (cap) BDC_TASK_* of the split (0 ok)
  int* pfx_id;                    // (cap, 2 PFX_LEVELS) the prefix (substation, bits) per level
  double* pfx_B;                  // (cap, R)  B_j
  double* pfx_C;                  // (cap, Cs) C_j over columns 0..C0+j
  uint8_t* oskip; // (Wb, NQ)      multi/injection case skipped by k_oscreen (cmax holds a bound)
  int* olist;     // (Wb, NQ)      the cases k_other evaluates, ascending
  int* ocnt;      // (Wb)
  int oscr;       // 1: k_oscreen runs (many cases over many candidates), else every case is
                  //    evaluated (oskip / olist unused)
  float* m0;      // (Wb, T)       FP32 N-0 max |n0|/rating (dominance-screen bound)
  float* scale;   // (Wb, SB, N1)  FP32 upper bound of max_{r in block} |LODF(r,c)|/rating_r
  float* B32;     // (Wb, b32_task_floats) FP32 B''/rating on monitored rows, 0 on dead rows,
                  //               in the tensor-core operand layout (b32_off)
  float* bmax;    // (Wb, rs)      max_r |B''(r,j)|/rating_r (float bits, atomicMax)
  unsigned long long* pairs;  // evaluated (single case, candidate) pairs, all tasks
  int* rsq;       // (Wb)          tasks whose winner band holds more than one candidate
  unsigned* rsq_n;  // their number (device counter, reset per wave)
  int screen;     // 1 = exact dominance screen on
  int rescore_full;  // 1 = k_rescore evaluates every class over every row (tests)
  int scale_tgfast;  // 1 = k_scale_tc rasterises task groups fastest (large D' tables)
  int rsel_cta;   // 1: winner report selection always CTA-per-task (test knob BDC_RSEL_CTA)
  int ptop;       // cases evaluated first (the TOP tile, ranked by screening key)
  int ranked;     // 1: top tile chosen by the screening key (screen on and N1 > ptop)
  float* s32;     // (Wb, N1, T)   n0[r_c][t] (pre-outage flow of each single case), FP32
                  //               (only when !g.s_mon; see s_at)
  float* rmax;    // (Wb, M)       max_t |n0s[m][t]| (g.s_mon: smax_c = rmax[sc_pos[c]] * sc_rat[c])
  uint32_t* bkey; // (Wb, N1)      ranking key max_t m0(t) + scale_c max_t |s(c,t)| (float bits)
  float* smax;    // (Wb, N1)      max_t |s(c,t)|
  int* top;       // (Wb, ptop)    the ptop cases with the largest bound, ascending index
  uint8_t* done;  // (Wb, N1)      1: TOP case (k_topk), 2: live case (k_live); both evaluated
                  //               for every candidate
  // multi-branch / injection cases as correction terms: F = n0 + sum_j Lo[j] So[j],
  // MT term slots per case q (multi: one per outaged branch, injection: 2), zero-padded
  float* Lo;      // (Wb, M, NQ, MT)  correction columns / rating on monitored rows
  float* So;      // (Wb, NQ, MT, T)  per-candidate multipliers
  int NTERM;      // NQ * MT, NQ = NM + NI
  double* n0b;    // (Wb, R)       winner's N-0 column (report scratch)
  double* n0m;    // (Wb, M)       the same on monitored positions
  double* Bmon;   // (Wb, rs, M)   B'' on monitored positions, FP64 (winner report)
  // winner report: listed cases and per-slot partial top-kg lists
  int* rlist;     // (Wb, N1)      single cases the FP64 report must visit, ascending
  int* rcnt;      // (Wb)          their number
  float* theta;   // (Wb)          report floor: kg-th largest exact case max - 2 eps (or -1)
  int nslot;      // RSEL_WARPS + ceil(N1 / RCW_MIN) partial lists per task
  int rcw;        // single cases per k_rsweep CTA (RCW or RCW_MIN)
  int* pcase;     // (Wb, nslot, KMAX) contingency order of each partial entry
  int* ppos;      // (Wb, nslot, KMAX) monitored position
  double* pflow;  // (Wb, nslot, KMAX)
  double* prel;   // (Wb, nslot, KMAX)  rel = -1 marks an empty entry
  double* pmax;   // (Wb, nslot)     FP64 max loading over the slot's cases
  // outputs (device)
  double* metric; int64_t* best; uint8_t* feasible;
  int* n0cnt; int* n0pos; double* n0flow; double* n0rel;
  int* n1cnt; int* n1case; int* n1pos; double* n1flow; double* n1rel;
  unsigned long long* lf;     // counters: [0] loadflows [1] bsdf [2] evaluated pairs
                              // [3] report cases [4] re-scored candidates [5] winners
                              // replaced by the re-score [6] tasks with a band > 1
  unsigned long long* bsdf;   // split applications counter
};

__device__ __forceinline__ bool is_dead(const int* dead, int nd, int row) {
  for (int i = 0; i < nd; ++i)
    if (dead[i] == row) return true;
  return false;
}

__device__ __forceinline__ void atomic_max_pos(uint32_t* addr, float v) {
  // v >= 0: IEEE order of non-negative floats equals unsigned order of their bits
  atomicMax(addr, __float_as_uint(v));
}

// One-sided Jacobi SVD (Hestenes) of an n x n matrix (row-major, n <= MMAX):
// returns the largest and smallest singular values.  Accurate to eps*sigma_max,
// which the islanding test sigma_min < 1e-8 max(1, sigma_max) needs
// (factors.py:398-399); an eigen-decomposition of A^T A would square the
// condition number and blur exactly that threshold.
__device__ inline void svd_minmax(const double* A, int n, double& smax, double& smin) {
  double U[MMAX * MMAX];
  for (int i = 0; i < n * n; ++i) U[i] = A[i];
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double al = 0, be = 0, ga = 0;
        for (int i = 0; i < n; ++i) {
          double x = U[i * n + p], y = U[i * n + q];
          al += x * x; be += y * y; ga += x * y;
        }
        if (ga == 0.0 || fabs(ga) <= 1e-17 * sqrt(al * be)) continue;
        rotated = true;
        double zeta = (be - al) / (2.0 * ga);
        double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < n; ++i) {
          double x = U[i * n + p], y = U[i * n + q];
          U[i * n + p] = c * x - s * y;
          U[i * n + q] = s * x + c * y;
        }
      }
    if (!rotated) break;
  }
  smax = 0.0; smin = 1e300;
  for (int j = 0; j < n; ++j) {
    double nrm = 0;
    for (int i = 0; i < n; ++i) nrm += U[i * n + j] * U[i * n + j];
    nrm = sqrt(nrm);
    smax = fmax(smax, nrm);
    smin = fmin(smin, nrm);
  }
}

// Gauss-Jordan inverse with partial pivoting (n <= MMAX).  Returns false if a
// pivot vanishes (callers only invert systems that passed svd_minmax).
__device__ inline bool invert_small(const double* A, int n, double* Ainv) {
  double M[MMAX * 2 * MMAX];
  const int w = 2 * n;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      M[i * w + j] = A[i * n + j];
      M[i * w + n + j] = (i == j) ? 1.0 : 0.0;
    }
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int i = c + 1; i < n; ++i)
      if (fabs(M[i * w + c]) > fabs(M[p * w + c])) p = i;
    if (M[p * w + c] == 0.0) return false;
    if (p != c)
      for (int j = 0; j < w; ++j) {
        double t = M[c * w + j]; M[c * w + j] = M[p * w + j]; M[p * w + j] = t;
      }
    double inv = 1.0 / M[c * w + c];
    for (int j = 0; j < w; ++j) M[c * w + j] *= inv;
    for (int i = 0; i < n; ++i) {
      if (i == c) continue;
      double f = M[i * w + c];
      if (f != 0.0)
        for (int j = 0; j < w; ++j) M[i * w + j] -= f * M[c * w + j];
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Ainv[i * n + j] = M[i * w + n + j];
  return true;
}

// FP64 N-0 flow of one row for one candidate, from the task's factors:
// n0 = f0 + B'' y_t, exactly 0 on disconnected rows (solver.py:575-595).
__device__ __forceinline__ double n0_at(const DevGrid& g, const Work& w, int b, int row, int t,
                                        int rt, const int* dead, int nd) {
  if (is_dead(dead, nd, row)) return 0.0;
  double v = g.f0[row];
  const double* Bm = w.Bm + (size_t)b * w.rs * g.R;
  const double* Y = w.Y + (size_t)b * w.rs * w.T;
  for (int j = 0; j < rt; ++j) v = fma(Bm[(size_t)j * g.R + row], Y[(size_t)j * w.T + t], v);
  return v;
}

// max(|a|, |b|, |c|) in one FMNMX3 (sm_100+ three-input max with the |.| modifier):
// the sweeps fold two rows into an accumulator per ALU-pipe instruction.
__device__ __forceinline__ float max3abs(float a, float b, float c) {
  float d;
  asm("max.abs.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// s(c, t) = n0[r_c][t] of single case c (FP32) and max_t |s(c, t)|, the same values in every
// kernel (solver.py:612-613).
__device__ __forceinline__ float s_at(const DevGrid& g, const Work& w, int b, int c, int t) {
  if (g.s_mon) return w.n0s[((size_t)b * g.M + g.sc_pos[c]) * w.T + t] * g.sc_rat[c];
  return w.s32[((size_t)b * g.N1 + c) * w.T + t];
}
// Is the multi/injection case q's cmax the exact FP32 maximum (k_other evaluated it), or the
// dominance bound k_oscreen left when it skipped the case?
__device__ __forceinline__ bool other_exact(const DevGrid& g, const Work& w, int b, int q) {
  return !w.oscr || !w.oskip[(size_t)b * (g.NM + g.NI) + q];
}
__device__ __forceinline__ float smax_at(const DevGrid& g, const Work& w, int b, int c) {
  if (g.s_mon) return w.rmax[(size_t)b * g.M + g.sc_pos[c]] * g.sc_rat[c];
  return w.smax[(size_t)b * g.N1 + c];
}

// cp.async helpers (global -> shared, zero-filling when !ok).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// Async copies global->shared; !ok stores zeros instead.  The zeros are a plain shared
// store rather than cp.async's src-size zero-fill: a runtime source size costs ~15 extra
// SASS instructions per copy (address re-alignment arithmetic), a predicated store one.
// Readers wait for the copy group and a barrier either way, so both are visible to them.
__device__ __forceinline__ void cp4(void* dst, const void* src, bool ok) {
  if (ok) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src));
  else *reinterpret_cast<uint32_t*>(dst) = 0u;
}
__device__ __forceinline__ void cp8(void* dst, const void* src, bool ok) {
  if (ok) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src));
  else *reinterpret_cast<uint2*>(dst) = make_uint2(0u, 0u);
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
  if (ok) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
  else *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }


// Dynamic shared-memory opt-in, per (device, kernel): cudaFuncSetAttribute applies to the
// current device only, so a process-wide "done" flag would leave a second device (or a
// second session on another device) without it.  Thread-safe; the lookup is a mutex and a
// small map, cheap next to a launch.
//   smem_opt_in(fn, bytes)  ensures the kernel may launch with `bytes` of dynamic smem;
//   smem_opt_in_max(fn)     opts in to everything the static part leaves free, returns it.
cudaError_t smem_opt_in(const void* fn, int bytes);
int smem_opt_in_max(const void* fn);

// Kernel launchers.
void launch_update(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s);
void launch_terms(const DevGrid& g, const Work& w, cudaStream_t s);  // multi/injection terms (k_terms)
void launch_n0(const DevGrid& g, const Work& w, cudaStream_t s);
// the single-branch N-1 stage in two parts: scales, top-k and the TOP tile (records ev[0..2]),
// then the exact screen's live cases (k_live, k_queue, k_pairs)
void launch_single_top(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s, cudaEvent_t* ev = nullptr);
void launch_single_screen(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s);
void launch_topk(const DevGrid& g, const Work& w, cudaStream_t s);
void launch_scale(const DevGrid& g, const Work& w, cudaStream_t s);
void launch_other(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s);
bool other_screened(const DevGrid& g, const Work& w);  // does k_oscreen run (Work::oscr)?
void launch_oexact(const DevGrid& g, const Work& w, cudaStream_t s);  // report prologue
void launch_select(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s);
void launch_report(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s);
void launch_rescore(const DevGrid& g, const DevCfg& c, const Work& w, cudaStream_t s);

// Device task generation (bdc_gen.cu, bdc_draw_tasks)
struct GenArgs {
  int64_t B;
  int T, E, D, n_splits, n_disc;
  uint32_t k0, k1;         // Philox key (the seed)
  const int32_t* attempt;  // (B) draw number per task, or null (0)
  const uint8_t* redraw;   // (B) 1 = draw this task's topology, or null (all)
  uint8_t* splits;         // (B, S, E)
  int64_t* discos;         // (B, D) or null
  uint8_t* inj;            // (B, T, K) or null (topology only)
};
cudaError_t launch_draw(const DevGrid& g, const GenArgs& a, cudaStream_t s);

// SPD solve A X = B on the device (bdc_chol.cu, bdc_spd_solve): A (n x n, row-major,
// overwritten by its Cholesky factor), B (n x m, overwritten by X); info (device int):
// 0, or the first non-positive pivot's column + 1
cudaError_t launch_spd_solve(double* A, int n, double* B, int m, int* info, cudaStream_t s);
void launch_probe(const DevGrid& g, const Work& w, double* n0, double* n1, uint8_t* ok,
                  cudaStream_t s);
int kernels_per_wave(const DevGrid& g, const Work& w);
int single_launches(const DevGrid& g, const Work& w);

}  // namespace bdc
