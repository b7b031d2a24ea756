/*
 * bdc.h -- C ABI of the B200 batched DC loadflow engine (libbdc.so).
 *
 * Plain pointers and sizes only: no torch, no C++ types cross this boundary.
 * Every entry point returns an int status (0 = ok); on failure the message is
 * available from bdc_last_error() (thread-local).  Nothing throws across it.
 *
 * Reference interfaces each entry point replaces (all in /root/reference/pkg):
 *
 *   bdc_session_create   <- batchdc_session.session_open
 *                           (bindings/src/batchdc_session/session.py:92-113)
 *                           with the base PTDF of batchdc.prepare_base_ptdf
 *                           (src/batchdc/factors.py:597-612) uploaded once.
 *   bdc_solve            <- batchdc_session.solve_batch (session.py:116-195)
 *                           and batchdc.solve_batch (src/batchdc/solver.py:970-1003):
 *                           split chain (_apply_splits :363), branch stage
 *                           (_branch_stage :381), injection stage
 *                           (_injection_stage :766), winner report (:652).
 *   bdc_probe_flows      <- batchdc.candidate_case_flows (solver.py:919-958):
 *                           every flow vector of one task, for parity checks.
 *   bdc_draw_tasks       <- batchdc.bench.random_tasks (src/batchdc/bench.py:33-91),
 *                           drawn on the device.
 *   bdc_spd_solve        <- the SPD solve of batchdc.factors.compute_ptdf
 *                           (src/batchdc/factors.py:161-216), on the device (8(f) row 3).
 *   bdc_scan_tasks       <- the rank / outage-cap checks of canonicalize_task and
 *                           _branch_stage (solver.py:148-197, 390-394), vectorised.
 *   bdc_session_destroy  <- (session lifetime end; the reference relies on GC)
 *   bdc_last_error, bdc_version, bdc_device_count -- plumbing.
 *
 * Array layouts (row-major, C order) are the session binding's
 * (session.py:9-19): splits (B,S,E) u8 0/1, disconnections (B,D) i64 with -1
 * for empty slots, injection_sets (B,T,K) u8 0/1.  The Python host layer
 * (paper_2501_17529_b200.session) performs the reference's up-front
 * validation before calling in; bdc_solve re-checks the invariants it relies
 * on and fails with BDC_EINVAL instead of reading out of range.
 */
#ifndef BDC_H_
#define BDC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BDC_OK 0
#define BDC_EINVAL 1   /* bad argument / unsupported size                      */
#define BDC_ECUDA 2    /* CUDA runtime error (no device, OOM, launch failure)   */
#define BDC_ELIMIT 3   /* engine limit exceeded (rank, top-k, elements ...)     */

/* Engine limits (compile-time sizes of on-chip buffers). */
#define BDC_MAX_RANK 32        /* k splits + d disconnections per task          */
#define BDC_MAX_ELEMENTS 32    /* branch elements per substation                */
#define BDC_MAX_MULTI 8        /* branches per multi-branch contingency         */
#define BDC_MAX_TOPK 32        /* topk_per_case and topk_global                 */

/* Per-task status codes written to BdcBatch.status. */
#define BDC_TASK_OK 0
#define BDC_TASK_DEGENERATE_SPLIT 1  /* status_arg = canonical split index     */
#define BDC_TASK_SINGULAR_SPLIT 2    /* status_arg = canonical split index     */
#define BDC_TASK_DISCONNECT_ISLAND 3 /* status_arg = outage index (sequential) or -1 (MODF) */
#define BDC_TASK_ISLAND_ERROR 4      /* islanding_policy = error; see islanded bitmap */
#define BDC_TASK_TOO_MANY_OUTAGES 5  /* batch-level ValidationError on the host */
#define BDC_TASK_DETACHED 6          /* internal consistency failure (never expected) */

typedef struct BdcSession BdcSession;

/* One grid, flattened (see paper_2501_17529_b200/ptdf.py:BaseTables). */
typedef struct {
  int32_t R, C0, M, S, E, K, N1, NM, NMB, NI, NC, NBR;
  int32_t static_col; /* -1 when the base carries no static column */
  const double* P0;          /* (R, C0)   */
  const double* P0T;         /* (C0, R)   */
  const int32_t* row_from;   /* (R)       base endpoint columns */
  const int32_t* row_to;     /* (R)       */
  const int32_t* branch_row; /* (NBR)     row of each branch, -1 if not retained */
  const double* f0;          /* (R)       base N-0 flows, every slot at home */
  const double* p_base;      /* (C0)      */
  const int32_t* mon_row;    /* (M)       */
  const double* rating;      /* (M)       */
  const int32_t* row_mon_pos;/* (R)       */
  const int32_t* sub_col;    /* (S)       */
  const int32_t* sub_count;  /* (S)       */
  const int32_t* sub_elem_row; /* (S, E)  */
  const double* sub_elem_b;  /* (S, E)    */
  const int32_t* slot_sub;   /* (K)       */
  const int32_t* slot_col;   /* (K)       */
  const double* slot_sp;     /* (K)       */
  const int32_t* sc_row;     /* (N1)      */
  const int32_t* sc_order;   /* (N1)      */
  const double* sc_delta;    /* (N1)      */
  const double* sc_dscale;   /* (N1)      max_m |D_base(mon_row[m], c)| / rating[m] */
  const double* D64;         /* (N1, R)   */
  const float* D32;          /* (M, N1)   */
  const int32_t* mc_start;   /* (NM+1)    */
  const int32_t* mc_order;   /* (NM)      */
  const int32_t* mb_row;     /* (NMB)     */
  const double* Dm64;        /* (NMB, R)  */
  const int32_t* ic_slot;    /* (NI)      */
  const int32_t* ic_col;     /* (NI)      */
  const double* ic_sp;       /* (NI)      */
  const int32_t* ic_order;   /* (NI)      */
} BdcGrid;

/* Device-time stages of bdc_solve (BdcBatch.stage_ms). */
#define BDC_STAGES 12
enum {
  BDC_STAGE_H2D = 0,      /* input copies + per-wave resets */
  BDC_STAGE_UPDATE = 1,   /* k_update: split chain, outages, case factors */
  BDC_STAGE_N0 = 2,       /* k_n0: N-0 contraction, screening data */
  BDC_STAGE_OTHER = 3,    /* k_terms + k_other (+ k_oscreen): multi-branch / injection cases */
  BDC_STAGE_SCALE = 4,    /* k_scale_tc: screening scales (tcgen05) */
  BDC_STAGE_TOPK = 5,     /* k_topk */
  BDC_STAGE_TOP = 6,      /* k_top: the TOP tile */
  BDC_STAGE_SCREEN = 7,   /* k_live + k_queue + k_pairs */
  BDC_STAGE_SELECT = 8,   /* k_select */
  BDC_STAGE_REPORT = 9,   /* k_rsel + k_rsweep + k_rmerge */
  BDC_STAGE_D2H = 10,     /* output copies */
  BDC_STAGE_SPARE = 11
};

/* SolveConfig (solver.py:61-91) fields the device needs. */
typedef struct {
  int32_t topk_per_case;
  int32_t topk_global;
  int32_t islanding_policy;    /* 0 penalize, 1 error */
  double islanding_penalty;
  int32_t multi_outage_method; /* 0 modf, 1 sequential */
  int32_t max_simultaneous_outages;
} BdcConfig;

/* One batch.  Input pointers are host memory unless inputs_on_device != 0;
 * output pointers are host memory unless outputs_on_device != 0.  Optional
 * outputs may be NULL. */
typedef struct {
  int64_t B;
  int32_t T, D;
  const uint8_t* splits;     /* (B, S, E)            */
  const int64_t* discos;     /* (B, D)  may be NULL when D == 0 */
  const uint8_t* inj;        /* (B, T, K)            */
  const int32_t* t_count;    /* (B) candidates per task (<= T), or NULL = T */
  int32_t max_rank;          /* max over tasks of (#non-trivial splits + #disconnections),
                                0 = unknown (engine assumes BDC_MAX_RANK) */
  int32_t inputs_on_device;
  int32_t outputs_on_device;
  void* stream;              /* cudaStream_t or NULL (engine-owned stream) */
  /* outputs */
  double* metric;            /* (B) NaN where infeasible            */
  int64_t* best;             /* (B) -1 where infeasible             */
  uint8_t* feasible;         /* (B)                                 */
  int32_t* status;           /* (B) BDC_TASK_*                      */
  int32_t* status_arg;       /* (B)                                 */
  int32_t* n_islanded;       /* (B)                                 */
  uint32_t* islanded_bits;   /* (B, ceil(NC/32)) case-order bitmap, optional */
  int32_t* n0_count;         /* (B)                                 */
  int32_t* n0_pos;           /* (B, topk_global) monitored position */
  double* n0_flow;           /* (B, topk_global)                    */
  double* n0_rel;            /* (B, topk_global)                    */
  int32_t* n1_count;         /* (B)                                 */
  int32_t* n1_case;          /* (B, topk_global) contingency order  */
  int32_t* n1_pos;           /* (B, topk_global)                    */
  double* n1_flow;           /* (B, topk_global)                    */
  double* n1_rel;            /* (B, topk_global)                    */
  float* cand_metric;        /* (B, T) FP32 screening metric per candidate, optional */
  int64_t* loadflows;        /* (1) T*(1+feasible cases) summed over feasible tasks */
  int64_t* bsdf_applications;/* (1) optional */
  int64_t* n1_pairs;         /* (1) optional: (single case, candidate) pairs the N-1
                                kernel evaluated; the rest were skipped by the exact
                                dominance screen (solver.py:798-822) */
  int64_t* report_cases;     /* (1) optional: single cases the FP64 winner report revisited
                                (summed over tasks) */
  int32_t screen;            /* 0 = brute force every pair, 1 = exact dominance screen */
  /* timing (filled by the engine; milliseconds of device time per stage, summed over waves) */
  float stage_ms[BDC_STAGES];  /* see BDC_STAGE_* */
  int32_t waves;
  int32_t kernel_launches;
  int64_t* rescore_stats;    /* (3) optional: [0] candidate classes (bitwise-equal rank
                                coefficients y_t) re-scored in FP64 (the winner's near-tie band,
                                solver.py:804-823), [1] tasks whose FP32 argmin the FP64
                                re-score replaced, [2] tasks with a band of > 1 */
  int64_t* split_shared;     /* (1) optional: split applications copied from another task of
                                the wave with the same split prefix (k_update's prefix memo,
                                tree.py:50-113) instead of computed */
} BdcBatch;

int bdc_device_count(int* count);
const char* bdc_version(void);
const char* bdc_last_error(void);

int bdc_session_create(const BdcGrid* grid, const BdcConfig* config, int device,
                       BdcSession** out);
int bdc_session_destroy(BdcSession* session);

/* Solve one batch (session.py:116-195).  Reentrant: concurrent calls on one
 * session are safe (each call owns its workspace and stream). */
int bdc_solve(BdcSession* session, BdcBatch* batch);

/* Flows of one task for every candidate (candidate_case_flows):
 * n0 (R, T) and n1 (NC, R, T) in contingency order, FP64, NaN rows for
 * islanded cases; case_ok (NC).  Host pointers.  The flows are written when
 * *status is BDC_TASK_OK or BDC_TASK_ISLAND_ERROR (then case_ok names the
 * islanded cases); other statuses leave them untouched. */
int bdc_probe_flows(BdcSession* session, const uint8_t* splits, const int64_t* discos,
                    int32_t D, const uint8_t* inj, int32_t T, double* n0, double* n1,
                    uint8_t* case_ok, int32_t* status, int32_t* status_arg);

/* Host-side scan of a batch's task arrays (no device work): the largest
 * rank k+d, disconnection count d and number of moved injection slots over
 * the tasks -- the quantities the engine limits and the workspace stride
 * depend on (replaces the per-task rank counting of canonicalize_task,
 * solver.py:148-197).  splits (B,S,E) u8, discos (B,D) i64 or NULL. */
int bdc_scan_tasks(BdcSession* session, const uint8_t* splits, const int64_t* discos,
                   int64_t B, int32_t D, int32_t* max_rank, int32_t* max_disc,
                   int32_t* max_active_slots);

/* Device-side random tasks (batchdc.bench.random_tasks, bench.py:33-91): the
 * reference's distribution drawn on the GPU into the session array layout.
 * All array pointers are DEVICE pointers: splits (B,S,E) u8, discos (B,D) i64
 * (NULL when D = 0), inj (B,T,K) u8 (NULL: topology only).  attempt (B) i32
 * (NULL = 0) is each task's draw number and redraw (B) u8 (NULL = every task)
 * selects the tasks whose topology is (re)drawn -- the caller's acceptance loop
 * redraws the tasks the engine reports as degenerate/singular/islanding
 * (bench.py:96-110).  Counter-based (Philox4x32-10): deterministic per seed.
 * Runs on `stream` (NULL: the default stream); no synchronisation. */
int bdc_draw_tasks(BdcSession* session, uint64_t seed, int64_t B, int32_t T, int32_t E, int32_t D,
                   int32_t n_splits, int32_t n_disconnections, const int32_t* attempt,
                   const uint8_t* redraw, uint8_t* splits, int64_t* discos, uint8_t* inj,
                   void* stream);

/* Dense SPD solve on the device (the base-PTDF setup, compute_ptdf factors.py:161-216,
 * i.e. scipy.linalg.solve(L, A^T, assume_a="pos") = LAPACK potrf + potrs): A (n x n,
 * row-major, lower triangle read, overwritten by its Cholesky factor) and B (n x m,
 * overwritten by A^-1 B) are DEVICE pointers; *info (device int) is set to 0 or to the
 * first non-positive pivot's column + 1 (the caller reads it after synchronising).
 * Runs on `stream` (NULL: the default stream). */
int bdc_spd_solve(int device, double* A, int32_t n, double* B, int32_t m, int32_t* info, void* stream);

/* Set the wave size cap (tasks per device wave); 0 = automatic. */
int bdc_session_set_wave(BdcSession* session, int64_t max_tasks_per_wave);

#ifdef __cplusplus
}
#endif
#endif /* BDC_H_ */
