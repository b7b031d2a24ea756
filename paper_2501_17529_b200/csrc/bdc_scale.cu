// bdc_scale.cu -- the screening scales of the single-branch N-1 stage on the tcgen05
// tensor cores.
//
// For every task, single case c and screening row block b (bdc_device.cuh) the
// dominance screen needs an upper bound of
//     max_{r in b} |L'(r,c)|,   L'(r,c) = L(r,c) / rating_r = (D'(r,c) + sum_j B'(r,j) W(c,j)) / den_c
// with D' = D_base / rating (a session table, case-major) and B' = B'' / rating (dead
// rows zeroed, written per task by k_n0).  The rank-r product sum_j B'(r,j) W(c,j) is a
// (cases x K) . (K x rows) GEMM per task, K = rank padded to 8: it runs as
// tcgen05.mma.kind::tf32 (M = 128 cases, N = 64 rows, K = 8 per instruction) into a
// TMEM accumulator, and the epilogue reads it back with tcgen05.ld (thread = case,
// columns = rows), adds D' from shared memory and folds max |.| per case and row block
// with FMNMX3 -- the reduction over rows never leaves the thread.
//
// Rigour: operands are rounded to TF32 (cvt.rna, relative error <= 2^-11 each), so the
// product terms carry <= 2^-10 relative error, accumulated and added in FP32.  The bound
//     |L~ - L| <= 2^-9 sum_j |W_cj| max_r |B'(r,j)| + (rt + 8) 2^-23 (max_r |D'(r,c)| + sum_j ...)
// is added before scaling by 1/|den_c| (the FP32 CUDA-core version needed only the
// second term).  The own row contributes 1/rating (L' = -1/rating there), dead rows
// nothing; both are masked out of the accumulated maxima.
//
// CTA = 128 cases x TB tasks (the D' tile staged once per row chunk serves all TB
// tasks); one elected thread issues the MMAs and commits them to an mbarrier.
#include "bdc_device.cuh"

#include <cstdlib>

#include <cuda.h>

#include <algorithm>

namespace bdc {

namespace {

constexpr int SM_CASES = 128;  // UMMA M
constexpr int SM_ROWS = 64;    // UMMA N: monitored rows per chunk
constexpr int DT_BYTES = SM_CASES * 32 * 4;  // one TMA tile of D': 128 cases x 32 rows FP32

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// K-major, no-swizzle canonical layout: 8-row x 16-byte core matrices; the two 16-byte
// K halves of a row group at +128 B (LBO), consecutive row groups at +256 B (SBO).
__device__ __forceinline__ int core_off(int row, int k) {  // byte offset of element (row, k), k < 8
  return (row >> 3) * 256 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint32_t a = smem_u32(p);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;  // leading byte offset (K direction)
  d |= (uint64_t)((256 >> 4) & 0x3FFF) << 32;  // stride byte offset (M/N direction)
  d |= (uint64_t)1 << 46;                      // descriptor version (sm_100)
  return d;                                    // base offset 0, SWIZZLE_NONE
}
// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = SM_ROWS
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(SM_ROWS >> 3) << 17) |
                            ((uint32_t)(SM_CASES >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, bool acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc ? 1 : 0));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace

// TB tasks per CTA, KB = K blocks of 8 rank terms (rank stride rs <= 8 KB).  256 threads:
// warp w reads TMEM lanes 32 (w % 4) .. +31 (the CTA's cases), warpgroup w / 4 takes one
// 32-row half of every 64-row chunk.  The D' tile and the B operands of chunk ch + 1 are
// in flight (cp.async, double buffer) while chunk ch is multiplied and reduced.
template <int TB, int KB>
__global__ void __launch_bounds__(2 * SM_CASES, 1) k_scale_tc(DevGrid g, Work w,
                                                               const __grid_constant__ CUtensorMap tmD) {
  constexpr int NT = 2 * SM_CASES;
  constexpr int TCOLS = TB * SM_ROWS;  // TMEM columns: one accumulator per task
  constexpr int NCOLS = TCOLS <= 32 ? 32 : (TCOLS <= 64 ? 64 : (TCOLS <= 128 ? 128 : (TCOLS <= 256 ? 256 : 512)));
  constexpr int ABYTES = SM_CASES * 32, BBYTES = SM_ROWS * 32;  // one K block of A / B
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, wg = wid >> 2;
  const int ci = (wid & 3) * 32 + lane;  // this thread's case within the tile (= TMEM lane)
  // raster: case tile fastest (a task group's B operands stay in L2 across its case tiles)
  // or, when the D' table outgrows L2, task group fastest (each D' slab is read from HBM
  // once and shared in L2 by every task group)
  const bool tgf = w.scale_tgfast != 0;
  const int c0 = (tgf ? blockIdx.y : blockIdx.x) * SM_CASES, c = c0 + ci;
  const int tb0 = (tgf ? blockIdx.x : blockIdx.y) * TB;
  const int rs = w.rs, M = g.M, N1 = g.N1, T = w.T;
  const int MB = screen_block_rows(M);
  extern __shared__ __align__(1024) unsigned char ssm_raw[];
  // the 128-byte swizzle repeats every 1024 bytes: the tiles start on a 1024-byte boundary
  unsigned char* ssm = ssm_raw + ((1024u - (smem_u32(ssm_raw) & 1023u)) & 1023u);
  // [2 buffers][2 row halves] TMA tiles of D' (128 cases x 32 rows, 128-byte swizzle)
  float* sD = reinterpret_cast<float*>(ssm);
  unsigned char* sA = ssm + 4 * DT_BYTES;             // [TB][KB] A tiles
  unsigned char* sBt = sA + TB * KB * ABYTES;         // [2][TB][KB] B tiles
  __shared__ __align__(8) uint64_t mbar;              // MMA completion
  __shared__ __align__(8) uint64_t full[2];           // TMA completion per buffer
  __shared__ uint32_t tmem_base;
  __shared__ int sdead[TB][RMAX];
  __shared__ int snd[TB], srt[TB];
  __shared__ float sm0[TB][SB];

  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "n"(NCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  if (tid < TB) {
    const int b = tb0 + tid;
    const bool on = b < w.Wb && w.status[b] == 0;
    snd[tid] = on ? w.ndead[b] : 0;
    srt[tid] = on ? w.rank[b] : -1;  // -1: slot idle
  }
  __syncthreads();
  // stage chunk ch into buffer bf (thread 0): two TMA tensor tiles of D' (rows x cases,
  // zero-filled out of bounds) and the tasks' B operand blocks as bulk copies (already in
  // the core-matrix layout, b32_off), all completing on full[bf]
  const size_t tf = b32_task_floats(rs, M);
  int nvalid = 0;
  for (int k = 0; k < TB; ++k) nvalid += srt[k] >= 0;
  auto issue = [&](int ch, int bf) {
    const int m0 = ch * SM_ROWS;
    const uint32_t bar = smem_u32(&full[bf]);
    const uint32_t bytes = 2u * DT_BYTES + (uint32_t)(nvalid * KB * BBYTES);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
    for (int h = 0; h < 2; ++h)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
              smem_u32(sD + (bf * 2 + h) * (DT_BYTES / 4))),
          "l"(&tmD), "r"(m0 + 32 * h), "r"(c0), "r"(bar)
          : "memory");
    unsigned char* Bt = sBt + bf * TB * KB * BBYTES;
    for (int k = 0; k < TB; ++k) {
      if (srt[k] < 0) continue;
      for (int kb = 0; kb < KB; ++kb) {
        const float* src = w.B32 + (size_t)(tb0 + k) * tf + ((size_t)ch * KB + kb) * 512;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                smem_u32(Bt + (k * KB + kb) * BBYTES)),
            "l"(src), "r"(BBYTES), "r"(bar)
            : "memory");
      }
    }
  };

  // chunk 0 is in flight while the tile's operands and bounds are prepared
  if (tid == 0) issue(0, 0);
  for (int i = tid; i < TB * RMAX; i += NT) {
    const int k = i / RMAX, d = i % RMAX;
    if (d < snd[k]) sdead[k][d] = g.row_mon_pos[w.dead[(size_t)(tb0 + k) * RMAX + d]];  // -1: unmonitored
  }
  // max_t m0_b(t) of each task and block (ranking key; folded by k_n0)
  if (tid < TB * SB) {
    const int k = tid / SB, blk = tid % SB;
    sm0[k][blk] = srt[k] >= 0 ? w.m0bx[(size_t)(tb0 + k) * SB + blk] : 0.f;
  }
  // A operands (warpgroup 0): W(c, j) of every task, TF32 (cvt.rna), zero past the rank
  if (wg == 0) {
#pragma unroll
    for (int k = 0; k < TB; ++k) {
      const int b = tb0 + k, rt = srt[k];
      const bool ok = c < N1 && rt >= 0 && w.sc_ok[(size_t)b * N1 + c];
#pragma unroll
      for (int kb = 0; kb < KB; ++kb)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = kb * 8 + jj;
          const float wv = (ok && j < rt) ? (float)w.Wsc[((size_t)b * N1 + c) * rs + j] : 0.f;
          *reinterpret_cast<uint32_t*>(sA + (k * KB + kb) * ABYTES + core_off(ci, jj)) = to_tf32(wv);
        }
    }
  }
  // own rows: the computed own-row value is |1 - den_c| / rating (D''(r_c, c) = 1 - den_c);
  // its true |L'| = 1/rating enters the bound at the end.  Scaled by 1/|den_c| the computed
  // value only loosens the bound when |1 - den_c| > |den_c|: masked out in that case only.
  const int ownp = c < N1 ? g.row_mon_pos[g.sc_row[c]] : -1;
  bool ownloose = false;
#pragma unroll
  for (int k = 0; k < TB; ++k)
    if (c < N1 && srt[k] >= 0 && w.sc_ok[(size_t)(tb0 + k) * N1 + c]) {
      const double den = w.den[(size_t)(tb0 + k) * N1 + c];
      ownloose |= fabs(1.0 - den) > 0.999 * fabs(den);
    }

  const int nchunks = (M + SM_ROWS - 1) / SM_ROWS;
  float mx[TB], mxb[TB][SB];  // running max of the current block; finished blocks
#pragma unroll
  for (int k = 0; k < TB; ++k) {
    mx[k] = 0.f;
#pragma unroll
    for (int bb = 0; bb < SB; ++bb) mxb[k][bb] = 0.f;
  }
  int curblk = -1;
  auto flush = [&]() {
#pragma unroll
    for (int k = 0; k < TB; ++k) {
#pragma unroll
      for (int bb = 0; bb < SB; ++bb)
        if (bb == curblk) mxb[k][bb] = fmaxf(mxb[k][bb], mx[k]);
      mx[k] = 0.f;
    }
  };
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = tmem_base;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int bf = ch & 1;
    // the other buffer was released at the end of the previous chunk
    if (tid == 0 && ch + 1 < nchunks) issue(ch + 1, bf ^ 1);
    mbar_wait(&full[bf], (ch >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (tid == 0) {
      const unsigned char* Bt = sBt + bf * TB * KB * BBYTES;
#pragma unroll
      for (int k = 0; k < TB; ++k)
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
          mma_tf32(tbase + k * SM_ROWS, smem_desc(sA + (k * KB + kb) * ABYTES),
                   smem_desc(Bt + (k * KB + kb) * BBYTES), kb > 0);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&mbar))
                   : "memory");
    }
    mbar_wait(&mbar, ch & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // epilogue: this warpgroup's 32-row half (a screening block holds whole halves)
    const int r0 = ch * SM_ROWS + wg * 32;
    // warps whose 32 cases all lie past N1 (the last case tile of G118: 24 of 128) skip
    // the epilogue: their accumulators are never read
    if (r0 < M && c0 + (wid & 3) * 32 < N1) {
      const int blk = r0 / MB;
      if (blk != curblk) {
        flush();
        curblk = blk;
      }
      // this thread's 32 rows of its case: one 128-byte row of the swizzled TMA tile
      // (16-byte chunk q lives at chunk q ^ (case & 7))
      const float* D = sD + (bf * 2 + wg) * (DT_BYTES / 4) + ci * 32;
      float dv[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 v4 = *reinterpret_cast<const float4*>(&D[4 * (q ^ (ci & 7))]);
        dv[4 * q] = v4.x; dv[4 * q + 1] = v4.y; dv[4 * q + 2] = v4.z; dv[4 * q + 3] = v4.w;
      }
      const int ownq = ownp - r0;
      const bool ownin = ownloose && ownq >= 0 && ownq < 32;
      const bool anyown = __any_sync(0xffffffffu, ownin);
#pragma unroll
      for (int k = 0; k < TB; ++k) {
        float acc[32];
        tmem_ld32(tbase + ((uint32_t)((wid & 3) * 32) << 16) + k * SM_ROWS + wg * 32, acc);
        if (srt[k] < 0) continue;
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          const float2 a2 = __fadd2_rn(make_float2(acc[q], acc[q + 1]), make_float2(dv[q], dv[q + 1]));
          acc[q] = a2.x; acc[q + 1] = a2.y;
        }
        // dead rows of the task -> excluded (their flow is exactly 0)
        for (int d = 0; d < snd[k]; ++d) {
          const int dq = sdead[k][d] - r0;
          if (dq >= 0 && dq < 32) {
#pragma unroll
            for (int q = 0; q < 32; ++q) acc[q] = (q == dq) ? 0.f : acc[q];
          }
        }
        if (anyown) {
#pragma unroll
          for (int q = 0; q < 32; ++q) acc[q] = (ownin && q == ownq) ? 0.f : acc[q];
        }
        float m = mx[k];
#pragma unroll
        for (int q = 0; q < 32; q += 2) m = max3abs(m, acc[q], acc[q + 1]);
        mx[k] = m;
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();  // TMEM and this chunk's buffers are free again
  }
  flush();
  __syncthreads();
  if (wid == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(NCOLS));
  // warpgroup 1 hands its block maxima over through the (now free) D' buffer
  float* sMx = sD;  // [SB][TB][128]
  if (wg == 1)
#pragma unroll
    for (int k = 0; k < TB; ++k)
#pragma unroll
      for (int bb = 0; bb < SB; ++bb) sMx[(bb * TB + k) * SM_CASES + ci] = mxb[k][bb];
  __syncthreads();
  if (wg != 0 || c >= N1) return;
  // warpgroup 0: combine the two halves' block maxima, scale, bound, ranking key
#pragma unroll
  for (int k = 0; k < TB; ++k) {
    const int b = tb0 + k, rt = srt[k];
    if (rt < 0) continue;
    const bool ok = w.sc_ok[(size_t)b * N1 + c] != 0;
    float aid = 0.f, rnd = 0.f;
    if (ok) {
      float wsum = 0.f;
      for (int j = 0; j < rt; ++j)
        wsum += (float)fabs(w.Wsc[((size_t)b * N1 + c) * rs + j]) * w.bmax[(size_t)b * rs + j];
      aid = (float)fabs(1.0 / w.den[(size_t)b * N1 + c]);
      const float gam = (float)(rt + 8) * 1.1920929e-7f;
      rnd = 0.001953125f * wsum + gam * ((float)g.sc_dscale[c] + wsum);  // 2^-9: tf32 products
    }
    bool owndead = false;
    for (int d = 0; d < snd[k]; ++d) owndead |= sdead[k][d] == ownp;
    float keyv = 0.f;
    const float smx = smax_at(g, w, b, c);
    for (int blk = 0; blk < SB; ++blk) {
      float U = 0.f;
      if (ok) {
        float mb = 0.f;
#pragma unroll
        for (int bb = 0; bb < SB; ++bb)
          if (bb == blk) mb = mxb[k][bb];
        mb = fmaxf(mb, sMx[(blk * TB + k) * SM_CASES + ci]);
        U = aid * (mb + rnd);
        if (ownp >= 0 && ownp / MB == blk && !owndead) U = fmaxf(U, (float)g.inv_rating[ownp]);
        U *= 1.f + 4e-6f;
      }
      w.scale[((size_t)b * SB + blk) * N1 + c] = U;
      keyv = fmaxf(keyv, sm0[k][blk] + U * smx);
    }
    w.bkey[(size_t)b * N1 + c] = ok ? __float_as_uint(keyv) : 0u;
  }
}

namespace {
template <int TB, int KB>
void launch_scale_tc_t(const DevGrid& g, const Work& w, cudaStream_t s) {
  size_t dyn = 1024 + 4 * (size_t)DT_BYTES + (size_t)TB * KB * (SM_CASES + 2 * SM_ROWS) * 32;
  static_assert(SB * TB * SM_CASES * 4 <= 4 * DT_BYTES, "block maxima fit the D' buffers");
  // at most 512 / NCOLS CTAs per SM fit their TMEM columns: size the shared memory so
  // that no more are resident (a CTA spinning in tcgen05.alloc would hold an SM slot)
  const int ncols = TB * SM_ROWS <= 64 ? 64 : (TB * SM_ROWS <= 128 ? 128 : (TB * SM_ROWS <= 256 ? 256 : 512));
  dyn = std::max(dyn, (size_t)(220 * 1024) / (size_t)(512 / ncols));
  smem_opt_in((const void*)k_scale_tc<TB, KB>, (int)dyn);
  const int nct = (g.N1 + SM_CASES - 1) / SM_CASES, ntg = (w.Wb + TB - 1) / TB;
  // D' = N1 x Mp FP32: beyond ~96 MB (G10k: 676 MB) it no longer stays in the 126 MB L2
  // while every task group streams it, so the task groups go fastest
  Work wr = w;
  const char* env = getenv("BDC_SCALE_RASTER");  // tests: 0 case tile / 1 task group fastest
  wr.scale_tgfast = env ? (env[0] == '1') : ((size_t)g.N1 * g.Mp * 4 > ((size_t)96 << 20));
  const dim3 grid(wr.scale_tgfast ? ntg : nct, wr.scale_tgfast ? nct : ntg);
  k_scale_tc<TB, KB><<<grid, 2 * SM_CASES, dyn, s>>>(g, wr, *g.tm_ds);
}
}  // namespace

void launch_scale(const DevGrid& g, const Work& w, cudaStream_t s) {
  // four tasks per CTA, two CTAs per SM.  Measured and not kept: eight tasks per CTA (one
  // CTA per SM for its 512 TMEM columns; G118 2.44 -> 4.22 ms) and two (four CTAs per SM,
  // each D' tile shared by half as many tasks; G118 2.64, G1k 3.69 -> 4.63, G3k 3.37 -> 4.31 ms)
  if (w.rs <= 8) launch_scale_tc_t<4, 1>(g, w, s);
  else if (w.rs <= 16) launch_scale_tc_t<2, 2>(g, w, s);
  else launch_scale_tc_t<1, 4>(g, w, s);
}

}  // namespace bdc
