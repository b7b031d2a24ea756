// bdc_capi.cu -- the C ABI (include/bdc.h): session lifetime, wave scheduling,
// host<->device staging.  No exceptions cross the boundary; every entry point
// returns a status and leaves a thread-local message for bdc_last_error().
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <cstdlib>
#include <cudaTypedefs.h>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "bdc_device.cuh"

using namespace bdc;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(BDC_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

template <class T>
cudaError_t upload(const T* src, size_t n, const T** dst, std::vector<void*>& owned) {
  *dst = nullptr;
  if (n == 0) return cudaSuccess;
  T* p = nullptr;
  cudaError_t e = cudaMalloc((void**)&p, n * sizeof(T));
  if (e != cudaSuccess) return e;
  owned.push_back(p);
  *dst = p;
  if (src) return cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice);
  return cudaMemset(p, 0, n * sizeof(T));
}

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

struct BdcSession {
  alignas(64) CUtensorMap tm_ds{};  // TMA descriptor of the screening table DsT
  int device = 0;
  DevGrid g{};
  DevCfg cfg{};
  std::vector<void*> owned;
  int64_t wave_cap = 0;
  size_t total_mem = 0;
  std::vector<int32_t> sub_count, slots_per_sub;  // host copies for bdc_scan_tasks
  std::vector<double> rating;                     // host copy: report loadings = |flow| / rating
  // pinned host staging for outputs bound for pageable host memory, reused across calls
  std::vector<std::pair<char*, size_t>> pin_free;
  // cached wave workspaces (one per concurrent call), reused across calls
  std::mutex ws_mu;
  std::vector<std::pair<char*, size_t>> ws_free;
};

namespace {
// Borrow a workspace of at least `bytes` from the session cache (or allocate one);
// returned to the cache when the call ends (the call synchronises its stream first).
struct WsLease {
  BdcSession* s;
  char* p = nullptr;
  size_t bytes = 0;
  WsLease(BdcSession* s_, size_t need) : s(s_) {
    {
      std::lock_guard<std::mutex> lk(s->ws_mu);
      for (size_t i = 0; i < s->ws_free.size(); ++i)
        if (s->ws_free[i].second >= need) {
          p = s->ws_free[i].first;
          bytes = s->ws_free[i].second;
          s->ws_free.erase(s->ws_free.begin() + i);
          return;
        }
    }
    if (cudaMalloc((void**)&p, need) != cudaSuccess) {
      cudaGetLastError();
      std::lock_guard<std::mutex> lk(s->ws_mu);  // drop smaller cached buffers and retry
      for (auto& f : s->ws_free) cudaFree(f.first);
      s->ws_free.clear();
      p = nullptr;
      if (cudaMalloc((void**)&p, need) != cudaSuccess) { cudaGetLastError(); p = nullptr; return; }
    }
    bytes = need;
  }
  ~WsLease() {
    if (!p) return;
    std::lock_guard<std::mutex> lk(s->ws_mu);
    s->ws_free.emplace_back(p, bytes);
  }
};
// Borrow pinned host memory of at least `need` bytes from the session cache.
struct PinLease {
  BdcSession* s;
  char* p = nullptr;
  size_t bytes = 0;
  PinLease(BdcSession* s_, size_t need) : s(s_) {
    {
      std::lock_guard<std::mutex> lk(s->ws_mu);
      for (size_t i = 0; i < s->pin_free.size(); ++i)
        if (s->pin_free[i].second >= need) {
          p = s->pin_free[i].first;
          bytes = s->pin_free[i].second;
          s->pin_free.erase(s->pin_free.begin() + i);
          return;
        }
    }
    if (cudaMallocHost((void**)&p, need) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return;
    }
    bytes = need;
  }
  ~PinLease() {
    if (!p) return;
    std::lock_guard<std::mutex> lk(s->ws_mu);
    s->pin_free.emplace_back(p, bytes);
  }
};
}  // namespace

namespace bdc {
namespace {
std::mutex g_optin_mu;
std::map<std::pair<int, const void*>, int> g_optin;  // (device, kernel) -> opted-in bytes
}  // namespace

cudaError_t smem_opt_in(const void* fn, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_optin_mu);
  int& have = g_optin[{dev, fn}];
  if (bytes <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

int smem_opt_in_max(const void* fn) {
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, fn);
  const int mx = optin - (int)fa.sharedSizeBytes;
  smem_opt_in(fn, mx);
  return mx;
}
}  // namespace bdc

extern "C" {

const char* bdc_version(void) { return "bdc-b200 0.1.0 (sm_100a)"; }

const char* bdc_last_error(void) { return g_err.c_str(); }

int bdc_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(BDC_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  *count = n;
  return BDC_OK;
}

int bdc_session_create(const BdcGrid* G, const BdcConfig* C, int device, BdcSession** out) {
  if (!G || !C || !out) return fail(BDC_EINVAL, "null argument");
  *out = nullptr;
  if (G->E > EMAX) return fail(BDC_ELIMIT, "substation has more than 32 branch elements");
  if (C->topk_per_case < 1 || C->topk_global < 1)
    return fail(BDC_EINVAL, "top-k limits must be >= 1");
  if (C->topk_per_case > KMAX || C->topk_global > KMAX)
    return fail(BDC_ELIMIT, "top-k limits above 32 are not supported by the engine");
  for (int q = 0; q < G->NM; ++q)
    if (G->mc_start[q + 1] - G->mc_start[q] > MMAX)
      return fail(BDC_ELIMIT, "multi-branch contingency with more than 8 branches");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(BDC_EINVAL, "device index out of range");
  CK(cudaSetDevice(device));
  auto* s = new BdcSession();
  s->device = device;
  DevGrid& g = s->g;
  g.R = G->R; g.C0 = G->C0; g.M = G->M; g.S = G->S; g.E = G->E; g.K = G->K;
  g.N1 = G->N1; g.NM = G->NM; g.NMB = G->NMB; g.NI = G->NI; g.NC = G->NC; g.NBR = G->NBR;
  g.static_col = G->static_col;
  g.MT = 2;
  for (int q = 0; q < G->NM; ++q)
    while (g.MT < G->mc_start[q + 1] - G->mc_start[q]) g.MT *= 2;
  std::vector<double> inv(G->M);
  for (int i = 0; i < G->M; ++i) inv[i] = 1.0 / G->rating[i];
  cudaError_t e = cudaSuccess;
  auto& o = s->owned;
#define UP(field, n) if (e == cudaSuccess) e = upload(G->field, (size_t)(n), &g.field, o)
  UP(P0, (size_t)G->R * G->C0);
  UP(P0T, (size_t)G->R * G->C0);
  UP(row_from, G->R);
  UP(row_to, G->R);
  UP(branch_row, G->NBR);
  UP(f0, G->R);
  UP(p_base, G->C0);
  UP(mon_row, G->M);
  UP(rating, G->M);
  UP(row_mon_pos, G->R);
  UP(sub_col, G->S);
  UP(sub_count, G->S);
  UP(sub_elem_row, (size_t)G->S * G->E);
  UP(sub_elem_b, (size_t)G->S * G->E);
  UP(slot_sub, G->K);
  UP(slot_col, G->K);
  UP(slot_sp, G->K);
  UP(sc_row, G->N1);
  UP(sc_order, G->N1);
  UP(sc_delta, G->N1);
  UP(sc_dscale, G->N1);
  UP(D64, (size_t)G->N1 * G->R);
  // D_base on monitored rows, rows padded to a multiple of 4 cases so every
  // chunk copy of the N-1 kernels is a 16-byte cp.async
  g.N1p = (G->N1 + 3) & ~3;
  if (e == cudaSuccess && (size_t)G->N1 * G->M > 0) {
    float* d = nullptr;
    e = cudaMalloc((void**)&d, (size_t)g.N1p * G->M * sizeof(float));
    if (e == cudaSuccess) {
      o.push_back(d);
      g.D32 = d;
      e = cudaMemset(d, 0, (size_t)g.N1p * G->M * sizeof(float));
      if (e == cudaSuccess)
        e = cudaMemcpy2D(d, (size_t)g.N1p * sizeof(float), G->D32, (size_t)G->N1 * sizeof(float),
                         (size_t)G->N1 * sizeof(float), G->M, cudaMemcpyHostToDevice);
    }
  }
  UP(mc_start, G->NM + 1);
  UP(mc_order, G->NM);
  UP(mb_row, G->NMB);
  UP(Dm64, (size_t)G->NMB * G->R);
  // D_base / rating on monitored rows, case-major, FP32, rows padded to a multiple of 4
  // (16-byte cp.async of the tensor-core screening kernel)
  g.Mp = (G->M + 3) & ~3;
  if (e == cudaSuccess && (size_t)G->N1 * G->M > 0) {
    std::vector<float> ds((size_t)G->N1 * g.Mp, 0.f);
    for (int c = 0; c < G->N1; ++c)
      for (int p = 0; p < G->M; ++p)
        ds[(size_t)c * g.Mp + p] = (float)(G->D64[(size_t)c * G->R + G->mon_row[p]] * (1.0 / G->rating[p]));
    e = upload(ds.data(), ds.size(), &g.DsT, o);
    if (e == cudaSuccess) {
      // TMA descriptor: dim 0 = monitored rows (contiguous), dim 1 = cases; boxes of
      // 32 rows x 128 cases with the 128-byte swizzle; out-of-range elements read as 0
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q{};
      e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
      if (e == cudaSuccess && (fn == nullptr || q != cudaDriverEntryPointSuccess)) e = cudaErrorNotSupported;
      if (e == cudaSuccess) {
        const cuuint64_t dims[2] = {(cuuint64_t)g.Mp, (cuuint64_t)G->N1};
        const cuuint64_t strides[1] = {(cuuint64_t)g.Mp * sizeof(float)};
        const cuuint32_t box[2] = {32, 128}, estr[2] = {1, 1};
        const CUresult r = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(
            &s->tm_ds, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)g.DsT, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) e = cudaErrorInvalidValue;
      }
    }
  }
  g.tm_ds = &s->tm_ds;
  {
    std::vector<int32_t> pos(G->N1 > 0 ? G->N1 : 1, -1);
    std::vector<float> rat(G->N1 > 0 ? G->N1 : 1, 0.f);
    int all = 1;
    for (int c = 0; c < G->N1; ++c) {
      const int p = G->row_mon_pos[G->sc_row[c]];
      pos[c] = p;
      rat[c] = p >= 0 ? (float)G->rating[p] : 0.f;
      all &= p >= 0;
    }
    g.s_mon = all;
    if (e == cudaSuccess) e = upload((const int32_t*)pos.data(), pos.size(), &g.sc_pos, o);
    if (e == cudaSuccess) e = upload((const float*)rat.data(), rat.size(), &g.sc_rat, o);
  }
  // D_base on monitored rows, case-major, for the winner report's coalesced sweeps
  if (e == cudaSuccess && (size_t)G->N1 * G->M > 0) {
    std::vector<double> dm((size_t)G->N1 * G->M);
    for (int c = 0; c < G->N1; ++c)
      for (int p = 0; p < G->M; ++p) dm[(size_t)c * G->M + p] = G->D64[(size_t)c * G->R + G->mon_row[p]];
    e = upload(dm.data(), dm.size(), &g.DM64, o);
  }
  UP(ic_slot, G->NI);
  UP(ic_col, G->NI);
  UP(ic_sp, G->NI);
  UP(ic_order, G->NI);
#undef UP
  if (e == cudaSuccess) e = upload((const double*)inv.data(), inv.size(), &g.inv_rating, o);
  s->rating.assign(G->rating, G->rating + G->M);
  if (e != cudaSuccess) {
    for (void* p : o) cudaFree(p);
    delete s;
    return fail(BDC_ECUDA, std::string("session upload: ") + cudaGetErrorString(e));
  }
  s->sub_count.assign(G->sub_count, G->sub_count + G->S);
  s->slots_per_sub.assign(G->S, 0);
  for (int k = 0; k < G->K; ++k)
    if (G->slot_sp[k] != 0.0 && G->slot_sub[k] >= 0 && G->slot_sub[k] < G->S) ++s->slots_per_sub[G->slot_sub[k]];
  s->cfg.kc = C->topk_per_case;
  s->cfg.kg = C->topk_global;
  s->cfg.policy = C->islanding_policy;
  s->cfg.method = C->multi_outage_method;
  s->cfg.maxout = C->max_simultaneous_outages;
  s->cfg.penalty = C->islanding_penalty;
  size_t fb = 0, tb = 0;
  cudaMemGetInfo(&fb, &tb);
  s->total_mem = tb;
  // keep freed workspace in the stream-ordered pool between calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = s;
  return BDC_OK;
}

int bdc_session_destroy(BdcSession* s) {
  if (!s) return BDC_OK;
  cudaSetDevice(s->device);
  for (void* p : s->owned) cudaFree(p);
  for (auto& f : s->ws_free) cudaFree(f.first);
  for (auto& f : s->pin_free) cudaFreeHost(f.first);
  delete s;
  return BDC_OK;
}

int bdc_scan_tasks(BdcSession* s, const uint8_t* splits, const int64_t* discos, int64_t B, int32_t D,
                   int32_t* max_rank, int32_t* max_disc, int32_t* max_active) {
  if (!s || (B > 0 && !splits && s->g.S > 0) || (D > 0 && B > 0 && !discos))
    return fail(BDC_EINVAL, "null argument");
  const int S = s->g.S, E = s->g.E > 0 ? s->g.E : 1;
  // chunks of tasks on host threads (a few ms per 10^5 tasks on one core)
  auto scan = [&](int64_t b0, int64_t b1, int32_t* out) {
    int32_t mr = 0, md = 0, ma = 0;
    for (int64_t b = b0; b < b1; ++b) {
      int k = 0, act = 0, d = 0;
      const uint8_t* sp = splits + (size_t)b * S * E;
      for (int si = 0; si < S; ++si) {
        const uint8_t* e = sp + (size_t)si * E;
        unsigned acc = 0;
        for (int j = 0; j < E; ++j) acc |= e[j];
        if (acc) { ++k; act += s->slots_per_sub[si]; }
      }
      for (int i = 0; i < D; ++i) d += discos[(size_t)b * D + i] >= 0;
      mr = std::max(mr, k + d);
      md = std::max(md, d);
      ma = std::max(ma, act);
    }
    out[0] = mr; out[1] = md; out[2] = ma;
  };
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(hw, B / 2048));
  std::vector<int32_t> res((size_t)nt * 3, 0);
  std::vector<std::thread> th;
  const int64_t per = (B + nt - 1) / nt;
  for (int i = 1; i < nt; ++i)
    th.emplace_back(scan, i * per, std::min<int64_t>(B, (i + 1) * per), &res[(size_t)i * 3]);
  scan(0, std::min<int64_t>(B, per), &res[0]);
  for (auto& t : th) t.join();
  int32_t mr = 0, md = 0, ma = 0;
  for (int i = 0; i < nt; ++i) {
    mr = std::max(mr, res[(size_t)i * 3]);
    md = std::max(md, res[(size_t)i * 3 + 1]);
    ma = std::max(ma, res[(size_t)i * 3 + 2]);
  }
  if (max_rank) *max_rank = mr;
  if (max_disc) *max_disc = md;
  if (max_active) *max_active = ma;
  return BDC_OK;
}

int bdc_draw_tasks(BdcSession* s, uint64_t seed, int64_t B, int32_t T, int32_t E, int32_t D, int32_t n_splits,
                   int32_t n_disc, const int32_t* attempt, const uint8_t* redraw, uint8_t* splits,
                   int64_t* discos, uint8_t* inj, void* stream) {
  if (!s) return fail(BDC_EINVAL, "null session");
  if (B < 0 || T < 0 || D < 0 || n_splits < 0 || n_disc < 0) return fail(BDC_EINVAL, "negative size");
  if (B == 0) return BDC_OK;
  if (!splits || (D > 0 && !discos))
    return fail(BDC_EINVAL, "missing output pointer");
  if (E < s->g.E) return fail(BDC_EINVAL, "split width E is smaller than the widest substation");
  if (n_splits > RMAX || n_disc > MMAX || n_disc > D) return fail(BDC_ELIMIT, "too many splits or disconnections");
  cudaError_t e = cudaSetDevice(s->device);
  if (e != cudaSuccess) return fail(BDC_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  GenArgs a{};
  a.B = B; a.T = T; a.E = E; a.D = D; a.n_splits = n_splits; a.n_disc = n_disc;
  a.k0 = (uint32_t)seed; a.k1 = (uint32_t)(seed >> 32);
  a.attempt = attempt; a.redraw = redraw; a.splits = splits; a.discos = discos; a.inj = inj;
  e = launch_draw(s->g, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(BDC_ECUDA, std::string("bdc_draw_tasks: ") + cudaGetErrorString(e));
  return BDC_OK;
}

int bdc_spd_solve(int device, double* A, int32_t n, double* B, int32_t m, int32_t* info, void* stream) {
  if (n < 0 || m < 0) return fail(BDC_EINVAL, "negative size");
  if (n == 0) return BDC_OK;
  if (!A || (m > 0 && !B) || !info) return fail(BDC_EINVAL, "missing pointer");
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = launch_spd_solve(A, n, B, m, info, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(BDC_ECUDA, std::string("bdc_spd_solve: ") + cudaGetErrorString(e));
  return BDC_OK;
}

int bdc_session_set_wave(BdcSession* s, int64_t cap) {
  if (!s) return fail(BDC_EINVAL, "null session");
  s->wave_cap = cap;
  return BDC_OK;
}

}  // extern "C"

namespace {

struct Layout {
  size_t off[128];
  int n = 0;
  size_t total = 0;
  size_t add(size_t bytes) {
    size_t o = total;
    off[n++] = o;
    total += al(bytes);
    return o;
  }
};

// Carve one allocation into the wave workspace; returns bytes needed.
size_t carve(const DevGrid& g, int Wb, int T, int D, int Ein, int rs, char* base, Work* w) {
  Layout L;
  const size_t B = Wb;
  const int Cs = g.C0 + rs;
  const int NCw = (g.NC + 31) / 32 > 0 ? (g.NC + 31) / 32 : 1;
  size_t o_spl = L.add(B * g.S * Ein), o_dis = L.add(B * (D > 0 ? D : 1) * 8), o_inj = L.add(B * T * (g.K > 0 ? g.K : 1));
  size_t o_tc = L.add(B * 4);
  // a second input buffer: host inputs of wave w + 1 are copied while wave w computes
  size_t o_spl2 = L.add(B * g.S * Ein), o_dis2 = L.add(B * (D > 0 ? D : 1) * 8), o_inj2 = L.add(B * T * (g.K > 0 ? g.K : 1));
  size_t o_tc2 = L.add(B * 4);
  size_t o_st = L.add(B * 4), o_sa = L.add(B * 4), o_rk = L.add(B * 4), o_ns = L.add(B * 4), o_nd = L.add(B * 4);
  size_t o_dead = L.add(B * RMAX * 4), o_ss = L.add(B * RMAX * 4), o_ni = L.add(B * 4), o_isl = L.add(B * NCw * 4);
  size_t o_B = L.add(B * rs * g.R * 8), o_C = L.add(B * rs * Cs * 8);
  size_t o_W = L.add(B * g.N1 * rs * 8), o_den = L.add(B * g.N1 * 8), o_ok = L.add(B * g.N1);
  size_t o_Wm = L.add(B * g.NMB * rs * 8), o_mi = L.add(B * g.NM * MMAX * MMAX * 8), o_mo = L.add(B * g.NM);
  size_t o_ca = L.add(B * g.NI * rs * 8), o_cb = L.add(B * g.NI * rs * 8);
  size_t o_Y = L.add(B * rs * T * 8), o_n0s = L.add(B * g.M * T * 4);
  size_t o_m32 = L.add(B * T * 4), o_n0b = L.add(B * g.R * 8), o_n0m = L.add(B * g.M * 8);
  size_t o_bmon = L.add(B * (size_t)rs * g.M * 8);
  size_t o_cmax = L.add(B * (size_t)(g.N1 + g.NM + g.NI) * T * 4);
  const size_t NTERM = ((size_t)g.NM + g.NI) * g.MT;
  size_t o_Lo = L.add(B * (size_t)g.M * NTERM * 4), o_So = L.add(B * NTERM * T * 4);
  size_t o_met = L.add(B * 8), o_best = L.add(B * 8), o_fe = L.add(B);
  size_t o_n0c = L.add(B * 4), o_n0p = L.add(B * KMAX * 4), o_n0f = L.add(B * KMAX * 8), o_n0r = L.add(B * KMAX * 8);
  size_t o_n1c = L.add(B * 4), o_n1k = L.add(B * KMAX * 4), o_n1p = L.add(B * KMAX * 4);
  size_t o_n1f = L.add(B * KMAX * 8), o_n1r = L.add(B * KMAX * 8);
  size_t o_m0 = L.add(B * T * 4), o_sc = L.add(B * (size_t)SB * g.N1 * 4);
  size_t o_m0b = L.add(B * (size_t)SB * T * 4), o_m0bx = L.add(B * (size_t)SB * 4);
  const size_t nqa = (size_t)std::max(1, g.NM + g.NI);
  size_t o_osk = L.add(B * nqa), o_ol = L.add(B * nqa * 4), o_oc = L.add(B * 4);
  const size_t nitems = B * (size_t)((g.N1 + TOPC - 1) / TOPC) * (size_t)((T + top_tile_cands(T) - 1) / top_tile_cands(T));
  size_t o_ll = L.add(B * (size_t)(g.N1 > 0 ? g.N1 : 1) * 4), o_lc = L.add(B * 4);
  size_t o_q = L.add((nitems > 0 ? nitems : 1) * 8);
  size_t o_s32 = L.add(g.s_mon ? 16 : B * (size_t)g.N1 * T * 4), o_bk = L.add(B * (size_t)g.N1 * 4);
  size_t o_rmx = L.add(B * (size_t)(g.M > 0 ? g.M : 1) * 4);
  size_t o_top = L.add(B * (size_t)TOPC * 4), o_done = L.add(B * (size_t)g.N1);
  const int nslot = RSEL_WARPS + (g.N1 + RCW_MIN - 1) / RCW_MIN;
  size_t o_rl = L.add(B * (size_t)(g.N1 > 0 ? g.N1 : 1) * 4), o_rc = L.add(B * 4), o_th = L.add(B * 4);
  size_t o_pc = L.add(B * nslot * KMAX * 4), o_pp = L.add(B * nslot * KMAX * 4);
  size_t o_pf = L.add(B * nslot * KMAX * 8), o_pr = L.add(B * nslot * KMAX * 8), o_pm = L.add(B * nslot * 8);
  size_t o_b32 = L.add(B * b32_task_floats(rs, g.M) * 4), o_bmx = L.add(B * (size_t)rs * 4);
  size_t o_smx = L.add(B * (size_t)g.N1 * 4);
  size_t o_lf = L.add(64), o_bs = L.add(16), o_rsq = L.add(B * 4);
  // prefix memo of the split chain (k_update): up to PFX_LEVELS entries per task.  Opt-in
  // (BDC_PREFIX=1): bit-identical and it shares 58 % of the split applications at G118, but
  // the probe / wait / copy costs more than the split it saves (G118 update 2.92 -> 3.62 ms,
  // G1k 3.44 -> 3.54 ms), so the flat chain is the default
  const char* pe = std::getenv("BDC_PREFIX");
  const bool pfx_on = pe && pe[0] == '1';
  size_t pcap = 0;
  if (pfx_on) { pcap = 1; while (pcap < (size_t)B * PFX_LEVELS) pcap <<= 1; }
  const size_t pc1 = pcap > 0 ? pcap : 1;
  size_t o_pk = L.add(pc1 * 8), o_pst = L.add(pc1 * 4), o_pfl = L.add(pc1 * 4), o_pid = L.add(pc1 * 2 * PFX_LEVELS * 4);
  size_t o_pB = L.add(pcap * (size_t)g.R * 8), o_pC = L.add(pcap * (size_t)Cs * 8);
  if (!base) return L.total;
  Work& x = *w;
  x.Wb = Wb; x.T = T; x.D = D; x.Ein = Ein; x.rs = rs; x.Cs = Cs; x.NCw = NCw;
  x.splits = (const uint8_t*)(base + o_spl);
  x.discos = (const int64_t*)(base + o_dis);
  x.inj = (const uint8_t*)(base + o_inj);
  x.tcount = (const int*)(base + o_tc);
  x.in2_splits = (const uint8_t*)(base + o_spl2);
  x.in2_discos = (const int64_t*)(base + o_dis2);
  x.in2_inj = (const uint8_t*)(base + o_inj2);
  x.in2_tcount = (const int*)(base + o_tc2);
  x.status = (int*)(base + o_st); x.sarg = (int*)(base + o_sa); x.rank = (int*)(base + o_rk);
  x.nsplit = (int*)(base + o_ns); x.ndead = (int*)(base + o_nd); x.dead = (int*)(base + o_dead);
  x.splitsub = (int*)(base + o_ss); x.nisl = (int*)(base + o_ni); x.isl = (uint32_t*)(base + o_isl);
  x.Bm = (double*)(base + o_B); x.Cm = (double*)(base + o_C);
  x.Wsc = (double*)(base + o_W); x.den = (double*)(base + o_den); x.sc_ok = (uint8_t*)(base + o_ok);
  x.Wm = (double*)(base + o_Wm); x.minv = (double*)(base + o_mi); x.mc_ok = (uint8_t*)(base + o_mo);
  x.cia = (double*)(base + o_ca); x.cib = (double*)(base + o_cb);
  x.Y = (double*)(base + o_Y); x.n0s = (float*)(base + o_n0s);
  x.m32 = (uint32_t*)(base + o_m32); x.n0b = (double*)(base + o_n0b); x.n0m = (double*)(base + o_n0m);
  x.Bmon = (double*)(base + o_bmon);
  x.cmax = (float*)(base + o_cmax);
  x.Lo = (float*)(base + o_Lo); x.So = (float*)(base + o_So); x.NTERM = (int)NTERM;
  x.metric = (double*)(base + o_met); x.best = (int64_t*)(base + o_best); x.feasible = (uint8_t*)(base + o_fe);
  x.n0cnt = (int*)(base + o_n0c); x.n0pos = (int*)(base + o_n0p); x.n0flow = (double*)(base + o_n0f);
  x.n0rel = (double*)(base + o_n0r);
  x.n1cnt = (int*)(base + o_n1c); x.n1case = (int*)(base + o_n1k); x.n1pos = (int*)(base + o_n1p);
  x.n1flow = (double*)(base + o_n1f); x.n1rel = (double*)(base + o_n1r);
  // counters, one 32-byte block zeroed per call: [0] loadflows [1] bsdf [2] evaluated pairs
  // [3] single cases revisited by the winner report
  x.lf = (unsigned long long*)(base + o_lf);
  x.bsdf = x.lf + 1;
  x.pairs = x.lf + 2;
  x.rsq = (int*)(base + o_rsq);
  x.rsq_n = (unsigned*)(base + o_bs) + 1;  // FP64 re-score queue length, zeroed per wave
  x.qcount = (unsigned*)(base + o_bs);  // k_pairs queue length, zeroed per wave
  x.m0 = (float*)(base + o_m0); x.scale = (float*)(base + o_sc);
  x.s32 = (float*)(base + o_s32); x.bkey = (uint32_t*)(base + o_bk); x.rmax = (float*)(base + o_rmx);
  x.top = (int*)(base + o_top); x.done = (uint8_t*)(base + o_done);
  x.ptop = TOPC;
  x.m0b = (float*)(base + o_m0b);
  x.m0bx = (float*)(base + o_m0bx);
  x.pfx_cap = (int)pcap;
  x.pfx_key = (unsigned long long*)(base + o_pk); x.pfx_state = (int*)(base + o_pst);
  x.pfx_fail = (int*)(base + o_pfl); x.pfx_id = (int*)(base + o_pid);
  x.pfx_B = (double*)(base + o_pB); x.pfx_C = (double*)(base + o_pC);
  x.oskip = (uint8_t*)(base + o_osk); x.olist = (int*)(base + o_ol); x.ocnt = (int*)(base + o_oc);
  x.llist = (int*)(base + o_ll); x.lcnt = (int*)(base + o_lc);
  x.queue = (int2*)(base + o_q);
  x.B32 = (float*)(base + o_b32); x.bmax = (float*)(base + o_bmx); x.smax = (float*)(base + o_smx);
  x.rlist = (int*)(base + o_rl); x.rcnt = (int*)(base + o_rc); x.theta = (float*)(base + o_th); x.nslot = nslot;
  {  // wide tiles when tasks alone fill the GPU (tests force either: BDC_RSWEEP_WIDE=0/1)
    const char* wide = std::getenv("BDC_RSWEEP_WIDE");
    x.rcw = wide ? (wide[0] == '1' ? RCW : RCW_MIN) : (Wb >= 1024 ? RCW : RCW_MIN);
  }
  x.pcase = (int*)(base + o_pc); x.ppos = (int*)(base + o_pp);
  x.pflow = (double*)(base + o_pf); x.prel = (double*)(base + o_pr); x.pmax = (double*)(base + o_pm);
  return L.total;
}

// Byte offsets of one wave's outputs in a pinned staging buffer.
struct OutLayout {
  size_t metric, best, feasible, status, sarg, nisl, isl, n0cnt, n1cnt;
  size_t n0pos, n0flow, n1case, n1pos, n1flow, cand;
  size_t build(int Wb, int kg, int NCw, int T) {
    size_t o = 0;
    auto add = [&](size_t bytes) { size_t r = o; o += (bytes + 255) & ~size_t(255); return r; };
    const size_t B = Wb;
    metric = add(B * 8); best = add(B * 8); feasible = add(B); status = add(B * 4); sarg = add(B * 4);
    nisl = add(B * 4); isl = add(B * NCw * 4); n0cnt = add(B * 4); n1cnt = add(B * 4);
    n0pos = add(B * kg * 4); n0flow = add(B * kg * 8); n1case = add(B * kg * 4); n1pos = add(B * kg * 4);
    n1flow = add(B * kg * 8); cand = add(B * (size_t)T * 4);
    return o;
  }
};

struct StreamGuard {
  cudaStream_t s = nullptr;
  bool own = false;
  ~StreamGuard() {
    if (own && s) cudaStreamDestroy(s);
  }
};

// Device-to-host (or device-to-device) copy of a wave's slice of one output.
template <class T>
cudaError_t out_copy(T* dst, const T* src, size_t n, int64_t off, bool on_dev, cudaStream_t st) {
  if (!dst || n == 0) return cudaSuccess;
  return cudaMemcpyAsync(dst + off, src, n * sizeof(T),
                         on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st);
}

// The wave workspace with its input pointers switched to input buffer `i` (0 or 1).
Work in_buf(const Work& w, int i) {
  Work x = w;
  if (i) {
    x.splits = w.in2_splits; x.discos = w.in2_discos; x.inj = w.in2_inj; x.tcount = w.in2_tcount;
  }
  return x;
}

}  // namespace

extern "C" int bdc_solve(BdcSession* s, BdcBatch* bt) {
  if (!s || !bt) return fail(BDC_EINVAL, "null argument");
  const DevGrid& g = s->g;
  const int64_t B = bt->B;
  const int T = bt->T, D = bt->D, Ein = g.E > 0 ? g.E : 1;
  for (int i = 0; i < BDC_STAGES; ++i) bt->stage_ms[i] = 0.f;
  bt->waves = 0;
  bt->kernel_launches = 0;
  if (B < 0 || T < 1 || D < 0) return fail(BDC_EINVAL, "bad batch dimensions");
  if (B == 0) {
    if (bt->loadflows) *bt->loadflows = 0;
    return BDC_OK;
  }
  if (!bt->splits || !bt->inj || (D > 0 && !bt->discos) || !bt->metric || !bt->best ||
      !bt->feasible || !bt->status)
    return fail(BDC_EINVAL, "missing required input or output pointer");
  if (T > 65535 * 128) return fail(BDC_ELIMIT, "too many candidates per task");
  const int rs = bt->max_rank > 0 ? (bt->max_rank < RMAX ? bt->max_rank : RMAX) : RMAX;
  CK(cudaSetDevice(s->device));
  StreamGuard sg;
  if (bt->stream) {
    sg.s = (cudaStream_t)bt->stream;
  } else {
    CK(cudaStreamCreateWithFlags(&sg.s, cudaStreamNonBlocking));
    sg.own = true;
  }
  cudaStream_t st = sg.s;

  // wave size: bounded by a workspace budget, the grid-z limit and the user cap
  // (a deterministic function of the batch shape and the device size, so repeated
  // calls reuse the session's cached workspace instead of re-mapping memory)
  size_t per = carve(g, 1, T, D, Ein, rs, nullptr, nullptr);
  size_t budget = std::min<size_t>(s->total_mem / 8, (size_t)16 << 30);
  int64_t Wb = (int64_t)(budget / per);
  if (Wb < 1) return fail(BDC_ELIMIT, "one task does not fit in device memory");
  Wb = std::min<int64_t>(Wb, 32768);
  if (s->wave_cap > 0) Wb = std::min<int64_t>(Wb, s->wave_cap);
  Wb = std::min<int64_t>(Wb, B);
  if (B > Wb) Wb = (B + ((B + Wb - 1) / Wb) - 1) / ((B + Wb - 1) / Wb);  // balance the waves
  Work w{};
  size_t bytes = carve(g, (int)Wb, T, D, Ein, rs, nullptr, nullptr);
  WsLease ws(s, bytes);
  if (!ws.p) return fail(BDC_ECUDA, "workspace allocation failed (" + std::to_string(bytes) + " bytes)");
  carve(g, (int)Wb, T, D, Ein, rs, ws.p, &w);
  w.screen = bt->screen ? 1 : 0;
  {
    const char* rc = std::getenv("BDC_RSEL_CTA");
    w.rsel_cta = (rc && rc[0] == '1') ? 1 : 0;
  }
  w.ranked = (w.screen && g.N1 > w.ptop) ? 1 : 0;
  w.oscr = other_screened(g, w) ? 1 : 0;
  CK(cudaMemsetAsync(w.lf, 0, 64, st));

  const int nwaves = (int)((B + Wb - 1) / Wb);
  constexpr int NE = BDC_STAGES + 1;  // events per wave
  std::vector<cudaEvent_t> ev((size_t)nwaves * NE);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  // side stream: the multi/injection correction terms (k_terms) next to the N-0 contraction,
  // and -- unscreened -- the multi/injection N-1 stream (k_other) next to the single-branch
  // scales / top-k / TOP tile; joined before the exact screen reads the candidates' lower
  // bounds.  Only on waves too small to fill the GPU (G10k, 64 topologies: 7.2 -> 6.6 ms);
  // on full waves the overlapped kernels slow each other down as much as they gain (G118
  // 20.0 -> 20.1 ms, G3k 17.8 -> 18.0).  Test knob BDC_SIDE=0/1 forces it.
  const char* side_env = std::getenv("BDC_SIDE");
  const bool side = (side_env ? side_env[0] == '1' : Wb < 512) && g.NM + g.NI > 0 && g.M > 0;
  constexpr int NS = 4;  // side events per wave: terms start/end, other start/end
  const bool terms = g.NM + g.NI > 0 && g.M > 0;  // k_terms timed apart (multi/injection stage)
  std::vector<cudaEvent_t> sev(terms ? (size_t)nwaves * NS : 0);
  for (auto& e : sev) CK(cudaEventCreate(&e));
  struct EvVecGuard {
    std::vector<cudaEvent_t>& v;
    ~EvVecGuard() { for (auto& e : v) cudaEventDestroy(e); }
  } sevg{sev};
  StreamGuard ss;
  if (side) {
    CK(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
    ss.own = true;
  }
  const bool ondev_in = bt->inputs_on_device != 0, ondev_out = bt->outputs_on_device != 0;
  const int kg = s->cfg.kg, NCw = w.NCw;
  // pinned staging for host outputs: two wave-sized buffers, unpacked by the host while
  // the next wave runs; report loadings are recomputed on the host as |flow| / rating
  // (true division, as the reference's np.abs(flows) / ratings, solver.py:293), so they are not copied
  OutLayout olay{};
  std::unique_ptr<PinLease> pin[2];
  cudaEvent_t wdone[2] = {nullptr, nullptr};
  int64_t staged_b0[2] = {0, 0};
  int staged_nb[2] = {0, 0};
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() { for (int i = 0; i < 2; ++i) if (e[i]) cudaEventDestroy(e[i]); }
  } evg{wdone};
  if (!ondev_out) {
    const size_t sb = olay.build((int)Wb, kg, NCw, bt->cand_metric ? T : 0);
    for (int i = 0; i < 2; ++i) {
      pin[i].reset(new PinLease(s, sb));
      if (!pin[i]->p) return fail(BDC_ECUDA, "pinned staging allocation failed");
      CK(cudaEventCreateWithFlags(&wdone[i], cudaEventDisableTiming));
    }
  }
  auto unpack = [&](int slot) -> cudaError_t {
    cudaError_t e = cudaEventSynchronize(wdone[slot]);
    if (e != cudaSuccess) return e;
    const char* hp = pin[slot]->p;
    const OutLayout& O = olay;
    const int64_t b0 = staged_b0[slot];
    const size_t nb = (size_t)staged_nb[slot];
    const double* rat = s->rating.data();
    const int M = (int)s->rating.size();
    // tasks [t0, t1) of the staged wave into the caller's arrays (first-touch page faults
    // and copies dominate for large waves: a few host threads share them)
    auto part = [&](size_t t0, size_t t1) {
      auto put = [&](void* dst, size_t off, size_t bpt) {
        if (dst) std::memcpy((char*)dst + (b0 + t0) * bpt, hp + off + t0 * bpt, (t1 - t0) * bpt);
      };
      put(bt->metric, O.metric, 8);
      put(bt->best, O.best, 8);
      put(bt->feasible, O.feasible, 1);
      put(bt->status, O.status, 4);
      put(bt->status_arg, O.sarg, 4);
      put(bt->n_islanded, O.nisl, 4);
      put(bt->islanded_bits, O.isl, (size_t)NCw * 4);
      put(bt->n0_count, O.n0cnt, 4);
      put(bt->n1_count, O.n1cnt, 4);
      put(bt->n0_pos, O.n0pos, (size_t)kg * 4);
      put(bt->n0_flow, O.n0flow, (size_t)kg * 8);
      put(bt->n1_case, O.n1case, (size_t)kg * 4);
      put(bt->n1_pos, O.n1pos, (size_t)kg * 4);
      put(bt->n1_flow, O.n1flow, (size_t)kg * 8);
      if (bt->cand_metric) put(bt->cand_metric, O.cand, (size_t)T * 4);
      auto rel = [&](double* dst, size_t pos_off, size_t flow_off) {
        if (!dst) return;
        const int32_t* pos = (const int32_t*)(hp + pos_off);
        const double* fl = (const double*)(hp + flow_off);
        double* d = dst + b0 * kg;
        for (size_t i = t0 * kg; i < t1 * (size_t)kg; ++i) {
          const int p = pos[i];
          d[i] = (p >= 0 && p < M) ? std::fabs(fl[i]) / rat[p] : 0.0;
        }
      };
      rel(bt->n0_rel, O.n0pos, O.n0flow);
      rel(bt->n1_rel, O.n1pos, O.n1flow);
    };
    const unsigned hw = std::max(1u, std::min(12u, std::thread::hardware_concurrency()));
    const size_t nt = std::max<size_t>(1, std::min<size_t>(hw, nb / 2048));
    const size_t per = (nb + nt - 1) / nt;
    std::vector<std::thread> th;
    for (size_t i = 1; i < nt; ++i) th.emplace_back(part, i * per, std::min(nb, (i + 1) * per));
    part(0, std::min(nb, per));
    for (auto& t : th) t.join();
    return cudaSuccess;
  };
  // host inputs with several waves: copies on their own stream into two input buffers
  const bool overlap_in = !ondev_in && nwaves > 1;
  StreamGuard cs;
  cudaEvent_t in_ready[2] = {nullptr, nullptr}, buf_free[2] = {nullptr, nullptr};
  struct EvGuard4 {
    cudaEvent_t* a; cudaEvent_t* b;
    ~EvGuard4() { for (int i = 0; i < 2; ++i) { if (a[i]) cudaEventDestroy(a[i]); if (b[i]) cudaEventDestroy(b[i]); } }
  } evg4{in_ready, buf_free};
  if (overlap_in) {
    CK(cudaStreamCreateWithFlags(&cs.s, cudaStreamNonBlocking));
    cs.own = true;
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&in_ready[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&buf_free[i], cudaEventDisableTiming));
    }
    CK(cudaEventRecord(buf_free[0], st));  // the caller's prior work on st precedes the copies
    CK(cudaStreamWaitEvent(cs.s, buf_free[0], 0));
  }
  const cudaMemcpyKind hk = ondev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const size_t sz_spl = (size_t)g.S * Ein, sz_inj = (size_t)T * g.K;
  // inputs of wave v into x's buffers on stream q (records in_ready when overlapping)
  auto copy_inputs = [&](const Work& x, int v, cudaStream_t q) -> cudaError_t {
    const int64_t v0 = (int64_t)v * Wb;
    const size_t m = (size_t)std::min<int64_t>(Wb, B - v0);
    cudaError_t e = cudaSuccess;
    if (sz_spl) e = cudaMemcpyAsync((void*)x.splits, bt->splits + v0 * sz_spl, m * sz_spl, hk, q);
    if (e == cudaSuccess && D > 0)
      e = cudaMemcpyAsync((void*)x.discos, bt->discos + v0 * D, m * D * 8, hk, q);
    if (e == cudaSuccess && sz_inj) e = cudaMemcpyAsync((void*)x.inj, bt->inj + v0 * sz_inj, m * sz_inj, hk, q);
    if (e == cudaSuccess && bt->t_count)
      e = cudaMemcpyAsync((void*)x.tcount, bt->t_count + v0, m * 4, hk, q);
    if (e == cudaSuccess && overlap_in) e = cudaEventRecord(in_ready[v & 1], q);
    return e;
  };
  int launches = 0;
  cudaError_t err = cudaSuccess;
  for (int wv = 0; wv < nwaves && err == cudaSuccess; ++wv) {
    const int64_t b0 = (int64_t)wv * Wb;
    const int nb = (int)std::min<int64_t>(Wb, B - b0);
    Work x = in_buf(w, wv & 1);
    x.Wb = nb;
    cudaEvent_t* E = &ev[(size_t)wv * NE];
    cudaEventRecord(E[0], st);
    if (!overlap_in) {
      err = copy_inputs(x, wv, st);
    } else {
      if (wv == 0) err = copy_inputs(x, 0, cs.s);
      if (err == cudaSuccess) err = cudaStreamWaitEvent(st, in_ready[wv & 1], 0);
    }
    if (!bt->t_count) x.tcount = nullptr;
    if (err == cudaSuccess) err = cudaMemsetAsync(x.m32, 0, (size_t)nb * T * 4, st);
    if (err == cudaSuccess) err = cudaMemsetAsync(x.m0, 0, (size_t)nb * T * 4, st);
    if (err == cudaSuccess) err = cudaMemsetAsync(x.m0b, 0, (size_t)nb * SB * T * 4, st);
    if (err == cudaSuccess) err = cudaMemsetAsync(x.m0bx, 0, (size_t)nb * SB * 4, st);
    if (err == cudaSuccess && x.pfx_cap) {  // an empty prefix table per wave
      err = cudaMemsetAsync(x.pfx_key, 0, (size_t)x.pfx_cap * 8, st);
      if (err == cudaSuccess) err = cudaMemsetAsync(x.pfx_state, 0, (size_t)x.pfx_cap * 4, st);
    }
    if (err == cudaSuccess) err = cudaMemsetAsync(x.qcount, 0, 8, st);  // k_pairs queue, re-score queue
    if (err == cudaSuccess) err = cudaMemsetAsync(x.lcnt, 0, (size_t)nb * 4, st);
    if (err == cudaSuccess) err = cudaMemsetAsync(x.bmax, 0, (size_t)nb * rs * 4, st);
    // zero padding of the tensor-core operand (rank slots past the task's rank, rows past M)
    if (err == cudaSuccess) err = cudaMemsetAsync(x.B32, 0, (size_t)nb * b32_task_floats(rs, g.M) * 4, st);
    if (err != cudaSuccess) break;
    cudaEventRecord(E[1], st);
    // events in execution order; stage_ms (bdc.h BDC_STAGE_*: 0 h2d, 1 update, 2 N-0,
    // 3 multi/injection N-1, 4 screening scales (tcgen05), 5 top-k, 6 TOP tile, 7 screen +
    // live cases, 8 select, 9 winner report, 10 d2h) from kExecStage below.  The
    // multi/injection cases run after the TOP tile so that their own dominance screen
    // (k_oscreen) sees the TOP cases' maxima.
    launch_update(g, s->cfg, x, st);
    cudaEventRecord(E[2], st);
    cudaEvent_t* S = terms ? &sev[(size_t)wv * NS] : nullptr;
    if (side) {  // S[0] follows k_update on the solve stream
      cudaEventRecord(S[0], st);
      cudaStreamWaitEvent(ss.s, S[0], 0);
      launch_terms(g, x, ss.s);
      cudaEventRecord(S[1], ss.s);
    } else if (terms) {  // inside the N-0 interval on the solve stream; moved to its stage below
      cudaEventRecord(S[0], st);
      launch_terms(g, x, st);
      cudaEventRecord(S[1], st);
    }
    launch_n0(g, x, st);
    cudaEventRecord(E[3], st);
    if (x.oscr) {
      launch_single_top(g, s->cfg, x, st, &E[4]);  // records E[4], E[5], E[6]
      if (side) cudaStreamWaitEvent(st, S[1], 0);
      launch_other(g, s->cfg, x, st);  // its screen reads the TOP tile's maxima
      cudaEventRecord(E[7], st);
    } else if (side) {  // the multi/injection stream next to the single-branch TOP path
      cudaStreamWaitEvent(ss.s, E[3], 0);  // reads the N-0 table
      cudaEventRecord(S[2], ss.s);
      launch_other(g, s->cfg, x, ss.s);
      cudaEventRecord(S[3], ss.s);
      cudaEventRecord(E[4], st);
      launch_single_top(g, s->cfg, x, st, &E[5]);  // records E[5], E[6], E[7]
      cudaStreamWaitEvent(st, S[3], 0);  // the screen's lower bounds include those cases
    } else {  // unscreened: the multi/injection stream first (the order measured faster)
      launch_other(g, s->cfg, x, st);
      cudaEventRecord(E[4], st);
      launch_single_top(g, s->cfg, x, st, &E[5]);  // records E[5], E[6], E[7]
    }
    launch_single_screen(g, s->cfg, x, st);
    cudaEventRecord(E[8], st);
    launch_select(g, s->cfg, x, st);
    cudaEventRecord(E[9], st);
    launch_report(g, s->cfg, x, st);
    cudaEventRecord(E[10], st);
    if (overlap_in && wv + 1 < nwaves) {
      // the next wave's inputs go into the other buffer once wave wv - 1 is done with it
      cudaEventRecord(buf_free[wv & 1], st);
      if (wv >= 1) cudaStreamWaitEvent(cs.s, buf_free[(wv + 1) & 1], 0);
      Work nx = in_buf(w, (wv + 1) & 1);
      if (err == cudaSuccess) err = copy_inputs(nx, wv + 1, cs.s);
    }
    launches += kernels_per_wave(g, x);
    err = cudaGetLastError();
    if (err != cudaSuccess) break;
    // outputs: straight into device buffers, or through pinned staging for host
    // (pageable) buffers -- the unpack of wave wv-1 overlaps the kernels of wave wv
    cudaError_t e2 = cudaSuccess;
    auto chk = [&](cudaError_t e) { if (e2 == cudaSuccess) e2 = e; };
    if (ondev_out) {
      chk(out_copy(bt->metric, x.metric, nb, b0, true, st));
      chk(out_copy(bt->best, x.best, nb, b0, true, st));
      chk(out_copy(bt->feasible, x.feasible, nb, b0, true, st));
      chk(out_copy(bt->status, x.status, nb, b0, true, st));
      chk(out_copy(bt->status_arg, x.sarg, nb, b0, true, st));
      chk(out_copy(bt->n_islanded, x.nisl, nb, b0, true, st));
      chk(out_copy(bt->islanded_bits, x.isl, (size_t)nb * NCw, b0 * NCw, true, st));
      chk(out_copy(bt->n0_count, x.n0cnt, nb, b0, true, st));
      chk(out_copy(bt->n1_count, x.n1cnt, nb, b0, true, st));
      // report entries: (task, kg) on device as in the user's arrays
      auto strided = [&](auto* dst, const auto* src, size_t elem) {
        if (!dst) return;
        chk(cudaMemcpy2DAsync(dst + b0 * kg, kg * elem, src, (size_t)kg * elem, (size_t)kg * elem, nb,
                              cudaMemcpyDeviceToDevice, st));
      };
      strided(bt->n0_pos, x.n0pos, 4);
      strided(bt->n0_flow, x.n0flow, 8);
      strided(bt->n0_rel, x.n0rel, 8);
      strided(bt->n1_case, x.n1case, 4);
      strided(bt->n1_pos, x.n1pos, 4);
      strided(bt->n1_flow, x.n1flow, 8);
      strided(bt->n1_rel, x.n1rel, 8);
      if (bt->cand_metric)
        chk(cudaMemcpyAsync(bt->cand_metric + b0 * T, x.m32, (size_t)nb * T * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      char* hp = pin[wv & 1]->p;
      const OutLayout& O = olay;
      chk(cudaMemcpyAsync(hp + O.metric, x.metric, (size_t)nb * 8, cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(hp + O.best, x.best, (size_t)nb * 8, cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(hp + O.feasible, x.feasible, (size_t)nb, cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(hp + O.status, x.status, (size_t)nb * 4, cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(hp + O.sarg, x.sarg, (size_t)nb * 4, cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(hp + O.nisl, x.nisl, (size_t)nb * 4, cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(hp + O.isl, x.isl, (size_t)nb * NCw * 4, cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(hp + O.n0cnt, x.n0cnt, (size_t)nb * 4, cudaMemcpyDeviceToHost, st));
      chk(cudaMemcpyAsync(hp + O.n1cnt, x.n1cnt, (size_t)nb * 4, cudaMemcpyDeviceToHost, st));
      auto strided = [&](size_t off, const void* src, size_t elem) {  // device stride is kg
        chk(cudaMemcpyAsync(hp + off, src, (size_t)nb * kg * elem, cudaMemcpyDeviceToHost, st));
      };
      strided(O.n0pos, x.n0pos, 4);
      strided(O.n0flow, x.n0flow, 8);
      strided(O.n1case, x.n1case, 4);
      strided(O.n1pos, x.n1pos, 4);
      strided(O.n1flow, x.n1flow, 8);
      if (bt->cand_metric) chk(cudaMemcpyAsync(hp + O.cand, x.m32, (size_t)nb * T * 4, cudaMemcpyDeviceToHost, st));
      chk(cudaEventRecord(wdone[wv & 1], st));
      staged_b0[wv & 1] = b0;
      staged_nb[wv & 1] = nb;
      if (wv > 0 && e2 == cudaSuccess) chk(unpack((wv - 1) & 1));
    }
    cudaEventRecord(E[11], st);
    cudaEventRecord(E[12], st);
    err = e2;
  }
  if (!ondev_out && err == cudaSuccess) err = unpack((nwaves - 1) & 1);
  unsigned long long counters[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (err == cudaSuccess) err = cudaMemcpyAsync(counters, w.lf, 64, cudaMemcpyDeviceToHost, st);
  cudaError_t es = cudaStreamSynchronize(st);
  if (err == cudaSuccess) err = es;
  // a copy of the next wave's inputs may still be in flight on the copy stream (error
  // break): it must land before the workspace goes back to the session cache
  if (overlap_in) {
    es = cudaStreamSynchronize(cs.s);
    if (err == cudaSuccess) err = es;
  }
  if (side) {  // likewise the side stream's kernels (an error break can leave them queued)
    es = cudaStreamSynchronize(ss.s);
    if (err == cudaSuccess) err = es;
  }
  if (err == cudaSuccess) {
    for (int wv = 0; wv < nwaves; ++wv) {
      cudaEvent_t* E = &ev[(size_t)wv * NE];
      // interval k (E[k] -> E[k+1], execution order) belongs to stage kExecStage[k]
      static constexpr int kScreened[BDC_STAGES] = {0, 1, 2, 4, 5, 6, 3, 7, 8, 9, 10, 11};
      static constexpr int kInOrder[BDC_STAGES] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11};
      const int* kExecStage = w.oscr ? kScreened : kInOrder;
      for (int k = 0; k < BDC_STAGES; ++k) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, E[k], E[k + 1]) == cudaSuccess) {
          bt->stage_ms[kExecStage[k]] += ms;
        }
      }
      if (terms) {  // k_terms (and, on the side stream, k_other) belong to the multi/injection stage
        const cudaEvent_t* S = &sev[(size_t)wv * NS];
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, S[0], S[1]) == cudaSuccess) {
          bt->stage_ms[BDC_STAGE_OTHER] += ms;
          if (!side) bt->stage_ms[BDC_STAGE_N0] -= ms;  // it ran inside the N-0 interval
        }
        if (side && !w.oscr && cudaEventElapsedTime(&ms, S[2], S[3]) == cudaSuccess)
          bt->stage_ms[BDC_STAGE_OTHER] += ms;
      }
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (err != cudaSuccess) return fail(BDC_ECUDA, std::string("bdc_solve: ") + cudaGetErrorString(err));
  if (bt->loadflows) *bt->loadflows = (int64_t)counters[0];
  if (bt->bsdf_applications) *bt->bsdf_applications = (int64_t)counters[1];
  if (bt->n1_pairs) *bt->n1_pairs = (int64_t)counters[2];
  if (bt->report_cases) *bt->report_cases = (int64_t)counters[3];
  if (bt->rescore_stats) {
    bt->rescore_stats[0] = (int64_t)counters[4];
    bt->rescore_stats[1] = (int64_t)counters[5];
    bt->rescore_stats[2] = (int64_t)counters[6];
  }
  if (bt->split_shared) {
    bt->split_shared[0] = (int64_t)counters[7];
  }
  bt->waves = nwaves;
  bt->kernel_launches = launches;
  return BDC_OK;
}

extern "C" int bdc_probe_flows(BdcSession* s, const uint8_t* splits, const int64_t* discos,
                               int32_t D, const uint8_t* inj, int32_t T, double* n0, double* n1,
                               uint8_t* case_ok, int32_t* status, int32_t* status_arg) {
  if (!s || !splits || !inj || !n0 || !n1 || !case_ok || !status || T < 1)
    return fail(BDC_EINVAL, "bad probe arguments");
  const DevGrid& g = s->g;
  const int Ein = g.E > 0 ? g.E : 1;
  CK(cudaSetDevice(s->device));
  StreamGuard sg;
  CK(cudaStreamCreateWithFlags(&sg.s, cudaStreamNonBlocking));
  sg.own = true;
  cudaStream_t st = sg.s;
  Work w{};
  size_t bytes = carve(g, 1, T, D, Ein, RMAX, nullptr, nullptr);
  char* ws = nullptr;
  double *dn0 = nullptr, *dn1 = nullptr;
  uint8_t* dok = nullptr;
  const size_t n1n = (size_t)g.NC * g.R * T;
  CK(cudaMalloc(&ws, bytes));
  carve(g, 1, T, D, Ein, RMAX, ws, &w);
  w.tcount = nullptr;
  cudaError_t e = cudaMalloc(&dn0, (size_t)g.R * T * 8);
  if (e == cudaSuccess) e = cudaMalloc(&dn1, n1n * 8 + 8);
  if (e == cudaSuccess) e = cudaMalloc(&dok, g.NC + 1);
  if (e == cudaSuccess) e = cudaMemsetAsync(w.lf, 0, 64, st);
  if (e == cudaSuccess && g.S) e = cudaMemcpyAsync((void*)w.splits, splits, (size_t)g.S * Ein, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && D) e = cudaMemcpyAsync((void*)w.discos, discos, (size_t)D * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && g.K) e = cudaMemcpyAsync((void*)w.inj, inj, (size_t)T * g.K, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(w.m32, 0, (size_t)T * 4, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(dok, 0, g.NC + 1, st);
  int hs[2] = {0, 0};
  if (e == cudaSuccess) {
    launch_update(g, s->cfg, w, st);
    e = cudaMemcpyAsync(hs, w.status, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hs + 1, w.sarg, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  // islanding_policy = "error" still evaluates every case (its case_ok flags name the
  // islanded cases the reference reports, solver.py:501-511)
  if (e == cudaSuccess && (hs[0] == BDC_TASK_OK || hs[0] == BDC_TASK_ISLAND_ERROR)) {
    launch_probe(g, w, dn0, dn1, dok, st);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(n0, dn0, (size_t)g.R * T * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && n1n) e = cudaMemcpyAsync(n1, dn1, n1n * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && g.NC) e = cudaMemcpyAsync(case_ok, dok, g.NC, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  cudaFree(ws);
  cudaFree(dn0);
  cudaFree(dn1);
  cudaFree(dok);
  if (e != cudaSuccess) return fail(BDC_ECUDA, std::string("bdc_probe_flows: ") + cudaGetErrorString(e));
  *status = hs[0];
  if (status_arg) *status_arg = hs[1];
  return BDC_OK;
}
