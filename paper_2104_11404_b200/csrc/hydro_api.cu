// hydro_api.cu -- the C ABI of include/hydro.h: argument checks, context/sample-plan
// setup (S0, untimed), and the launch sequences of the hot path (S1-S9).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <vector>

#include "../../include/hydro.h"
#include "force2d.cuh"
#include "force2d_pl.cuh"
#include "fom.cuh"
#include "offline.cuh"
#include "force_kernel.cuh"
#include "hydro_internal.h"
#include "rom_kernels.cuh"

namespace {

std::atomic<int64_t> g_launches{0};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t tables, status, mq, off, slot, evec, cnt, total;
};

bool supported(int dim, int k, int q) {
  return (dim == 2 || dim == 3) && ((k == 2 && q == 4) || (k == 3 && q == 6));
}

int ipow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

bool layout_for(const hydro_mesh_desc *d, Layout *L) {
  if (!d || !supported(d->dim, d->order_h1, d->nq1d) || d->n_elem <= 0 || d->n_nodes <= 0)
    return false;
  const int64_t nd = ipow(d->order_h1 + 1, d->dim), nq = ipow(d->nq1d, d->dim);
  if (d->n_elem * nd >= (int64_t)1 << 31) return false;  // int32 slots
  size_t o = 0;
  L->tables = o; o = align256(o + sizeof(double) * HYDRO_TAB_DOUBLES);
  L->status = o; o = align256(o + sizeof(hydro_devstatus));
  L->mq = o;     o = align256(o + sizeof(double) * (size_t)(d->n_elem * nq));
  L->off = o;    o = align256(o + sizeof(int32_t) * (size_t)(d->n_nodes + 1));
  L->slot = o;   o = align256(o + sizeof(int32_t) * (size_t)(d->n_elem * nd));
  L->evec = o;   o = align256(o + sizeof(double) * (size_t)(d->n_elem * nd * d->dim));
  L->cnt = o;    o = align256(o + sizeof(uint32_t) * (size_t)(d->n_nodes + 1));  // + done counter
  L->total = o;
  return true;
}

#define CUDA_OK(x)                                   \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) {                         \
      fprintf(stderr, "hydro: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return HYDRO_ERR_CUDA;                         \
    }                                                \
  } while (0)

// device tables [w(q) | B(q*n) | G(q*n) | Bl(q*m)]
void pack_tables(const hydro_tables_t &T, std::vector<double> &out) {
  const int q = T.q, n = T.k + 1, m = T.k;
  out.assign(HYDRO_TAB_DOUBLES, 0.0);
  size_t o = 0;
  for (int i = 0; i < q; ++i) out[o++] = T.w[i];
  for (int i = 0; i < q; ++i)
    for (int a = 0; a < n; ++a) out[o++] = T.B[i][a];
  for (int i = 0; i < q; ++i)
    for (int a = 0; a < n; ++a) out[o++] = T.G[i][a];
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < m; ++j) out[o++] = T.Bl[i][j];
}

}  // namespace

struct hydro_ctx {
  hydro_mesh_desc d;
  int nd, ne, nq;
  char *ws;
  Layout L;
  double *tab;            // device packed tables
  hydro_devstatus *st;
  double *mq;
  int32_t *off, *slot;
  double *evec;
  unsigned *cnt;          // [n_nodes] arrival counters, then the CTA done counter
  std::vector<int32_t> h_elem_nodes;  // host copy (sample plans)
};

struct hydro_sample {
  hydro_ctx *ctx;
  int B;
  int64_t n_cl, n_cl_nodes, n_s0_nodes, n_s0;
  int64_t n_slots;
  std::vector<int32_t> h_closure;
  std::vector<int64_t> h_cl_nodes, h_s0_nodes;
  int32_t *elem_nodes = nullptr, *elem_gid = nullptr, *slot = nullptr, *off = nullptr,
          *ftw_row = nullptr, *anode = nullptr;
  int32_t *s0_elem = nullptr;  // [n_s0] closure-local element of each S0 row (inverse of ftw_row)
  unsigned *cnt = nullptr;  // [n_s0_nodes][B] arrival counters, then the done counter
  double *evec = nullptr;
  hydro_devstatus *st = nullptr;
};

namespace {

// --- profiling: event pairs around the force kernel (bench.py's live roofline)
// While a stream is being captured into a CUDA graph the pair is recorded as external
// event-record nodes (they then time every replay of the graph) and kept in `captured`.
struct ProfState {
  std::atomic<bool> on{false};
  std::mutex mu;  // guards the three lists (calls may come from several host threads)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending, pool, captured;
};
ProfState g_prof;

// 2D Q2 kernel choice (hydro_set_2d_kernel): 0 size-based, 1 element per thread, 2 point per
// thread (generic), 3 point per lane with q1 per warp (force2d_pl)
std::atomic<int> g_kernel_2d{0};

std::pair<cudaEvent_t, cudaEvent_t> prof_pair() {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  if (!g_prof.pool.empty()) {
    auto p = g_prof.pool.back();
    g_prof.pool.pop_back();
    return p;
  }
  std::pair<cudaEvent_t, cudaEvent_t> p;
  cudaEventCreate(&p.first);
  cudaEventCreate(&p.second);
  return p;
}

template <int DIM, int K, int Q, bool VISC, int MODE, bool BATCHED, bool HAS_W>
hydro_status launch_force_k(const hk::Params &P, cudaStream_t s) {
  constexpr int NF = hk::nfields<MODE, HAS_W>();
  using G = hk::Geo<DIM, K, Q, NF>;
  constexpr int UPC = hk::units_per_cta<DIM, G::EPB, MODE, BATCHED>();
  const int64_t grid = ((int64_t)P.n_units + G::EPB * UPC - 1) / (G::EPB * UPC);
  if (grid <= 0) return HYDRO_OK;
  constexpr bool SPEC2D = DIM == 2 && K == 2 && Q == 4 && MODE != hk::MODE_MQ && MODE != hk::MODE_FTW;
  using G2 = hk::G2<NF>;
  // one-thread-per-element 2D kernel only when there are enough elements to fill the GPU;
  // small meshes (C0: 64 elements) run a point-per-thread kernel (16x the threads);
  // hydro_set_2d_kernel overrides the choice (the tests run both paths)
  const int k2d = g_kernel_2d.load(std::memory_order_relaxed);
  const bool use2d = SPEC2D && (k2d == 1 || (k2d == 0 && P.n_units >= 148 * G2::UPB * 2));
  constexpr bool SPEC2L = SPEC2D && !HAS_W;
  // small meshes (C0) and w == v: one lane per point, q1 per warp (C0 force call 14.1 -> 11.3 us;
  // on C1 the element kernel stays ahead, 43.0 vs 45.5 us: profiles/ab/r02_ab21_2d_lane.txt)
  const bool use2l = SPEC2L && (k2d == 3 || (k2d == 0 && !use2d));
  void (*kern)(const hk::Params) = hk::force_kernel<DIM, K, Q, VISC, MODE, BATCHED, HAS_W>;
  size_t smem = G::SMEM;
  int nt = G::NT;
  int64_t grid2 = grid;
  if constexpr (SPEC2D) {
    if (use2d) {
      kern = hk::force2d_kernel<VISC, MODE, BATCHED, HAS_W>;
      smem = G2::SMEM;
      nt = G2::NT;
      grid2 = ((int64_t)P.n_units + G2::UPB - 1) / G2::UPB;  // G2::TPE threads per unit
    }
  }
  if constexpr (SPEC2L) {
    if (use2l) {
      kern = hk::force2d_pl_kernel<VISC, MODE, BATCHED>;
      smem = hk::G2L::SMEM;
      nt = hk::G2L::NT;
      grid2 = ((int64_t)P.n_units + hk::G2L::UPB - 1) / hk::G2L::UPB;
    }
  }
  const int kidx = use2l ? 2 : (use2d ? 1 : 0);
  // the dynamic shared-memory opt-in is a per-device function attribute: once per device
  // and kernel (bit d of the mask for device d)
  static std::atomic<unsigned long long> attr_done[3];
  {
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done[kidx].load(std::memory_order_acquire) & bit)) {
      CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_done[kidx].fetch_or(bit, std::memory_order_acq_rel);
    }
  }
  std::pair<cudaEvent_t, cudaEvent_t> ev;
  const bool prof = g_prof.on && (MODE == hk::MODE_FORCE || MODE == hk::MODE_DT);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (prof) {
    ev = prof_pair();
    CUDA_OK(cudaStreamIsCapturing(s, &cap));
    if (cap == cudaStreamCaptureStatusActive)
      CUDA_OK(cudaEventRecordWithFlags(ev.first, s, cudaEventRecordExternal));
    else
      CUDA_OK(cudaEventRecord(ev.first, s));
  }
  kern<<<(unsigned)grid2, nt, smem, s>>>(P);
  g_launches++;
  if (prof) {
    if (cap == cudaStreamCaptureStatusActive) {
      CUDA_OK(cudaEventRecordWithFlags(ev.second, s, cudaEventRecordExternal));
      std::lock_guard<std::mutex> lk(g_prof.mu);
      g_prof.captured.push_back(ev);
    } else {
      CUDA_OK(cudaEventRecord(ev.second, s));
      std::lock_guard<std::mutex> lk(g_prof.mu);
      g_prof.pending.push_back(ev);
    }
  }
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

// Instantiated variants: FORCE x {visc} x {batched} x {w given}; DT x {visc} (full mode,
// no w); MQ (setup).
template <int DIM, int K, int Q>
hydro_status launch_force_t(int mode, bool visc, bool batched, bool has_w, const hk::Params &P,
                            cudaStream_t s) {
  using namespace hk;
  if (mode == MODE_MQ) return launch_force_k<DIM, K, Q, false, MODE_MQ, false, false>(P, s);
  if (mode == MODE_FTW)
    return batched ? launch_force_k<DIM, K, Q, false, MODE_FTW, true, false>(P, s)
                   : launch_force_k<DIM, K, Q, false, MODE_FTW, false, false>(P, s);
  if (mode == MODE_DT) {
    if (batched || has_w) return HYDRO_ERR_ARG;
    return visc ? launch_force_k<DIM, K, Q, true, MODE_DT, false, false>(P, s)
                : launch_force_k<DIM, K, Q, false, MODE_DT, false, false>(P, s);
  }
#define HK_F(V, BA, W) launch_force_k<DIM, K, Q, V, MODE_FORCE, BA, W>(P, s)
  if (visc) {
    if (batched) return has_w ? HK_F(true, true, true) : HK_F(true, true, false);
    return has_w ? HK_F(true, false, true) : HK_F(true, false, false);
  }
  if (batched) return has_w ? HK_F(false, true, true) : HK_F(false, true, false);
  return has_w ? HK_F(false, false, true) : HK_F(false, false, false);
#undef HK_F
}

hydro_status launch_force(int dim, int k, int mode, bool visc, bool batched, bool has_w,
                          const hk::Params &P0, cudaStream_t s) {
  hk::Params P = P0;
  P.b_shift = -1;
  for (int sh = 0; sh < 31; ++sh)
    if (P.B == (1 << sh)) { P.b_shift = sh; break; }
  if (dim == 2 && k == 2) return launch_force_t<2, 2, 4>(mode, visc, batched, has_w, P, s);
  if (dim == 3 && k == 2) return launch_force_t<3, 2, 4>(mode, visc, batched, has_w, P, s);
  if (dim == 2 && k == 3) return launch_force_t<2, 3, 6>(mode, visc, batched, has_w, P, s);
  if (dim == 3 && k == 3) return launch_force_t<3, 3, 6>(mode, visc, batched, has_w, P, s);
  return HYDRO_ERR_UNSUPPORTED;
}

// Dependent launch of the assembly / dt-finalisation kernel with programmatic stream
// serialisation: it is scheduled while the force kernel drains (griddepcontrol) and waits
// on-device for the force grid's results, so the second launch's latency is hidden.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

hydro_status launch_assemble(int dim, int64_t n_nodes, int B, const int32_t *off,
                             const double *evec, double *F1, hydro_devstatus *st, double *dt,
                             cudaStream_t s) {
  const int threads = 256;
  int64_t blocks = (n_nodes * B + threads - 1) / threads;
  if (blocks < 1) blocks = 1;
  cudaError_t e;
  if (dim == 2)
    e = launch_pdl(hk::assemble_kernel<2>, dim3((unsigned)blocks), dim3(threads), s, n_nodes, B, off,
                   evec, F1, st, dt);
  else
    e = launch_pdl(hk::assemble_kernel<3>, dim3((unsigned)blocks), dim3(threads), s, n_nodes, B, off,
                   evec, F1, st, dt);
  g_launches++;
  CUDA_OK(e);
  return HYDRO_OK;
}

void fill_tables_ptrs(hk::Params &P, const hydro_ctx *c) {
  const int q = c->d.nq1d, n = c->d.order_h1 + 1;
  P.tab_w = c->tab;
  P.tab_B = c->tab + q;
  P.tab_G = c->tab + q + q * n;
  P.tab_Bl = c->tab + q + 2 * q * n;
}

}  // namespace

extern "C" {

hydro_status hydro_profile_enable(int on) {
  g_prof.on = on != 0;
  return HYDRO_OK;
}

hydro_status hydro_profile_read(double *total_ms, int64_t *count) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  double tot = 0.0;
  int64_t n = 0;
  for (auto &p : g_prof.pending) {
    CUDA_OK(cudaEventSynchronize(p.second));
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, p.first, p.second));
    tot += ms;
    ++n;
    g_prof.pool.push_back(p);
  }
  g_prof.pending.clear();
  if (total_ms) *total_ms = tot;
  if (count) *count = n;
  return HYDRO_OK;
}

#ifdef HYDRO_COUNT_ROT
hydro_status hydro_debug_rot_counts(unsigned long long *out /* host [12] */, int reset) {
  CUDA_OK(cudaMemcpyFromSymbol(out, hk::g_rot_count, 2 * sizeof(unsigned long long)));
  CUDA_OK(cudaMemcpyFromSymbol(out + 2, hk::g_sweep_count, 8 * sizeof(unsigned long long)));
  CUDA_OK(cudaMemcpyFromSymbol(out + 10, hk::g_rerun_count, 2 * sizeof(unsigned long long)));
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    CUDA_OK(cudaMemcpyToSymbol(hk::g_rot_count, z, 2 * sizeof(unsigned long long)));
    CUDA_OK(cudaMemcpyToSymbol(hk::g_sweep_count, z, sizeof(z)));
    CUDA_OK(cudaMemcpyToSymbol(hk::g_rerun_count, z, 2 * sizeof(unsigned long long)));
  }
  return HYDRO_OK;
}
#endif

hydro_status hydro_profile_read_captured(double *total_ms, int64_t *count) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  double tot = 0.0;
  int64_t n = 0;
  for (auto &p : g_prof.captured) {
    CUDA_OK(cudaEventSynchronize(p.second));
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, p.first, p.second));
    tot += ms;
    ++n;
  }
  if (total_ms) *total_ms = tot;
  if (count) *count = n;
  return HYDRO_OK;
}

hydro_status hydro_profile_release_captured(void) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  for (auto &p : g_prof.captured) g_prof.pool.push_back(p);
  g_prof.captured.clear();
  return HYDRO_OK;
}

hydro_status hydro_selftest_ieee_fast(uint64_t seed, int64_t n, int op, int dist,
                                      unsigned long long *counts, hydro_stream_t stream) {
  if (n < 0 || op < 0 || op > 2 || dist < 0 || dist > 1 || !counts) return HYDRO_ERR_ARG;
  hk::selftest_ieee_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(seed, n, op, dist, counts);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

hydro_status hydro_set_2d_kernel(int choice) {
  if (choice < 0 || choice > 3) return HYDRO_ERR_ARG;
  g_kernel_2d.store(choice);
  return HYDRO_OK;
}

const char *hydro_version(void) { return "hydro-b200 0.1 (sm_100a, FP64)"; }

int64_t hydro_launch_count(void) { return g_launches.load(); }

hydro_status hydro_basis_tables(int k, int q, double *xi, double *w, double *B, double *G,
                                double *Bl) {
  hydro_tables_t T;
  if (hydro_make_tables(k, q, &T)) return HYDRO_ERR_ARG;
  for (int i = 0; i < q; ++i) {
    if (xi) xi[i] = T.xi[i];
    if (w) w[i] = T.w[i];
    for (int a = 0; a <= k; ++a) {
      if (B) B[i * (k + 1) + a] = T.B[i][a];
      if (G) G[i * (k + 1) + a] = T.G[i][a];
    }
    for (int j = 0; j < k; ++j)
      if (Bl) Bl[i * k + j] = T.Bl[i][j];
  }
  return HYDRO_OK;
}

size_t hydro_ctx_workspace_bytes(const hydro_mesh_desc *desc) {
  Layout L;
  if (!layout_for(desc, &L)) return 0;
  return L.total;
}

hydro_status hydro_ctx_create(const hydro_mesh_desc *desc, void *workspace, size_t ws_bytes,
                              hydro_stream_t stream, hydro_ctx **out) {
  if (!desc || !out) return HYDRO_ERR_ARG;
  *out = nullptr;
  if (!supported(desc->dim, desc->order_h1, desc->nq1d)) return HYDRO_ERR_UNSUPPORTED;
  if (!desc->elem_nodes || !desc->x0 || !desc->rho0) return HYDRO_ERR_ARG;
  Layout L;
  if (!layout_for(desc, &L)) return HYDRO_ERR_ARG;
  if (!workspace || ws_bytes < L.total || ((uintptr_t)workspace & 255)) return HYDRO_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  hydro_ctx *c = new hydro_ctx();
  c->d = *desc;
  c->nd = ipow(desc->order_h1 + 1, desc->dim);
  c->ne = ipow(desc->order_h1, desc->dim);
  c->nq = ipow(desc->nq1d, desc->dim);
  c->ws = (char *)workspace;
  c->L = L;
  c->tab = (double *)(c->ws + L.tables);
  c->st = (hydro_devstatus *)(c->ws + L.status);
  c->mq = (double *)(c->ws + L.mq);
  c->off = (int32_t *)(c->ws + L.off);
  c->slot = (int32_t *)(c->ws + L.slot);
  c->evec = (double *)(c->ws + L.evec);
  c->cnt = (unsigned *)(c->ws + L.cnt);
  auto fail = [&](hydro_status st) { delete c; return st; };
  // tables
  hydro_tables_t T;
  if (hydro_make_tables(desc->order_h1, desc->nq1d, &T)) return fail(HYDRO_ERR_ARG);
  std::vector<double> packed;
  pack_tables(T, packed);
  if (desc->order_h1 == 2 && desc->nq1d == 4) {
    // __constant__ copy for the one-thread-per-element 2D kernel and the blocked 3D stages
    static_assert(sizeof(hk::Tab24) == sizeof(double) * (4 + 12 + 12 + 8), "Tab24 layout");
    if (cudaMemcpyToSymbolAsync(hk::c_t24, packed.data(), sizeof(hk::Tab24), 0,
                                cudaMemcpyHostToDevice, s) != cudaSuccess)
      return fail(HYDRO_ERR_CUDA);
  }
  if (desc->order_h1 == 3 && desc->nq1d == 6) {
    // __constant__ copy for the register-blocked 3D stages of force_kernel (Q3/Q2)
    static_assert(sizeof(hk::Tab36) == sizeof(double) * (6 + 24 + 24 + 18), "Tab36 layout");
    if (cudaMemcpyToSymbolAsync(hk::c_t36, packed.data(), sizeof(hk::Tab36), 0,
                                cudaMemcpyHostToDevice, s) != cudaSuccess)
      return fail(HYDRO_ERR_CUDA);
  }
  if (cudaMemcpyAsync(c->tab, packed.data(), sizeof(double) * HYDRO_TAB_DOUBLES, cudaMemcpyHostToDevice, s) !=
      cudaSuccess)
    return fail(HYDRO_ERR_CUDA);
  // status block
  hydro_devstatus hst;
  hst.dt_key = 0xFFF0000000000000ull;  // key(+inf) = bits(+inf) | sign bit
  hst.first_bad = ~0ull;
  hst.nan_flag = 0;
  hst.nan_sticky = 0;
  // node -> slot CSR on the host (setup, untimed): slots of a node ordered by element
  const int64_t E = desc->n_elem, NN = desc->n_nodes, nd = c->nd;
  c->h_elem_nodes.resize((size_t)(E * nd));
  if (cudaMemcpyAsync(c->h_elem_nodes.data(), desc->elem_nodes, sizeof(int32_t) * E * nd,
                      cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return fail(HYDRO_ERR_CUDA);
  std::vector<int32_t> off((size_t)NN + 1, 0), slot((size_t)(E * nd));
  for (int64_t i = 0; i < E * nd; ++i) {
    const int32_t nde = c->h_elem_nodes[(size_t)i];
    if (nde < 0 || nde >= NN) return fail(HYDRO_ERR_ARG);
    off[(size_t)nde + 1]++;
  }
  for (int64_t i = 0; i < NN; ++i) off[(size_t)i + 1] += off[(size_t)i];
  {
    std::vector<int32_t> pos(off.begin(), off.end() - 1);
    for (int64_t i = 0; i < E * nd; ++i) slot[(size_t)i] = pos[(size_t)c->h_elem_nodes[(size_t)i]]++;
  }
  if (cudaMemsetAsync(c->cnt, 0, sizeof(uint32_t) * (size_t)(NN + 1), s) != cudaSuccess ||
      cudaMemcpyAsync(c->st, &hst, sizeof(hst), cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(c->off, off.data(), sizeof(int32_t) * (NN + 1), cudaMemcpyHostToDevice, s) !=
          cudaSuccess ||
      cudaMemcpyAsync(c->slot, slot.data(), sizeof(int32_t) * E * nd, cudaMemcpyHostToDevice, s) !=
          cudaSuccess)
    return fail(HYDRO_ERR_CUDA);
  // m_q = rho0_K detJ0 (density elimination) with the contract formulas
  hk::Params P;
  std::memset(&P, 0, sizeof(P));
  P.n_units = (int32_t)E;
  P.B = 1;
  P.ld_nodes = NN;
  P.elem_nodes = desc->elem_nodes;
  P.x = desc->x0;
  P.rho0 = desc->rho0;
  P.mq_out = c->mq;
  P.st = c->st;
  fill_tables_ptrs(P, c);
  hydro_status r = launch_force(desc->dim, desc->order_h1, hk::MODE_MQ, false, false, false, P, s);
  if (r != HYDRO_OK) return fail(r);
  if (cudaStreamSynchronize(s) != cudaSuccess) return fail(HYDRO_ERR_CUDA);
  *out = c;
  return HYDRO_OK;
}

hydro_status hydro_ctx_destroy(hydro_ctx *ctx) {
  delete ctx;
  return HYDRO_OK;
}

static hydro_status force_common(hydro_ctx *c, int mode, const double *x, const double *v,
                                 const double *e, const double *w, const double *gamma,
                                 hydro_visc visc, hydro_cfl cfl, double *F1, double *FTw,
                                 double *dt, cudaStream_t s, double *S_store = nullptr) {
  if (!c || !x || !v || !e || !gamma) return HYDRO_ERR_ARG;
  if (mode == hk::MODE_FORCE && (!F1 || !FTw)) return HYDRO_ERR_ARG;
  hk::Params P;
  std::memset(&P, 0, sizeof(P));
  P.n_units = (int32_t)c->d.n_elem;
  P.B = 1;
  P.ld_nodes = c->d.n_nodes;
  P.elem_nodes = c->d.elem_nodes;
  P.x = x; P.v = v; P.w = w; P.e = e; P.gamma = gamma; P.mq = c->mq; P.rho0 = c->d.rho0;
  P.q1 = visc.q1; P.q2 = visc.q2; P.alpha = cfl.alpha; P.alpha_mu = cfl.alpha_mu;
  P.visc = visc.enabled;
  P.evec = c->evec;
  P.slot = c->slot;
  P.FTw = FTw;
  P.st = c->st;
  P.anode = c->d.elem_nodes;  // full mode: assembly nodes are the mesh nodes
  P.off = c->off;
  P.cnt = c->cnt;
  P.done = c->cnt + c->d.n_nodes;
  P.F1 = F1;
  P.n_asm = c->d.n_nodes;
  P.dt_out = dt;
  P.S_store = S_store;
  fill_tables_ptrs(P, c);
  hydro_status r = launch_force(c->d.dim, c->d.order_h1, mode, visc.enabled != 0, false, w != nullptr, P, s);
  if (r != HYDRO_OK) return r;
  if (mode == hk::MODE_FORCE)
    return launch_assemble(c->d.dim, c->d.n_nodes, 1, c->off, c->evec, F1, c->st, dt, s);
  CUDA_OK(launch_pdl(hk::finalize_dt_kernel, dim3(1), dim3(32), s, 1, c->st, dt));
  g_launches++;
  return HYDRO_OK;
}

hydro_status hydro_force_full(hydro_ctx *ctx, const double *x, const double *v, const double *e,
                              const double *w, const double *gamma, hydro_visc visc,
                              hydro_cfl cfl, double *F1, double *FTw, double *dt,
                              hydro_stream_t stream) {
  return force_common(ctx, hk::MODE_FORCE, x, v, e, w, gamma, visc, cfl, F1, FTw, dt,
                      (cudaStream_t)stream);
}

hydro_status hydro_dt_estimate(hydro_ctx *ctx, const double *x, const double *v, const double *e,
                               const double *gamma, hydro_visc visc, hydro_cfl cfl, double *dt,
                               hydro_stream_t stream) {
  return force_common(ctx, hk::MODE_DT, x, v, e, nullptr, gamma, visc, cfl, nullptr, nullptr, dt,
                      (cudaStream_t)stream);
}

size_t hydro_force_stress_bytes(const hydro_ctx *c) {
  if (!c) return 0;
  return sizeof(double) * (size_t)c->d.n_elem * c->d.dim * c->d.dim * c->nq;
}

hydro_status hydro_force_full_store(hydro_ctx *ctx, const double *x, const double *v, const double *e,
                                    const double *gamma, hydro_visc visc, hydro_cfl cfl, double *F1,
                                    double *FTw, double *dt, double *S, hydro_stream_t stream) {
  if (!S) return HYDRO_ERR_ARG;
  return force_common(ctx, hk::MODE_FORCE, x, v, e, nullptr, gamma, visc, cfl, F1, FTw, dt,
                      (cudaStream_t)stream, S);
}

hydro_status hydro_force_transpose(hydro_ctx *c, const double *S, const double *w, double *FTw,
                                   hydro_stream_t stream) {
  if (!c || !S || !w || !FTw) return HYDRO_ERR_ARG;
  hk::Params P;
  std::memset(&P, 0, sizeof(P));
  P.n_units = (int32_t)c->d.n_elem;
  P.B = 1;
  P.ld_nodes = c->d.n_nodes;
  P.elem_nodes = c->d.elem_nodes;
  P.x = w;
  P.FTw = FTw;
  P.S_load = S;
  fill_tables_ptrs(P, c);
  return launch_force(c->d.dim, c->d.order_h1, hk::MODE_FTW, false, false, false, P, (cudaStream_t)stream);
}

static hydro_status status_sync_impl(hydro_devstatus *st, int B, cudaStream_t s,
                                     int64_t *first_bad) {
  CUDA_OK(cudaStreamSynchronize(s));
  CUDA_OK(cudaGetLastError());
  std::vector<hydro_devstatus> h((size_t)B);
  CUDA_OK(cudaMemcpy(h.data(), st, sizeof(hydro_devstatus) * B, cudaMemcpyDeviceToHost));
  unsigned long long bad = ~0ull;
  bool nan = false;
  for (auto &x : h) {
    bad = std::min(bad, x.first_bad);
    nan = nan || x.nan_sticky || x.nan_flag;
    x.first_bad = ~0ull;
    x.nan_sticky = 0;
  }
  CUDA_OK(cudaMemcpy(st, h.data(), sizeof(hydro_devstatus) * B, cudaMemcpyHostToDevice));
  if (first_bad) *first_bad = bad == ~0ull ? -1 : (int64_t)bad;
  if (bad != ~0ull) return HYDRO_ERR_TANGLED;
  if (nan) return HYDRO_ERR_NONFINITE;
  return HYDRO_OK;
}

hydro_status hydro_status_sync(hydro_ctx *ctx, hydro_stream_t stream, int64_t *first_bad_elem) {
  if (!ctx) return HYDRO_ERR_ARG;
  return status_sync_impl(ctx->st, 1, (cudaStream_t)stream, first_bad_elem);
}

// ------------------------------------------------------------------------------ ROM
hydro_status hydro_sample_create(hydro_ctx *c, const int32_t *sample_elems, int64_t n_sample,
                                 int B, hydro_sample **out) {
  if (!c || !sample_elems || n_sample <= 0 || B <= 0 || !out) return HYDRO_ERR_ARG;
  *out = nullptr;
  const int64_t E = c->d.n_elem, NN = c->d.n_nodes, nd = c->nd, ne = c->ne;
  for (int64_t i = 0; i < n_sample; ++i) {
    if (sample_elems[i] < 0 || sample_elems[i] >= E) return HYDRO_ERR_ARG;
    if (i && sample_elems[i] <= sample_elems[i - 1]) return HYDRO_ERR_ARG;  // sorted unique
  }
  const int32_t *en = c->h_elem_nodes.data();
  std::vector<char> s0node((size_t)NN, 0), clnode((size_t)NN, 0);
  std::vector<int64_t> s0idx((size_t)E, -1);
  for (int64_t i = 0; i < n_sample; ++i) {
    const int64_t K = sample_elems[i];
    s0idx[(size_t)K] = i;
    for (int a = 0; a < nd; ++a) s0node[(size_t)en[K * nd + a]] = 1;
  }
  hydro_sample *p = new hydro_sample();
  p->ctx = c;
  p->B = B;
  p->n_s0 = n_sample;
  for (int64_t K = 0; K < E; ++K) {
    bool hit = false;
    for (int a = 0; a < nd && !hit; ++a) hit = s0node[(size_t)en[K * nd + a]] != 0;
    if (hit) {
      p->h_closure.push_back((int32_t)K);
      for (int a = 0; a < nd; ++a) clnode[(size_t)en[K * nd + a]] = 1;
    }
  }
  std::vector<int64_t> local((size_t)NN, -1), s0local((size_t)NN, -1);
  for (int64_t i = 0; i < NN; ++i) {
    if (clnode[(size_t)i]) { local[(size_t)i] = (int64_t)p->h_cl_nodes.size(); p->h_cl_nodes.push_back(i); }
    if (s0node[(size_t)i]) { s0local[(size_t)i] = (int64_t)p->h_s0_nodes.size(); p->h_s0_nodes.push_back(i); }
  }
  p->n_cl = (int64_t)p->h_closure.size();
  p->n_cl_nodes = (int64_t)p->h_cl_nodes.size();
  p->n_s0_nodes = (int64_t)p->h_s0_nodes.size();
  // local tables; slots (CSR over S0 nodes, ordered by closure element)
  std::vector<int32_t> len((size_t)(p->n_cl * nd)), gid((size_t)p->n_cl), frow((size_t)p->n_cl),
      slot((size_t)(p->n_cl * nd), -1), off((size_t)p->n_s0_nodes + 1, 0),
      anode((size_t)(p->n_cl * nd), -1);
  for (int64_t l = 0; l < p->n_cl; ++l) {
    const int64_t K = p->h_closure[(size_t)l];
    gid[(size_t)l] = (int32_t)K;
    frow[(size_t)l] = (int32_t)s0idx[(size_t)K];
    for (int a = 0; a < nd; ++a) {
      const int32_t g = en[K * nd + a];
      len[(size_t)(l * nd + a)] = (int32_t)local[(size_t)g];
      anode[(size_t)(l * nd + a)] = (int32_t)s0local[(size_t)g];
      if (s0local[(size_t)g] >= 0) off[(size_t)s0local[(size_t)g] + 1]++;
    }
  }
  for (int64_t i = 0; i < p->n_s0_nodes; ++i) off[(size_t)i + 1] += off[(size_t)i];
  p->n_slots = off[(size_t)p->n_s0_nodes];
  {
    std::vector<int32_t> pos(off.begin(), off.end() - 1);
    for (int64_t l = 0; l < p->n_cl; ++l)
      for (int a = 0; a < nd; ++a) {
        const int64_t sl = s0local[(size_t)en[(int64_t)p->h_closure[(size_t)l] * nd + a]];
        if (sl >= 0) slot[(size_t)(l * nd + a)] = pos[(size_t)sl]++;
      }
  }
  (void)ne;
  std::vector<int32_t> s0el((size_t)(p->n_s0 > 0 ? p->n_s0 : 1), 0);
  for (int64_t l = 0; l < p->n_cl; ++l)
    if (frow[(size_t)l] >= 0) s0el[(size_t)frow[(size_t)l]] = (int32_t)l;
  auto fail = [&](hydro_status st) { hydro_sample_destroy(p); return st; };
  const size_t evec_bytes = sizeof(double) * (size_t)p->n_slots * c->d.dim * B;
  if (cudaMalloc(&p->elem_nodes, sizeof(int32_t) * len.size()) != cudaSuccess ||
      cudaMalloc(&p->elem_gid, sizeof(int32_t) * gid.size()) != cudaSuccess ||
      cudaMalloc(&p->ftw_row, sizeof(int32_t) * frow.size()) != cudaSuccess ||
      cudaMalloc(&p->slot, sizeof(int32_t) * slot.size()) != cudaSuccess ||
      cudaMalloc(&p->off, sizeof(int32_t) * off.size()) != cudaSuccess ||
      cudaMalloc(&p->evec, evec_bytes > 0 ? evec_bytes : 8) != cudaSuccess ||
      cudaMalloc(&p->st, sizeof(hydro_devstatus) * B) != cudaSuccess ||
      cudaMalloc(&p->anode, sizeof(int32_t) * anode.size()) != cudaSuccess ||
      cudaMalloc(&p->s0_elem, sizeof(int32_t) * s0el.size()) != cudaSuccess ||
      cudaMalloc(&p->cnt, sizeof(uint32_t) * (size_t)(p->n_s0_nodes * B + 1)) != cudaSuccess ||
      cudaMemset(p->cnt, 0, sizeof(uint32_t) * (size_t)(p->n_s0_nodes * B + 1)) != cudaSuccess)
    return fail(HYDRO_ERR_CUDA);
  std::vector<hydro_devstatus> hst((size_t)B);
  for (auto &h : hst) { h.dt_key = 0xFFF0000000000000ull; h.first_bad = ~0ull; h.nan_flag = 0; h.nan_sticky = 0; }
  if (cudaMemcpy(p->elem_nodes, len.data(), sizeof(int32_t) * len.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->elem_gid, gid.data(), sizeof(int32_t) * gid.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->ftw_row, frow.data(), sizeof(int32_t) * frow.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->slot, slot.data(), sizeof(int32_t) * slot.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->off, off.data(), sizeof(int32_t) * off.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->anode, anode.data(), sizeof(int32_t) * anode.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->s0_elem, s0el.data(), sizeof(int32_t) * s0el.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->st, hst.data(), sizeof(hydro_devstatus) * B, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(HYDRO_ERR_CUDA);
  *out = p;
  return HYDRO_OK;
}

hydro_status hydro_sample_destroy(hydro_sample *p) {
  if (!p) return HYDRO_OK;
  cudaFree(p->elem_nodes); cudaFree(p->elem_gid); cudaFree(p->ftw_row); cudaFree(p->slot);
  cudaFree(p->off); cudaFree(p->evec); cudaFree(p->st); cudaFree(p->anode); cudaFree(p->cnt);
  cudaFree(p->s0_elem);
  delete p;
  return HYDRO_OK;
}

hydro_status hydro_sample_info(const hydro_sample *p, int64_t *n_closure_elem,
                               int64_t *n_closure_nodes, int64_t *n_s0_nodes, int64_t *s_v,
                               int64_t *s_e) {
  if (!p) return HYDRO_ERR_ARG;
  if (n_closure_elem) *n_closure_elem = p->n_cl;
  if (n_closure_nodes) *n_closure_nodes = p->n_cl_nodes;
  if (n_s0_nodes) *n_s0_nodes = p->n_s0_nodes;
  if (s_v) *s_v = p->n_s0_nodes * p->ctx->d.dim;
  if (s_e) *s_e = p->n_s0 * p->ctx->ne;
  return HYDRO_OK;
}

hydro_status hydro_sample_lists(const hydro_sample *p, int32_t *closure_elems,
                                int64_t *closure_nodes, int64_t *s0_nodes) {
  if (!p) return HYDRO_ERR_ARG;
  if (closure_elems) std::copy(p->h_closure.begin(), p->h_closure.end(), closure_elems);
  if (closure_nodes) std::copy(p->h_cl_nodes.begin(), p->h_cl_nodes.end(), closure_nodes);
  if (s0_nodes) std::copy(p->h_s0_nodes.begin(), p->h_s0_nodes.end(), s0_nodes);
  return HYDRO_OK;
}

static hydro_status sampled_common(hydro_sample *p, const double *x_S, const double *v_S,
                                   const double *e_S, const double *w_S, const double *gamma,
                                   hydro_visc visc, hydro_cfl cfl, double *F1_rows,
                                   double *FTw_rows, double *dt, hydro_stream_t stream,
                                   double *S_store) {
  if (!p || !x_S || !v_S || !e_S || !gamma || !F1_rows || !FTw_rows) return HYDRO_ERR_ARG;
  hydro_ctx *c = p->ctx;
  cudaStream_t s = (cudaStream_t)stream;
  hk::Params P;
  std::memset(&P, 0, sizeof(P));
  if (p->n_cl * (int64_t)p->B >= ((int64_t)1 << 31)) return HYDRO_ERR_ARG;
  P.n_units = (int32_t)(p->n_cl * p->B);
  P.B = p->B;
  P.ld_nodes = p->n_cl_nodes;
  P.elem_nodes = p->elem_nodes;
  P.elem_gid = p->elem_gid;
  P.x = x_S; P.v = v_S; P.w = w_S; P.e = e_S; P.gamma = gamma; P.mq = c->mq; P.rho0 = c->d.rho0;
  P.q1 = visc.q1; P.q2 = visc.q2; P.alpha = cfl.alpha; P.alpha_mu = cfl.alpha_mu;
  P.visc = visc.enabled;
  P.evec = p->evec;
  P.slot = p->slot;
  P.FTw = FTw_rows;
  P.ftw_row = p->ftw_row;
  P.st = p->st;
  P.anode = p->anode;
  P.off = p->off;
  P.cnt = p->cnt;
  P.done = p->cnt + p->n_s0_nodes * p->B;
  P.F1 = F1_rows;
  P.n_asm = p->n_s0_nodes;
  P.dt_out = dt;
  P.S_store = S_store;
  fill_tables_ptrs(P, c);
  hydro_status r = launch_force(c->d.dim, c->d.order_h1, hk::MODE_FORCE, visc.enabled != 0, p->B > 1,
                                w_S != nullptr, P, s);
  if (r != HYDRO_OK) return r;
  return launch_assemble(c->d.dim, p->n_s0_nodes, p->B, p->off, p->evec, F1_rows, p->st, dt, s);
}

hydro_status hydro_force_sampled(hydro_sample *p, const double *x_S, const double *v_S,
                                 const double *e_S, const double *w_S, const double *gamma,
                                 hydro_visc visc, hydro_cfl cfl, double *F1_rows,
                                 double *FTw_rows, double *dt, hydro_stream_t stream) {
  return sampled_common(p, x_S, v_S, e_S, w_S, gamma, visc, cfl, F1_rows, FTw_rows, dt, stream,
                        nullptr);
}

size_t hydro_sample_stress_bytes(const hydro_sample *p) {
  if (!p) return 0;
  const hydro_ctx *c = p->ctx;
  // only the S0 elements' point stresses are kept: F^T w is needed at their L2 rows only
  return sizeof(double) * (size_t)(p->n_s0 > 0 ? p->n_s0 : 1) * p->B * c->d.dim * c->d.dim * c->nq;
}

hydro_status hydro_force_sampled_store(hydro_sample *p, const double *x_S, const double *v_S,
                                       const double *e_S, const double *gamma, hydro_visc visc,
                                       hydro_cfl cfl, double *F1_rows, double *FTw_rows, double *dt,
                                       double *S, hydro_stream_t stream) {
  if (!S) return HYDRO_ERR_ARG;
  return sampled_common(p, x_S, v_S, e_S, nullptr, gamma, visc, cfl, F1_rows, FTw_rows, dt, stream, S);
}

hydro_status hydro_sample_force_transpose(hydro_sample *p, const double *S, const double *w_S,
                                          double *FTw_rows, hydro_stream_t stream) {
  if (!p || !S || !w_S || !FTw_rows) return HYDRO_ERR_ARG;
  hydro_ctx *c = p->ctx;
  if (p->n_cl * (int64_t)p->B >= ((int64_t)1 << 31)) return HYDRO_ERR_ARG;
  hk::Params P;
  std::memset(&P, 0, sizeof(P));
  if (p->n_s0 == 0) return HYDRO_OK;
  P.n_units = (int32_t)(p->n_s0 * p->B);  // units: (S0 row, instance)
  P.B = p->B;
  P.ld_nodes = p->n_cl_nodes;
  P.elem_nodes = p->elem_nodes;
  P.elem_gid = p->elem_gid;
  P.unit_elem = p->s0_elem;
  P.x = w_S;
  P.FTw = FTw_rows;
  P.S_load = S;
  fill_tables_ptrs(P, c);
  return launch_force(c->d.dim, c->d.order_h1, hk::MODE_FTW, false, p->B > 1, false, P,
                      (cudaStream_t)stream);
}

hydro_status hydro_sample_status_sync(hydro_sample *p, hydro_stream_t stream,
                                      int64_t *first_bad_elem) {
  if (!p) return HYDRO_ERR_ARG;
  return status_sync_impl(p->st, p->B, (cudaStream_t)stream, first_bad_elem);
}

}  // extern "C"

namespace {

template <int NKS, int WM, int MINB>
hydro_status launch_lift_mma_t(int64_t rows, int n, int B, const double *Phi, const double *os, int os_batched,
                               const double *Y, double *out, cudaStream_t s) {
  static std::atomic<int> sms{0};
  if (sms.load() == 0) {
    int dev = 0, v = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    sms.store(v);
  }
  constexpr int RT = 8 * 8 * WM;
  const int64_t tiles = (rows + RT - 1) / RT;
  const int64_t g = std::min<int64_t>(tiles, (int64_t)sms.load() * MINB);   // persistent CTAs
  dim3 grid((unsigned)g, (unsigned)((B + 63) / 64));
  hk::lift_mma_kernel<NKS, WM, MINB><<<grid, hk::LIFT_MMA_THREADS, 0, s>>>(rows, n, B, Phi, os, os_batched, Y, out);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

template <int NKS>
hydro_status launch_lift_mma(int64_t rows, int n, int B, const double *Phi, const double *os, int os_batched,
                             const double *Y, double *out, cudaStream_t s) {
  return os_batched ? launch_lift_mma_t<NKS, 1, 4>(rows, n, B, Phi, os, os_batched, Y, out, s)
                    : launch_lift_mma_t<NKS, 2, 2>(rows, n, B, Phi, os, os_batched, Y, out, s);
}

template <int MT, bool P8>
hydro_status launch_project_mma3(int n, int64_t s_rows, int B, int G, int64_t chunk, const double *P,
                                 const double *f, double *part, double *r, cudaStream_t s) {
  constexpr size_t smem = sizeof(double) * hk::PROJ3_PS *
                          (MT * 8 * hk::PROJ3_SPS + hk::PROJ3_PK * hk::PROJ3_SFS);
  static std::atomic<unsigned long long> attr_done{0};
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_done.load() & bit)) {
    CUDA_OK(cudaFuncSetAttribute(hk::project_mma3_kernel<MT, P8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_done.fetch_or(bit);
  }
  hk::project_mma3_kernel<MT, P8><<<G, 256, smem, s>>>(n, s_rows, B, chunk, P, f, part);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  const int nB = n * B;
  hk::project_mma_reduce_kernel<<<(nB + hk::PROJ_RED_OUT - 1) / hk::PROJ_RED_OUT, 256, 0, s>>>(nB, G, part, r);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

template <int MT, bool AT = false>
hydro_status launch_project_mma(int n, int64_t s_rows, int B, int G, int64_t chunk, const double *P,
                                const double *f, double *part, double *r, cudaStream_t s,
                                int64_t lda = -1, int64_t ldf = -1) {
  constexpr size_t smem = sizeof(double) * 4 * MT * 4 * 2 * 32;
  static std::atomic<unsigned long long> attr_done{0};
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_done.load() & bit)) {
    CUDA_OK(cudaFuncSetAttribute(hk::project_mma_kernel<MT, AT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_done.fetch_or(bit);
  }
  hk::project_mma_kernel<MT, AT><<<G, hk::PROJ_MMA_THREADS, smem, s>>>(
      n, s_rows, B, chunk, P, lda >= 0 ? lda : s_rows, f, ldf >= 0 ? ldf : B, part);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  const int nB = n * B;
  hk::project_mma_reduce_kernel<<<(nB + hk::PROJ_RED_OUT - 1) / hk::PROJ_RED_OUT, 256, 0, s>>>(nB, G, part, r);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

}  // namespace

extern "C" {

hydro_status hydro_rom_lift(int64_t rows, int n, int B, const double *Phi, const double *os,
                            int os_batched, const double *Y, double *out, hydro_stream_t stream) {
  if (rows < 0 || n <= 0 || n > 256 || B <= 0) return HYDRO_ERR_ARG;
  if (rows == 0) return HYDRO_OK;   // nothing to lift (the row pointers may be NULL)
  if (!Phi || !os || !Y || !out) return HYDRO_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  // the FP64 tensor-pipe kernel (n <= 64); os/out rows of 16-byte aligned pairs
  const bool aligned = ((uintptr_t)out % 16 == 0) && (!os_batched || (uintptr_t)os % 16 == 0) && B % 2 == 0;
  if (aligned && n <= 64) {
    const int nks = (n + 3) / 4;
    if (nks <= 2) return launch_lift_mma<2>(rows, n, B, Phi, os, os_batched, Y, out, st);
    if (nks <= 4) return launch_lift_mma<4>(rows, n, B, Phi, os, os_batched, Y, out, st);
    if (nks <= 8) return launch_lift_mma<8>(rows, n, B, Phi, os, os_batched, Y, out, st);
    if (nks <= 10) return launch_lift_mma<10>(rows, n, B, Phi, os, os_batched, Y, out, st);
    return launch_lift_mma<16>(rows, n, B, Phi, os, os_batched, Y, out, st);
  }
  // the FMA kernel stages Y's column block and the Phi rows: (n LIFT_CB + LIFT_RT (n + 1))
  // doubles, up to the device's opt-in maximum (n <= 224 on B200)
  const size_t smem = sizeof(double) * (size_t)(n * hk::LIFT_CB + hk::LIFT_RT * (n + 1));
  static std::atomic<unsigned long long> attr_done{0};
  if (smem > 48 * 1024) {
    int dev = 0, optin = 0;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (smem > (size_t)optin) return HYDRO_ERR_ARG;
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
      CUDA_OK(cudaFuncSetAttribute(hk::lift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
      attr_done.fetch_or(bit);
    }
  }
  dim3 grid((unsigned)((rows + hk::LIFT_RT - 1) / hk::LIFT_RT), (unsigned)((B + hk::LIFT_CB - 1) / hk::LIFT_CB));
  hk::lift_kernel<<<grid, hk::LIFT_THREADS, smem, st>>>(rows, n, B, Phi, os, os_batched, Y, out);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

// split-K groups of the projection: the tensor-pipe kernel (n <= 40, B <= 64) uses up to
// 2 CTAs per SM with >= 128 rows each; the fallback up to 8 per SM with >= 256 rows each
static int project_groups(int n, int64_t s_rows, int B) {
  const bool mma = n <= 40 && B <= 64;
  int64_t g = mma ? (s_rows + 127) / 128 : (s_rows + 255) / 256;
  const int64_t cap = mma ? 148 * std::max(2, hk::PROJ3_MINB) : 148 * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

size_t hydro_rom_project_workspace_bytes(int n, int64_t s_rows, int B) {
  if (n <= 0 || B <= 0 || s_rows < 0) return 0;
  return sizeof(double) * (size_t)project_groups(n, s_rows, B) * n * B;
}

hydro_status hydro_rom_project(int n, int64_t s_rows, int B, const double *P, const double *f,
                               double *r, void *workspace, size_t ws_bytes, hydro_stream_t stream) {
  if (n <= 0 || n > hk::PROJ_MAXN || B <= 0 || B > hk::PROJ_MAXB || s_rows < 0 || !r)
    return HYDRO_ERR_ARG;
  if (s_rows == 0)   // an empty sample: the empty sum (P and f may be NULL)
    return cudaMemsetAsync(r, 0, sizeof(double) * (size_t)n * B, (cudaStream_t)stream) == cudaSuccess
               ? HYDRO_OK : HYDRO_ERR_CUDA;
  if (!P || !f) return HYDRO_ERR_ARG;
  const int G = project_groups(n, s_rows, B);
  if (!workspace || ws_bytes < sizeof(double) * (size_t)G * n * B) return HYDRO_ERR_WORKSPACE;
  int64_t chunk = std::max<int64_t>((s_rows + G - 1) / G, 1);
  cudaStream_t s = (cudaStream_t)stream;
  double *part = (double *)workspace;
  if (n <= 40 && B % 2 == 0 && ((uintptr_t)P % 16) == 0 && ((uintptr_t)f % 16) == 0) {
    constexpr int PK = hk::PROJ3_PK;
    chunk = (chunk + PK - 1) / PK * PK;
    const int G3 = (int)((s_rows + chunk - 1) / chunk);
    const int mt = (n + 7) / 8;
#define HK_P3(MT)                                                                      \
  return s_rows % 2 ? launch_project_mma3<MT, true>(n, s_rows, B, G3, chunk, P, f, part, r, s) \
                    : launch_project_mma3<MT, false>(n, s_rows, B, G3, chunk, P, f, part, r, s)
    if (mt == 1) HK_P3(1);
    if (mt == 2) HK_P3(2);
    if (mt == 3) HK_P3(3);
    if (mt == 4) HK_P3(4);
    HK_P3(5);
#undef HK_P3
  }
  if (n <= 40) {
    const int mt = (n + 7) / 8;
    if (mt == 1) return launch_project_mma<1>(n, s_rows, B, G, chunk, P, f, part, r, s);
    if (mt == 2) return launch_project_mma<2>(n, s_rows, B, G, chunk, P, f, part, r, s);
    if (mt == 3) return launch_project_mma<3>(n, s_rows, B, G, chunk, P, f, part, r, s);
    if (mt == 4) return launch_project_mma<4>(n, s_rows, B, G, chunk, P, f, part, r, s);
    return launch_project_mma<5>(n, s_rows, B, G, chunk, P, f, part, r, s);
  }
  hk::project_partial_kernel<<<G, hk::PROJ_THREADS, 0, s>>>(n, s_rows, B, chunk, P, f, part);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  hk::project_reduce_kernel<<<(n * B + 255) / 256, 256, 0, s>>>(n, B, G, part, r);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}


// ------------------------------------------------------------------------------ FOM step
}  // extern "C"

struct hydro_fom {
  hydro_ctx *c = nullptr;
  int64_t n = 0;  // dim * n_nodes
  double *mask = nullptr, *dinv = nullptr, *Minv = nullptr, *csum = nullptr, *wm = nullptr;
  double *Mblk = nullptr;  // M_E,K blocks (hydro_mass_e_apply)
  double *r = nullptr, *z = nullptr, *p = nullptr, *Ap = nullptr, *part = nullptr, *sc = nullptr;
  double *F1 = nullptr, *F1x = nullptr, *FTw = nullptr, *FTx = nullptr, *dv = nullptr;
  double *vh = nullptr, *eh = nullptr, *xh = nullptr, *v1 = nullptr, *vbar = nullptr,
         *dts = nullptr, *S = nullptr;
  double *xb = nullptr, *vb = nullptr, *eb = nullptr;  // state backup of the step controller
  bool have_dv = false;  // dv holds the previous solve's solution (warm start of the step's CG)
  std::vector<void *> allocs;
  double *colbuf = nullptr;  // mass_columns' transpose scratch, grown on demand (freed on destroy)
  size_t colbuf_doubles = 0;
};

namespace {

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <int DIM, int K, int Q>
hydro_status mass_apply_t(hydro_fom *f, const double *in, double *out, const double *mask, int mode,
                          int invert, cudaStream_t s) {
  hydro_ctx *c = f->c;
  hk::MassParams P;
  P.n_elem = (int32_t)c->d.n_elem;
  P.n_nodes = c->d.n_nodes;
  P.elem_nodes = c->d.elem_nodes;
  P.slot = c->slot;
  P.mq = c->mq;
  P.in = in;
  P.evec = c->evec;
  P.mode = mode;
  P.tab_w = c->tab;
  P.tab_B = c->tab + Q;
  constexpr int NT = DIM == 3 ? (Q == 4 ? 64 : 224) : 64;
  hk::mass_apply_kernel<DIM, K, Q><<<(unsigned)c->d.n_elem, NT, 0, s>>>(P);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  hk::assemble_masked_kernel<DIM><<<blocks_for(c->d.n_nodes, 256), 256, 0, s>>>(
      c->d.n_nodes, c->off, c->evec, mask, out, invert);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

// Element part of M_V in (contributions into the context's slot buffer), 3D Q2 fast kernel
// or the generic one.
hydro_status mass_apply_elements(hydro_fom *f, const double *in, cudaStream_t s) {
  const hydro_mesh_desc &d = f->c->d;
  hydro_ctx *c = f->c;
  if (d.dim == 3 && d.order_h1 == 2 && f->wm) {
    const int64_t threads = d.n_elem * 3 * 4;
    hk::mass_apply3_q2_kernel<<<blocks_for(threads, 256), 256, 0, s>>>(
        (int32_t)d.n_elem, d.n_nodes, d.elem_nodes, c->slot, f->wm, in, c->evec);
    g_launches++;
    CUDA_OK(cudaGetLastError());
    return HYDRO_OK;
  }
  hk::MassParams P;
  P.n_elem = (int32_t)d.n_elem;
  P.n_nodes = d.n_nodes;
  P.elem_nodes = d.elem_nodes;
  P.slot = c->slot;
  P.mq = c->mq;
  P.in = in;
  P.evec = c->evec;
  P.mode = 0;
  P.tab_w = c->tab;
  P.tab_B = c->tab + d.nq1d;
  if (d.dim == 2 && d.order_h1 == 2) hk::mass_apply_kernel<2, 2, 4><<<(unsigned)d.n_elem, 64, 0, s>>>(P);
  else if (d.dim == 3 && d.order_h1 == 2) hk::mass_apply_kernel<3, 2, 4><<<(unsigned)d.n_elem, 64, 0, s>>>(P);
  else if (d.dim == 2 && d.order_h1 == 3) hk::mass_apply_kernel<2, 3, 6><<<(unsigned)d.n_elem, 64, 0, s>>>(P);
  else hk::mass_apply_kernel<3, 3, 6><<<(unsigned)d.n_elem, 224, 0, s>>>(P);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

hydro_status mass_apply(hydro_fom *f, const double *in, double *out, const double *mask, int mode,
                        int invert, cudaStream_t s) {
  const hydro_mesh_desc &d = f->c->d;
  if (mode == 0 && d.dim == 3 && d.order_h1 == 2 && f->wm) {
    hydro_ctx *c = f->c;
    const int64_t threads = d.n_elem * 3 * 4;
    hk::mass_apply3_q2_kernel<<<blocks_for(threads, 256), 256, 0, s>>>(
        (int32_t)d.n_elem, d.n_nodes, d.elem_nodes, c->slot, f->wm, in, c->evec);
    g_launches++;
    CUDA_OK(cudaGetLastError());
    hk::assemble_masked_kernel<3><<<blocks_for(d.n_nodes, 256), 256, 0, s>>>(d.n_nodes, c->off, c->evec,
                                                                             mask, out, invert);
    g_launches++;
    CUDA_OK(cudaGetLastError());
    return HYDRO_OK;
  }
  if (d.dim == 2 && d.order_h1 == 2) return mass_apply_t<2, 2, 4>(f, in, out, mask, mode, invert, s);
  if (d.dim == 3 && d.order_h1 == 2) return mass_apply_t<3, 2, 4>(f, in, out, mask, mode, invert, s);
  if (d.dim == 2 && d.order_h1 == 3) return mass_apply_t<2, 3, 6>(f, in, out, mask, mode, invert, s);
  if (d.dim == 3 && d.order_h1 == 3) return mass_apply_t<3, 3, 6>(f, in, out, mask, mode, invert, s);
  return HYDRO_ERR_UNSUPPORTED;
}

hydro_status dot(hydro_fom *f, int64_t n, const double *a, const double *b, double *out,
                 cudaStream_t s) {
  hk::dot_partial_kernel<<<hk::DOT_BLOCKS, hk::DOT_THREADS, 0, s>>>(n, a, b, f->part);
  hk::dot_final_kernel<<<1, 256, 0, s>>>(f->part, out);
  g_launches += 2;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

hydro_status mass_e_update(hydro_fom *f, const double *a, const double *rhs, double scale,
                           double *out, cudaStream_t s, const double *blocks = nullptr) {
  const double *Mb = blocks ? blocks : f->Minv;
  const hydro_ctx *c = f->c;
  const int ne = c->ne;
  const int64_t n = c->d.n_elem * ne;
  const unsigned g = blocks_for(n, 256);
  const int32_t E = (int32_t)c->d.n_elem;
  if (ne == 4) hk::mass_e_update_kernel<4><<<g, 256, 0, s>>>(E, Mb, a, rhs, scale, out);
  else if (ne == 8) hk::mass_e_update_kernel<8><<<g, 256, 0, s>>>(E, Mb, a, rhs, scale, out);
  else if (ne == 9) hk::mass_e_update_kernel<9><<<g, 256, 0, s>>>(E, Mb, a, rhs, scale, out);
  else if (ne == 27) hk::mass_e_update_kernel<27><<<g, 256, 0, s>>>(E, Mb, a, rhs, scale, out);
  else return HYDRO_ERR_UNSUPPORTED;
  g_launches++;
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

// PCG with the Jacobi preconditioner on the free dofs.  Stops when the preconditioned
// residual norm relative to the right-hand side's, sqrt(r.z / b.D^-1 b), is <= tol.
// warm: x holds the initial guess (constrained components zero), else x0 = 0 -- the two
// coincide in their first residual when x = 0.
hydro_status pcg(hydro_fom *f, const double *b, double *x, double tol, int max_iter, int *iters,
                 double *relres, cudaStream_t s, bool warm = false) {
  const int64_t n = f->n;
  const unsigned g = blocks_for(n, 256);
  // r = mask b, z = D^-1 r (= p), x = 0; the reference norm b.D^-1 b is r.z of this state
  hk::cg_init_kernel<<<g, 256, 0, s>>>(n, b, f->mask, f->dinv, warm ? f->Ap : x, f->r, f->z, f->p);
  g_launches++;
  CUDA_OK(cudaGetLastError());
  hydro_status st = dot(f, n, f->r, f->z, f->sc + 5, s);
  if (st != HYDRO_OK) return st;
  if (warm) {
    // r = mask (b - M x), z = D^-1 r, p = z
    const hydro_mesh_desc &d = f->c->d;
    if ((st = mass_apply_elements(f, x, s)) != HYDRO_OK) return st;
    if (d.dim == 3)
      hk::assemble_dot_kernel<3><<<hk::DOT_BLOCKS, hk::DOT_THREADS, 0, s>>>(
          d.n_nodes, f->c->off, f->c->evec, f->mask, x, f->Ap, f->part);
    else
      hk::assemble_dot_kernel<2><<<hk::DOT_BLOCKS, hk::DOT_THREADS, 0, s>>>(
          d.n_nodes, f->c->off, f->c->evec, f->mask, x, f->Ap, f->part);
    hk::cg_residual_kernel<<<g, 256, 0, s>>>(n, f->Ap, f->dinv, f->r, f->z, f->p);
    g_launches += 2;
    CUDA_OK(cudaGetLastError());
  }
  if ((st = dot(f, n, f->r, f->z, f->sc + 0, s)) != HYDRO_OK) return st;
  double h[6];
  CUDA_OK(cudaMemcpyAsync(h, f->sc, 6 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  const double rz0 = h[0], bz = h[5];
  int it = 0;
  double rel = bz > 0.0 ? sqrt(rz0 / bz) : 0.0;
  if (rz0 > 0.0 && rel > tol) {
    rel = 1.0;
    const hydro_mesh_desc &d = f->c->d;
    while (it < max_iter) {
      // Ap = M p (element kernel into the slots, then fused masked assembly + p.Ap partials)
      if ((st = mass_apply_elements(f, f->p, s)) != HYDRO_OK) return st;
      if (d.dim == 3)
        hk::assemble_dot_kernel<3><<<hk::DOT_BLOCKS, hk::DOT_THREADS, 0, s>>>(
            d.n_nodes, f->c->off, f->c->evec, f->mask, f->p, f->Ap, f->part);
      else
        hk::assemble_dot_kernel<2><<<hk::DOT_BLOCKS, hk::DOT_THREADS, 0, s>>>(
            d.n_nodes, f->c->off, f->c->evec, f->mask, f->p, f->Ap, f->part);
      // r.z alternates between sc[0] and sc[8] (read by all CTAs / written by one: fom.cuh)
      const int rz_in = (it & 1) ? 8 : 0, rz_out = (it & 1) ? 0 : 8;
      hk::cg_xr_dot_fused_kernel<<<hk::DOT_BLOCKS, hk::DOT_THREADS, 0, s>>>(
          n, f->sc, rz_in, f->part, f->p, f->Ap, f->dinv, x, f->r, f->z, f->part + hk::DOT_BLOCKS);
      hk::cg_p_fused_kernel<<<hk::DOT_BLOCKS, hk::DOT_THREADS, 0, s>>>(n, f->sc, rz_in, rz_out,
                                                                      f->part + hk::DOT_BLOCKS, f->z, f->p);
      g_launches += 3;
      CUDA_OK(cudaGetLastError());
      ++it;
      if (it % 4 == 0 || it == max_iter) {
        double rz = 0.0;
        CUDA_OK(cudaMemcpyAsync(&rz, f->sc + rz_out, sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        rel = sqrt(rz / bz);
        if (!(rel > tol)) break;
      }
    }
  }
  if (iters) *iters = it;
  if (relres) *relres = rel;
  return HYDRO_OK;
}

}  // namespace

extern "C" {

hydro_status hydro_fom_create(hydro_ctx *c, const int64_t *bc_dofs, int64_t n_bc,
                              hydro_stream_t stream, hydro_fom **out) {
  if (!c || !out || n_bc < 0 || (n_bc > 0 && !bc_dofs)) return HYDRO_ERR_ARG;
  *out = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  hydro_fom *f = new hydro_fom();
  f->c = c;
  const int dim = c->d.dim;
  const int64_t NN = c->d.n_nodes, E = c->d.n_elem, ne = c->ne;
  f->n = dim * NN;
  std::vector<double> mask((size_t)f->n, 1.0);
  for (int64_t i = 0; i < n_bc; ++i) {
    if (bc_dofs[i] < 0 || bc_dofs[i] >= f->n) { delete f; return HYDRO_ERR_ARG; }
    mask[(size_t)bc_dofs[i]] = 0.0;
  }
  auto fail = [&](hydro_status st) { hydro_fom_destroy(f); return st; };
  auto alloc = [&](double **ptr, size_t count) {
    void *q = nullptr;
    if (cudaMalloc(&q, sizeof(double) * (count > 0 ? count : 1)) != cudaSuccess) return false;
    f->allocs.push_back(q);
    *ptr = (double *)q;
    return true;
  };
  const size_t n = (size_t)f->n, nE = (size_t)(E * ne);
  if (!alloc(&f->mask, n) || !alloc(&f->dinv, n) || !alloc(&f->Minv, nE * ne) ||
      !alloc(&f->csum, nE) || !alloc(&f->r, n) || !alloc(&f->z, n) || !alloc(&f->p, n) ||
      !alloc(&f->Ap, n) || !alloc(&f->part, 2 * hk::DOT_BLOCKS) || !alloc(&f->sc, 16) ||
      !alloc(&f->F1, n) || !alloc(&f->F1x, n) || !alloc(&f->FTw, nE) || !alloc(&f->FTx, nE) ||
      !alloc(&f->dv, n) || !alloc(&f->vh, n) || !alloc(&f->eh, nE) || !alloc(&f->xh, n) ||
      !alloc(&f->v1, n) || !alloc(&f->vbar, n) || !alloc(&f->dts, 2) ||
      !alloc(&f->xb, n) || !alloc(&f->vb, n) || !alloc(&f->eb, nE) ||
      !alloc(&f->S, hydro_force_stress_bytes(c) / sizeof(double)) || !alloc(&f->Mblk, nE * (size_t)c->ne))
    return fail(HYDRO_ERR_CUDA);
  if (cudaMemcpyAsync(f->mask, mask.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return fail(HYDRO_ERR_CUDA);
  if (dim == 3 && c->d.order_h1 == 2) {
    // w_q m_q for the register-resident 3D Q2 mass kernel, and its constant table
    const int64_t nq = 64;
    if (!alloc(&f->wm, (size_t)(E * nq))) return fail(HYDRO_ERR_CUDA);
    hk::wm_setup_kernel<<<blocks_for(E * nq, 256), 256, 0, s>>>(E, 4, 3, c->tab, c->mq, f->wm);
    g_launches++;
    double hB[12];
    if (cudaMemcpyAsync(hB, c->tab + 4, sizeof(hB), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess ||
        cudaMemcpyToSymbolAsync(hk::c_mB24, hB, sizeof(hB), 0, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return fail(HYDRO_ERR_CUDA);
  }
  // Jacobi preconditioner: 1 / diag(M_V) on the free dofs, 0 on the constrained ones
  hydro_status st = mass_apply(f, nullptr, f->dinv, f->mask, 1, 1, s);
  if (st != HYDRO_OK) return fail(st);
  // M_E,K^{-1} and the internal-energy weights
  const int q = c->d.nq1d, nn = c->d.order_h1 + 1;
  const double *tw = c->tab, *tBl = c->tab + q + 2 * q * nn;
  const unsigned g = blocks_for(E, 64);
  if (dim == 2 && c->d.order_h1 == 2)
    hk::mass_e_setup_kernel<2, 2, 4><<<g, 64, 0, s>>>((int32_t)E, c->mq, tw, tBl, f->Minv, f->csum, f->Mblk);
  else if (dim == 3 && c->d.order_h1 == 2)
    hk::mass_e_setup_kernel<3, 2, 4><<<g, 64, 0, s>>>((int32_t)E, c->mq, tw, tBl, f->Minv, f->csum, f->Mblk);
  else if (dim == 2 && c->d.order_h1 == 3)
    hk::mass_e_setup_kernel<2, 3, 6><<<g, 64, 0, s>>>((int32_t)E, c->mq, tw, tBl, f->Minv, f->csum, f->Mblk);
  else
    hk::mass_e_setup_kernel<3, 3, 6><<<g, 64, 0, s>>>((int32_t)E, c->mq, tw, tBl, f->Minv, f->csum, f->Mblk);
  g_launches++;
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return fail(HYDRO_ERR_CUDA);
  *out = f;
  return HYDRO_OK;
}

hydro_status hydro_fom_destroy(hydro_fom *f) {
  if (!f) return HYDRO_OK;
  for (void *q : f->allocs) cudaFree(q);
  cudaFree(f->colbuf);
  delete f;
  return HYDRO_OK;
}

hydro_status hydro_mass_v_apply(hydro_fom *f, const double *in, double *out, hydro_stream_t stream) {
  if (!f || !in || !out) return HYDRO_ERR_ARG;
  return mass_apply(f, in, out, nullptr, 0, 0, (cudaStream_t)stream);
}

hydro_status hydro_mass_v_solve(hydro_fom *f, const double *rhs, double *sol, double rel_tol,
                                int max_iter, int *iters, double *relres, hydro_stream_t stream) {
  if (!f || !rhs || !sol || max_iter < 0 || !(rel_tol >= 0.0)) return HYDRO_ERR_ARG;
  return pcg(f, rhs, sol, rel_tol, max_iter, iters, relres, (cudaStream_t)stream);
}

hydro_status hydro_mass_e_solve(hydro_fom *f, const double *rhs, double *sol, hydro_stream_t stream) {
  if (!f || !rhs || !sol) return HYDRO_ERR_ARG;
  hydro_status st;
  cudaStream_t s = (cudaStream_t)stream;
  // sol = 0 + 1 * Minv rhs  (the zero vector: FTx scratch cleared first)
  const size_t nE = (size_t)(f->c->d.n_elem * f->c->ne);
  CUDA_OK(cudaMemsetAsync(f->FTx, 0, sizeof(double) * nE, s));
  if ((st = mass_e_update(f, f->FTx, rhs, 1.0, sol, s)) != HYDRO_OK) return st;
  return HYDRO_OK;
}

hydro_status hydro_mass_e_apply(hydro_fom *f, const double *in, double *out, hydro_stream_t stream) {
  if (!f || !in || !out) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nE = (size_t)(f->c->d.n_elem * f->c->ne);
  CUDA_OK(cudaMemsetAsync(f->FTx, 0, sizeof(double) * nE, s));
  return mass_e_update(f, f->FTx, in, 1.0, out, s, f->Mblk);
}

hydro_status hydro_fom_energy(hydro_fom *f, const double *v, const double *e, double *kinetic,
                              double *internal, hydro_stream_t stream) {
  if (!f || !v || !e) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  hydro_status st;
  if ((st = mass_apply(f, v, f->Ap, nullptr, 0, 0, s)) != HYDRO_OK) return st;
  if ((st = dot(f, f->n, v, f->Ap, f->sc + 6, s)) != HYDRO_OK) return st;
  if ((st = dot(f, f->c->d.n_elem * f->c->ne, f->csum, e, f->sc + 7, s)) != HYDRO_OK) return st;
  double h[2];
  CUDA_OK(cudaMemcpyAsync(h, f->sc + 6, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  if (kinetic) *kinetic = 0.5 * h[0];
  if (internal) *internal = h[1];
  return HYDRO_OK;
}

hydro_status hydro_rk2avg_step(hydro_fom *f, double *x, double *v, double *e, const double *gamma,
                               hydro_visc visc, hydro_cfl cfl, double dt, double cg_tol,
                               int cg_max_iter, double *dt_est, int *cg_iters,
                               hydro_stream_t stream) {
  if (!f || !x || !v || !e || !gamma || !(dt > 0.0)) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  hydro_ctx *c = f->c;
  const int64_t n = f->n, nE = c->d.n_elem * c->ne;
  const unsigned g = blocks_for(n, 256);
  hydro_status st;
  int it1 = 0, it2 = 0;
  double rel1 = 0.0, rel2 = 0.0;
  // ---- stage 1: F(U^n) (F.1, dt, and the point stresses S_q for the transposed product)
  if ((st = force_common(c, hk::MODE_FORCE, x, v, e, nullptr, gamma, visc, cfl, f->F1, f->FTx,
                         f->dts + 0, s, f->S)) != HYDRO_OK) return st;
  // the CG of each stage starts from the previous solve's solution (the accelerations of
  // consecutive stages differ by O(dt)); the stopping test is relative to the rhs either way
  if ((st = pcg(f, f->F1, f->dv, cg_tol, cg_max_iter, &it1, &rel1, s, f->have_dv)) != HYDRO_OK)
    return st;
  f->have_dv = true;
  hk::axpy_kernel<<<g, 256, 0, s>>>(n, v, -0.5 * dt, f->dv, f->mask, f->vh);    // v^{n+1/2}
  g_launches++;
  if ((st = hydro_force_transpose(c, f->S, f->vh, f->FTw, stream)) != HYDRO_OK) return st;  // F(U^n)^T v^{n+1/2}
  if ((st = mass_e_update(f, e, f->FTw, 0.5 * dt, f->eh, s)) != HYDRO_OK) return st;
  hk::axpy_kernel<<<g, 256, 0, s>>>(n, x, 0.5 * dt, f->vh, nullptr, f->xh);    // x^{n+1/2}
  g_launches++;
  // ---- stage 2: F(U^{n+1/2})
  if ((st = force_common(c, hk::MODE_FORCE, f->xh, f->vh, f->eh, nullptr, gamma, visc, cfl, f->F1,
                         f->FTx, f->dts + 1, s, f->S)) != HYDRO_OK) return st;
  if ((st = pcg(f, f->F1, f->dv, cg_tol, cg_max_iter, &it2, &rel2, s, true)) != HYDRO_OK) return st;
  hk::axpy_kernel<<<g, 256, 0, s>>>(n, v, -dt, f->dv, f->mask, f->v1);         // v^{n+1}
  hk::avg_kernel<<<g, 256, 0, s>>>(n, v, f->v1, f->vbar);                       // vbar
  g_launches += 2;
  if ((st = hydro_force_transpose(c, f->S, f->vbar, f->FTw, stream)) != HYDRO_OK) return st;  // F(U^{n+1/2})^T vbar
  if ((st = mass_e_update(f, e, f->FTw, dt, e, s)) != HYDRO_OK) return st;     // e^{n+1}
  hk::axpy_kernel<<<g, 256, 0, s>>>(n, x, dt, f->vbar, nullptr, x);            // x^{n+1}
  g_launches++;
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaMemcpyAsync(v, f->v1, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  double h[2];
  CUDA_OK(cudaMemcpyAsync(h, f->dts, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  // min of the stage estimates, NaN if either is NaN (or a CG residual is: an invalid state)
  const bool nan = h[0] != h[0] || h[1] != h[1] || rel1 != rel1 || rel2 != rel2;
  if (dt_est) *dt_est = nan ? std::numeric_limits<double>::quiet_NaN() : std::fmin(h[0], h[1]);
  if (cg_iters) *cg_iters = it1 + it2;
  (void)nE;
  if (!nan && (rel1 > cg_tol || rel2 > cg_tol)) return HYDRO_ERR_NOT_CONVERGED;
  return HYDRO_OK;
}


// Per-instance validity of the last evaluation(s) since the previous read (tangled element or
// non-finite estimate), then the status words are reset: a rejected trial step must not
// leave its condition behind.  bad[b] = 1 for an invalid instance.
static hydro_status read_reset_status(hydro_devstatus *st, int B, cudaStream_t s,
                                      std::vector<char> &bad) {
  std::vector<hydro_devstatus> h((size_t)B);
  CUDA_OK(cudaMemcpyAsync(h.data(), st, sizeof(hydro_devstatus) * B, cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  bad.assign((size_t)B, 0);
  bool any = false;
  for (int b = 0; b < B; ++b) {
    hydro_devstatus &x = h[(size_t)b];
    if (x.first_bad != ~0ull || x.nan_sticky || x.nan_flag) { bad[(size_t)b] = 1; any = true; }
    x.first_bad = ~0ull;
    x.nan_sticky = 0;
  }
  if (any) {
    CUDA_OK(cudaMemcpyAsync(st, h.data(), sizeof(hydro_devstatus) * B, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaStreamSynchronize(s));
  }
  return HYDRO_OK;
}

hydro_status hydro_fom_advance(hydro_fom *f, double *x, double *v, double *e, const double *gamma,
                               hydro_visc visc, hydro_cfl cfl, hydro_dt_ctrl ctrl, double t0,
                               double t_final, double *dt, int max_steps, double cg_tol,
                               int cg_max_iter, double *t_out, int *steps, int *rejected,
                               hydro_stream_t stream) {
  if (!f || !x || !v || !e || !gamma || !dt || !(*dt > 0.0) || !(t_final >= t0) || max_steps < 0 ||
      !(ctrl.beta1 > 0.0 && ctrl.beta1 < 1.0) || !(ctrl.beta2 >= 1.0) || !(ctrl.gamma > 0.0))
    return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = f->n, nE = f->c->d.n_elem * f->c->ne;
  double t = t0, h = *dt;
  int ns = 0, nr = 0;
  hydro_status st = HYDRO_OK;
  // (1) advance with dt, get the estimate; (2) dt >= estimate: dt <- beta1 dt,
  // redo the step from the saved state; (3) dt <= gamma * estimate: dt <- beta2 dt; (4) next.
  // The step that reaches t_final is shortened to land on it.
  while (t < t_final && ns < max_steps) {
    const double h_try = (t_final - t < h) ? t_final - t : h;
    CUDA_OK(cudaMemcpyAsync(f->xb, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemcpyAsync(f->vb, v, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemcpyAsync(f->eb, e, sizeof(double) * nE, cudaMemcpyDeviceToDevice, s));
    double est = 0.0;
    if ((st = hydro_rk2avg_step(f, x, v, e, gamma, visc, cfl, h_try, cg_tol, cg_max_iter, &est,
                                nullptr, stream)) != HYDRO_OK)
      break;
    std::vector<char> bad;
    if ((st = read_reset_status(f->c->st, 1, s, bad)) != HYDRO_OK) break;
#ifdef HYDRO_DEBUG_ADV
    fprintf(stderr, "adv t=%.17g h_try=%.17g est=%.17g bad=%d ns=%d nr=%d\n", t, h_try, est, (int)bad[0], ns, nr);
#endif
    // rejected (too large, or invalid: tangled / NaN estimate, DESIGN R26): restore, retry
    if (bad[0] || !(est == est) || h_try >= est) {
      CUDA_OK(cudaMemcpyAsync(x, f->xb, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      CUDA_OK(cudaMemcpyAsync(v, f->vb, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      CUDA_OK(cudaMemcpyAsync(e, f->eb, sizeof(double) * nE, cudaMemcpyDeviceToDevice, s));
      h = ctrl.beta1 * h_try;
      ++nr;
      if (nr > 10000) { st = HYDRO_ERR_NONFINITE; break; }  // no admissible step found
      continue;
    }
    t = (h_try == t_final - t) ? t_final : t + h_try;
    ++ns;
    h = (h_try <= ctrl.gamma * est) ? ctrl.beta2 * h_try : h_try;
  }
  CUDA_OK(cudaStreamSynchronize(s));
  *dt = h;
  if (t_out) *t_out = t;
  if (steps) *steps = ns;
  if (rejected) *rejected = nr;
  return st;
}

hydro_status hydro_fom_stage_state(hydro_fom *f, double *x_half, double *v_half, double *e_half,
                                   hydro_stream_t stream) {
  if (!f) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = f->n, nE = f->c->d.n_elem * f->c->ne;
  if (x_half) CUDA_OK(cudaMemcpyAsync(x_half, f->xh, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  if (v_half) CUDA_OK(cudaMemcpyAsync(v_half, f->vh, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  if (e_half) CUDA_OK(cudaMemcpyAsync(e_half, f->eh, sizeof(double) * nE, cudaMemcpyDeviceToDevice, s));
  return HYDRO_OK;
}

// ------------------------------------------------------------------------------ ROM step
}  // extern "C"

struct hydro_rom {
  hydro_sample *p = nullptr;
  int B = 0, nx = 0, nv = 0, ne = 0, os_flags = 0;
  int64_t rows_h1 = 0, rows_l2 = 0, s_v = 0, s_e = 0;
  const double *Phi_x = nullptr, *Phi_v = nullptr, *Phi_e = nullptr;
  const double *x_os = nullptr, *v_os = nullptr, *e_os = nullptr;
  const double *R_v = nullptr, *R_e = nullptr, *C_xv = nullptr, *c_x = nullptr;
  double *xS = nullptr, *vS = nullptr, *eS = nullptr, *wS = nullptr, *F1r = nullptr,
         *F1x = nullptr, *FTr = nullptr, *FTx = nullptr, *rv = nullptr, *re = nullptr,
         *rx = nullptr, *Yv_h = nullptr, *Ye_h = nullptr, *Yx_h = nullptr, *Yv1 = nullptr,
         *Yvb = nullptr, *dt1 = nullptr, *dt2 = nullptr, *wsv = nullptr, *wse = nullptr,
         *S = nullptr;
  double *Yxb = nullptr, *Yvb_ = nullptr, *Yeb = nullptr, *hdev = nullptr, *est = nullptr,
         *keep = nullptr;  // step-controller state (backup of the reduced coordinates)
  size_t wsv_bytes = 0, wse_bytes = 0;
  std::vector<void *> allocs;
};

extern "C" {

hydro_status hydro_rom_create(hydro_sample *p, int nx, int nv, int ne, const double *Phi_x_S,
                              const double *Phi_v_S, const double *Phi_e_S, const double *x_os_S,
                              const double *v_os_S, const double *e_os_S, int os_batched_flags,
                              const double *R_v, const double *R_e, const double *C_xv,
                              const double *c_x, hydro_rom **out) {
  if (!p || !out || nx <= 0 || nv <= 0 || ne <= 0 || nx > 256 || nv > hk::PROJ_MAXN ||
      ne > hk::PROJ_MAXN || nv > 256 || !Phi_x_S || !Phi_v_S || !Phi_e_S || !x_os_S || !v_os_S ||
      !e_os_S || !R_v || !R_e || !C_xv || !c_x || p->B > hk::PROJ_MAXB)
    return HYDRO_ERR_ARG;
  *out = nullptr;
  hydro_rom *r = new hydro_rom();
  r->p = p;
  r->B = p->B;
  r->nx = nx; r->nv = nv; r->ne = ne;
  r->os_flags = os_batched_flags;
  const hydro_ctx *c = p->ctx;
  r->rows_h1 = (int64_t)c->d.dim * p->n_cl_nodes;
  r->rows_l2 = p->n_cl * c->ne;
  r->s_v = p->n_s0_nodes * c->d.dim;
  r->s_e = p->n_s0 * c->ne;
  r->Phi_x = Phi_x_S; r->Phi_v = Phi_v_S; r->Phi_e = Phi_e_S;
  r->x_os = x_os_S; r->v_os = v_os_S; r->e_os = e_os_S;
  r->R_v = R_v; r->R_e = R_e; r->C_xv = C_xv; r->c_x = c_x;
  auto fail = [&](hydro_status st) { hydro_rom_destroy(r); return st; };
  auto alloc = [&](double **ptr, size_t count) {
    void *q = nullptr;
    if (cudaMalloc(&q, sizeof(double) * (count > 0 ? count : 1)) != cudaSuccess) return false;
    r->allocs.push_back(q);
    *ptr = (double *)q;
    return true;
  };
  const size_t B = (size_t)r->B, h1 = (size_t)r->rows_h1 * B, l2 = (size_t)r->rows_l2 * B;
  r->wsv_bytes = hydro_rom_project_workspace_bytes(nv, r->s_v, r->B);
  r->wse_bytes = hydro_rom_project_workspace_bytes(ne, r->s_e, r->B);
  if (!alloc(&r->xS, h1) || !alloc(&r->vS, h1) || !alloc(&r->eS, l2) || !alloc(&r->wS, h1) ||
      !alloc(&r->F1r, (size_t)r->s_v * B) || !alloc(&r->F1x, (size_t)r->s_v * B) ||
      !alloc(&r->FTr, (size_t)r->s_e * B) || !alloc(&r->FTx, (size_t)r->s_e * B) ||
      !alloc(&r->rv, (size_t)nv * B) || !alloc(&r->re, (size_t)ne * B) || !alloc(&r->rx, (size_t)nx * B) ||
      !alloc(&r->Yv_h, (size_t)nv * B) || !alloc(&r->Ye_h, (size_t)ne * B) ||
      !alloc(&r->Yx_h, (size_t)nx * B) || !alloc(&r->Yv1, (size_t)nv * B) ||
      !alloc(&r->Yvb, (size_t)nv * B) || !alloc(&r->dt1, B) || !alloc(&r->dt2, B) ||
      !alloc(&r->wsv, r->wsv_bytes / 8 + 1) || !alloc(&r->wse, r->wse_bytes / 8 + 1) ||
      !alloc(&r->Yxb, (size_t)nx * B) || !alloc(&r->Yvb_, (size_t)nv * B) ||
      !alloc(&r->Yeb, (size_t)ne * B) || !alloc(&r->hdev, B) || !alloc(&r->est, B) ||
      !alloc(&r->keep, B) ||
      !alloc(&r->S, hydro_sample_stress_bytes(p) / sizeof(double)))
    return fail(HYDRO_ERR_CUDA);
  *out = r;
  return HYDRO_OK;
}

hydro_status hydro_rom_destroy(hydro_rom *r) {
  if (!r) return HYDRO_OK;
  for (void *q : r->allocs) cudaFree(q);
  delete r;
  return HYDRO_OK;
}

hydro_status hydro_rom_rk2avg_step(hydro_rom *r, double *Yx, double *Yv, double *Ye,
                                   const double *gamma, hydro_visc visc, hydro_cfl cfl,
                                   const double *dt, double *dt_est, hydro_stream_t stream) {
  if (!r || !Yx || !Yv || !Ye || !gamma || !dt) return HYDRO_ERR_ARG;
  const int B = r->B;
  hydro_status st;
  auto lift = [&](const double *Phi, const double *os, int batched, int64_t rows, int n,
                  const double *Y, double *o) {
    return hydro_rom_lift(rows, n, B, Phi, os, batched, Y, o, stream);
  };
  auto proj = [&](const double *P, int n, int64_t s_rows, const double *f, double *o, double *ws,
                  size_t wsb) {
    return hydro_rom_project(n, s_rows, B, P, f, o, ws, wsb, stream);
  };
  auto axpy = [&](int64_t n, const double *a, double sc, const double *rr, double *o) {
    hk::rom_axpy_kernel<<<blocks_for(n * B, 256), 256, 0, (cudaStream_t)stream>>>(n, B, a, sc, dt, rr, o);
    g_launches++;
    return cudaGetLastError() == cudaSuccess ? HYDRO_OK : HYDRO_ERR_CUDA;
  };
  const int fx = r->os_flags & 1, fv = (r->os_flags >> 1) & 1, fe = (r->os_flags >> 2) & 1;
  const int fc = (r->os_flags >> 3) & 1;   // c_x per instance ([nx][B]: previous-window offsets)
#define RS(call) do { if ((st = (call)) != HYDRO_OK) return st; } while (0)
  // ---- stage 1 at the lifted U~^n
  RS(lift(r->Phi_x, r->x_os, fx, r->rows_h1, r->nx, Yx, r->xS));
  RS(lift(r->Phi_v, r->v_os, fv, r->rows_h1, r->nv, Yv, r->vS));
  RS(lift(r->Phi_e, r->e_os, fe, r->rows_l2, r->ne, Ye, r->eS));
  RS(hydro_force_sampled_store(r->p, r->xS, r->vS, r->eS, gamma, visc, cfl, r->F1r, r->FTx, r->dt1, r->S, stream));
  RS(proj(r->R_v, r->nv, r->s_v, r->F1r, r->rv, r->wsv, r->wsv_bytes));
  RS(axpy(r->nv, Yv, -0.5, r->rv, r->Yv_h));                                   // vhat^{n+1/2}
  RS(lift(r->Phi_v, r->v_os, fv, r->rows_h1, r->nv, r->Yv_h, r->wS));          // v~^{n+1/2}
  RS(hydro_sample_force_transpose(r->p, r->S, r->wS, r->FTr, stream));
  RS(proj(r->R_e, r->ne, r->s_e, r->FTr, r->re, r->wse, r->wse_bytes));
  RS(axpy(r->ne, Ye, 0.5, r->re, r->Ye_h));                                    // ehat^{n+1/2}
  RS(lift(r->C_xv, r->c_x, fc, r->nx, r->nv, r->Yv_h, r->rx));                 // c_x + C_xv vhat
  RS(axpy(r->nx, Yx, 0.5, r->rx, r->Yx_h));                                    // xhat^{n+1/2}
  // ---- stage 2 at U~^{n+1/2} (its velocity is wS)
  RS(lift(r->Phi_x, r->x_os, fx, r->rows_h1, r->nx, r->Yx_h, r->xS));
  RS(lift(r->Phi_e, r->e_os, fe, r->rows_l2, r->ne, r->Ye_h, r->eS));
  RS(hydro_force_sampled_store(r->p, r->xS, r->wS, r->eS, gamma, visc, cfl, r->F1r, r->FTx, r->dt2, r->S, stream));
  RS(proj(r->R_v, r->nv, r->s_v, r->F1r, r->rv, r->wsv, r->wsv_bytes));
  RS(axpy(r->nv, Yv, -1.0, r->rv, r->Yv1));                                    // vhat^{n+1}
  hk::avg_kernel<<<blocks_for((int64_t)r->nv * B, 256), 256, 0, (cudaStream_t)stream>>>(
      (int64_t)r->nv * B, Yv, r->Yv1, r->Yvb);
  g_launches++;
  RS(lift(r->Phi_v, r->v_os, fv, r->rows_h1, r->nv, r->Yvb, r->vS));           // v~bar
  RS(hydro_sample_force_transpose(r->p, r->S, r->vS, r->FTr, stream));
  RS(proj(r->R_e, r->ne, r->s_e, r->FTr, r->re, r->wse, r->wse_bytes));
  RS(axpy(r->ne, Ye, 1.0, r->re, Ye));                                         // ehat^{n+1}
  RS(lift(r->C_xv, r->c_x, fc, r->nx, r->nv, r->Yvb, r->rx));
  RS(axpy(r->nx, Yx, 1.0, r->rx, Yx));                                         // xhat^{n+1}
  CUDA_OK(cudaMemcpyAsync(Yv, r->Yv1, sizeof(double) * (size_t)r->nv * B, cudaMemcpyDeviceToDevice,
                          (cudaStream_t)stream));
  if (dt_est) {
    hk::min2_kernel<<<blocks_for(B, 128), 128, 0, (cudaStream_t)stream>>>(B, r->dt1, r->dt2, dt_est);
    g_launches++;
  }
#undef RS
  CUDA_OK(cudaGetLastError());
  return HYDRO_OK;
}

hydro_status hydro_rom_advance(hydro_rom *r, double *Yx, double *Yv, double *Ye,
                               const double *gamma, hydro_visc visc, hydro_cfl cfl,
                               hydro_dt_ctrl ctrl, double t0, double t_final, double *dt,
                               int max_iters, double *t_out, int *steps, int *rejected,
                               int *iters, hydro_stream_t stream) {
  if (!r || !Yx || !Yv || !Ye || !gamma || !dt || !(t_final >= t0) || max_iters < 0 ||
      !(ctrl.beta1 > 0.0 && ctrl.beta1 < 1.0) || !(ctrl.beta2 >= 1.0) || !(ctrl.gamma > 0.0))
    return HYDRO_ERR_ARG;
  const int B = r->B;
  for (int b = 0; b < B; ++b)
    if (!(dt[b] > 0.0)) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<double> t((size_t)B, t0), h(dt, dt + B), htry((size_t)B), est((size_t)B),
      keep((size_t)B);
  std::vector<int> ns((size_t)B, 0), nr((size_t)B, 0);
  int it = 0;
  hydro_status st = HYDRO_OK;
  const size_t bx = sizeof(double) * (size_t)r->nx * B, bv = sizeof(double) * (size_t)r->nv * B,
               be = sizeof(double) * (size_t)r->ne * B;
  // PAPER P:549-566 per instance (each instance is an independent simulation): instances
  // step together with their own trial dt; a rejected instance (dt >= its estimate) is
  // restored from the copy and retried with beta1*dt; finished instances ride along with a
  // zero step and are restored too, so their coordinates stay bit-identical.
  while (it < max_iters) {
    bool any = false;
    for (int b = 0; b < B; ++b) {
      const bool act = t[(size_t)b] < t_final;
      any = any || act;
      htry[(size_t)b] = act ? ((t_final - t[(size_t)b] < h[(size_t)b]) ? t_final - t[(size_t)b]
                                                                       : h[(size_t)b])
                            : 0.0;
    }
    if (!any) break;
    CUDA_OK(cudaMemcpyAsync(r->Yxb, Yx, bx, cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemcpyAsync(r->Yvb_, Yv, bv, cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemcpyAsync(r->Yeb, Ye, be, cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemcpyAsync(r->hdev, htry.data(), sizeof(double) * B, cudaMemcpyHostToDevice, s));
    if ((st = hydro_rom_rk2avg_step(r, Yx, Yv, Ye, gamma, visc, cfl, r->hdev, r->est, stream)) !=
        HYDRO_OK)
      break;
    CUDA_OK(cudaMemcpyAsync(est.data(), r->est, sizeof(double) * B, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    std::vector<char> bad;
    if ((st = read_reset_status(r->p->st, B, s, bad)) != HYDRO_OK) break;
    ++it;
    for (int b = 0; b < B; ++b) {
      const size_t i = (size_t)b;
      keep[i] = 0.0;
      if (htry[i] == 0.0) continue;  // finished instance
      if (bad[i] || !(est[i] == est[i]) || htry[i] >= est[i]) {  // too large or invalid (R26)
        if (nr[i] >= 10000) st = HYDRO_ERR_NONFINITE;               // no admissible step found
        h[i] = ctrl.beta1 * htry[i];
        ++nr[i];
        continue;
      }
      keep[i] = 1.0;
      t[i] = (htry[i] == t_final - t[i]) ? t_final : t[i] + htry[i];
      ++ns[i];
      h[i] = (htry[i] <= ctrl.gamma * est[i]) ? ctrl.beta2 * htry[i] : htry[i];
    }
    CUDA_OK(cudaMemcpyAsync(r->keep, keep.data(), sizeof(double) * B, cudaMemcpyHostToDevice, s));
    hk::rom_select_kernel<<<blocks_for((int64_t)r->nx * B, 256), 256, 0, s>>>(r->nx, B, r->keep, r->Yxb, Yx);
    hk::rom_select_kernel<<<blocks_for((int64_t)r->nv * B, 256), 256, 0, s>>>(r->nv, B, r->keep, r->Yvb_, Yv);
    hk::rom_select_kernel<<<blocks_for((int64_t)r->ne * B, 256), 256, 0, s>>>(r->ne, B, r->keep, r->Yeb, Ye);
    g_launches += 3;
    CUDA_OK(cudaGetLastError());
    if (st != HYDRO_OK) break;
  }
  CUDA_OK(cudaStreamSynchronize(s));
  for (int b = 0; b < B; ++b) {
    dt[b] = h[(size_t)b];
    if (t_out) t_out[b] = t[(size_t)b];
    if (steps) steps[b] = ns[(size_t)b];
    if (rejected) rejected[b] = nr[(size_t)b];
  }
  if (iters) *iters = it;
  return st;
}

}  // extern "C"

// ------------------------------------------------------------------------------ offline (NEXT-3)
namespace {

// Symmetric eigen-decomposition of a small dense matrix (host): Householder reduction to
// tridiagonal form with the reflections accumulated, then the implicit-shift QL iteration on
// the tridiagonal with the rotations applied to the accumulated basis (O(n^3); the cyclic
// Jacobi used before took ~6 ms for the 64 x 64 snapshot Gram matrix).  A [n][n] row-major in,
// eigenvalues lam[n] descending, eigenvectors V [n][n] (column c = eigenvector c), each with
// its largest-magnitude component positive.  Backward stable: eigenvalue errors ~ n eps ||A||.
void sym_eig_host(int n, std::vector<double> A, std::vector<double> &lam, std::vector<double> &V) {
  auto a = [&](int i, int j) -> double & { return A[(size_t)i * n + j]; };
  V.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
  auto z = [&](int i, int j) -> double & { return V[(size_t)i * n + j]; };
  std::vector<double> d((size_t)n), e((size_t)n, 0.0), v((size_t)n), pv((size_t)n);
  // Householder: for column k, reflect A[k+1:, k] onto a multiple of e_{k+1}; A <- H A H, Z <- Z H
  for (int k = 0; k + 2 < n; ++k) {
    double nx = 0.0;
    for (int i = k + 1; i < n; ++i) nx += a(i, k) * a(i, k);
    nx = std::sqrt(nx);
    if (nx == 0.0) continue;
    const double x0 = a(k + 1, k);
    const double alpha = x0 >= 0.0 ? -nx : nx;
    for (int i = 0; i <= k; ++i) v[(size_t)i] = 0.0;
    for (int i = k + 1; i < n; ++i) v[(size_t)i] = a(i, k);
    v[(size_t)k + 1] -= alpha;
    double vv = 0.0;
    for (int i = k + 1; i < n; ++i) vv += v[(size_t)i] * v[(size_t)i];
    if (vv == 0.0) continue;
    const double beta = 2.0 / vv;
    // p = beta A v, q = p - (beta v^T p / 2) v, A <- A - v q^T - q v^T (rows/cols >= k)
    double vp = 0.0;
    for (int i = k; i < n; ++i) {
      double acc = 0.0;
      for (int j = k + 1; j < n; ++j) acc += a(i, j) * v[(size_t)j];
      pv[(size_t)i] = beta * acc;
      vp += v[(size_t)i] * pv[(size_t)i];
    }
    const double kk = 0.5 * beta * vp;
    for (int i = k; i < n; ++i) pv[(size_t)i] -= kk * v[(size_t)i];
    for (int i = k; i < n; ++i)
      for (int j = k; j < n; ++j) a(i, j) -= v[(size_t)i] * pv[(size_t)j] + pv[(size_t)i] * v[(size_t)j];
    for (int i = 0; i < n; ++i) {  // Z <- Z (I - beta v v^T)
      double acc = 0.0;
      for (int j = k + 1; j < n; ++j) acc += z(i, j) * v[(size_t)j];
      acc *= beta;
      for (int j = k + 1; j < n; ++j) z(i, j) -= acc * v[(size_t)j];
    }
  }
  for (int i = 0; i < n; ++i) d[(size_t)i] = a(i, i);
  for (int i = 0; i + 1 < n; ++i) e[(size_t)i] = a(i + 1, i);   // e[i]: between i and i+1
  // implicit-shift QL on (d, e); e[n-1] = 0
  const double eps = std::numeric_limits<double>::epsilon();
  for (int l = 0; l < n; ++l) {
    for (int iter = 0; iter < 60; ++iter) {
      int m = l;
      for (; m < n - 1; ++m) {
        const double dd = std::fabs(d[(size_t)m]) + std::fabs(d[(size_t)m + 1]);
        if (std::fabs(e[(size_t)m]) <= eps * dd) break;
      }
      if (m == l) break;
      double g = (d[(size_t)l + 1] - d[(size_t)l]) / (2.0 * e[(size_t)l]);
      double r = std::hypot(g, 1.0);
      g = d[(size_t)m] - d[(size_t)l] + e[(size_t)l] / (g + (g >= 0.0 ? r : -r));
      double sn = 1.0, c = 1.0, p = 0.0;
      int i = m - 1;
      bool deflated = false;
      for (; i >= l; --i) {
        const double f = sn * e[(size_t)i], b = c * e[(size_t)i];
        r = std::hypot(f, g);
        e[(size_t)i + 1] = r;
        if (r == 0.0) {  // underflow: the subdiagonal split
          d[(size_t)i + 1] -= p;
          e[(size_t)m] = 0.0;
          deflated = true;
          break;
        }
        sn = f / r;
        c = g / r;
        g = d[(size_t)i + 1] - p;
        r = (d[(size_t)i] - g) * sn + 2.0 * c * b;
        p = sn * r;
        d[(size_t)i + 1] = g + p;
        g = c * r - b;
        for (int k = 0; k < n; ++k) {
          const double zf = z(k, i + 1);
          z(k, i + 1) = sn * z(k, i) + c * zf;
          z(k, i) = c * z(k, i) - sn * zf;
        }
      }
      if (deflated) continue;
      d[(size_t)l] -= p;
      e[(size_t)l] = g;
      e[(size_t)m] = 0.0;
    }
  }
  for (int i = 0; i < n; ++i) a(i, i) = d[(size_t)i];
  std::vector<int> order((size_t)n);
  for (int i = 0; i < n; ++i) order[(size_t)i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return a(x, x) > a(y, y); });
  std::vector<double> Vs((size_t)n * n);
  lam.resize((size_t)n);
  for (int c = 0; c < n; ++c) {
    const int o = order[(size_t)c];
    lam[(size_t)c] = a(o, o);
    int imax = 0;
    for (int k = 1; k < n; ++k)
      if (std::fabs(V[(size_t)k * n + o]) > std::fabs(V[(size_t)imax * n + o])) imax = k;
    const double sg = V[(size_t)imax * n + o] < 0.0 ? -1.0 : 1.0;
    for (int k = 0; k < n; ++k) Vs[(size_t)k * n + c] = sg * V[(size_t)k * n + o];
  }
  V.swap(Vs);
}

// Solve A x = b (n x n, row-major) by LU with partial pivoting (host; DEIM's small systems).
bool lu_solve_host(int n, std::vector<double> A, std::vector<double> &b) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(A[(size_t)i * n + k]) > std::fabs(A[(size_t)p * n + k])) p = i;
    if (A[(size_t)p * n + k] == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A[(size_t)k * n + j], A[(size_t)p * n + j]);
      std::swap(b[(size_t)k], b[(size_t)p]);
    }
    for (int i = k + 1; i < n; ++i) {
      const double l = A[(size_t)i * n + k] / A[(size_t)k * n + k];
      for (int j = k; j < n; ++j) A[(size_t)i * n + j] -= l * A[(size_t)k * n + j];
      b[(size_t)i] -= l * b[(size_t)k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double acc = b[(size_t)i];
    for (int j = i + 1; j < n; ++j) acc -= A[(size_t)i * n + j] * b[(size_t)j];
    b[(size_t)i] = acc / A[(size_t)i * n + i];
  }
  return true;
}

// Least squares min |A x - b|_2 (rows x n, row-major, rows >= n) by Householder QR (host; the
// oversampled greedy's small gappy fits).  x = first n entries of b on return.
bool lstsq_host(int rows, int n, std::vector<double> A, std::vector<double> &b) {
  for (int k = 0; k < n; ++k) {
    double nrm = 0.0;
    for (int i = k; i < rows; ++i) nrm += A[(size_t)i * n + k] * A[(size_t)i * n + k];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) return false;
    const double a = A[(size_t)k * n + k] > 0 ? -nrm : nrm;   // R_kk
    std::vector<double> w((size_t)rows, 0.0);
    for (int i = k; i < rows; ++i) w[(size_t)i] = A[(size_t)i * n + k];
    w[(size_t)k] -= a;
    double ww = 0.0;
    for (int i = k; i < rows; ++i) ww += w[(size_t)i] * w[(size_t)i];
    if (ww > 0.0) {
      for (int j = k; j < n; ++j) {
        double d = 0.0;
        for (int i = k; i < rows; ++i) d += w[(size_t)i] * A[(size_t)i * n + j];
        const double f = 2.0 * d / ww;
        for (int i = k; i < rows; ++i) A[(size_t)i * n + j] -= f * w[(size_t)i];
      }
      double d = 0.0;
      for (int i = k; i < rows; ++i) d += w[(size_t)i] * b[(size_t)i];
      const double f = 2.0 * d / ww;
      for (int i = k; i < rows; ++i) b[(size_t)i] -= f * w[(size_t)i];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double acc = b[(size_t)i];
    for (int j = i + 1; j < n; ++j) acc -= A[(size_t)i * n + j] * b[(size_t)j];
    if (A[(size_t)i * n + i] == 0.0) return false;
    b[(size_t)i] = acc / A[(size_t)i * n + i];
  }
  return true;
}

// A per-device scratch buffer of the offline routines (split-K partials), kept between calls
// and grown on demand; the routines using it synchronise their stream before returning, and
// the lock serialises host threads for the duration of a call.
struct Scratch {
  std::mutex mu;
  double *p[64] = {};
  size_t n[64] = {};
  double *get(size_t need) {  // call with mu held
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    dev &= 63;
    if (n[dev] < need) {
      cudaFree(p[dev]);
      p[dev] = nullptr;
      n[dev] = 0;
      if (cudaMalloc(&p[dev], sizeof(double) * need) != cudaSuccess) return nullptr;
      n[dev] = need;
    }
    return p[dev];
  }
};
Scratch g_gram_scratch;
Scratch g_deim_scratch;   // Q-DEIM / DEIM: transposed basis, norms, pivots
void transpose(int64_t N, int64_t m, const double *A, double *At, cudaStream_t s);

int sm_count() {
  static std::atomic<int> sms{0};
  if (sms.load() == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return 148;
    sms.store(v);
  }
  return sms.load();
}

// G (device [n][n], full) = the Gram matrix of A's n vectors of length N on the FP64 tensor pipe
// (gram_mma_kernel, split-K over ~2 CTAs per SM, fixed-order reduce); synchronous.
// kfast: A(i, k) = A[i * ld + k] (snapshot rows), else A[k * ld + i] (basis columns).
hydro_status gram_mma(int n, int64_t N, int64_t ld, bool kfast, const double *A, double *G, cudaStream_t s) {
  const int tiles = (n + hk::GMMA_T - 1) / hk::GMMA_T;
  const int64_t kblocks = (N + hk::GMMA_KB - 1) / hk::GMMA_KB;
  int64_t chunks = std::max<int64_t>(1, (int64_t)sm_count() * 2 / ((int64_t)tiles * tiles));
  chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, kblocks / 4));
  const int64_t chunk = (kblocks + chunks - 1) / chunks * hk::GMMA_KB;
  chunks = (N + chunk - 1) / chunk;
  std::lock_guard<std::mutex> lk(g_gram_scratch.mu);
  double *part = g_gram_scratch.get((size_t)chunks * n * n);
  if (!part) return HYDRO_ERR_CUDA;
  const dim3 grid((unsigned)chunks, (unsigned)tiles, (unsigned)tiles);
  if (kfast) hk::gram_mma_kernel<true><<<grid, 256, 0, s>>>(n, N, chunk, ld, A, part);
  else hk::gram_mma_kernel<false><<<grid, 256, 0, s>>>(n, N, chunk, ld, A, part);
  const int nn = n * n;
  hk::project_mma_reduce_kernel<<<(nn + hk::PROJ_RED_OUT - 1) / hk::PROJ_RED_OUT, 256, 0, s>>>(nn, (int)chunks, part, G);
  g_launches += 2;
  const bool ok = cudaGetLastError() == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess;
  return ok ? HYDRO_OK : HYDRO_ERR_CUDA;
}

// out[r][c] (row stride ldo) = sum_k A(r, k) Y[k][c], r < rows, c < B <= 64, K <= 64, on the FP64
// tensor pipe (tall_mma_kernel); A(r, k) = at ? A[k * lda + r] : A[r * lda + k].  Asynchronous.
// In place (out == A, !at, ldo == lda) is allowed.
template <bool AT>
hydro_status tall_mma(int64_t rows, int K, int B, const double *A, int64_t lda, const double *Y, double *out,
                      int64_t ldo, cudaStream_t s) {
  if (K <= 0 || K > 64 || B <= 0 || B > 64) return HYDRO_ERR_ARG;
  const int64_t tiles = (rows + 127) / 128;
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count() * 2));
  if (K <= 8) hk::tall_mma_kernel<AT, 2><<<g, 256, 0, s>>>(rows, K, B, A, lda, Y, out, ldo);
  else if (K <= 16) hk::tall_mma_kernel<AT, 4><<<g, 256, 0, s>>>(rows, K, B, A, lda, Y, out, ldo);
  else if (K <= 32) hk::tall_mma_kernel<AT, 8><<<g, 256, 0, s>>>(rows, K, B, A, lda, Y, out, ldo);
  else hk::tall_mma_kernel<AT, 16><<<g, 256, 0, s>>>(rows, K, B, A, lda, Y, out, ldo);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? HYDRO_OK : HYDRO_ERR_CUDA;
}

}  // namespace

extern "C" {

hydro_status hydro_pod(const double *S, int ns, int64_t N, double eps, int max_k, double *Phi,
                       double *sigma, int *k_out, hydro_stream_t stream) {
  if (!S || ns <= 0 || ns > 4096 || N <= 0 || !(eps > 0.0 && eps <= 1.0) || max_k <= 0 ||
      max_k > hk::POD_MAXK || !Phi || !k_out)
    return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int chunks = (int)std::min<int64_t>(hk::GRAM_CHUNKS, (N + hk::GRAM_KT - 1) / hk::GRAM_KT);
  const int64_t chunk = (N + chunks - 1) / chunks;
  const int tiles = (ns + hk::GRAM_T - 1) / hk::GRAM_T;
  double *part = nullptr, *G = nullptr, *W = nullptr;
  hydro_status st = HYDRO_OK;
  auto cleanup = [&]() { cudaFree(part); cudaFree(G); cudaFree(W); };
  if ((!(ns <= 64 && max_k <= 64) && cudaMalloc(&part, sizeof(double) * (size_t)chunks * ns * ns) != cudaSuccess) ||
      cudaMalloc(&G, sizeof(double) * (size_t)ns * ns) != cudaSuccess) {
    cleanup();
    return HYDRO_ERR_CUDA;
  }
  // G = S S^T (the snapshot Gram matrix; S holds one snapshot per row), on the FP64 tensor pipe
  // when the snapshot count allows the tall basis formation below (ns <= 64), else the tiled
  // FMA kernel
  const bool mma = ns <= 64 && max_k <= 64;
  if (mma) {
    if (gram_mma(ns, N, N, true, S, G, s) != HYDRO_OK) { cleanup(); return HYDRO_ERR_CUDA; }
  } else {
    hk::gram_partial_kernel<<<dim3((unsigned)chunks, (unsigned)tiles, (unsigned)tiles), hk::GRAM_T * hk::GRAM_T, 0, s>>>(
        ns, N, chunk, N, 1, S, part);
    hk::gram_reduce_kernel<<<(ns * ns + 255) / 256, 256, 0, s>>>(ns, chunks, part, G);
    g_launches += 2;
  }
  std::vector<double> hG((size_t)ns * ns), lam, V;
  if (cudaGetLastError() != cudaSuccess ||
      cudaMemcpyAsync(hG.data(), G, sizeof(double) * hG.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {
    cleanup();
    return HYDRO_ERR_CUDA;
  }
  // G = V Lambda V^T; singular values of S^T: sigma = sqrt(lambda)
  sym_eig_host(ns, hG, lam, V);
  std::vector<double> sg((size_t)ns);
  double tot = 0.0;
  for (int i = 0; i < ns; ++i) { sg[(size_t)i] = std::sqrt(std::max(lam[(size_t)i], 0.0)); tot += sg[(size_t)i]; }
  if (sigma) std::copy(sg.begin(), sg.end(), sigma);
  // energy criterion: the smallest k with sum_{i<=k} sigma_i / sum sigma_i >= eps
  int k = ns;
  double run = 0.0;
  for (int i = 0; i < ns; ++i) {
    run += sg[(size_t)i];
    if (tot > 0.0 && run / tot >= eps) { k = i + 1; break; }
  }
  if (k > max_k) k = max_k;
  // Directions the Gram route cannot resolve are dropped: lambda_i <= ns eps lambda_1 is
  // rounding noise of S S^T (a rank-deficient snapshot set gives ~1e-16 lambda_1 there, not
  // 0), and S^T v_i / sigma_i would be garbage.  eps = 1 keeps the numerically nonzero ones.
  const double lam_floor = (double)ns * std::numeric_limits<double>::epsilon() * std::max(lam[0], 0.0);
  while (k > 0 && !(lam[(size_t)k - 1] > lam_floor)) --k;
  *k_out = k;
  if (k == 0) { cleanup(); return HYDRO_OK; }
  // Phi = S^T V_k Sigma_k^-1  ([N][k]; the left singular vectors)
  std::vector<double> hW((size_t)ns * k);
  for (int j = 0; j < ns; ++j)
    for (int c = 0; c < k; ++c) hW[(size_t)j * k + c] = V[(size_t)j * ns + c] / sg[(size_t)c];
  if (cudaMalloc(&W, sizeof(double) * hW.size()) != cudaSuccess ||
      cudaMemcpyAsync(W, hW.data(), sizeof(double) * hW.size(), cudaMemcpyHostToDevice, s) != cudaSuccess) {
    cleanup();
    return HYDRO_ERR_CUDA;
  }
  if (mma) {  // Phi = S^T W on the tensor pipe (A read transposed from the snapshot rows)
    if (tall_mma<true>(N, ns, k, S, N, W, Phi, max_k, s) != HYDRO_OK) { cleanup(); return HYDRO_ERR_CUDA; }
  } else {
    hk::snapshot_combine_kernel<<<blocks_for(N, 128), 128, 0, s>>>(ns, N, k, max_k, S, W, Phi);
    g_launches++;
  }
  if (cudaGetLastError() != cudaSuccess) { cleanup(); return HYDRO_ERR_CUDA; }
  // One CholQR pass: the Gram route leaves Phi orthonormal only to ~eps (sigma_1/sigma_k)^2;
  // Phi <- Phi R^-1 with R^T R = Phi^T Phi restores it to rounding (same span).
  {
    double *P2 = nullptr, *Rinv = nullptr, *G2 = nullptr;
    bool chol_fail = false;
    const int ch = (int)std::min<int64_t>(hk::GRAM_CHUNKS, (N + hk::GRAM_KT - 1) / hk::GRAM_KT);
    const int64_t chs = (N + ch - 1) / ch;
    const int kt = (k + hk::GRAM_T - 1) / hk::GRAM_T;
    bool ok = (mma || cudaMalloc(&P2, sizeof(double) * (size_t)ch * k * k) == cudaSuccess) &&
              cudaMalloc(&G2, sizeof(double) * (size_t)k * k) == cudaSuccess &&
              cudaMalloc(&Rinv, sizeof(double) * (size_t)k * k) == cudaSuccess;
    std::vector<double> C((size_t)k * k, 0.0), Ri((size_t)k * k, 0.0);
    if (ok && mma) {  // Phi^T Phi on the tensor pipe (the basis columns)
      ok = gram_mma(k, N, max_k, false, Phi, G2, s) == HYDRO_OK &&
           cudaMemcpyAsync(C.data(), G2, sizeof(double) * C.size(), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
           cudaStreamSynchronize(s) == cudaSuccess;
    } else if (ok) {  // Phi^T Phi: the same tiled Gram kernel on the columns of the row-major basis
      hk::gram_partial_kernel<<<dim3((unsigned)ch, (unsigned)kt, (unsigned)kt), hk::GRAM_T * hk::GRAM_T, 0, s>>>(
          k, N, chs, 1, max_k, Phi, P2);
      hk::gram_reduce_kernel<<<(k * k + 255) / 256, 256, 0, s>>>(k, ch, P2, G2);
      g_launches += 2;
      ok = cudaGetLastError() == cudaSuccess &&
           cudaMemcpyAsync(C.data(), G2, sizeof(double) * C.size(), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
           cudaStreamSynchronize(s) == cudaSuccess;
    }
    if (ok) {
      // upper Cholesky R (C = R^T R), then R^-1 by back substitution
      std::vector<double> R((size_t)k * k, 0.0);
      for (int i = 0; i < k && ok; ++i) {
        double d = C[(size_t)i * k + i];
        for (int p = 0; p < i; ++p) d -= R[(size_t)p * k + i] * R[(size_t)p * k + i];
        if (!(d > 0.0)) { ok = false; chol_fail = true; break; }
        R[(size_t)i * k + i] = std::sqrt(d);
        for (int j = i + 1; j < k; ++j) {
          double v = C[(size_t)i * k + j];
          for (int p = 0; p < i; ++p) v -= R[(size_t)p * k + i] * R[(size_t)p * k + j];
          R[(size_t)i * k + j] = v / R[(size_t)i * k + i];
        }
      }
      for (int c = 0; c < k && ok; ++c) {  // column c of R^-1: R x = e_c
        for (int i = c; i >= 0; --i) {
          double v = (i == c) ? 1.0 : 0.0;
          for (int j = i + 1; j <= c; ++j) v -= R[(size_t)i * k + j] * Ri[(size_t)j * k + c];
          Ri[(size_t)i * k + c] = v / R[(size_t)i * k + i];
        }
      }
    }
    if (ok) {
      ok = cudaMemcpyAsync(Rinv, Ri.data(), sizeof(double) * Ri.size(), cudaMemcpyHostToDevice, s) == cudaSuccess;
      if (mma) {  // Phi <- Phi R^-1 in place on the tensor pipe
        ok = ok && tall_mma<false>(N, k, k, Phi, max_k, Rinv, Phi, max_k, s) == HYDRO_OK;
      } else {
        hk::right_mult_kernel<<<blocks_for(N, 128), 128, 0, s>>>(N, k, max_k, Rinv, Phi);
        g_launches++;
      }
      ok = ok && cudaGetLastError() == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess;
    }
    cudaFree(P2); cudaFree(Rinv); cudaFree(G2);
    if (!ok) st = chol_fail ? HYDRO_ERR_NONFINITE : HYDRO_ERR_CUDA;
  }
  cleanup();
  return st;
}

hydro_status hydro_deim(const double *U, int64_t N, int m, int64_t *idx, hydro_stream_t stream) {
  if (!U || N <= 0 || m <= 0 || m > N || m > 4096 || !idx) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  // device scratch (kept between calls): c [m], block maxima [DEIM_BLOCKS], their rows
  std::unique_lock<std::mutex> lk(g_deim_scratch.mu);
  double *c = g_deim_scratch.get((size_t)m + 2 * hk::DEIM_BLOCKS);
  if (!c) return HYDRO_ERR_CUDA;
  double *bval = c + m;
  int64_t *bidx = (int64_t *)(bval + hk::DEIM_BLOCKS);
  auto cleanup = [&]() {};
  std::vector<double> rows((size_t)m * m), hv(hk::DEIM_BLOCKS), hc((size_t)m);
  std::vector<int64_t> hi(hk::DEIM_BLOCKS);
  hydro_status st = HYDRO_OK;
  for (int j = 0; j < m; ++j) {
    if (j > 0) {  // c = (P^T U_{<j})^-1 P^T u_j
      std::vector<double> A((size_t)j * j), b((size_t)j);
      for (int a = 0; a < j; ++a) {
        for (int q = 0; q < j; ++q) A[(size_t)a * j + q] = rows[(size_t)a * m + q];
        b[(size_t)a] = rows[(size_t)a * m + j];
      }
      if (!lu_solve_host(j, A, b)) { st = HYDRO_ERR_NONFINITE; break; }
      std::copy(b.begin(), b.end(), hc.begin());
      if (cudaMemcpyAsync(c, hc.data(), sizeof(double) * j, cudaMemcpyHostToDevice, s) != cudaSuccess) {
        st = HYDRO_ERR_CUDA;
        break;
      }
    }
    hk::deim_residual_kernel<<<hk::DEIM_BLOCKS, hk::DEIM_THREADS, 0, s>>>(N, m, j, U, c, bval, bidx);
    g_launches++;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(hv.data(), bval, sizeof(double) * hk::DEIM_BLOCKS, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(hi.data(), bidx, sizeof(int64_t) * hk::DEIM_BLOCKS, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      st = HYDRO_ERR_CUDA;
      break;
    }
    double best = -1.0;
    int64_t p = -1;
    for (int q = 0; q < hk::DEIM_BLOCKS; ++q)  // blocks cover ascending row ranges
      if (hi[(size_t)q] >= 0 && hv[(size_t)q] > best) { best = hv[(size_t)q]; p = hi[(size_t)q]; }
    if (p < 0) { st = HYDRO_ERR_NONFINITE; break; }
    idx[j] = p;
    if (cudaMemcpyAsync(rows.data() + (size_t)j * m, U + p * m, sizeof(double) * m, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      st = HYDRO_ERR_CUDA;
      break;
    }
  }
  cleanup();
  return st;
}

}  // extern "C"

namespace {

// [N][m] row-major -> [m][N] (tiled, coalesced both ways)
void transpose(int64_t N, int64_t m, const double *A, double *At, cudaStream_t s) {
  const int64_t tiles = ((N + 31) / 32) * ((m + 31) / 32);
  hk::transpose_kernel<<<(unsigned)tiles, dim3(32, 8), 0, s>>>(N, m, A, At);
  g_launches++;
}

// W = M Phi for the n columns of Phi [N][n] (field 1: M_V, 2: M_E): one tiled transpose to
// [n][N] so every column is a contiguous vector for the mass operator, n applications into
// a second [n][N] buffer, one transpose back.  (Column-by-column strided copies read a
// 32-byte sector per 8-byte value: 110 us per C2 column, profiles/fom/r01_fom_step_v3_*.)
hydro_status mass_columns(hydro_fom *F, int field, int64_t N, int n, const double *Phi, double *W,
                          cudaStream_t s) {
  const size_t need = (size_t)N * n * 2;
  if (F->colbuf_doubles < need) {  // grow the FOM's scratch (kept for the next call)
    cudaStreamSynchronize(s);
    cudaFree(F->colbuf);
    F->colbuf = nullptr;
    F->colbuf_doubles = 0;
    if (cudaMalloc(&F->colbuf, sizeof(double) * need) != cudaSuccess) return HYDRO_ERR_CUDA;
    F->colbuf_doubles = need;
  }
  double *T = F->colbuf;
  double *T2 = T + (size_t)N * n;
  transpose(N, n, Phi, T, s);
  hydro_status st = HYDRO_OK;
  for (int j = 0; j < n && st == HYDRO_OK; ++j)
    st = field == 1 ? mass_apply(F, T + (size_t)j * N, T2 + (size_t)j * N, nullptr, 0, 0, s)
                    : hydro_mass_e_apply(F, T + (size_t)j * N, T2 + (size_t)j * N, s);
  if (st == HYDRO_OK) transpose(n, N, T2, W, s);
  if (st == HYDRO_OK && cudaGetLastError() != cudaSuccess) st = HYDRO_ERR_CUDA;
  return st;
}

}  // namespace

extern "C" {

// Q-DEIM for m <= 64 by column-norm downdating (qdeim_dd_kernel): one read of U^T per pivot;
// the transposed copy and the norms live in a per-device scratch kept between calls.
static hydro_status qdeim_downdate(const double *U, int64_t N, int m, int64_t *idx, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_deim_scratch.mu);
  double *buf = g_deim_scratch.get((size_t)N * m + 2 * (size_t)N + (size_t)m * m + 2 * hk::DEIM_BLOCKS);
  if (!buf) return HYDRO_ERR_CUDA;
  double *Ut = buf, *nu = Ut + (size_t)N * m, *nu0 = nu + N, *Q = nu0 + N, *bval = Q + (size_t)m * m;
  int64_t *bidx = (int64_t *)(bval + hk::DEIM_BLOCKS);
  transpose(N, m, U, Ut, s);
  std::vector<double> hv(hk::DEIM_BLOCKS), row((size_t)m), hq((size_t)m * m);
  std::vector<int64_t> hi(hk::DEIM_BLOCKS);
  for (int k = 0; k < m; ++k) {
    hk::qdeim_dd_kernel<64><<<hk::DEIM_BLOCKS, hk::DEIM_THREADS, 0, s>>>(N, m, k, Q, Ut, nu, nu0, bval, bidx);
    g_launches++;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(hv.data(), bval, sizeof(double) * hk::DEIM_BLOCKS, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(hi.data(), bidx, sizeof(int64_t) * hk::DEIM_BLOCKS, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return HYDRO_ERR_CUDA;
    double best = -1.0;
    int64_t p = -1;
    for (int b = 0; b < hk::DEIM_BLOCKS; ++b)  // blocks cover ascending row ranges
      if (hi[(size_t)b] >= 0 && hv[(size_t)b] > best) { best = hv[(size_t)b]; p = hi[(size_t)b]; }
    if (p < 0 || !(best > 0.0)) return HYDRO_ERR_NONFINITE;
    idx[k] = p;
    if (k + 1 == m) break;
    // q_k = the pivot row's residual (MGS against q_0 .. q_{k-1}), normalised
    if (cudaMemcpyAsync(row.data(), U + p * m, sizeof(double) * m, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return HYDRO_ERR_CUDA;
    for (int l = 0; l < k; ++l) {
      const double *ql = hq.data() + (size_t)l * m;
      double d = 0.0;
      for (int j = 0; j < m; ++j) d = std::fma(row[(size_t)j], ql[j], d);
      for (int j = 0; j < m; ++j) row[(size_t)j] = std::fma(-d, ql[j], row[(size_t)j]);
    }
    double n2 = 0.0;
    for (int j = 0; j < m; ++j) n2 += row[(size_t)j] * row[(size_t)j];
    if (!(n2 > 0.0)) return HYDRO_ERR_NONFINITE;
    const double inv = 1.0 / std::sqrt(n2);
    for (int j = 0; j < m; ++j) hq[(size_t)k * m + j] = row[(size_t)j] * inv;
    if (cudaMemcpyAsync(Q + (size_t)k * m, hq.data() + (size_t)k * m, sizeof(double) * m, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return HYDRO_ERR_CUDA;
    hk::mark_chosen_kernel<<<1, 1, 0, s>>>(nu, p);
    g_launches++;
  }
  return cudaStreamSynchronize(s) == cudaSuccess ? HYDRO_OK : HYDRO_ERR_CUDA;
}

hydro_status hydro_qdeim(const double *U, int64_t N, int m, int64_t *idx, hydro_stream_t stream) {
  if (!U || N <= 0 || m <= 0 || m > N || m > 4096 || !idx) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (m <= 64) return qdeim_downdate(U, N, m, idx, s);
  double *Rt = nullptr, *q = nullptr, *bval = nullptr;
  int64_t *bidx = nullptr;
  auto cleanup = [&]() { cudaFree(Rt); cudaFree(q); cudaFree(bval); cudaFree(bidx); };
  if (cudaMalloc(&Rt, sizeof(double) * (size_t)N * m) != cudaSuccess ||
      cudaMalloc(&q, sizeof(double) * (size_t)m) != cudaSuccess ||
      cudaMalloc(&bval, sizeof(double) * hk::DEIM_BLOCKS) != cudaSuccess ||
      cudaMalloc(&bidx, sizeof(int64_t) * hk::DEIM_BLOCKS) != cudaSuccess) {
    cleanup();
    return HYDRO_ERR_CUDA;
  }
  transpose(N, m, U, Rt, s);
  std::vector<double> hv(hk::DEIM_BLOCKS), row((size_t)m);
  std::vector<int64_t> hi(hk::DEIM_BLOCKS);
  hydro_status st = HYDRO_OK;
  for (int k = 0; k < m; ++k) {
    hk::qdeim_step_kernel<<<hk::DEIM_BLOCKS, hk::DEIM_THREADS, 0, s>>>(N, m, q, Rt, bval, bidx, k == 0);
    g_launches++;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(hv.data(), bval, sizeof(double) * hk::DEIM_BLOCKS, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(hi.data(), bidx, sizeof(int64_t) * hk::DEIM_BLOCKS, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      st = HYDRO_ERR_CUDA;
      break;
    }
    double best = -1.0;
    int64_t p = -1;
    for (int b = 0; b < hk::DEIM_BLOCKS; ++b)  // blocks cover ascending row ranges
      if (hi[(size_t)b] >= 0 && hv[(size_t)b] > best) { best = hv[(size_t)b]; p = hi[(size_t)b]; }
    if (p < 0 || !(best > 0.0)) { st = HYDRO_ERR_NONFINITE; break; }
    idx[k] = p;
    if (k + 1 == m) break;
    // q = R[p] / |R[p]| for the next step (row p of the column-major residual: stride N)
    if (cudaMemcpy2DAsync(row.data(), sizeof(double), Rt + p, sizeof(double) * (size_t)N, sizeof(double),
                          (size_t)m, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      st = HYDRO_ERR_CUDA;
      break;
    }
    double n2 = 0.0;
    for (int j = 0; j < m; ++j) n2 += row[(size_t)j] * row[(size_t)j];
    const double inv = 1.0 / std::sqrt(n2);
    for (int j = 0; j < m; ++j) row[(size_t)j] *= inv;
    if (cudaMemcpyAsync(q, row.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      st = HYDRO_ERR_CUDA;
      break;
    }
  }
  cudaStreamSynchronize(s);
  cleanup();
  return st;
}

}  // extern "C"

extern "C" {

hydro_status hydro_deim_oversampled(const double *U, int64_t N, int m, int n_s, int64_t *idx,
                                    hydro_stream_t stream) {
  if (!U || N <= 0 || m <= 0 || m > 4096 || n_s < m || n_s > N || n_s > 65536 || !idx) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  // device scratch (kept between calls): |residual| of the current column (kept for its further
  // picks) [N], c [m], block maxima and their rows [DEIM_BLOCKS], the chosen-row mask [N bytes]
  std::unique_lock<std::mutex> lk(g_deim_scratch.mu);
  double *absr = g_deim_scratch.get((size_t)N + m + 2 * hk::DEIM_BLOCKS + ((size_t)N + 7) / 8);
  if (!absr) return HYDRO_ERR_CUDA;
  double *c = absr + N, *bval = c + m;
  int64_t *bidx = (int64_t *)(bval + hk::DEIM_BLOCKS);
  unsigned char *mask = (unsigned char *)(bidx + hk::DEIM_BLOCKS);
  if (cudaMemsetAsync(mask, 0, (size_t)N, s) != cudaSuccess) return HYDRO_ERR_CUDA;
  auto cleanup = [&]() {};
  std::vector<double> rows((size_t)n_s * m), hv(hk::DEIM_BLOCKS);
  std::vector<int64_t> hi(hk::DEIM_BLOCKS);
  const unsigned char one = 1;
  hydro_status st = HYDRO_OK;
  int got = 0;
  for (int j = 0; j < m && st == HYDRO_OK; ++j) {
    if (j > 0) {  // c = argmin |U[I, <j] c - U[I, j]|_2 over the current sample set I
      std::vector<double> A((size_t)got * j), b((size_t)got);
      for (int a = 0; a < got; ++a) {
        for (int q = 0; q < j; ++q) A[(size_t)a * j + q] = rows[(size_t)a * m + q];
        b[(size_t)a] = rows[(size_t)a * m + j];
      }
      if (!lstsq_host(got, j, A, b)) { st = HYDRO_ERR_NONFINITE; break; }
      if (cudaMemcpyAsync(c, b.data(), sizeof(double) * j, cudaMemcpyHostToDevice, s) != cudaSuccess) {
        st = HYDRO_ERR_CUDA;
        break;
      }
    }
    const int n_add = n_s / m + (j < n_s % m ? 1 : 0);
    for (int t = 0; t < n_add; ++t) {  // the n_add largest |residual| rows outside I, in order
      if (absr && t > 0)   // further picks of column j: arg-max of the kept |residual|
        hk::argmax_masked_kernel<<<hk::DEIM_BLOCKS, hk::DEIM_THREADS, 0, s>>>(N, absr, mask, bval, bidx);
      else
        hk::deim_residual_kernel<<<hk::DEIM_BLOCKS, hk::DEIM_THREADS, 0, s>>>(N, m, j, U, c, bval, bidx, mask, absr);
      g_launches++;
      if (cudaGetLastError() != cudaSuccess ||
          cudaMemcpyAsync(hv.data(), bval, sizeof(double) * hk::DEIM_BLOCKS, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaMemcpyAsync(hi.data(), bidx, sizeof(int64_t) * hk::DEIM_BLOCKS, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess) {
        st = HYDRO_ERR_CUDA;
        break;
      }
      double best = -1.0;
      int64_t p = -1;
      for (int q = 0; q < hk::DEIM_BLOCKS; ++q)  // blocks cover ascending row ranges
        if (hi[(size_t)q] >= 0 && hv[(size_t)q] > best) { best = hv[(size_t)q]; p = hi[(size_t)q]; }
      if (p < 0) { st = HYDRO_ERR_NONFINITE; break; }
      idx[got] = p;
      if (cudaMemcpyAsync(mask + p, &one, 1, cudaMemcpyHostToDevice, s) != cudaSuccess ||
          cudaMemcpyAsync(rows.data() + (size_t)got * m, U + p * m, sizeof(double) * m, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess) {
        st = HYDRO_ERR_CUDA;
        break;
      }
      ++got;
    }
  }
  cudaStreamSynchronize(s);
  cleanup();
  return st;
}

}  // extern "C"

namespace {

// G (device [na][nx]) = A^T X over N rows; A, X row-major with leading dimensions lda, ldx.
hydro_status xprod(int64_t N, int na, const double *A, int64_t lda, int nx, const double *X, int64_t ldx,
                   double *G, cudaStream_t s) {
  if (na <= 40 && nx <= 64) {
    // the FP64 tensor-pipe split-K kernel with A read transposed (A^T X), fixed-order reduce
    int64_t g = (N + 127) / 128;
    if (g > 148 * 2) g = 148 * 2;
    if (g < 1) g = 1;
    const int64_t chunk = (N + g - 1) / g;
    // the split-K partials: a per-device scratch kept between calls (grown on demand); the
    // call is synchronous, the mutex serialises host threads
    static std::mutex mu;
    static double *scratch[64] = {};
    static size_t scratch_n[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return HYDRO_ERR_CUDA;
    dev &= 63;
    const size_t need = (size_t)g * na * nx;
    if (scratch_n[dev] < need) {
      cudaFree(scratch[dev]);
      scratch[dev] = nullptr;
      scratch_n[dev] = 0;
      if (cudaMalloc(&scratch[dev], sizeof(double) * need) != cudaSuccess) return HYDRO_ERR_CUDA;
      scratch_n[dev] = need;
    }
    double *part = scratch[dev];
    const int mt = (na + 7) / 8;
    hydro_status st;
    if (mt == 1) st = launch_project_mma<1, true>(na, N, nx, (int)g, chunk, A, X, part, G, s, lda, ldx);
    else if (mt == 2) st = launch_project_mma<2, true>(na, N, nx, (int)g, chunk, A, X, part, G, s, lda, ldx);
    else if (mt == 3) st = launch_project_mma<3, true>(na, N, nx, (int)g, chunk, A, X, part, G, s, lda, ldx);
    else if (mt == 4) st = launch_project_mma<4, true>(na, N, nx, (int)g, chunk, A, X, part, G, s, lda, ldx);
    else st = launch_project_mma<5, true>(na, N, nx, (int)g, chunk, A, X, part, G, s, lda, ldx);
    const bool ok = st == HYDRO_OK && cudaStreamSynchronize(s) == cudaSuccess;
    return ok ? HYDRO_OK : (st != HYDRO_OK ? st : HYDRO_ERR_CUDA);
  }
  const int chunks = (int)std::min<int64_t>(hk::GRAM_CHUNKS, (N + hk::GRAM_KT - 1) / hk::GRAM_KT);
  const int64_t chunk = (N + chunks - 1) / chunks;
  double *part = nullptr;
  if (cudaMalloc(&part, sizeof(double) * (size_t)chunks * na * nx) != cudaSuccess) return HYDRO_ERR_CUDA;
  hk::xprod_partial_kernel<<<dim3((unsigned)chunks, (unsigned)((na + hk::GRAM_T - 1) / hk::GRAM_T),
                                  (unsigned)((nx + hk::GRAM_T - 1) / hk::GRAM_T)),
                             hk::GRAM_T * hk::GRAM_T, 0, s>>>(na, nx, N, chunk, A, lda, X, ldx, part);
  hk::xprod_reduce_kernel<<<(na * nx + 255) / 256, 256, 0, s>>>(na, nx, chunks, part, G);
  g_launches += 2;
  const bool ok = cudaGetLastError() == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess;
  cudaFree(part);
  return ok ? HYDRO_OK : HYDRO_ERR_CUDA;
}

// Ri = R^-1 of an upper triangular k x k R (row-major, host), by back substitution.
void upper_inv(int k, const std::vector<double> &R, std::vector<double> &Ri) {
  Ri.assign((size_t)k * k, 0.0);
  for (int c = 0; c < k; ++c)  // column c of R^-1: R x = e_c
    for (int i = c; i >= 0; --i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int j = i + 1; j <= c; ++j) v -= R[(size_t)i * k + j] * Ri[(size_t)j * k + c];
      Ri[(size_t)i * k + c] = v / R[(size_t)i * k + i];
    }
}

// Upper Cholesky factor R of the SPD k x k matrix C (C = R^T R) and its inverse Ri (both
// row-major, host).  false if a pivot is not positive (C not numerically SPD).
bool chol_upper_inv(int k, const std::vector<double> &C, std::vector<double> &R, std::vector<double> &Ri) {
  R.assign((size_t)k * k, 0.0);
  Ri.assign((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) {
    double d = C[(size_t)i * k + i];
    for (int p = 0; p < i; ++p) d -= R[(size_t)p * k + i] * R[(size_t)p * k + i];
    if (!(d > 0.0)) return false;
    R[(size_t)i * k + i] = std::sqrt(d);
    for (int j = i + 1; j < k; ++j) {
      double v = C[(size_t)i * k + j];
      for (int p = 0; p < i; ++p) v -= R[(size_t)p * k + i] * R[(size_t)p * k + j];
      R[(size_t)i * k + j] = v / R[(size_t)i * k + i];
    }
  }
  upper_inv(k, R, Ri);
  return true;
}

}  // namespace

extern "C" {

hydro_status hydro_window_ops(hydro_fom *fom, int field, int64_t N, int n_new, int n_old, int B,
                              const double *Phi_new, const double *Phi_old, const double *os_new,
                              const double *os_old, double *T, double *c, hydro_stream_t stream) {
  if (N <= 0 || n_new <= 0 || n_old <= 0 || B <= 0 || n_new > 1024 || n_old > 1024 || B > 65536 ||
      !Phi_new || !Phi_old || !os_new || !os_old || !T || !c || field < 0 || field > 2)
    return HYDRO_ERR_ARG;
  const bool oblique = fom && field > 0;
  if (oblique) {
    const int64_t want = field == 1 ? fom->n : fom->c->d.n_elem * fom->c->ne;
    if (N != want) return HYDRO_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  double *W = nullptr, *d = nullptr, *G = nullptr, *tmp = nullptr;
  auto cleanup = [&]() { cudaFree(W); cudaFree(d); cudaFree(G); cudaFree(tmp); };
  const size_t gsz = (size_t)n_new * (n_new + n_old + B);
  if (cudaMalloc(&d, sizeof(double) * (size_t)N * B) != cudaSuccess ||
      cudaMalloc(&G, sizeof(double) * gsz) != cudaSuccess) {
    cleanup();
    return HYDRO_ERR_CUDA;
  }
  hydro_status st = HYDRO_OK;
  const double *Wp = Phi_new;
  if (oblique) {  // W = M Phi_new, column by column through the FOM's own mass operators
    if (cudaMalloc(&W, sizeof(double) * (size_t)N * n_new) != cudaSuccess) {
      cleanup();
      return HYDRO_ERR_CUDA;
    }
    st = mass_columns(fom, field, N, n_new, Phi_new, W, s);
    Wp = W;
  }
  if (st == HYDRO_OK) {
    hk::sub_kernel<<<blocks_for(N * B, 256), 256, 0, s>>>(N * B, os_old, os_new, d);
    g_launches++;
    if (cudaGetLastError() != cudaSuccess) st = HYDRO_ERR_CUDA;
  }
  // G = [W^T Phi_old | W^T d | W^T Phi_new]
  double *G2 = G, *G3 = G + (size_t)n_new * n_old, *G1 = G3 + (size_t)n_new * B;
  if (st == HYDRO_OK) st = xprod(N, n_new, Wp, n_new, n_old, Phi_old, n_old, G2, s);
  if (st == HYDRO_OK) st = xprod(N, n_new, Wp, n_new, B, d, B, G3, s);
  if (st == HYDRO_OK && oblique) st = xprod(N, n_new, Wp, n_new, n_new, Phi_new, n_new, G1, s);
  if (st == HYDRO_OK && !oblique) {
    if (cudaMemcpyAsync(T, G2, sizeof(double) * (size_t)n_new * n_old, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(c, G3, sizeof(double) * (size_t)n_new * B, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      st = HYDRO_ERR_CUDA;
  } else if (st == HYDRO_OK) {  // T = Mhat^-1 (W^T Phi_old), c = Mhat^-1 (W^T d), Mhat = W^T Phi_new
    std::vector<double> h(gsz);
    if (cudaMemcpyAsync(h.data(), G, sizeof(double) * gsz, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      st = HYDRO_ERR_CUDA;
    } else {
      const double *h1 = h.data() + (size_t)n_new * (n_old + B);
      std::vector<double> A(h1, h1 + (size_t)n_new * n_new), out((size_t)n_new * (n_old + B)), b((size_t)n_new);
      const int nr = n_old + B;
      for (int col = 0; col < nr && st == HYDRO_OK; ++col) {
        const double *src = col < n_old ? h.data() : h.data() + (size_t)n_new * n_old;
        const int ld = col < n_old ? n_old : B, cc = col < n_old ? col : col - n_old;
        for (int i = 0; i < n_new; ++i) b[(size_t)i] = src[(size_t)i * ld + cc];
        if (!lu_solve_host(n_new, A, b)) { st = HYDRO_ERR_NONFINITE; break; }
        for (int i = 0; i < n_new; ++i) out[(size_t)i * nr + col] = b[(size_t)i];
      }
      if (st == HYDRO_OK) {
        std::vector<double> hT((size_t)n_new * n_old), hc((size_t)n_new * B);
        for (int i = 0; i < n_new; ++i) {
          for (int j = 0; j < n_old; ++j) hT[(size_t)i * n_old + j] = out[(size_t)i * nr + j];
          for (int j = 0; j < B; ++j) hc[(size_t)i * B + j] = out[(size_t)i * nr + n_old + j];
        }
        if (cudaMemcpyAsync(T, hT.data(), sizeof(double) * hT.size(), cudaMemcpyHostToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(c, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
          st = HYDRO_ERR_CUDA;
      }
    }
  }
  cudaStreamSynchronize(s);
  cleanup();
  return st;
}

hydro_status hydro_gappy_pinv(const double *U, int64_t N, int m, const int64_t *rows, int64_t s_rows,
                              double *P, hydro_stream_t stream) {
  if (!U || N <= 0 || m <= 0 || m > hk::POD_MAXK || !rows || s_rows <= 0 || s_rows > INT32_MAX || !P)
    return HYDRO_ERR_ARG;
  for (int64_t i = 0; i < s_rows; ++i)
    if (rows[i] < 0 || rows[i] >= N) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t *d_rows = nullptr;
  double *Q = nullptr, *G = nullptr, *Rinv = nullptr;
  auto cleanup = [&]() { cudaFree(d_rows); cudaFree(Q); cudaFree(G); cudaFree(Rinv); };
  if (cudaMalloc(&d_rows, sizeof(int64_t) * (size_t)s_rows) != cudaSuccess ||
      cudaMalloc(&Q, sizeof(double) * (size_t)s_rows * m) != cudaSuccess ||
      cudaMalloc(&G, sizeof(double) * (size_t)m * m) != cudaSuccess ||
      cudaMalloc(&Rinv, sizeof(double) * (size_t)m * m) != cudaSuccess ||
      cudaMemcpyAsync(d_rows, rows, sizeof(int64_t) * (size_t)s_rows, cudaMemcpyHostToDevice, s) != cudaSuccess) {
    cleanup();
    return HYDRO_ERR_CUDA;
  }
  // Q = U[rows, :]
  hk::gather_rows_kernel<<<blocks_for(s_rows * m, 256), 256, 0, s>>>((int)s_rows, m, d_rows, U, m, Q);
  g_launches++;
  if (s_rows < m) {
    // fewer sampled rows than basis columns (a wide U[rows], s < m <= 128): the minimum-norm
    // pseudo-inverse A^+ = Q R^-T from A^T = Q R (m x s, two Gram-Schmidt passes), on the host
    const int sr = (int)s_rows;
    std::vector<double> A((size_t)sr * m), Qt((size_t)sr * m), R((size_t)sr * sr, 0.0), Pm((size_t)m * sr);
    hydro_status st0 = HYDRO_OK;
    if (cudaMemcpyAsync(A.data(), Q, sizeof(double) * A.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      st0 = HYDRO_ERR_CUDA;
    // column j of A^T is row j of A: orthonormalise the rows of A (Qt[j] = q_j, length m)
    for (int j = 0; j < sr && st0 == HYDRO_OK; ++j) {
      std::vector<double> v(A.begin() + (size_t)j * m, A.begin() + (size_t)(j + 1) * m);
      for (int pass = 0; pass < 2; ++pass)
        for (int i = 0; i < j; ++i) {
          double d = 0.0;
          for (int k = 0; k < m; ++k) d += Qt[(size_t)i * m + k] * v[(size_t)k];
          R[(size_t)i * sr + j] += d;
          for (int k = 0; k < m; ++k) v[(size_t)k] -= d * Qt[(size_t)i * m + k];
        }
      double nrm = 0.0;
      for (int k = 0; k < m; ++k) nrm += v[(size_t)k] * v[(size_t)k];
      nrm = std::sqrt(nrm);
      if (!(nrm > 0.0)) { st0 = HYDRO_ERR_NONFINITE; break; }
      R[(size_t)j * sr + j] = nrm;
      for (int k = 0; k < m; ++k) Qt[(size_t)j * m + k] = v[(size_t)k] / nrm;
    }
    if (st0 == HYDRO_OK) {  // P = Q R^-T: P[k][j] = sum_i Q[k][i] (R^-1)[j][i]
      std::vector<double> Ri;
      upper_inv(sr, R, Ri);
      for (int k = 0; k < m; ++k)
        for (int j = 0; j < sr; ++j) {
          double acc = 0.0;
          for (int i = j; i < sr; ++i) acc += Qt[(size_t)i * m + k] * Ri[(size_t)j * sr + i];
          Pm[(size_t)k * sr + j] = acc;
        }
      if (cudaMemcpyAsync(P, Pm.data(), sizeof(double) * Pm.size(), cudaMemcpyHostToDevice, s) != cudaSuccess ||
          cudaStreamSynchronize(s) != cudaSuccess)
        st0 = HYDRO_ERR_CUDA;
    }
    cleanup();
    return st0;
  }
  // CholQR2: Q <- Q R1^-1, Q <- Q R2^-1 (Q^T Q = R^T R each pass), R = R2 R1
  std::vector<double> C((size_t)m * m), R, Ri, Racc((size_t)m * m, 0.0);
  for (int i = 0; i < m; ++i) Racc[(size_t)i * m + i] = 1.0;
  hydro_status st = cudaGetLastError() == cudaSuccess ? HYDRO_OK : HYDRO_ERR_CUDA;
  for (int pass = 0; pass < 2 && st == HYDRO_OK; ++pass) {
    st = xprod(s_rows, m, Q, m, m, Q, m, G, s);
    if (st != HYDRO_OK) break;
    if (cudaMemcpyAsync(C.data(), G, sizeof(double) * C.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      st = HYDRO_ERR_CUDA;
      break;
    }
    if (!chol_upper_inv(m, C, R, Ri)) { st = HYDRO_ERR_NONFINITE; break; }  // U[rows] rank-deficient
    std::vector<double> Rn((size_t)m * m, 0.0);  // R_pass * Racc (both upper triangular)
    for (int i = 0; i < m; ++i)
      for (int j = i; j < m; ++j) {
        double acc = 0.0;
        for (int k = i; k <= j; ++k) acc += R[(size_t)i * m + k] * Racc[(size_t)k * m + j];
        Rn[(size_t)i * m + j] = acc;
      }
    Racc.swap(Rn);
    if (cudaMemcpyAsync(Rinv, Ri.data(), sizeof(double) * Ri.size(), cudaMemcpyHostToDevice, s) != cudaSuccess) {
      st = HYDRO_ERR_CUDA;
      break;
    }
    hk::right_mult_kernel<<<blocks_for(s_rows, 128), 128, 0, s>>>(s_rows, m, m, Rinv, Q);
    g_launches++;
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) st = HYDRO_ERR_CUDA;
  }
  if (st == HYDRO_OK) {  // P = R^-1 Q^T
    upper_inv(m, Racc, Ri);
    if (cudaMemcpyAsync(Rinv, Ri.data(), sizeof(double) * Ri.size(), cudaMemcpyHostToDevice, s) != cudaSuccess) {
      st = HYDRO_ERR_CUDA;
    } else {
      hk::pinv_apply_kernel<<<blocks_for(s_rows, 128), 128, 0, s>>>(s_rows, m, Rinv, Q, P);
      g_launches++;
      if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) st = HYDRO_ERR_CUDA;
    }
  }
  cleanup();
  return st;
}

hydro_status hydro_rom_window_offset(int64_t rows, int n_prev, int B, const double *Phi_prev,
                                     const double *os_prev, int os_prev_batched, const double *Y_prev,
                                     double *os_new, int n_new, double *Y_new, hydro_stream_t stream) {
  if (rows < 0 || n_prev <= 0 || B <= 0 || n_new < 0 || (n_new > 0 && !Y_new) || !os_new) return HYDRO_ERR_ARG;
  // Eq. previous_os: os_w = os_{w-1} + Phi_{w-1} yhat_{w-1}(t_{w-1})  (the lift of the final state)
  hydro_status st = hydro_rom_lift(rows, n_prev, B, Phi_prev, os_prev, os_prev_batched, Y_prev, os_new, stream);
  if (st != HYDRO_OK) return st;
  // yhat_w(t_{w-1}) = Phi_w^T (os_{w-1} + Phi_{w-1} yhat_{w-1} - os_w) = 0
  if (n_new > 0) CUDA_OK(cudaMemsetAsync(Y_new, 0, sizeof(double) * (size_t)n_new * B, (cudaStream_t)stream));
  return HYDRO_OK;
}

hydro_status hydro_basis_tproduct(int64_t N, int n, int B, const double *Phi, const double *X, double *out,
                                  hydro_stream_t stream) {
  if (N <= 0 || n <= 0 || B <= 0 || n > 1024 || B > 65536 || !Phi || !X || !out) return HYDRO_ERR_ARG;
  return xprod(N, n, Phi, n, B, X, B, out, (cudaStream_t)stream);
}

}  // extern "C"

namespace {

// eta = | (I - M Phi Mhat^-1 Phi^T P) f |_2 with P f = U (U[Z,:])^+ f[Z]  (one field of the
// Theorem-2 integrand).  f: device [N]; Phi [N][n]; U [N][m]; Z host [s].
hydro_status indicator_field(hydro_fom *F, int field, int64_t N, const double *f, int n, const double *Phi,
                             int m, const double *U, int s_rows, const int64_t *Z, double *eta,
                             cudaStream_t s) {
  double *W = nullptr, *tmp = nullptr, *G = nullptr, *gat = nullptr, *y = nullptr;
  int64_t *dZ = nullptr;
  auto cleanup = [&]() { cudaFree(W); cudaFree(tmp); cudaFree(G); cudaFree(gat); cudaFree(y); cudaFree(dZ); };
  if (cudaMalloc(&W, sizeof(double) * (size_t)N * n) != cudaSuccess ||
      cudaMalloc(&tmp, sizeof(double) * (size_t)N * 2) != cudaSuccess ||
      cudaMalloc(&G, sizeof(double) * std::max<size_t>((size_t)n * (n + 1), (size_t)N)) != cudaSuccess ||
      cudaMalloc(&gat, sizeof(double) * (size_t)s_rows * (m + 1)) != cudaSuccess ||
      cudaMalloc(&y, sizeof(double) * (size_t)(m > n ? m : n)) != cudaSuccess ||
      cudaMalloc(&dZ, sizeof(int64_t) * (size_t)s_rows) != cudaSuccess) {
    cleanup();
    return HYDRO_ERR_CUDA;
  }
  hydro_status st = HYDRO_OK;
  const unsigned g = blocks_for(N, 256);
  // P f: least-squares fit of the sampled rows
  std::vector<double> hU((size_t)s_rows * m), hf((size_t)s_rows);
  if (cudaMemcpyAsync(dZ, Z, sizeof(int64_t) * s_rows, cudaMemcpyHostToDevice, s) != cudaSuccess) st = HYDRO_ERR_CUDA;
  if (st == HYDRO_OK) {
    hk::gather_rows_kernel<<<(s_rows * m + 255) / 256, 256, 0, s>>>(s_rows, m, dZ, U, m, gat);
    hk::gather_rows_kernel<<<(s_rows + 255) / 256, 256, 0, s>>>(s_rows, 1, dZ, f, 1, gat + (size_t)s_rows * m);
    g_launches += 2;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(hU.data(), gat, sizeof(double) * hU.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(hf.data(), gat + (size_t)s_rows * m, sizeof(double) * s_rows, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      st = HYDRO_ERR_CUDA;
  }
  if (st == HYDRO_OK && !lstsq_host(s_rows, m, hU, hf)) st = HYDRO_ERR_NONFINITE;
  if (st == HYDRO_OK) {  // tmp = U a
    if (cudaMemcpyAsync(y, hf.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s) != cudaSuccess) st = HYDRO_ERR_CUDA;
    hk::gemv_kernel<<<g, 256, 0, s>>>(N, m, U, m, y, nullptr, -1.0, tmp);
    g_launches++;
  }
  // W = M Phi
  if (st == HYDRO_OK) st = mass_columns(F, field, N, n, Phi, W, s);
  // [Mhat | b] = Phi^T [W | U a]
  if (st == HYDRO_OK) st = xprod(N, n, Phi, n, n, W, n, G, s);
  if (st == HYDRO_OK) st = xprod(N, n, Phi, n, 1, tmp, 1, G + (size_t)n * n, s);
  std::vector<double> hG((size_t)n * (n + 1));
  if (st == HYDRO_OK &&
      (cudaMemcpyAsync(hG.data(), G, sizeof(double) * hG.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
       cudaStreamSynchronize(s) != cudaSuccess))
    st = HYDRO_ERR_CUDA;
  if (st == HYDRO_OK) {
    std::vector<double> A(hG.begin(), hG.begin() + (size_t)n * n), b(hG.begin() + (size_t)n * n, hG.end());
    if (!lu_solve_host(n, A, b)) st = HYDRO_ERR_NONFINITE;
    else if (cudaMemcpyAsync(y, b.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s) != cudaSuccess)
      st = HYDRO_ERR_CUDA;
  }
  if (st == HYDRO_OK) {  // r = f - W z;  eta = |r|
    hk::gemv_kernel<<<g, 256, 0, s>>>(N, n, W, n, y, f, 1.0, tmp + N);
    g_launches++;
    st = dot(F, N, tmp + N, tmp + N, F->sc + 5, s);
  }
  double h = 0.0;
  if (st == HYDRO_OK &&
      (cudaMemcpyAsync(&h, F->sc + 5, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
       cudaStreamSynchronize(s) != cudaSuccess))
    st = HYDRO_ERR_CUDA;
  if (st == HYDRO_OK) *eta = std::sqrt(h);
  cudaStreamSynchronize(s);
  cleanup();
  return st;
}

}  // namespace

extern "C" {

hydro_status hydro_rom_indicator(hydro_fom *fom, const double *x, const double *v, const double *e,
                                 const double *gamma, hydro_visc visc, hydro_cfl cfl, int nv,
                                 const double *Phi_v, int ne, const double *Phi_e, int m1, const double *U1,
                                 int s1, const int64_t *Z1, int m2, const double *U2, int s2,
                                 const int64_t *Z2, double *eta, hydro_stream_t stream) {
  if (!fom || !x || !v || !e || !gamma || !Phi_v || !Phi_e || !U1 || !U2 || !Z1 || !Z2 || !eta ||
      nv <= 0 || ne <= 0 || m1 <= 0 || m2 <= 0 || s1 < m1 || s2 < m2 || nv > 1024 || ne > 1024 ||
      m1 > 4096 || m2 > 4096)
    return HYDRO_ERR_ARG;
  const int64_t NV = fom->n, NE = fom->c->d.n_elem * fom->c->ne;
  for (int i = 0; i < s1; ++i)
    if (Z1[i] < 0 || Z1[i] >= NV) return HYDRO_ERR_ARG;
  for (int i = 0; i < s2; ++i)
    if (Z2[i] < 0 || Z2[i] >= NE) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  hydro_status st = force_common(fom->c, hk::MODE_FORCE, x, v, e, v, gamma, visc, cfl, fom->F1, fom->FTw,
                                 fom->dts, s);
  if (st != HYDRO_OK) return st;
  std::vector<char> bad;
  if ((st = read_reset_status(fom->c->st, 1, s, bad)) != HYDRO_OK) return st;
  if (bad[0]) return HYDRO_ERR_TANGLED;
  if ((st = indicator_field(fom, 1, NV, fom->F1, nv, Phi_v, m1, U1, s1, Z1, &eta[0], s)) != HYDRO_OK) return st;
  return indicator_field(fom, 2, NE, fom->FTw, ne, Phi_e, m2, U2, s2, Z2, &eta[1], s);
}

}  // extern "C"

extern "C" {

hydro_status hydro_index_copy_add(int64_t n, int dim, const double *src, int64_t ld_src,
                                  const int64_t *src_idx, double *dst, int64_t ld_dst,
                                  const int64_t *dst_idx, int add, hydro_stream_t stream) {
  if (n < 0 || dim <= 0 || dim > 3 || ld_src < 0 || ld_dst < 0) return HYDRO_ERR_ARG;
  if (n == 0) return HYDRO_OK;
  if (!src || !dst) return HYDRO_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  hk::index_copy_add_kernel<<<blocks_for(n * dim, 256), 256, 0, s>>>(n, dim, src, ld_src, src_idx, dst, ld_dst,
                                                                      dst_idx, add);
  g_launches++;
  return cudaGetLastError() == cudaSuccess ? HYDRO_OK : HYDRO_ERR_CUDA;
}

}  // extern "C"
