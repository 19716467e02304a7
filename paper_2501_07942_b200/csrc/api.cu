// C-ABI entry points (include/ttgbf.h).  Each entry point launches ONE
// kernel with one 256-thread CTA per item (filter or TT) on the caller's
// stream; per-item status codes land in device memory.
//
// Built by nvcc for sm_100a this is the product library libttgbf.so.
// Built by g++ with -DENGINE_HOSTSIM (tests only) the same source becomes
// libttgbf_hostsim.so, whose "launch" loops over items on the CPU with a
// one-thread CTA; the product package never loads it.
#include "bodies.cuh"

#ifdef __CUDACC__
#include <cuda_runtime.h>
#define LAMBDA [=] __device__
#else
#include <vector>
#define LAMBDA [=]
#endif

using namespace tg;

// The device build compiles this file once per part (-DTTGBF_API_PART=1..4,
// in parallel: build.py); part 0 (host emulation) holds every entry point.
#ifndef TTGBF_API_PART
#define TTGBF_API_PART 0
#endif
#define API_PART(k) (TTGBF_API_PART == 0 || TTGBF_API_PART == (k))

namespace {

#ifdef __CUDACC__
template <class F>
__global__ void __launch_bounds__(BLOCK_THREADS, CTAS_PER_SM) k_items(F f, int count) {
  extern __shared__ double smem[];
  const Ctx c = make_ctx(smem, threadIdx.x, blockDim.x);
  if ((int)blockIdx.x < count) f(c, (int)blockIdx.x, smem);
}

template <class F>
int launch(int count, F f, void* stream) {
  if (count <= 0) return TTGBF_OK;
  const size_t smem = (size_t)SMEM_DOUBLES * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(k_items<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return TTGBF_E_CUDA;
  k_items<F><<<count, BLOCK_THREADS, smem, (cudaStream_t)stream>>>(f, count);
  e = cudaGetLastError();
  return e == cudaSuccess ? TTGBF_OK : TTGBF_E_CUDA;
}
#else
template <class F>
int launch(int count, F f, void*) {
  std::vector<double> smem(SMEM_DOUBLES);
  for (int i = 0; i < count; ++i) {
    const Ctx c = make_ctx(smem.data(), 0, 1);
    f(c, i, smem.data());
  }
  return TTGBF_OK;
}
#endif

}  // namespace

extern "C" {

#if API_PART(1)
int ttgbf_version(void) { return 1; }
int ttgbf_block_threads(void) { return BLOCK_THREADS; }
int64_t ttgbf_smem_bytes(void) { return (int64_t)SMEM_DOUBLES * 8; }
int ttgbf_ctas_per_sm(void) { return CTAS_PER_SM; }

const char* ttgbf_status_string(int s) {
  switch (s) {
    case TTGBF_OK: return "ok";
    case TTGBF_E_ARG: return "invalid argument / shape";
    case TTGBF_E_NONFINITE: return "evaluator returned a non-finite value";
    case TTGBF_E_DEGENERATE: return "TT weights carry no probability mass";
    case TTGBF_E_WORKSPACE: return "per-filter workspace exhausted";
    case TTGBF_E_CACHE: return "evaluator cache capacity exhausted";
    case TTGBF_E_CUDA: return "CUDA error";
    case TTGBF_E_LINALG: return "singular matrix";
    case TTGBF_E_DENSE_GUARD: return "dense guard exceeded";
    case TTGBF_E_STATE_CAP: return "TT larger than the per-filter state slab";
    default: return "unknown status";
  }
}

// ---------------------------------------------------------------- stages
int ttgbf_filter_prior(const ttgbf_model* model, const ttgbf_gauss* prior, ttgbf_grid_cfg gcfg,
                       ttgbf_cross_cfg xcfg, const ttgbf_filter_io* io, int nfilt, const int32_t* probes,
                       int nprobes, ttgbf_tt* state_hdr, double* state, int64_t state_cap, void* ws,
                       int64_t ws_bytes, ttgbf_diag* diag, void* stream) {
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    if (!io[i].active) return;
    Arena ar = make_arena(ws, ws_bytes, i);
    ttgbf_diag* dg = diag + i;
    if (c.leader()) { dg->clipped_mass = 0.0; dg->outlier = 0; }
    c.sync();
    int st = stage_prior(c, ar, *model, *prior, gcfg, xcfg, io[i], probes, nprobes, state_hdr + i,
                         state + (int64_t)i * state_cap, state_cap, dg, make_stage_smem(smem));
    if (c.leader()) { dg->status = st; dg->ws_peak = (int64_t)ar.peak; }
  };
  return launch(nfilt, f, stream);
}

int ttgbf_filter_measure(const ttgbf_model* model, ttgbf_grid_cfg gcfg, ttgbf_cross_cfg xcfg,
                         const ttgbf_filter_io* io, int nfilt, const int32_t* probes, int nprobes,
                         const int32_t* seeds, int nseeds, ttgbf_tt* state_hdr, double* state,
                         int64_t state_cap, void* ws, int64_t ws_bytes, ttgbf_diag* diag, void* stream) {
  auto f = LAMBDA(const Ctx& c0, int i, double* smem) {
    if (!io[i].active) return;
    Arena ar = make_arena(ws, ws_bytes, i);
    ttgbf_diag* dg = diag + i;
    Ctx c = c0;
    c.prof = dg->prof;
    if (c.leader()) {
      dg->clipped_mass = 0.0; dg->outlier = 0; dg->mass_before_norm = NAN;
      for (int q = 0; q < 32; ++q) dg->prof[q] = 0;
      for (int q = 0; q < 8; ++q) dg->cycles[q] = 0;
    }
    c.sync();
    int st = stage_measure(c, ar, *model, gcfg, xcfg, io[i], probes, nprobes, seeds, nseeds, state_hdr + i,
                           state + (int64_t)i * state_cap, state_cap, dg, make_stage_smem(smem));
    if (c.leader()) { dg->status = st; dg->ws_peak = (int64_t)ar.peak; }
  };
  return launch(nfilt, f, stream);
}
#endif

#if API_PART(2)
int ttgbf_filter_time_update(const ttgbf_model* model, ttgbf_grid_cfg gcfg, ttgbf_cross_cfg xcfg,
                             const ttgbf_filter_io* io, int nfilt, const int32_t* probes, int nprobes,
                             const int32_t* seeds, int nseeds, ttgbf_tt* state_hdr, double* state,
                             int64_t state_cap, void* ws, int64_t ws_bytes, ttgbf_diag* diag, void* stream) {
  auto f = LAMBDA(const Ctx& c0, int i, double* smem) {
    if (!io[i].active) return;
    Arena ar = make_arena(ws, ws_bytes, i);
    ttgbf_diag* dg = diag + i;
    Ctx c = c0;
    c.prof = dg->prof;
    int st = stage_time(c, ar, *model, gcfg, xcfg, io[i], probes, nprobes, seeds, nseeds, state_hdr + i,
                        state + (int64_t)i * state_cap, state_cap, dg, make_stage_smem(smem));
    if (c.leader()) {
      dg->status = st;
      if ((int64_t)ar.peak > dg->ws_peak) dg->ws_peak = (int64_t)ar.peak;
    }
  };
  return launch(nfilt, f, stream);
}

int ttgbf_filter_time_update_std(const ttgbf_model* model, ttgbf_grid_cfg gcfg, ttgbf_cross_cfg xcfg,
                                 const ttgbf_filter_io* io, int nfilt, const int32_t* probes, int nprobes,
                                 ttgbf_tt* state_hdr, double* state, int64_t state_cap, void* ws, int64_t ws_bytes,
                                 ttgbf_diag* diag, void* stream) {
  auto f = LAMBDA(const Ctx& c0, int i, double* smem) {
    if (!io[i].active) return;
    Arena ar = make_arena(ws, ws_bytes, i);
    ttgbf_diag* dg = diag + i;
    Ctx c = c0;
    c.prof = dg->prof;
    int st = stage_time_std(c, ar, *model, gcfg, xcfg, io[i], probes, nprobes, state_hdr + i,
                            state + (int64_t)i * state_cap, state_cap, dg, make_stage_smem(smem));
    if (c.leader()) {
      dg->status = st;
      if ((int64_t)ar.peak > dg->ws_peak) dg->ws_peak = (int64_t)ar.peak;
    }
  };
  return launch(nfilt, f, stream);
}
#endif

#if API_PART(3)
int ttgbf_filter_run(const ttgbf_model* model, const ttgbf_gauss* prior, ttgbf_grid_cfg gcfg, ttgbf_cross_cfg xcfg,
                     ttgbf_run_cfg rcfg, ttgbf_filter_io* io, int32_t* kstep, const double* Z, int nfilt,
                     const int32_t* probes, int nprobes, const int32_t* seeds, int nseeds, ttgbf_tt* state_hdr,
                     double* state, int64_t state_cap, void* ws, int64_t ws_bytes, int32_t* sched,
                     int nslots, ttgbf_diag* diag, ttgbf_step_rec* rec, void* stream) {
  if (rcfg.steps < 0 || rcfg.kf < 1 || nslots < 1 || nfilt < 1) return TTGBF_E_ARG;
  const int64_t total = (int64_t)nfilt * rcfg.steps;
  auto f = LAMBDA(const Ctx& c, int slot, double* smem) {
    Arena ar = make_arena(ws, ws_bytes, slot);
    int32_t* cursor = sched;
    int32_t* ndone = sched + 1;
    int32_t* lock = sched + 2;
    int32_t* done = sched + 2 + nfilt;
    const int b = model->b;
    while (true) {
      int fsel = -1;
      if (c.leader()) {
        while (true) {
#if ENGINE_DEVICE
          if (*(volatile int32_t*)ndone >= total) break;
          const int g = (int)((unsigned)atomicAdd(cursor, 1) % (unsigned)nfilt);
          if (*(volatile int32_t*)(done + g) >= rcfg.steps) continue;
          if (atomicCAS(&lock[g], 0, 1) != 0) continue;
          __threadfence();   // acquire: drop stale L1 lines of this filter's state
          if (*(volatile int32_t*)(done + g) >= rcfg.steps) { atomicExch(&lock[g], 0); continue; }
          fsel = g;
          break;
#else
          if (*ndone >= total) break;
          const int g = (int)((unsigned)((*cursor)++) % (unsigned)nfilt);
          if (done[g] >= rcfg.steps || lock[g]) continue;
          lock[g] = 1;
          fsel = g;
          break;
#endif
        }
      }
      fsel = (int)bcast_i(c, fsel);
      if (fsel < 0) break;
      const int i = fsel;
      ttgbf_diag* dg = diag + i;
      Ctx cc = c;
      cc.prof = dg->prof;
      const int sidx = done[i];
      int st = stage_run_step(cc, ar, *model, *prior, gcfg, xcfg, rcfg, io + i, kstep + i,
                              Z + (int64_t)i * rcfg.kf * b, probes, nprobes, seeds, nseeds, state_hdr + i,
                              state + (int64_t)i * state_cap, state_cap, dg, rec + (int64_t)i * rcfg.steps + sidx,
                              make_stage_smem(smem));
      if (c.leader()) {
        dg->status = st;
        if ((int64_t)ar.peak > dg->ws_peak) dg->ws_peak = (int64_t)ar.peak;
      }
      c.sync();
      if (c.leader()) {
#if ENGINE_DEVICE
        __threadfence();
        done[i] = sidx + 1;
        __threadfence();
        atomicAdd(ndone, 1);
        atomicExch(&lock[i], 0);
#else
        done[i] = sidx + 1;
        *ndone += 1;
        lock[i] = 0;
#endif
      }
      c.sync();
    }
  };
  return launch(nslots < nfilt ? nslots : nfilt, f, stream);
}
#endif

#if API_PART(4)
// ---------------------------------------------------------------- TT primitives
int ttgbf_tt_round(const ttgbf_tt* in_hdr, const double* in, int64_t in_cap, int count, double tol, int max_rank,
                   ttgbf_tt* out_hdr, double* out, int64_t out_cap, void* ws, int64_t ws_bytes, int32_t* status,
                   void* stream) {
  if (tol < 0.0) return TTGBF_E_ARG;
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    Arena ar = make_arena(ws, ws_bytes, i);
    int st = body_round(c, ar, in_hdr + i, in + (int64_t)i * in_cap, tol, max_rank, out_hdr + i,
                        out + (int64_t)i * out_cap, out_cap, make_stage_smem(smem).sm);
    if (c.leader()) status[i] = st;
  };
  return launch(count, f, stream);
}

int ttgbf_tt_hadamard(const ttgbf_tt* a_hdr, const double* a, int64_t a_cap, const ttgbf_tt* b_hdr, const double* b,
                      int64_t b_cap, int count, ttgbf_tt* out_hdr, double* out, int64_t out_cap, void* ws,
                      int64_t ws_bytes, int32_t* status, void* stream) {
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    (void)smem;
    Arena ar = make_arena(ws, ws_bytes, i);
    int st = body_hadamard(c, ar, a_hdr + i, a + (int64_t)i * a_cap, b_hdr + i, b + (int64_t)i * b_cap,
                           out_hdr + i, out + (int64_t)i * out_cap, out_cap);
    if (c.leader()) status[i] = st;
  };
  return launch(count, f, stream);
}

int ttgbf_tt_fft_convolve(const ttgbf_tt* k_hdr, const double* k, int64_t k_cap, const ttgbf_tt* w_hdr,
                          const double* w, int64_t w_cap, int count, double tol, int max_rank, ttgbf_tt* out_hdr,
                          double* out, int64_t out_cap, void* ws, int64_t ws_bytes, int32_t* status, void* stream) {
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    Arena ar = make_arena(ws, ws_bytes, i);
    int st = body_fftconv(c, ar, k_hdr + i, k + (int64_t)i * k_cap, w_hdr + i, w + (int64_t)i * w_cap, tol,
                          max_rank, out_hdr + i, out + (int64_t)i * out_cap, out_cap, make_stage_smem(smem).sm);
    if (c.leader()) status[i] = st;
  };
  return launch(count, f, stream);
}

int ttgbf_tt_interpolate(const ttgbf_tt* in_hdr, const double* in, int64_t in_cap, int count,
                         const ttgbf_axis* old_axes, const ttgbf_axis* new_axes, ttgbf_tt* out_hdr, double* out,
                         int64_t out_cap, void* ws, int64_t ws_bytes, int32_t* status, void* stream) {
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    (void)smem;
    Arena ar = make_arena(ws, ws_bytes, i);
    const int d = in_hdr[i].d;
    int st = body_interp(c, ar, in_hdr + i, in + (int64_t)i * in_cap, old_axes + (int64_t)i * d,
                         new_axes + (int64_t)i * d, out_hdr + i, out + (int64_t)i * out_cap, out_cap);
    if (c.leader()) status[i] = st;
  };
  return launch(count, f, stream);
}

int ttgbf_tt_eval_many(const ttgbf_tt* hdr, const double* data, int64_t cap, int count, const int32_t* idx, int64_t K,
                       double* out, void* ws, int64_t ws_bytes, int32_t* status, void* stream) {
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    const int d = hdr[i].d;
    Arena ar = make_arena(ws, ws_bytes, i);
    int st = body_eval_many(c, ar, hdr + i, data + (int64_t)i * cap, idx + (int64_t)i * K * d, K,
                            out + (int64_t)i * K, make_stage_smem(smem).sm);
    if (c.leader()) status[i] = st;
  };
  return launch(count, f, stream);
}

int ttgbf_tt_eval_at_points(const ttgbf_tt* hdr, const double* data, int64_t cap, int count, const ttgbf_axis* axes,
                            const double* pts, int64_t K, double* out, void* ws, int64_t ws_bytes, int32_t* status,
                            void* stream) {
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    Arena ar = make_arena(ws, ws_bytes, i);
    const int d = hdr[i].d;
    int st = body_eval_points(c, ar, hdr + i, data + (int64_t)i * cap, axes + (int64_t)i * d,
                              pts + (int64_t)i * K * d, K, out + (int64_t)i * K, make_stage_smem(smem).sm);
    if (c.leader()) status[i] = st;
  };
  return launch(count, f, stream);
}

int ttgbf_tt_sum_moments(const ttgbf_tt* hdr, const double* data, int64_t cap, int count, const ttgbf_axis* axes,
                         double* out, void* ws, int64_t ws_bytes, int32_t* status, void* stream) {
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    (void)smem;
    Arena ar = make_arena(ws, ws_bytes, i);
    const int d = hdr[i].d;
    int st = body_moments(c, ar, hdr + i, data + (int64_t)i * cap, axes + (int64_t)i * d,
                          out + (int64_t)i * TTGBF_NMOM);
    if (c.leader()) status[i] = st;
  };
  return launch(count, f, stream);
}

int ttgbf_greedy_cross(int kind, const ttgbf_model* model, const ttgbf_gauss* prior, ttgbf_cross_cfg xcfg,
                       const ttgbf_filter_io* io, int count, const int32_t* seeds, int nseeds, ttgbf_tt* out_hdr,
                       double* out, int64_t out_cap, void* ws, int64_t ws_bytes, ttgbf_diag* diag, void* stream) {
  if (kind < 0 || kind > 2) return TTGBF_E_ARG;
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    Arena ar = make_arena(ws, ws_bytes, i);
    int st = body_cross(c, ar, kind, *model, prior, xcfg, io[i], seeds, nseeds, out_hdr + i,
                        out + (int64_t)i * out_cap, out_cap, diag + i, make_stage_smem(smem));
    if (c.leader()) { diag[i].status = st; diag[i].ws_peak = (int64_t)ar.peak; }
  };
  return launch(count, f, stream);
}

int ttgbf_negative_mass(const ttgbf_tt* hdr, const double* data, int64_t cap, int count, const ttgbf_axis* axes,
                        int64_t guard, const int32_t* probes, int nprobes, double* out, void* ws, int64_t ws_bytes,
                        int32_t* status, void* stream) {
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    Arena ar = make_arena(ws, ws_bytes, i);
    const int d = hdr[i].d;
    int st = body_negmass(c, ar, hdr + i, data + (int64_t)i * cap, axes + (int64_t)i * d, guard, probes, nprobes,
                          out + i, make_stage_smem(smem).sm);
    if (c.leader()) status[i] = st;
  };
  return launch(count, f, stream);
}

int ttgbf_eval_blackbox(int kind, const ttgbf_model* model, const ttgbf_gauss* prior, const ttgbf_filter_io* io,
                        const ttgbf_tt* tt_hdr, const double* tt, int64_t tt_cap, int count, const int32_t* idx,
                        int64_t K, double* out, void* ws, int64_t ws_bytes, int32_t* status, void* stream) {
  if (kind < TTGBF_BB_GAUSS || kind > TTGBF_BB_REALIGN) return TTGBF_E_ARG;
  if (kind == TTGBF_BB_GAUSS && prior == nullptr) return TTGBF_E_ARG;
  if (kind == TTGBF_BB_REALIGN && (tt_hdr == nullptr || tt == nullptr)) return TTGBF_E_ARG;
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    Arena ar = make_arena(ws, ws_bytes, i);
    const int d = model->d;
    int st = body_eval_bb(c, ar, kind, *model, prior, io[i], tt_hdr ? tt_hdr + i : nullptr,
                          tt ? tt + (int64_t)i * tt_cap : nullptr, idx + (int64_t)i * K * d, K,
                          out + (int64_t)i * K, make_stage_smem(smem).sm);
    if (c.leader()) status[i] = st;
  };
  return launch(count, f, stream);
}

int ttgbf_rng_draws(int kind, uint64_t* state6, const int32_t* shape, int d, int64_t K, int64_t pop, int64_t size,
                    int64_t* out, void* ws, int64_t ws_bytes, int32_t* status, void* stream) {
  auto f = LAMBDA(const Ctx& c, int i, double* smem) {
    Arena ar = make_arena(ws, ws_bytes, i);
    XShared* sh = make_stage_smem(smem).xs;
    double* sm = make_stage_smem(smem).sm;
    auto body = [&]() -> int {
      if (c.leader()) {
        sh->rng.s_lo = state6[0]; sh->rng.s_hi = state6[1]; sh->rng.i_lo = state6[2]; sh->rng.i_hi = state6[3];
        sh->rng.has32 = (uint32_t)state6[4]; sh->rng.u32 = (uint32_t)state6[5];
      }
      c.sync();
      PcgJump* jt;
      ALLOC(jt, PcgJump, 1, ar);
      if (c.leader()) pcg_make_jump(sh->rng, jt);
      c.sync();
      if (kind == 0) {
        int64_t* tmp;
        int32_t* o32;
        ALLOC(tmp, int64_t, K * d + 1, ar);
        ALLOC(o32, int32_t, K * d + 1, ar);
        warp_integers(c, &sh->rng, jt, shape, d, K, o32, tmp);
        for (int64_t e = c.tid; e < K * d; e += c.nt) out[e] = o32[e];
      } else {
        int32_t* disp;
        int64_t *touch, *draws;
        uint8_t* flags;
        uint32_t* gset;
        ALLOC(disp, int32_t, pop + 16, ar);
        ALLOC(touch, int64_t, size + 16, ar);
        ALLOC(draws, int64_t, size + 16, ar);
        ALLOC(flags, uint8_t, size + 16, ar);
        ALLOC(gset, uint32_t, 8 * (size + 16) + 64, ar);
        par_fill_i32(c, disp, pop + 16, -1);
        c.sync();
        warp_choice(c, &sh->rng, jt, pop, size, out, disp, touch, draws, flags, reinterpret_cast<uint32_t*>(sm),
                    2 * SMEM_SCRATCH_DOUBLES, gset);
        double bad = 0.0;
        for (int64_t q = c.tid; q < pop; q += c.nt)
          if (disp[q] != -1) bad = 1.0;   // the displacement map must be restored
        if (block_max(c, bad) > 0.0) return E_ARG;
      }
      c.sync();
      if (c.leader()) {
        state6[0] = sh->rng.s_lo; state6[1] = sh->rng.s_hi; state6[2] = sh->rng.i_lo; state6[3] = sh->rng.i_hi;
        state6[4] = sh->rng.has32; state6[5] = sh->rng.u32;
      }
      return OK;
    };
    const int st = body();
    if (c.leader()) status[i] = st;
  };
  return launch(1, f, stream);
}
#endif

#if API_PART(1)
int64_t ttgbf_sizeof(int which) {
  switch (which) {
    case 0: return (int64_t)sizeof(ttgbf_axis);
    case 1: return (int64_t)sizeof(ttgbf_tt);
    case 2: return (int64_t)sizeof(ttgbf_cross_cfg);
    case 3: return (int64_t)sizeof(ttgbf_grid_cfg);
    case 4: return (int64_t)sizeof(ttgbf_diag);
    case 5: return (int64_t)sizeof(ttgbf_model);
    case 6: return (int64_t)sizeof(ttgbf_gauss);
    case 7: return (int64_t)sizeof(ttgbf_filter_io);
    case 8: return (int64_t)sizeof(ttgbf_run_cfg);
    case 9: return (int64_t)sizeof(ttgbf_step_rec);
    default: return -1;
  }
}
#endif

}  // extern "C"

#ifdef ENGINE_HOSTSIM
// Test-only hooks (host emulation build): numpy-stream draws through the
// same warp-parallel code the device cross uses.
extern "C" int ttgbf_test_draws(int kind, uint64_t* state6, const int* shape, int d, int64_t K, int64_t pop,
                                int64_t size, int64_t* out) {
  std::vector<double> smem(SMEM_DOUBLES);
  const Ctx c = make_ctx(smem.data(), 0, 1);
  Pcg64 g;
  g.s_lo = state6[0]; g.s_hi = state6[1]; g.i_lo = state6[2]; g.i_hi = state6[3];
  g.has32 = (uint32_t)state6[4]; g.u32 = (uint32_t)state6[5];
  PcgJump jt;
  pcg_make_jump(g, &jt);
  if (kind == 0) {
    std::vector<int64_t> tmp(K * d);
    std::vector<int32_t> o32(K * d);
    warp_integers(c, &g, &jt, shape, d, K, o32.data(), tmp.data());
    for (int64_t e = 0; e < K * d; ++e) out[e] = o32[e];
  } else {
    std::vector<int32_t> disp(pop + 16, -1);
    std::vector<int64_t> touch(size + 16), draws(size + 16);
    std::vector<uint8_t> flags(size + 16);
    std::vector<uint32_t> gset(4 * (size + 16) + 64);
    warp_choice(c, &g, &jt, pop, size, out, disp.data(), touch.data(), draws.data(), flags.data(),
                reinterpret_cast<uint32_t*>(smem.data() + SMEM_RED + SMEM_XBLK), 2 * SMEM_SCRATCH_DOUBLES, gset.data());
    for (int64_t q = 0; q < pop; ++q)
      if (disp[q] != -1) return 99;   // displacement map must be restored
  }
  state6[0] = g.s_lo; state6[1] = g.s_hi; state6[2] = g.i_lo; state6[3] = g.i_hi;
  state6[4] = g.has32; state6[5] = g.u32;
  return 0;
}
#endif

#ifdef ENGINE_HOSTSIM
// Test-only: blocked QR of A (m x n col-major, overwritten) and Q (m x k) = Q [I; 0].
extern "C" int ttgbf_test_qr(double* A, int m, int n, double* Q, void* ws, int64_t ws_bytes) {
  std::vector<double> smem(SMEM_DOUBLES);
  const Ctx c = make_ctx(smem.data(), 0, 1);
  Arena ar = make_arena(ws, ws_bytes, 0);
  const int k = m < n ? m : n;
  std::vector<double> tau(k), Ts(((k + NB - 1) / NB) * NB * NB);
  int st = geqrf_nb(c, ar, A, m, m, n, tau.data(), Ts.data(), smem.data() + SMEM_RED + SMEM_XBLK);
  if (st) return st;
  for (int64_t e = 0; e < (int64_t)m * k; ++e) Q[e] = ((e % m) == (e / m)) ? 1.0 : 0.0;
  return apply_q(c, ar, A, m, m, k, Ts.data(), false, Q, m, k, smem.data() + SMEM_RED + SMEM_XBLK);
}
#endif

#ifdef ENGINE_HOSTSIM
extern "C" int ttgbf_test_qr_apply(double* A, int m, int n, double* X, int nc, void* ws, int64_t ws_bytes) {
  std::vector<double> smem(SMEM_DOUBLES);
  const Ctx c = make_ctx(smem.data(), 0, 1);
  Arena ar = make_arena(ws, ws_bytes, 0);
  const int k = m < n ? m : n;
  std::vector<double> tau(k), Ts(((k + NB - 1) / NB) * NB * NB);
  int st = geqrf_nb(c, ar, A, m, m, n, tau.data(), Ts.data(), smem.data() + SMEM_RED + SMEM_XBLK);
  if (st) return st;
  return apply_q(c, ar, A, m, m, k, Ts.data(), false, X, m, nc, smem.data() + SMEM_RED + SMEM_XBLK);
}
#endif

#ifdef ENGINE_HOSTSIM
// Test-only: the cross's core solve lstsq(A, B) (gelsy emulation) for an r x r
// A and r x nrhs B, both col-major; X r x nrhs col-major; *rank the rank used.
extern "C" int ttgbf_test_lstsq(const double* A, const double* B, int r, int nrhs, double* X, int* rank) {
  std::vector<double> smem(SMEM_DOUBLES);
  const Ctx c = make_ctx(smem.data(), 0, 1);
  std::vector<double> W((size_t)r * r), W2((size_t)r * r), tau(r), tau2(r), cn(r + 1);
  std::vector<int> jpvt(r);
  return lstsq_pivoted(c, A, 1, r, r, B, r, nrhs, X, r, W.data(), W2.data(), tau.data(), tau2.data(), jpvt.data(),
                       cn.data(), rank);
}
#endif
