// numpy-compatible random draws on the device.
//
// The reference drives its cross with numpy.random.Generator(PCG64)
// (tt_algorithms.py:488) and draws with `integers(0, shape, size=(K, d))`
// and `choice(n, size, replace=False)`.  Reproducing those streams exactly
// makes the device cross replay the reference's decisions.  Restated here:
//   * PCG64 (XSL-RR 128/64): state = state*M + inc; out = rotr(hi^lo, hi>>58)
//   * next_uint32 buffers the high half of a 64-bit draw (low half first)
//   * bounded draws on [0, rng] with rng < 2^32 use Lemire's multiply-shift
//     with rejection threshold (2^32 - 1 - rng) mod (rng + 1)  (lower is 32-bit)
//   * choice without replacement: Floyd's algorithm with a linear-probing set
//     sized to the next power of two above 1.2*size, followed by a
//     Fisher-Yates shuffle of the result; or, when pop > 10000 and
//     size > pop/50, a tail Fisher-Yates of arange(pop).
// Validated against numpy itself by tests/test_rng.py.
// All functions here are SERIAL: call them from the CTA leader only.
#pragma once
#include "common.cuh"

namespace tg {

typedef unsigned __int128 u128;

struct Pcg64 {
  uint64_t s_lo, s_hi, i_lo, i_hi;   // 128-bit state and increment
  uint32_t has32;
  uint32_t u32;
};

HD uint64_t pcg_next64(Pcg64& g) {
  const u128 mult = (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;
  u128 s = (((u128)g.s_hi) << 64) | g.s_lo;
  u128 inc = (((u128)g.i_hi) << 64) | g.i_lo;
  s = s * mult + inc;
  g.s_lo = (uint64_t)s;
  g.s_hi = (uint64_t)(s >> 64);
  uint64_t x = g.s_hi ^ g.s_lo;
  unsigned r = (unsigned)(g.s_hi >> 58);
  return (x >> r) | (x << ((64u - r) & 63u));
}

HD uint32_t pcg_next32(Pcg64& g) {
  if (g.has32) {
    g.has32 = 0;
    return g.u32;
  }
  uint64_t n = pcg_next64(g);
  g.has32 = 1;
  g.u32 = (uint32_t)(n >> 32);
  return (uint32_t)n;
}

// uniform integer on [0, rng] (closed), rng < 2^32 for every draw we make.
HD uint64_t pcg_bounded(Pcg64& g, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFull) return pcg_next32(g);
  const uint32_t excl = (uint32_t)rng + 1u;
  uint64_t m = (uint64_t)pcg_next32(g) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t th = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % excl;
    while (left < th) {
      m = (uint64_t)pcg_next32(g) * excl;
      left = (uint32_t)m;
    }
  }
  return m >> 32;
}

// rng.integers(0, shape, size=(K, d)) -> row-major int32 out[K*d]
HD void pcg_integers(Pcg64& g, const int* shape, int d, int64_t K, int32_t* out) {
  for (int64_t i = 0; i < K; ++i)
    for (int k = 0; k < d; ++k) out[i * d + k] = (int32_t)pcg_bounded(g, (uint64_t)(shape[k] - 1));
}

HD uint64_t gen_mask(uint64_t m) {
  m |= m >> 1; m |= m >> 2; m |= m >> 4; m |= m >> 8; m |= m >> 16; m |= m >> 32;
  return m;
}

// Workspace (in uint64 words) needed by pcg_choice for (pop, size).
HD int64_t choice_ws_words(int64_t pop, int64_t size) {
  if (pop > 10000 && size > pop / 50) {
    uint64_t m = gen_mask((uint64_t)(4 * size + 8));
    return (int64_t)(2 * (m + 1));
  }
  uint64_t m = gen_mask((uint64_t)(1.2 * (double)size));
  return (int64_t)(m + 1);
}

// rng.choice(pop, size=size, replace=False) -> out[size] (int64)
HD void pcg_choice(Pcg64& g, int64_t pop, int64_t size, int64_t* out, uint64_t* ws) {
  if (pop > 10000 && size > pop / 50) {
    // tail shuffle of a virtual arange(pop): sparse map position -> value
    const uint64_t mask = gen_mask((uint64_t)(4 * size + 8));
    uint64_t* keys = ws;
    uint64_t* vals = ws + (mask + 1);
    for (uint64_t i = 0; i <= mask; ++i) keys[i] = ~0ull;
    auto find = [&](uint64_t pos) -> uint64_t {
      uint64_t h = (pos * 0x9E3779B97F4A7C15ull) >> 11;
      uint64_t loc = h & mask;
      while (keys[loc] != ~0ull && keys[loc] != pos) loc = (loc + 1) & mask;
      return loc;
    };
    auto get = [&](uint64_t pos) -> uint64_t {
      uint64_t loc = find(pos);
      return keys[loc] == ~0ull ? pos : vals[loc];
    };
    auto put = [&](uint64_t pos, uint64_t v) {
      uint64_t loc = find(pos);
      keys[loc] = pos;
      vals[loc] = v;
    };
    int64_t first = pop - size;
    if (first < 1) first = 1;
    for (int64_t i = pop - 1; i >= first; --i) {
      uint64_t j = pcg_bounded(g, (uint64_t)i);
      uint64_t vj = get(j), vi = get((uint64_t)i);
      put(j, vi);
      put((uint64_t)i, vj);
    }
    for (int64_t t = 0; t < size; ++t) out[t] = (int64_t)get((uint64_t)(pop - size + t));
    return;
  }
  const uint64_t mask = gen_mask((uint64_t)(1.2 * (double)size));
  uint64_t* hs = ws;
  for (uint64_t i = 0; i <= mask; ++i) hs[i] = ~0ull;
  for (int64_t j = pop - size; j < pop; ++j) {
    uint64_t val = pcg_bounded(g, (uint64_t)j);
    uint64_t loc = val & mask;
    while (hs[loc] != ~0ull && hs[loc] != val) loc = (loc + 1) & mask;
    if (hs[loc] == ~0ull) {
      hs[loc] = val;
      out[j - pop + size] = (int64_t)val;
    } else {
      loc = (uint64_t)j & mask;
      while (hs[loc] != ~0ull) loc = (loc + 1) & mask;
      hs[loc] = (uint64_t)j;
      out[j - pop + size] = j;
    }
  }
  for (int64_t i = size - 1; i >= 1; --i) {
    int64_t j = (int64_t)pcg_bounded(g, (uint64_t)i);
    int64_t t = out[j];
    out[j] = out[i];
    out[i] = t;
  }
}

// Cooperative form of pcg_choice with identical output and stream use.
// All CTA threads call it; warp 0 does the work (lane 0 draws).
//  * tail shuffle: the virtual arange(pop) lives in `disp` (pop int32 entries,
//    -1 = untouched; restored to -1 on return).  Draws are made 32 at a
//    time, the 32 pairs of displacement loads are issued by 32 lanes at once,
//    then lane 0 resolves the batch in order against its own pending stores.
//  * Floyd: the probing set lives in shared memory when it fits (sset).
// jb: >= 128 int64 of shared scratch; touch: >= size int64 (global).
HDN void choice_coop(const Ctx& c, Pcg64* g, int64_t pop, int64_t size, int64_t* out, int32_t* disp,
                     uint64_t* sset, int64_t sset_words, uint64_t* gset, int64_t* jb, int64_t* touch) {
#if ENGINE_DEVICE
  const int lane = c.tid & 31;
  const bool w0 = c.tid < 32;
  const int stride = 32;
#else
  const int lane = 0;
  const bool w0 = true;
  const int stride = 1;
#endif
  if (pop > 10000 && size > pop / 50) {
    int64_t first = pop - size;
    if (first < 1) first = 1;
    const int64_t nsteps = pop - first;
    if (w0) {
      int64_t* ld = jb + 32;
      int64_t* ldi = jb + 64;
      for (int64_t i0 = pop - 1; i0 >= first; i0 -= 32) {
        const int cnt = (int)lmin(32, i0 - first + 1);
        if (lane == 0)
          for (int t = 0; t < cnt; ++t) jb[t] = (int64_t)pcg_bounded(*g, (uint64_t)(i0 - t));
#if ENGINE_DEVICE
        __syncwarp();
#endif
        for (int t = lane; t < cnt; t += stride) {
          ld[t] = disp[jb[t]];
          ldi[t] = disp[i0 - t];
        }
#if ENGINE_DEVICE
        __syncwarp();
#endif
        if (lane == 0) {
          int64_t sp[32], sv[32];
          int ns = 0;
          for (int t = 0; t < cnt; ++t) {
            const int64_t i = i0 - t, j = jb[t];
            int64_t vj = ld[t] < 0 ? j : ld[t];
            int64_t vi = ldi[t] < 0 ? i : ldi[t];
            for (int q = ns - 1; q >= 0; --q)
              if (sp[q] == j) { vj = sv[q]; break; }
            for (int q = ns - 1; q >= 0; --q)
              if (sp[q] == i) { vi = sv[q]; break; }
            int q = 0;
            while (q < ns && sp[q] != j) ++q;
            sp[q] = j;
            sv[q] = vi;
            if (q == ns) ++ns;
            if (i >= pop - size) out[i - (pop - size)] = vj;
            touch[(pop - 1) - i] = j;
          }
          for (int q = 0; q < ns; ++q) disp[sp[q]] = (int32_t)sv[q];
        }
#if ENGINE_DEVICE
        __syncwarp();
#endif
      }
    }
    c.sync();
    for (int64_t q = c.tid; q < nsteps; q += c.nt) disp[touch[q]] = -1;
    c.sync();
    return;
  }
  if (c.leader()) {
    const uint64_t mask = gen_mask((uint64_t)(1.2 * (double)size));
    uint64_t* hs = (int64_t)(mask + 1) <= sset_words ? sset : gset;
    for (uint64_t i = 0; i <= mask; ++i) hs[i] = ~0ull;
    for (int64_t j = pop - size; j < pop; ++j) {
      uint64_t val = pcg_bounded(*g, (uint64_t)j);
      uint64_t loc = val & mask;
      while (hs[loc] != ~0ull && hs[loc] != val) loc = (loc + 1) & mask;
      if (hs[loc] == ~0ull) {
        hs[loc] = val;
        out[j - pop + size] = (int64_t)val;
      } else {
        loc = (uint64_t)j & mask;
        while (hs[loc] != ~0ull) loc = (loc + 1) & mask;
        hs[loc] = (uint64_t)j;
        out[j - pop + size] = j;
      }
    }
    for (int64_t i = size - 1; i >= 1; --i) {
      int64_t j = (int64_t)pcg_bounded(*g, (uint64_t)i);
      int64_t t = out[j];
      out[j] = out[i];
      out[i] = t;
    }
  }
  c.sync();
}

}  // namespace tg
