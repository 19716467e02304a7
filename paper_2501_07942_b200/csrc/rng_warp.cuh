// Warp-parallel numpy-compatible draws (same streams as rng.cuh, bit-exact).
//
// Every draw sequence the cross makes has bounds that do not depend on the
// drawn values (integers: shape per column; Floyd: j = pop-size..pop-1 then
// the shuffle i = size-1..1; tail shuffle: i = pop-1..first).  So a warp can
// produce the 32-bit PCG64 stream 64 values at a time by jump-ahead
// (state_{m+k} = A_k state_m + C_k, k = 1..32), evaluate 32 Lemire draws in
// parallel, and fall back to lane 0 only for the rare rejection.  The final
// generator state (incl. numpy's buffered high half) is restored from the
// source state of the last value consumed.
//
// On the host emulation the 32 "lanes" are looped; the logic is identical.
#pragma once
#include "rng.cuh"

namespace tg {

struct PcgJump {
  uint64_t a_lo[32], a_hi[32], c_lo[32], c_hi[32];   // k = 1..32 at index k-1
};

HD void pcg_make_jump(const Pcg64& g, PcgJump* j) {
  const u128 mult = (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;
  const u128 inc = (((u128)g.i_hi) << 64) | g.i_lo;
  u128 A = mult, C = inc;
  for (int k = 0; k < 32; ++k) {
    j->a_lo[k] = (uint64_t)A; j->a_hi[k] = (uint64_t)(A >> 64);
    j->c_lo[k] = (uint64_t)C; j->c_hi[k] = (uint64_t)(C >> 64);
    A = A * mult;
    C = C * mult + inc;
  }
}

constexpr int DB_CAP = 128;
struct DrawBuf {          // shared memory
  uint32_t v[DB_CAP];     // pending 32-bit values
  uint64_t slo[DB_CAP];   // source state (after the 64-bit output they came from)
  uint64_t shi[DB_CAP];
  uint32_t half[DB_CAP];  // 0 = low half (high half follows), 1 = high half / buffered
  int head, count;
  int last_slot_valid;
  uint64_t last_lo, last_hi;
  uint32_t last_half, last_next;
};

#if ENGINE_DEVICE
#define LANE_LOOP(l) for (int l = (c.tid & 31), _once = 0; _once < 1; ++_once)
#else
#define LANE_LOOP(l) for (int l = 0; l < 32; ++l)
#endif

HD uint64_t xsl_rr(uint64_t hi, uint64_t lo) {
  uint64_t x = hi ^ lo;
  unsigned r = (unsigned)(hi >> 58);
  return (x >> r) | (x << ((64u - r) & 63u));
}

// Append 64 fresh values (32 outputs) after compacting the buffer.  Warp 0.
HDN void db_refill(const Ctx& c, DrawBuf* db, uint64_t* base_lo, uint64_t* base_hi, const PcgJump* jt) {
  // compact: move pending values to the front
  if (c.leader() || !ENGINE_DEVICE) {
    if (db->head > 0) {
      for (int q = 0; q < db->count; ++q) {
        db->v[q] = db->v[db->head + q];
        db->slo[q] = db->slo[db->head + q];
        db->shi[q] = db->shi[db->head + q];
        db->half[q] = db->half[db->head + q];
      }
      db->head = 0;
    }
  }
#if ENGINE_DEVICE
  __syncwarp();
#endif
  const int cnt0 = db->count;
  const u128 base = (((u128)*base_hi) << 64) | *base_lo;
  uint64_t last_lo = 0, last_hi = 0;
  LANE_LOOP(l) {
    const u128 A = (((u128)jt->a_hi[l]) << 64) | jt->a_lo[l];
    const u128 C = (((u128)jt->c_hi[l]) << 64) | jt->c_lo[l];
    const u128 st = A * base + C;
    const uint64_t slo = (uint64_t)st, shi = (uint64_t)(st >> 64);
    const uint64_t o = xsl_rr(shi, slo);
    const int q = cnt0 + 2 * l;
    db->v[q] = (uint32_t)o;
    db->v[q + 1] = (uint32_t)(o >> 32);
    db->slo[q] = slo; db->shi[q] = shi; db->half[q] = 0;
    db->slo[q + 1] = slo; db->shi[q + 1] = shi; db->half[q + 1] = 1;
    if (l == 31) { last_lo = slo; last_hi = shi; }
  }
#if ENGINE_DEVICE
  last_lo = __shfl_sync(0xffffffffu, last_lo, 31);
  last_hi = __shfl_sync(0xffffffffu, last_hi, 31);
  __syncwarp();
#endif
  *base_lo = last_lo;
  *base_hi = last_hi;
  if (c.leader() || !ENGINE_DEVICE) db->count = cnt0 + 64;
#if ENGINE_DEVICE
  __syncwarp();
#endif
}

// Lemire draw from value x with inclusive bound b (b < 2^32-1, b > 0):
// returns true and *res if accepted.
HD bool lemire_try(uint32_t x, uint64_t b, uint64_t* res) {
  const uint32_t excl = (uint32_t)b + 1u;
  const uint64_t m = (uint64_t)x * excl;
  const uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t th = (uint32_t)(0xFFFFFFFFu - (uint32_t)b) % excl;
    if (left < th) return false;
  }
  *res = m >> 32;
  return true;
}

HD void db_pop(DrawBuf* db) {
  const int q = db->head;
  db->last_slot_valid = 1;
  db->last_lo = db->slo[q];
  db->last_hi = db->shi[q];
  db->last_half = db->half[q];
  db->last_next = db->v[q];   // value consumed (numpy keeps it as the stale buffer)
  db->head++;
  db->count--;
}

// n bounded draws out[t] = bounded(bound(t)), bound(t) in [0, 2^32-2].
// All CTA threads call; warp 0 works.  g is updated to the numpy state.
template <class Bound>
HDN void warp_draws(const Ctx& c, Pcg64* g, const PcgJump* jt, int64_t n, Bound bound, int64_t* out,
                    DrawBuf* db) {
  const bool w0 = !ENGINE_DEVICE || c.tid < 32;
  if (w0 && n > 0) {
    uint64_t base_lo = g->s_lo, base_hi = g->s_hi;
    if (c.leader() || !ENGINE_DEVICE) {
      db->head = 0;
      db->count = 0;
      db->last_slot_valid = 0;
      if (g->has32) {
        db->v[0] = g->u32;
        db->slo[0] = g->s_lo;
        db->shi[0] = g->s_hi;
        db->half[0] = 1;
        db->count = 1;
      }
    }
#if ENGINE_DEVICE
    __syncwarp();
#endif
    int64_t t = 0;
    while (t < n) {
      if (db->count < 40) db_refill(c, db, &base_lo, &base_hi, jt);
      const int m = (int)lmin(32, n - t);
      // parallel phase: lane l draws t+l with value head+l (no rejection assumed)
      unsigned rejmask = 0;
      LANE_LOOP(l) {
        bool rej = false;
        uint64_t res = 0;
        if (l < m) {
          const uint64_t b = bound(t + l);
          if (b == 0) rej = true;          // consumes nothing: handle serially
          else rej = !lemire_try(db->v[db->head + l], b, &res);
          if (!rej) out[t + l] = (int64_t)res;
        }
#if ENGINE_DEVICE
        rejmask = __ballot_sync(0xffffffffu, rej && l < m);
#else
        if (rej && l < m) rejmask |= (1u << l);
#endif
      }
      int f = m;
      if (rejmask) {
#if ENGINE_DEVICE
        f = __ffs(rejmask) - 1;
#else
        f = 0;
        while (!((rejmask >> f) & 1u)) ++f;
#endif
      }
      // accept draws t..t+f-1 (lanes >= f may have written provisional outs; they are redrawn)
      if (c.leader() || !ENGINE_DEVICE) {
        for (int q = 0; q < f; ++q) db_pop(db);
      }
#if ENGINE_DEVICE
      __syncwarp();
#endif
      t += f;
      if (f < m) {
        // serial draw for index t on lane 0 (rejection or zero bound)
        bool done = false;
        while (!done) {
          if (db->count < 2) db_refill(c, db, &base_lo, &base_hi, jt);
          if (c.leader() || !ENGINE_DEVICE) {
            const uint64_t b = bound(t);
            if (b == 0) {
              out[t] = 0;
              done = true;
            } else {
              while (db->count > 0) {
                uint64_t res;
                const bool ok = lemire_try(db->v[db->head], b, &res);
                db_pop(db);
                if (ok) { out[t] = (int64_t)res; done = true; break; }
              }
            }
          }
#if ENGINE_DEVICE
          __syncwarp();
          done = __shfl_sync(0xffffffffu, (int)done, 0);
          __syncwarp();
#endif
        }
        t += 1;
      }
    }
    // restore numpy state from the last consumed value
    if ((c.leader() || !ENGINE_DEVICE) && db->last_slot_valid) {
      g->s_lo = db->last_lo;
      g->s_hi = db->last_hi;
      if (db->last_half == 0) {   // low half consumed: numpy buffers the high half
        g->has32 = 1;
        g->u32 = db->v[db->head];
      } else {
        g->has32 = 0;
        g->u32 = db->last_next;
      }
    }
  }
  c.sync();
}

struct BoundCols {
  const int* shape;
  int d;
  HD uint64_t operator()(int64_t t) const { return (uint64_t)(shape[t % d] - 1); }
};
struct BoundUp {   // j = lo + t
  int64_t lo;
  HD uint64_t operator()(int64_t t) const { return (uint64_t)(lo + t); }
};
struct BoundDown {  // i = hi - t
  int64_t hi;
  HD uint64_t operator()(int64_t t) const { return (uint64_t)(hi - t); }
};

// rng.integers(0, shape, size=(K, d)) -> out32 (K*d), via an int64 scratch
HDN void warp_integers(const Ctx& c, Pcg64* g, const PcgJump* jt, const int* shape, int d, int64_t K,
                       int32_t* out32, int64_t* tmp, DrawBuf* db) {
  warp_draws(c, g, jt, K * d, BoundCols{shape, d}, tmp, db);
  for (int64_t e = c.tid; e < K * d; e += c.nt) out32[e] = (int32_t)tmp[e];
  c.sync();
}

// Warp-batched resolution of a Fisher-Yates swap sequence: step t swaps
// positions I(t) > ... (decreasing) and J(t) <= I(t).  Values of untouched
// positions come from get(pos); set(pos, v) writes; fin(t, pos_i, v) receives
// the final value of position I(t) (never touched again).  Lanes load the 32
// steps' operands at once; in-batch dependencies are resolved by shuffles.
template <class IFn, class JFn, class Get, class Set, class Fin>
HD void swap_resolve(const Ctx& c, int64_t ns, IFn I, JFn J, Get get, Set set, Fin fin) {
  const bool w0 = !ENGINE_DEVICE || c.tid < 32;
  if (!w0) return;
  for (int64_t t0 = 0; t0 < ns; t0 += 32) {
    const int m = (int)lmin(32, ns - t0);
#if ENGINE_DEVICE
    const int l = c.tid & 31;
    const bool act = l < m;
    const int64_t i = act ? I(t0 + l) : -1;
    const int64_t j = act ? J(t0 + l) : -2;
    const int64_t ldj = act ? get(j) : 0;
    const int64_t ldi = act ? get(i) : 0;
    int wj = -1, wi = -1, later = 0;
    for (int q = 0; q < 32; ++q) {
      const int64_t jq = __shfl_sync(0xffffffffu, j, q);
      if (q < l && q < m) {
        if (jq == j) wj = q;
        if (jq == i) wi = q;
      }
      if (q > l && q < m && jq == j) later = 1;
    }
    int64_t vi = ldi;
    for (int it = 0; it < 32; ++it) {
      const int64_t src = __shfl_sync(0xffffffffu, vi, wi < 0 ? l : wi);
      const int64_t nv = wi < 0 ? ldi : src;
      const bool ch = nv != vi;
      vi = nv;
      if (!__any_sync(0xffffffffu, ch)) break;
    }
    const int64_t viw = __shfl_sync(0xffffffffu, vi, wj < 0 ? l : wj);
    const int64_t vj = wj < 0 ? ldj : viw;
    if (act) {
      if (!later) set(j, vi);
      fin(t0 + l, i, vj);
    }
    __syncwarp();
#else
    int64_t Iv[32], Jv[32], VI[32], LDJ[32], LDI[32];
    for (int l = 0; l < m; ++l) {
      Iv[l] = I(t0 + l);
      Jv[l] = J(t0 + l);
      LDJ[l] = get(Jv[l]);
      LDI[l] = get(Iv[l]);
    }
    for (int l = 0; l < m; ++l) {
      int wi = -1;
      for (int q = 0; q < l; ++q) if (Jv[q] == Iv[l]) wi = q;
      VI[l] = wi < 0 ? LDI[l] : VI[wi];
    }
    for (int l = 0; l < m; ++l) {
      int wj = -1, later = 0;
      for (int q = 0; q < l; ++q) if (Jv[q] == Jv[l]) wj = q;
      for (int q = l + 1; q < m; ++q) if (Jv[q] == Jv[l]) later = 1;
      const int64_t vj = wj < 0 ? LDJ[l] : VI[wj];
      if (!later) set(Jv[l], VI[l]);
      fin(t0 + l, Iv[l], vj);
    }
#endif
  }
}

// rng.choice(pop, size, replace=False) with pre-drawn bounds.
// disp: >= pop int32 all -1 (restored); touch, draws: >= size int64;
// flags: >= size bytes; sset: shared scratch (sset_words32 uint32);
// gset: global scratch >= 2*(gen_mask(1.2*size)+1) uint32.
HDN void warp_choice(const Ctx& c, Pcg64* g, const PcgJump* jt, int64_t pop, int64_t size, int64_t* out,
                     int32_t* disp, int64_t* touch, int64_t* draws, uint8_t* flags, uint32_t* sset,
                     int64_t sset_words32, uint32_t* gset, DrawBuf* db) {
  if (pop > 10000 && size > pop / 50) {
    int64_t first = pop - size;
    if (first < 1) first = 1;
    const int64_t ns = pop - first;
    warp_draws(c, g, jt, ns, BoundDown{pop - 1}, draws, db);   // draw t: j for i = pop-1-t
    const int64_t lo = pop - size;
    swap_resolve(
        c, ns, [=](int64_t t) { return pop - 1 - t; }, [=](int64_t t) { return draws[t]; },
        [=](int64_t pos) { const int32_t v = disp[pos]; return v < 0 ? pos : (int64_t)v; },
        [=](int64_t pos, int64_t v) { disp[pos] = (int32_t)v; },
        [=](int64_t t, int64_t pos, int64_t v) {
          if (pos >= lo) out[pos - lo] = v;
          touch[t] = draws[t];
        });
    c.sync();
    for (int64_t q = c.tid; q < ns; q += c.nt) disp[touch[q]] = -1;
    c.sync();
    return;
  }
  // Floyd: draws val_t for j_t = pop-size+t, then the shuffle draws (i = size-1..1)
  warp_draws(c, g, jt, size, BoundUp{pop - size}, draws, db);
  int64_t* sdraws = touch;
  warp_draws(c, g, jt, size > 1 ? size - 1 : 0, BoundDown{size - 1}, sdraws, db);
  // first occurrence of each value: open addressing, key = value, payload = min t
  const uint64_t mask = gen_mask((uint64_t)(1.2 * (double)size));
  const int64_t tsz = (int64_t)mask + 1;
  uint32_t* keys = (2 * tsz <= sset_words32) ? sset : gset;
  uint32_t* mins = keys + tsz;
  for (int64_t q = c.tid; q < tsz; q += c.nt) { keys[q] = 0xFFFFFFFFu; mins[q] = 0xFFFFFFFFu; }
  c.sync();
  for (int64_t t = c.tid; t < size; t += c.nt) {
    const uint32_t v = (uint32_t)draws[t];
    uint64_t h = v & mask;
    while (true) {
#if ENGINE_DEVICE
      const uint32_t old = atomicCAS(&keys[h], 0xFFFFFFFFu, v);
      if (old == 0xFFFFFFFFu || old == v) { atomicMin(&mins[h], (uint32_t)t); break; }
#else
      if (keys[h] == 0xFFFFFFFFu || keys[h] == v) {
        keys[h] = v;
        if ((uint32_t)t < mins[h]) mins[h] = (uint32_t)t;
        break;
      }
#endif
      h = (h + 1) & mask;
    }
  }
  c.sync();
  // provisional outputs; flag steps that may collide (duplicate value or a
  // value in the j-range pop-size..)
  const int64_t jlo = pop - size;
  for (int64_t t = c.tid; t < size; t += c.nt) {
    const uint32_t v = (uint32_t)draws[t];
    uint64_t h = v & mask;
    while (keys[h] != v) h = (h + 1) & mask;
    const bool rare = mins[h] < (uint32_t)t || (int64_t)v >= jlo;
    flags[t] = rare ? 2 : 0;
    out[t] = (int64_t)v;
  }
  c.sync();
  // in-order resolution of the rare steps (leader): collided[t] lives in flags bit 0
  if (c.leader()) {
    for (int64_t t = 0; t < size; ++t) {
      if (!(flags[t] & 2)) continue;
      const uint32_t v = (uint32_t)draws[t];
      uint64_t h = v & mask;
      while (keys[h] != v) h = (h + 1) & mask;
      bool coll = mins[h] < (uint32_t)t;
      if (!coll && (int64_t)v >= jlo) {
        const int64_t sidx = (int64_t)v - jlo;
        coll = sidx < t && (flags[sidx] & 1);
      }
      if (coll) {
        out[t] = jlo + t;
        flags[t] |= 1;
      }
    }
  }
  c.sync();
  // Fisher-Yates shuffle of out[0..size): step q swaps i = size-1-q and j = sdraws[q]
  swap_resolve(
      c, size > 1 ? size - 1 : 0, [=](int64_t q) { return size - 1 - q; }, [=](int64_t q) { return sdraws[q]; },
      [=](int64_t pos) { return out[pos]; }, [=](int64_t pos, int64_t v) { out[pos] = v; },
      [=](int64_t, int64_t pos, int64_t v) { out[pos] = v; });
  c.sync();
}

}  // namespace tg
