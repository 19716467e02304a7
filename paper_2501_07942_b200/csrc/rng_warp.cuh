// Warp-parallel numpy-compatible draws (same streams as rng.cuh, bit-exact).
//
// Every draw sequence the cross makes has bounds that do not depend on the
// drawn values (integers: shape per column; Floyd: j = pop-size..pop-1 then
// the shuffle i = size-1..1; tail shuffle: i = pop-1..first).  So a warp can
// address the 32-bit PCG64 stream by position: lane l computes value P + l
// by jump-ahead (state_{m+k} = A_k state_m + C_k, k = 1..32) from a running
// base, 32 Lemire draws are evaluated in parallel, and only the rare
// rejection is resolved one value at a time.  The final generator state
// (incl. numpy's buffered high half) is that of the last value consumed.
//
// On the host emulation the 32 "lanes" are looped; the logic is identical.
#pragma once
#include "rng.cuh"

namespace tg {

constexpr int JMAX = 160;   // jump table: k = 1..JMAX steps (a CTA looks 128 outputs ahead)
struct PcgJump {
  uint64_t a_lo[JMAX], a_hi[JMAX], c_lo[JMAX], c_hi[JMAX];   // k = 1..JMAX at index k-1
};

HD void pcg_make_jump(const Pcg64& g, PcgJump* j) {
  const u128 mult = (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;
  const u128 inc = (((u128)g.i_hi) << 64) | g.i_lo;
  u128 A = mult, C = inc;
  for (int k = 0; k < JMAX; ++k) {
    j->a_lo[k] = (uint64_t)A; j->a_hi[k] = (uint64_t)(A >> 64);
    j->c_lo[k] = (uint64_t)C; j->c_hi[k] = (uint64_t)(C >> 64);
    A = A * mult;
    C = C * mult + inc;
  }
}

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

// Position-addressed view of the 32-bit numpy stream: value p of the
// current call is the buffered high half g.u32 (p = 0 when g.has32), else
// half (p - off) % 2 of 64-bit output o = (p - off) / 2, whose source state
// is g.s advanced o + 1 steps.  `base` holds g.s advanced `ob` steps; any
// state within 32 steps of it is one jump-table multiply-add away.  All
// lanes keep identical copies (uniform updates), so no serial bookkeeping.
struct StreamPos {
  u128 g0;          // g.s at entry
  u128 base;        // g.s advanced ob steps
  int64_t ob;
  int off;          // 1 if the call starts with a buffered half
  uint32_t u32_0;   // that buffered half
};

HD u128 jump_k(const PcgJump* jt, u128 s, int k) {   // k in [1, JMAX]
  const u128 A = (((u128)jt->a_hi[k - 1]) << 64) | jt->a_lo[k - 1];
  const u128 C = (((u128)jt->c_hi[k - 1]) << 64) | jt->c_lo[k - 1];
  return A * s + C;
}

// state after `steps` steps from g0 (steps >= ob), rebasing base forward
HD u128 sp_state(StreamPos& sp, const PcgJump* jt, int64_t steps) {
  while (steps - sp.ob > 32) { sp.base = jump_k(jt, sp.base, 32); sp.ob += 32; }
  return steps == sp.ob ? sp.base : jump_k(jt, sp.base, (int)(steps - sp.ob));
}

// same, without moving base (per-thread lookahead, steps - ob in [0, JMAX])
HD u128 sp_peek(const StreamPos& sp, const PcgJump* jt, int64_t steps) {
  return steps == sp.ob ? sp.base : jump_k(jt, sp.base, (int)(steps - sp.ob));
}

HD uint32_t sp_value(const StreamPos& sp, const PcgJump* jt, int64_t p) {
  if (p < sp.off) return sp.u32_0;
  const int64_t o = (p - sp.off) >> 1;
  const u128 st = sp_peek(sp, jt, o + 1);
  const uint64_t out = xsl_rr((uint64_t)(st >> 64), (uint64_t)st);
  return ((p - sp.off) & 1) ? (uint32_t)(out >> 32) : (uint32_t)out;
}

// move base so that value p (and the next 32 values) are peekable
HD void sp_seek(StreamPos& sp, const PcgJump* jt, int64_t p) {
  const int64_t o = p < sp.off ? 0 : (p - sp.off) >> 1;
  while (o - sp.ob > 32) { sp.base = jump_k(jt, sp.base, 32); sp.ob += 32; }
  if (o > sp.ob) { sp.base = jump_k(jt, sp.base, (int)(o - sp.ob)); sp.ob = o; }
}

// n bounded draws out[t] = bounded(bound(t)), bound(t) in [0, 2^32-2].
// All CTA threads work: per round thread l evaluates draw t + l from stream
// value P + l (jump-ahead from a common base, at most 129 outputs away), the
// first rejection or zero bound in the round (CTA min) ends the accepted run
// and is resolved on its own, identically by every thread.  Values written
// beyond the first rejection are rewritten by later rounds.  g is left as
// numpy leaves it.
template <class Bound>
HDN void warp_draws(const Ctx& c, Pcg64* g, const PcgJump* jt, int64_t n, Bound bound, int64_t* out) {
  if (n > 0) {
    StreamPos sp;
    sp.g0 = (((u128)g->s_hi) << 64) | g->s_lo;
    sp.base = sp.g0;
    sp.ob = 0;
    sp.off = g->has32 ? 1 : 0;
    sp.u32_0 = g->u32;
    int64_t P = 0;   // stream values consumed
    int64_t t = 0;
    while (t < n) {
      // base at the output holding value P: values P .. P + nt - 1 are <= nt/2 + 1 steps away
      const int64_t o = P < sp.off ? 0 : (P - sp.off) >> 1;
      while (o - sp.ob > JMAX) { sp.base = jump_k(jt, sp.base, JMAX); sp.ob += JMAX; }
      if (o > sp.ob) { sp.base = jump_k(jt, sp.base, (int)(o - sp.ob)); sp.ob = o; }
      const int m = (int)lmin(c.nt, n - t);
      int first = m;
      for (int l = c.tid; l < m; l += c.nt) {
        const uint64_t b = bound(t + l);
        uint64_t res = 0;
        const bool rej = b == 0 || !lemire_try(sp_value(sp, jt, P + l), b, &res);
        if (rej) first = imin(first, l);
        else out[t + l] = (int64_t)res;
      }
      const int f = (int)(-block_max(c, -(double)first));
      t += f;
      P += f;
      if (f < m) {
        // draw t: zero bound (no value consumed) or Lemire rejection loop
        const uint64_t b = bound(t);
        if (b == 0) {
          if (c.leader()) out[t] = 0;
        } else {
          while (true) {
            const int64_t o2 = P < sp.off ? 0 : (P - sp.off) >> 1;
            while (o2 - sp.ob > JMAX) { sp.base = jump_k(jt, sp.base, JMAX); sp.ob += JMAX; }
            if (o2 > sp.ob) { sp.base = jump_k(jt, sp.base, (int)(o2 - sp.ob)); sp.ob = o2; }
            uint64_t res = 0;
            const bool ok = lemire_try(sp_value(sp, jt, P), b, &res);
            ++P;
            if (ok) {
              if (c.leader()) out[t] = (int64_t)res;
              break;
            }
          }
        }
        t += 1;
      }
    }
    // numpy state after the last consumed value
    if (P > 0 && P - 1 >= sp.off) {
      const int64_t o = (P - 1 - sp.off) >> 1;
      const bool low = ((P - 1 - sp.off) & 1) == 0;
      const u128 st = sp_state(sp, jt, o + 1);
      const uint64_t outv = xsl_rr((uint64_t)(st >> 64), (uint64_t)st);
      if (c.leader()) {
        g->s_lo = (uint64_t)st;
        g->s_hi = (uint64_t)(st >> 64);
        g->has32 = low ? 1u : 0u;          // low half consumed: high half buffered
        g->u32 = (uint32_t)(outv >> 32);   // buffered half, or the stale consumed one
      }
    } else if (P > 0) {                    // only the buffered half was consumed
      if (c.leader()) g->has32 = 0;
    }
  }
  c.sync();
}

struct BoundCols {
  const int* shape;
  int d;
  HD uint64_t operator()(int64_t t) const { return (uint64_t)(shape[(int)t % d] - 1); }   // t < 2^31
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
                       int32_t* out32, int64_t* tmp) {
  warp_draws(c, g, jt, K * d, BoundCols{shape, d}, tmp);
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

HDN int64_t scan_offsets(const Ctx& c, int64_t mine, int64_t* total);   // cache.cuh

// rng.choice(pop, size, replace=False) with pre-drawn bounds.
// disp: >= pop int32 all -1 (restored); touch, draws: >= size int64;
// flags: >= size bytes; sset: shared scratch (sset_words32 uint32);
// gset: global scratch >= 2*(gen_mask(1.2*size)+1) uint32.
HDN void warp_choice(const Ctx& c, Pcg64* g, const PcgJump* jt, int64_t pop, int64_t size, int64_t* out,
                     int32_t* disp, int64_t* touch, int64_t* draws, uint8_t* flags, uint32_t* sset,
                     int64_t sset_words32, uint32_t* gset) {
  if (pop > 10000 && size > pop / 50) {
    int64_t first = pop - size;
    if (first < 1) first = 1;
    const int64_t ns = pop - first;
    warp_draws(c, g, jt, ns, BoundDown{pop - 1}, draws);   // draw t: j for i = pop-1-t
    const int64_t lo = pop - size;
    // Step t puts the value found at j_t into position i_t = pop-1-t and the
    // value of i_t into j_t.  A step whose j_t is drawn once and lies below
    // the i-range [first, pop) never meets another step: nobody else writes
    // j_t before it reads it (so it reads j_t itself), and what it writes
    // there is never read.  Those steps (the bulk: pop >> ns) are resolved by
    // all threads at once; only the steps with a repeated j or a j inside
    // the i-range are replayed in order (they read positions that only steps
    // of the same kind write).
    for (int64_t t = c.tid; t < ns; t += c.nt) flags[t] = draws[t] >= first ? 1 : 0;
    c.sync();
    for (int64_t t = c.tid; t < ns; t += c.nt) {
      const int64_t j = draws[t];
#if ENGINE_DEVICE
      const int32_t prev = atomicCAS(&disp[j], -1, -2 - (int32_t)t);
#else
      const int32_t prev = disp[j];
      if (prev == -1) disp[j] = -2 - (int32_t)t;
#endif
      if (prev != -1) { flags[t] = 1; flags[-2 - prev] = 1; }   // both the claimer and the repeat
    }
    c.sync();
    for (int64_t t = c.tid; t < ns; t += c.nt) disp[draws[t]] = -1;
    c.sync();
    // in-order list of the interacting steps (touch[0..nc))
    const int64_t chunk = (ns + c.nt - 1) / c.nt;
    const int64_t t0 = lmin(ns, chunk * c.tid), t1 = lmin(ns, t0 + chunk);
    int64_t mine = 0;
    for (int64_t t = t0; t < t1; ++t) {
      if (flags[t]) ++mine;
      else if (pop - 1 - t >= lo) out[pop - 1 - t - lo] = draws[t];
    }
    int64_t nc = 0;
    int64_t off = scan_offsets(c, mine, &nc);
    for (int64_t t = t0; t < t1; ++t)
      if (flags[t]) touch[off++] = t;
    c.sync();
    swap_resolve(
        c, nc, [=](int64_t q) { return pop - 1 - touch[q]; }, [=](int64_t q) { return draws[touch[q]]; },
        [=](int64_t pos) { const int32_t v = disp[pos]; return v < 0 ? pos : (int64_t)v; },
        [=](int64_t pos, int64_t v) { disp[pos] = (int32_t)v; },
        [=](int64_t, int64_t pos, int64_t v) {
          if (pos >= lo) out[pos - lo] = v;
        });
    c.sync();
    for (int64_t q = c.tid; q < nc; q += c.nt) disp[draws[touch[q]]] = -1;
    c.sync();
    return;
  }
  // Floyd: draws val_t for j_t = pop-size+t, then the shuffle draws (i = size-1..1)
  warp_draws(c, g, jt, size, BoundUp{pop - size}, draws);
  int64_t* sdraws = touch;
  warp_draws(c, g, jt, size > 1 ? size - 1 : 0, BoundDown{size - 1}, sdraws);
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
  // Floyd's collisions: step t collides when its value was drawn before, or
  // when the value is the j of an earlier step that itself collided (and so
  // inserted its j).  That chain only walks to smaller t over read-only data,
  // so every flagged step resolves itself independently.
  for (int64_t t = c.tid; t < size; t += c.nt) {
    if (!(flags[t] & 2)) continue;
    int64_t cur = t;
    bool coll = false;
    while (true) {
      const uint32_t v = (uint32_t)draws[cur];
      uint64_t h = v & mask;
      while (keys[h] != v) h = (h + 1) & mask;
      if (mins[h] < (uint32_t)cur) { coll = true; break; }
      if ((int64_t)v < jlo) break;
      const int64_t sidx = (int64_t)v - jlo;
      if (sidx >= cur) break;
      cur = sidx;
    }
    if (coll) out[t] = jlo + t;
  }
  c.sync();
  // Fisher-Yates shuffle of out[0..size): step q swaps i = size-1-q and j = sdraws[q]
#if ENGINE_DEVICE
  if (size >= 64 && size <= 4096 && 2 * size + (size + 1) / 2 <= sset_words32) {
    // All steps at once.  Position i_q is final after step q and receives
    // V(j_q, q), the value at j_q just before step q.  A position p is
    // written before its own step only by the steps that drew j = p, each
    // moving A(q') = V(i_q', q') there; so with the writers of every position
    // listed in step order,
    //   A(q) = A(latest q' < q with j_q' = i_q)   or out[i_q] if none,
    //   F(q) = A(q) if j_q = i_q, else A(latest q' < q with j_q' = j_q) or out[j_q].
    // The chains only walk to earlier steps (short: a position is drawn
    // ~ln(size/i) times).
    const int ns = (int)size - 1;
    int* cnt = reinterpret_cast<int*>(sset);       // writers per position, then fill cursor
    int* start = cnt + size;                       // list offsets
    uint16_t* list = reinterpret_cast<uint16_t*>(start + size);   // writer steps by position, ascending
    for (int pq = c.tid; pq < (int)size; pq += c.nt) cnt[pq] = 0;
    c.sync();
    for (int q = c.tid; q < ns; q += c.nt) atomicAdd(&cnt[(int)sdraws[q]], 1);
    c.sync();
    {
      const int chunk = ((int)size + c.nt - 1) / c.nt;
      const int p0 = imin((int)size, chunk * c.tid), p1 = imin((int)size, p0 + chunk);
      int64_t mine = 0;
      for (int pq = p0; pq < p1; ++pq) mine += cnt[pq];
      int64_t tot;
      int64_t off = scan_offsets(c, mine, &tot);
      for (int pq = p0; pq < p1; ++pq) {
        start[pq] = (int)off;
        off += cnt[pq];
        cnt[pq] = 0;
      }
    }
    c.sync();
    for (int q = c.tid; q < ns; q += c.nt) {
      const int j = (int)sdraws[q];
      list[start[j] + atomicAdd(&cnt[j], 1)] = (uint16_t)q;
    }
    c.sync();
    for (int pq = c.tid; pq < (int)size; pq += c.nt) {
      const int nq = cnt[pq];
      uint16_t* l = list + start[pq];
      for (int a = 1; a < nq; ++a) {   // insertion sort (lists of 1-3 steps)
        const uint16_t x = l[a];
        int b2 = a - 1;
        while (b2 >= 0 && l[b2] > x) { l[b2 + 1] = l[b2]; --b2; }
        l[b2 + 1] = x;
      }
    }
    c.sync();
    auto latest = [&](int pq, int q) -> int {   // latest writer of position pq before step q
      const uint16_t* l = list + start[pq];
      for (int k = cnt[pq] - 1; k >= 0; --k)
        if ((int)l[k] < q) return (int)l[k];
      return -1;
    };
    auto before = [&](int q) -> int64_t {       // A(q) = V(i_q, q)
      int x = q;
      while (true) {
        const int pa = latest((int)size - 1 - x, x);
        if (pa < 0) break;
        x = pa;
      }
      return out[size - 1 - x];
    };
    for (int q = c.tid; q <= ns; q += c.nt) {
      int64_t f;
      if (q == ns) {                            // position 0 is never an i: its last writer decides
        const int pf = latest(0, ns);
        f = pf >= 0 ? before(pf) : out[0];
      } else {
        const int i = (int)size - 1 - q, j = (int)sdraws[q];
        if (j == i) {
          f = before(q);
        } else {
          const int pf = latest(j, q);
          f = pf >= 0 ? before(pf) : out[j];
        }
      }
      draws[q] = f;
    }
    c.sync();
    for (int q = c.tid; q <= ns; q += c.nt) out[q == ns ? 0 : size - 1 - q] = draws[q];
    c.sync();
    return;
  }
#endif
  swap_resolve(
      c, size > 1 ? size - 1 : 0, [=](int64_t q) { return size - 1 - q; }, [=](int64_t q) { return sdraws[q]; },
      [=](int64_t pos) { return out[pos]; }, [=](int64_t pos, int64_t v) { out[pos] = v; },
      [=](int64_t, int64_t pos, int64_t v) { out[pos] = v; });
  c.sync();
}

}  // namespace tg
