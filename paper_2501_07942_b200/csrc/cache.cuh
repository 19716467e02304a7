// Memoised, counted, finiteness-checked evaluator (device form of
// _CachedEvaluator, tt_algorithms.py:137-208).
//
// Keys are the multi-index bit-packed lexicographically (index 0 most
// significant) into 128 bits, so key order == C-order flat-index order (the
// reference's `ravel_multi_index`, which overflows int64 at 129^10 -- the
// packed key does not).  Misses of one call are deduplicated, sorted
// ascending and appended in that order: insertion order is what
// `sample_cache` draws positions from, so it must match the reference.
#pragma once
#include "common.cuh"
#include "models.cuh"
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
#include <stdio.h>
#endif

namespace tg {

struct Key {
  uint64_t hi, lo;
};
HD bool key_lt(const Key& a, const Key& b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }
HD bool key_eq(const Key& a, const Key& b) { return a.hi == b.hi && a.lo == b.lo; }

HD uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct Cache {
  int d;
  int bits;
  int n[MAXD];
  int64_t cap;
  int64_t count;
  int64_t calls;
  double max_abs;
  uint64_t tmask;
  Key* keys;
  double* vals;
  int32_t* table;
};

HD Key pack_key(int d, int bits, const int32_t* idx) {
  Key k{0, 0};
  for (int j = 0; j < d; ++j) {
    k.hi = (k.hi << bits) | (k.lo >> (64 - bits));
    k.lo = (k.lo << bits) | (uint64_t)(uint32_t)idx[j];
  }
  return k;
}
HD void unpack_key(int d, int bits, Key k, int32_t* idx) {
  const uint64_t m = (1ull << bits) - 1;
  for (int j = d - 1; j >= 0; --j) {
    idx[j] = (int32_t)(k.lo & m);
    k.lo = (k.lo >> bits) | (k.hi << (64 - bits));
    k.hi >>= bits;
  }
}

HD int64_t cache_lookup(const Cache& C, const Key& k) {
  uint64_t h = mix64(k.hi ^ mix64(k.lo)) & C.tmask;
  while (true) {
    const int32_t e = C.table[h];
    if (e < 0) return -1;
    if (key_eq(C.keys[e], k)) return e;
    h = (h + 1) & C.tmask;
  }
}

HD void cache_insert(Cache& C, const Key& k, int32_t e) {
  uint64_t h = mix64(k.hi ^ mix64(k.lo)) & C.tmask;
  while (true) {
#if ENGINE_DEVICE
    const int32_t prev = atomicCAS(&C.table[h], -1, e);
    if (prev == -1) return;
#else
    if (C.table[h] == -1) { C.table[h] = e; return; }
#endif
    h = (h + 1) & C.tmask;
  }
}

// Allocate and clear a cache for `cap` entries.
HDN int cache_init(const Ctx& c, Arena& ar, Cache*& C, int d, const int* n, int64_t cap) {
  ALLOC(C, Cache, 1, ar);
  int maxn = 1;
  for (int k = 0; k < d; ++k) maxn = imax(maxn, n[k]);
  int bits = 1;
  while ((1 << bits) < maxn) ++bits;
  if (bits * d > 128) return E_ARG;
  uint64_t tsz = 1;
  while (tsz < (uint64_t)(2 * cap)) tsz <<= 1;
  Key* keys;
  double* vals;
  int32_t* table;
  ALLOC(keys, Key, cap, ar);
  ALLOC(vals, double, cap, ar);
  ALLOC(table, int32_t, tsz, ar);
  par_fill_i32(c, table, (int64_t)tsz, -1);
  if (c.leader()) {
    C->d = d;
    C->bits = bits;
    for (int k = 0; k < d; ++k) C->n[k] = n[k];
    C->cap = cap;
    C->count = 0;
    C->calls = 0;
    C->max_abs = 0.0;
    C->tmask = tsz - 1;
    C->keys = keys;
    C->vals = vals;
    C->table = table;
  }
  c.sync();
  return OK;
}

constexpr int64_t RANK_SORT_MAX = 256;   // cache_eval: rank sort below, bitonic above

// In-place CTA bitonic sort of P (power of two) keys.
HDN void bitonic_sort(const Ctx& c, Key* a, int64_t P) {
  for (int64_t k = 2; k <= P; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = c.tid; i < P; i += c.nt) {
        const int64_t l = i ^ j;
        if (l > i) {
          const bool asc = (i & k) == 0;
          const Key x = a[i], y = a[l];
          if (asc ? key_lt(y, x) : key_lt(x, y)) { a[i] = y; a[l] = x; }
        }
      }
      c.sync();
    }
  }
}

// Order-preserving compaction helper: thread t owns the contiguous range
// [t*chunk, (t+1)*chunk); returns this thread's output offset and the total.
HDN int64_t scan_offsets(const Ctx& c, int64_t mine, int64_t* total) {
#if ENGINE_DEVICE
  // exclusive block scan: warp inclusive scan by shuffles, then warp totals
  const int lane = c.tid & 31, w = c.tid >> 5, nw = (c.nt + 31) >> 5;
  int64_t* wt = reinterpret_cast<int64_t*>(c.red) + 64;   // nw warp totals
  int64_t x = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) wt[w] = x;
  __syncthreads();
  int64_t base = 0, tot = 0;
  for (int i = 0; i < nw; ++i) {
    if (i < w) base += wt[i];
    tot += wt[i];
  }
  __syncthreads();
  *total = tot;
  return base + x - mine;
#else
  (void)c;
  *total = mine;
  return 0;
#endif
}

// Evaluate K multi-indices (int32, K x d) through the cache; out[K].
// presorted: idx is already in strictly ascending key order (no duplicates),
// so the misses need no sort (Cartesian fibre blocks enumerated in order).
HDN int cache_eval(const Ctx& c, Arena& ar, Cache* C, const EvalSpec& spec, const int32_t* idx,
                          int64_t K, double* out, double* sm, bool presorted = false) {
  const int d = C->d, bits = C->bits;
  PROF(c, 2);
  size_t mk = ar.mark();
  int64_t* pos;
  ALLOC(pos, int64_t, K > 0 ? K : 1, ar);
  Key* mkeys;
  ALLOC(mkeys, Key, K > 0 ? K : 1, ar);
  // 1. lookup
  const int64_t chunk = (K + c.nt - 1) / c.nt;
  const int64_t lo = lmin(K, (int64_t)c.tid * chunk), hi = lmin(K, lo + chunk);
  int64_t nmiss = 0;
  for (int64_t p = lo; p < hi; ++p) {
    const Key k = pack_key(d, bits, idx + p * d);
    const int64_t e = cache_lookup(*C, k);
    pos[p] = e;
    if (e < 0) ++nmiss;
  }
  int64_t total;
  int64_t off = scan_offsets(c, nmiss, &total);
  for (int64_t p = lo; p < hi; ++p)
    if (pos[p] < 0) mkeys[off++] = pack_key(d, bits, idx + p * d);
  c.sync();
  if (total > 0) {
    // 2. sort + dedup (skipped for presorted blocks: compaction kept the order)
    int64_t P = 1;
    while (P < total) P <<= 1;
    Key* sk = mkeys;
    if (!presorted && total <= RANK_SORT_MAX && (!ENGINE_DEVICE || total <= c.nt) && total * (int64_t)sizeof(Key) <= (int64_t)(SMEM_SCRATCH_DOUBLES * sizeof(double))) {
      // few misses: stable rank sort (one barrier) instead of the bitonic
      // network's log^2 P barrier-separated stages; equal keys end adjacent
      PROF(c, 0);
      Key* ks = reinterpret_cast<Key*>(sm);
      for (int64_t i = c.tid; i < total; i += c.nt) ks[i] = mkeys[i];
      c.sync();
#if ENGINE_DEVICE
      // L = 2^k lanes share one key's comparisons (L * total <= blockDim)
      int L = 1;
      while (L < 32 && 2 * L * total <= c.nt) L <<= 1;
      {
        const int i = c.tid / L, sub = c.tid % L;
        const bool act = i < total;
        const Key ki = ks[act ? i : 0];
        int rank = 0;
        if (act)
          for (int j = sub; j < (int)total; j += L) {
            const Key kj = ks[j];
            rank += (key_lt(kj, ki) || (j < i && key_eq(kj, ki))) ? 1 : 0;
          }
        for (int o = L >> 1; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
        if (act && sub == 0) mkeys[rank] = ki;
      }
#else
      for (int64_t i = c.tid; i < total; i += c.nt) {
        const Key ki = ks[i];
        int64_t rank = 0;
        for (int64_t j = 0; j < total; ++j) {
          const Key kj = ks[j];
          rank += (key_lt(kj, ki) || (j < i && key_eq(kj, ki))) ? 1 : 0;
        }
        mkeys[rank] = ki;
      }
#endif
      c.sync();
    } else if (!presorted) {
      PROF(c, 0);
      const bool in_smem = P * (int64_t)sizeof(Key) <= (int64_t)(SMEM_SCRATCH_DOUBLES * sizeof(double));
      if (in_smem) {
        sk = reinterpret_cast<Key*>(sm);
      } else {
        ALLOC(sk, Key, P, ar);
      }
      for (int64_t i = c.tid; i < P; i += c.nt) sk[i] = (i < total) ? mkeys[i] : Key{~0ull, ~0ull};
      c.sync();
      bitonic_sort(c, sk, P);
      if (in_smem) {   // move back to global: sm is reused by the evaluator
        for (int64_t i = c.tid; i < total; i += c.nt) mkeys[i] = sk[i];
        c.sync();
        sk = mkeys;
      }
    }
    const int64_t ch2 = (total + c.nt - 1) / c.nt;
    const int64_t lo2 = lmin(total, (int64_t)c.tid * ch2), hi2 = lmin(total, lo2 + ch2);
    int64_t nu = 0;
    for (int64_t i = lo2; i < hi2; ++i)
      if (i == 0 || !key_eq(sk[i], sk[i - 1])) ++nu;
    int64_t M;
    int64_t o2 = scan_offsets(c, nu, &M);
    const int64_t base = C->count;
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
    fprintf(stderr, "EV K=%lld M=%lld\n", (long long)K, (long long)M);
#endif
    if (base + M > C->cap) { ar.release(mk); return E_CACHE; }
    for (int64_t i = lo2; i < hi2; ++i)
      if (i == 0 || !key_eq(sk[i], sk[i - 1])) C->keys[base + (o2++)] = sk[i];
    c.sync();
    // 3. evaluate the new entries
    int32_t* uidx;
    ALLOC(uidx, int32_t, M * d, ar);
    for (int64_t j = c.tid; j < M; j += c.nt) unpack_key(d, bits, C->keys[base + j], uidx + j * d);
    c.sync();
    double* nv = C->vals + base;
    PROF(c, 1);
    if (spec.kind == EV_REALIGN) {
      // pull the predictive nodes back once: coords = F^{-1} y (filters.py:973)
      double* coords;
      ALLOC(coords, double, M * d, ar);
      for (int64_t e = c.tid; e < M * d; e += c.nt) coords[e] = realign_coord(spec, uidx + (e / d) * d, (int)(e % d));
      c.sync();
      PointSlice<PtsFn> ps{&spec.conv, spec.geo, PtsFn{coords, d}, 0, 0.0};
      CK(tt_eval_bucketed(c, ar, spec.conv, M, ps, nv, sm));
    } else {
      for (int64_t j = c.tid; j < M; j += c.nt) nv[j] = eval_point(spec, uidx + j * d);
    }
    c.sync();
    double vmax = 0.0, bad = 0.0;
    for (int64_t j = c.tid; j < M; j += c.nt) {
      const double v = nv[j];
      if (!isfinite(v)) bad = 1.0;
      else vmax = fmax(vmax, fabs(v));
    }
    bad = block_max(c, bad);
    vmax = block_max(c, vmax);
    if (bad > 0.0) { ar.release(mk); return E_NONFINITE; }
    for (int64_t j = c.tid; j < M; j += c.nt) cache_insert(*C, C->keys[base + j], (int32_t)(base + j));
    c.sync();
    if (c.leader()) {
      C->count = base + M;
      C->calls += M;
      if (M > 0) C->max_abs = fmax(C->max_abs, vmax);
    }
    c.sync();
    for (int64_t p = lo; p < hi; ++p)
      if (pos[p] < 0) pos[p] = cache_lookup(*C, pack_key(d, bits, idx + p * d));
  }
  for (int64_t p = lo; p < hi; ++p) out[p] = C->vals[pos[p]];
  c.sync();
  ar.release(mk);
  return OK;
}

}  // namespace tg
