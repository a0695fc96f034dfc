/*
 * CPU oracle for the ShockHash hot path — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference algorithm, used by tests/ (as the
 * checker), __graft_entry__.smoke() and bench.py's cpu_baseline leg; never
 * by the product path.  Each function cites the reference it restates
 * (/root/reference/pkg/src/shockhash/...).  It is pinned against golden
 * vectors produced by the real reference (tests/golden/, make_golden.py) in
 * tests/test_oracle.py.
 *
 * Build: make -C oracle   (gcc -O3 -fopenmp, -> oracle/_build/libshk_oracle.so)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define GOLDEN 0x9E3779B97F4A7C15ull
#define MUL1 0xBF58476D1CE4E5B9ull
#define MUL2 0x94D049BB133111EBull
enum { T_LEAF = 1, T_SPLITBIT = 2, T_SPLIT = 3, T_BUCKET = 4, T_RSTART = 5, T_RPAT0 = 6, T_RPAT1 = 7 };

/* _pure.py:32-72 */
uint64_t o_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * MUL1;
  z = (z ^ (z >> 27)) * MUL2;
  return z ^ (z >> 31);
}
uint64_t o_seed_mixer(uint64_t s, uint64_t tag) { return o_mix64(s + tag * GOLDEN); }
uint64_t o_remix(uint64_t hi, uint64_t lo, uint64_t s, uint64_t tag) {
  return o_mix64(o_mix64(hi ^ o_seed_mixer(s, tag)) ^ lo);
}
uint64_t o_hash_range(uint64_t v, uint64_t m) { return ((v >> 32) * m) >> 32; }
static inline void pair_x(uint64_t hi, uint64_t lo, uint64_t x, int n, int* a, int* b) {
  uint64_t v = o_mix64(o_mix64(hi ^ x) ^ lo);
  int h0 = (int)(((v >> 32) * (uint64_t)n) >> 32);
  int h1 = (int)(((v & 0xFFFFFFFFull) * (uint64_t)(n - 1)) >> 32);
  *a = h0;
  *b = h1 + (h1 >= h0);
}
void o_leaf_pair(uint64_t hi, uint64_t lo, uint64_t s, int n, int* a, int* b) {
  if (n == 1) {
    *a = *b = 0;
    return;
  }
  pair_x(hi, lo, o_seed_mixer(s, T_LEAF), n, a, b);
}
int o_split_bit(uint64_t hi, uint64_t lo, uint64_t s) { return (int)(o_remix(hi, lo, s, T_SPLITBIT) >> 63); }

/* _pure.py:553-569 */
int o_leaf_cell(uint64_t hi, uint64_t lo, int64_t q, int m, int mode, int64_t ck, int choice) {
  int a, b;
  if (mode == 0) {
    o_leaf_pair(hi, lo, (uint64_t)q, m, &a, &b);
    return choice ? b : a;
  }
  int64_t base = q / m, r = q % m;
  int64_t sa = (mode == 2 && ck && m > 32) ? base - base % ck : base;
  if (o_split_bit(hi, lo, (uint64_t)sa) == 0) {
    o_leaf_pair(hi, lo, (uint64_t)sa, m, &a, &b);
    return choice ? b : a;
  }
  o_leaf_pair(hi, lo, (uint64_t)base, m, &a, &b);
  return (int)(((choice ? b : a) + r) % m);
}

/* union-find with pseudotree flags, _pure.py:95-147 */
typedef struct {
  int parent[64], size[64];
  uint8_t pseudo[64];
} UF;
static int uf_find(UF* u, int x) {
  int r = x;
  while (u->parent[r] != r) r = u->parent[r];
  while (u->parent[x] != r) {
    int nx = u->parent[x];
    u->parent[x] = r;
    x = nx;
  }
  return r;
}
static int pf_accepts(const int* h0, const int* h1, int k, int n) {
  UF u;
  for (int i = 0; i < n; ++i) {
    u.parent[i] = i;
    u.size[i] = 1;
    u.pseudo[i] = 0;
  }
  for (int i = 0; i < k; ++i) {
    int a = uf_find(&u, h0[i]), b = uf_find(&u, h1[i]);
    if (a == b) {
      if (u.pseudo[a]) return 0;
      u.pseudo[a] = 1;
      continue;
    }
    if (u.pseudo[a] && u.pseudo[b]) return 0;
    if (u.size[a] < u.size[b]) {
      int t = a;
      a = b;
      b = t;
    }
    u.parent[b] = a;
    u.size[a] += u.size[b];
    u.pseudo[a] |= u.pseudo[b];
  }
  return 1;
}

/* search_plain, _pure.py:154-189; out = (seed, evals, passes, checks, a_evals) */
void o_search_plain(const uint64_t* hi, const uint64_t* lo, int n, int64_t max_seed, int64_t* out) {
  if (n == 1) {
    out[0] = 0, out[1] = 1, out[2] = 1, out[3] = 1, out[4] = 0;
    return;
  }
  uint64_t full = n == 64 ? ~0ull : ((1ull << n) - 1);
  int h0[64], h1[64];
  int64_t evals = 0, passes = 0;
  for (int64_t s = 0; s < max_seed; ++s) {
    uint64_t x = o_seed_mixer((uint64_t)s, T_LEAF), mask = 0;
    for (int i = 0; i < n; ++i) {
      pair_x(hi[i], lo[i], x, n, &h0[i], &h1[i]);
      mask |= (1ull << h0[i]) | (1ull << h1[i]);
    }
    evals += n;
    if (mask != full) continue;
    ++passes;
    if (pf_accepts(h0, h1, n, n)) {
      out[0] = s, out[1] = evals, out[2] = passes, out[3] = passes, out[4] = 0;
      return;
    }
  }
  out[0] = -1, out[1] = evals, out[2] = passes, out[3] = passes, out[4] = 0;
}

/* search_rotate, _pure.py:192-270 */
void o_search_rotate(const uint64_t* hi, const uint64_t* lo, int n, int64_t ck, int64_t max_seed, int64_t* out) {
  if (n == 1) {
    out[0] = 0, out[1] = 1, out[2] = 1, out[3] = 1, out[4] = 0;
    return;
  }
  uint64_t full = n == 64 ? ~0ull : ((1ull << n) - 1);
  int ai[64], bi[64], a0[64], a1[64], b0[64], b1[64], h0[64], h1[64];
  int na = 0, nb = 0;
  uint64_t mask_a = 0;
  int64_t evals = 0, passes = 0, aev = 0;
  int64_t max_base = max_seed / n + 1;
  if (max_seed < 0) max_base = (max_seed - (n - 1)) / n + 1; /* Python floor division */
  for (int64_t base = 0; base < max_base; ++base) {
    int64_t sa = ck ? base - base % ck : base;
    if (base == 0 || ck == 0 || base % ck == 0) {
      uint64_t xb = o_seed_mixer((uint64_t)sa, T_SPLITBIT), xa = o_seed_mixer((uint64_t)sa, T_LEAF);
      na = nb = 0;
      mask_a = 0;
      for (int i = 0; i < n; ++i) {
        if (o_mix64(o_mix64(hi[i] ^ xb) ^ lo[i]) >> 63)
          bi[nb++] = i;
        else
          ai[na++] = i;
      }
      evals += n;
      for (int j = 0; j < na; ++j) {
        pair_x(hi[ai[j]], lo[ai[j]], xa, n, &a0[j], &a1[j]);
        mask_a |= (1ull << a0[j]) | (1ull << a1[j]);
      }
      evals += na;
      aev += na;
    }
    uint64_t xg = o_seed_mixer((uint64_t)base, T_LEAF), mask_b = 0;
    for (int j = 0; j < nb; ++j) {
      pair_x(hi[bi[j]], lo[bi[j]], xg, n, &b0[j], &b1[j]);
      mask_b |= (1ull << b0[j]) | (1ull << b1[j]);
    }
    evals += nb;
    for (int r = 0; r < n; ++r) {
      uint64_t rot = r ? (((mask_b << r) | (mask_b >> (n - r))) & full) : mask_b;
      if ((mask_a | rot) != full) continue;
      ++passes;
      for (int j = 0; j < na; ++j) h0[j] = a0[j], h1[j] = a1[j];
      for (int j = 0; j < nb; ++j) h0[na + j] = (b0[j] + r) % n, h1[na + j] = (b1[j] + r) % n;
      if (pf_accepts(h0, h1, n, n)) {
        int64_t q = base * n + r;
        out[0] = q >= max_seed ? -1 : q, out[1] = evals, out[2] = passes, out[3] = passes, out[4] = aev;
        return;
      }
    }
  }
  out[0] = -1, out[1] = evals, out[2] = passes, out[3] = passes, out[4] = aev;
}

/* orient, pseudoforest.py:149-201 (stack peel, then cycles from the
 * lowest-index key).  Returns f bits; -1 in *ok if not a pseudoforest. */
uint64_t o_orient(const int* eu, const int* ev, int n, int* ok) {
  int deg[64] = {0}, alive[64], stack[256], sp = 0;
  uint64_t f = 0;
  int h0[64], h1[64];
  for (int k = 0; k < n; ++k) h0[k] = eu[k], h1[k] = ev[k];
  *ok = pf_accepts(h0, h1, n, n);
  if (!*ok) return 0;
  for (int k = 0; k < n; ++k) {
    deg[eu[k]]++;
    deg[ev[k]]++;
    alive[k] = 1;
  }
  for (int u = 0; u < n; ++u)
    if (deg[u] == 1) stack[sp++] = u;
  while (sp) {
    int u = stack[--sp];
    if (deg[u] != 1) continue;
    int k = -1;
    for (int j = 0; j < n; ++j)
      if (alive[j] && (eu[j] == u || ev[j] == u)) {
        k = j;
        break;
      }
    if (eu[k] != u) f |= 1ull << k;
    alive[k] = 0;
    deg[eu[k]]--;
    deg[ev[k]]--;
    int other = eu[k] == u ? ev[k] : eu[k];
    if (deg[other] == 1 && sp < 256) stack[sp++] = other;
  }
  for (int k0 = 0; k0 < n; ++k0) {
    if (!alive[k0]) continue;
    alive[k0] = 0;
    int u0 = eu[k0], node = ev[k0];
    while (node != u0) {
      int k = -1;
      for (int j = 0; j < n; ++j)
        if (alive[j] && (eu[j] == node || ev[j] == node)) {
          k = j;
          break;
        }
      if (k < 0) break;
      if (eu[k] != node) f |= 1ull << k;
      alive[k] = 0;
      node = eu[k] == node ? ev[k] : eu[k];
    }
  }
  return f;
}

/* split_seed_search, _pure.py:311-345 */
void o_split_search(const uint64_t* hi, const uint64_t* lo, int64_t m, const int64_t* sizes, int fan,
                    int64_t max_seed, int64_t* seed, int64_t* evals) {
  int64_t bounds[64], counts[64], acc = 0, ev = 0;
  for (int j = 0; j < fan; ++j) bounds[j] = (acc += sizes[j]);
  for (int64_t s = 0; s < max_seed; ++s) {
    uint64_t x = o_seed_mixer((uint64_t)s, T_SPLIT);
    for (int j = 0; j < fan; ++j) counts[j] = 0;
    int ok = 1;
    for (int64_t i = 0; i < m; ++i) {
      uint64_t v = o_mix64(o_mix64(hi[i] ^ x) ^ lo[i]);
      int64_t r = (int64_t)(((v >> 32) * (uint64_t)m) >> 32);
      int p = 0;
      while (r >= bounds[p]) ++p;
      if (++counts[p] > sizes[p]) {
        ok = 0;
        ev += i + 1;
        break;
      }
    }
    if (ok) {
      *seed = s;
      *evals = ev + m;
      return;
    }
  }
  *seed = -1;
  *evals = ev;
}

void o_split_parts(const uint64_t* hi, const uint64_t* lo, int64_t m, uint64_t seed, const int64_t* sizes, int fan,
                   int64_t* parts) {
  uint64_t x = o_seed_mixer(seed, T_SPLIT);
  for (int64_t i = 0; i < m; ++i) {
    uint64_t r = ((o_mix64(o_mix64(hi[i] ^ x) ^ lo[i]) >> 32) * (uint64_t)m) >> 32;
    int64_t acc = 0;
    int p = 0;
    for (; p < fan; ++p) {
      acc += sizes[p];
      if ((int64_t)r < acc) break;
    }
    parts[i] = p;
  }
}

/* ribbon, _pure.py:354-435 (on-the-fly elimination in row order) */
void o_ribbon_rows(const uint64_t* hi, const uint64_t* lo, int64_t N, int64_t m, uint64_t seed, int64_t* st,
                   uint64_t* p0, uint64_t* p1) {
  uint64_t xs = o_seed_mixer(seed, T_RSTART), x0 = o_seed_mixer(seed, T_RPAT0), x1 = o_seed_mixer(seed, T_RPAT1);
  for (int64_t i = 0; i < N; ++i) {
    st[i] = (int64_t)o_hash_range(o_mix64(o_mix64(hi[i] ^ xs) ^ lo[i]), (uint64_t)(m - 127));
    p0[i] = o_mix64(o_mix64(hi[i] ^ x0) ^ lo[i]) | 1;
    p1[i] = o_mix64(o_mix64(hi[i] ^ x1) ^ lo[i]);
  }
}

/* returns 1 and fills words on success, 0 if inconsistent */
int o_ribbon_solve(const int64_t* st, const uint64_t* p0, const uint64_t* p1, const uint8_t* rhs, int64_t N,
                   int64_t m, uint64_t* words) {
  u128* slot = (u128*)calloc((size_t)m, sizeof(u128));
  uint8_t* sb = (uint8_t*)calloc((size_t)m, 1);
  uint8_t* occ = (uint8_t*)calloc((size_t)m, 1);
  uint8_t* sol = (uint8_t*)calloc((size_t)m + 128, 1);
  int good = 1;
  for (int64_t i = 0; i < N && good; ++i) {
    int64_t s = st[i];
    u128 p = ((u128)p1[i] << 64) | p0[i];
    int b = rhs[i] & 1;
    for (;;) {
      if (!occ[s]) {
        occ[s] = 1;
        slot[s] = p;
        sb[s] = (uint8_t)b;
        break;
      }
      p ^= slot[s];
      b ^= sb[s];
      if (p == 0) {
        if (b) good = 0;
        break;
      }
      uint64_t l = (uint64_t)p;
      int t = l ? __builtin_ctzll(l) : 64 + __builtin_ctzll((uint64_t)(p >> 64));
      p >>= t;
      s += t;
    }
  }
  if (good) {
    for (int64_t s = m - 1; s >= 0; --s) {
      if (!occ[s]) continue;
      u128 p = slot[s] >> 1;
      int acc = sb[s];
      int64_t j = s + 1;
      while (p) {
        if ((uint64_t)p & 1) acc ^= sol[j];
        p >>= 1;
        ++j;
      }
      sol[s] = (uint8_t)acc;
    }
    int64_t nw = (m + 63) / 64;
    memset(words, 0, (size_t)nw * 8);
    for (int64_t s = 0; s < m; ++s)
      if (sol[s]) words[s >> 6] |= 1ull << (s & 63);
  }
  free(slot);
  free(sb);
  free(occ);
  free(sol);
  return good;
}

static int parity_window(const uint64_t* w, int64_t nw, int64_t s, uint64_t p0, uint64_t p1) {
  int64_t i = s >> 6;
  int sh = (int)(s & 63);
  uint64_t a = i < nw ? w[i] : 0, b = i + 1 < nw ? w[i + 1] : 0, c = i + 2 < nw ? w[i + 2] : 0;
  uint64_t v0 = sh ? (a >> sh) | (b << (64 - sh)) : a, v1 = sh ? (b >> sh) | (c << (64 - sh)) : b;
  return (__builtin_popcountll(v0 & p0) + __builtin_popcountll(v1 & p1)) & 1;
}

void o_ribbon_query(const int64_t* st, const uint64_t* p0, const uint64_t* p1, int64_t N, const uint64_t* w,
                    int64_t nw, uint8_t* out) {
  for (int64_t i = 0; i < N; ++i) out[i] = (uint8_t)parity_window(w, nw, st[i], p0[i], p1[i]);
}

/* Rice decode, _pure.py:456-482 / _core.pyx:575-623; returns 1 on overrun */
int o_rice_decode(const uint64_t* words, int64_t bit_len, int64_t* pos, int g, int64_t* out) {
  int64_t q = 0, p = *pos, nw = (bit_len + 63) >> 6;
  for (;;) {
    if (p >= bit_len) return 1;
    int64_t i = p >> 6;
    int sh = (int)(p & 63);
    uint64_t c = words[i] >> sh;
    if (sh && i + 1 < nw) c |= words[i + 1] << (64 - sh);
    int64_t avail = bit_len - p < 64 ? bit_len - p : 64;
    int t = ~c ? __builtin_ctzll(~c) : 64;
    if (t >= avail) {
      q += avail;
      p += avail;
      continue;
    }
    q += t;
    p += t + 1;
    break;
  }
  uint64_t rem = 0;
  if (g) {
    if (p + g > bit_len) return 1;
    int64_t i = p >> 6;
    int sh = (int)(p & 63);
    uint64_t c = words[i] >> sh;
    if (sh && i + 1 < nw) c |= words[i + 1] << (64 - sh);
    rem = c & ((1ull << g) - 1);
    p += g;
  }
  *out = (int64_t)(((uint64_t)q << g) | rem);
  *pos = p;
  return 0;
}

/* ---- plan (recsplit.py:45-67) and the per-bucket construction ---------- */
static int o_plan(int64_t m, int n, int64_t* sizes) { /* returns fanout, 0 = leaf */
  if (m <= n) return 0;
  int64_t unit;
  if (n <= 24) {
    unit = n;
  } else if (m <= 4 * (int64_t)n || m <= 12 * (int64_t)n) {
    int64_t part = m <= 4 * (int64_t)n ? n : 4 * (int64_t)n, k = 0, mm = m;
    while (mm >= part) sizes[k++] = part, mm -= part;
    if (mm) sizes[k++] = mm;
    return (int)k;
  } else {
    unit = 12 * (int64_t)n;
  }
  int64_t left = unit * ((m + 2 * unit - 1) / (2 * unit));
  if (left < 1) left = 1;
  if (left > m - 1) left = m - 1;
  sizes[0] = left;
  sizes[1] = m - left;
  return 2;
}

typedef struct {
  uint64_t h, l;
} K2;

static int k2cmp_part(const void* a, const void* b) { (void)a, (void)b; return 0; }

/* One bucket (recsplit.py:499-520 + _build_split/_build_leaf): preorder
 * seeds into seeds[]/gs[] (returns node count), choice bits per key, keys
 * permuted in place.  split_g[m] and leaf_g[m] are host-computed tables. */
static int64_t o_build_bucket(K2* keys, int64_t cnt, int n, int mode, int ck, const int32_t* leaf_g,
                              const int32_t* split_g, int64_t* seeds, int32_t* gs, uint8_t* choice,
                              int64_t* stats) {
  int64_t stack[4096][2], sp = 0, nn = 0;
  uint64_t hi[64], lo[64];
  uint64_t* thi = (uint64_t*)malloc((size_t)(cnt + 1) * 8);
  uint64_t* tlo = (uint64_t*)malloc((size_t)(cnt + 1) * 8);
  int64_t* parts = (int64_t*)malloc((size_t)(cnt + 1) * 8);
  K2* tmp = (K2*)malloc((size_t)(cnt + 1) * sizeof(K2));
  stack[sp][0] = 0, stack[sp][1] = cnt, ++sp;
  while (sp) {
    --sp;
    int64_t s0 = stack[sp][0], s1 = stack[sp][1], m = s1 - s0;
    int64_t sizes[64];
    int fan = o_plan(m, n, sizes);
    if (fan == 0) {
      for (int64_t i = 0; i < m; ++i) hi[i] = keys[s0 + i].h, lo[i] = keys[s0 + i].l;
      int64_t t[5];
      int eff_ck = m > 32 ? ck : 0;
      if (mode == 0)
        o_search_plain(hi, lo, (int)m, (int64_t)1 << 40, t);
      else
        o_search_rotate(hi, lo, (int)m, eff_ck, (int64_t)1 << 40, t);
      if (t[0] < 0) nn = -1 - nn; /* exhausted: flagged by a negative count */
      if (nn < 0) break;
      seeds[nn] = t[0];
      gs[nn] = leaf_g[m];
      ++nn;
      stats[0] += t[1], stats[1] += t[2], stats[2] += t[3], stats[3] += t[4];
      int eu[64], ev[64], ok;
      for (int64_t i = 0; i < m; ++i) {
        int a, b;
        if (mode == 0 || m == 1) {
          o_leaf_pair(hi[i], lo[i], (uint64_t)t[0], (int)m, &a, &b);
        } else {
          int64_t base = t[0] / m, r = t[0] % m, sa = eff_ck ? base - base % eff_ck : base;
          if (o_split_bit(hi[i], lo[i], (uint64_t)sa) == 0) {
            o_leaf_pair(hi[i], lo[i], (uint64_t)sa, (int)m, &a, &b);
          } else {
            o_leaf_pair(hi[i], lo[i], (uint64_t)base, (int)m, &a, &b);
            a = (int)((a + r) % m);
            b = (int)((b + r) % m);
          }
        }
        eu[i] = a, ev[i] = b;
      }
      uint64_t f = o_orient(eu, ev, (int)m, &ok);
      for (int64_t i = 0; i < m; ++i) choice[s0 + i] = (uint8_t)((f >> i) & 1);
    } else {
      for (int64_t i = 0; i < m; ++i) thi[i] = keys[s0 + i].h, tlo[i] = keys[s0 + i].l;
      int64_t seed, ev;
      o_split_search(thi, tlo, m, sizes, fan, (int64_t)1 << 40, &seed, &ev);
      if (seed < 0) {
        nn = -1 - nn;
        break;
      }
      seeds[nn] = seed;
      gs[nn] = split_g[m];
      ++nn;
      stats[4] += ev;
      o_split_parts(thi, tlo, m, (uint64_t)seed, sizes, fan, parts);
      int64_t w = 0;
      for (int p = 0; p < fan; ++p)
        for (int64_t i = 0; i < m; ++i)
          if (parts[i] == p) tmp[w++] = keys[s0 + i];
      memcpy(keys + s0, tmp, (size_t)m * sizeof(K2));
      int64_t bnd[65];
      bnd[0] = s0;
      for (int p = 0; p < fan; ++p) bnd[p + 1] = bnd[p] + sizes[p];
      for (int p = fan - 1; p >= 0; --p) stack[sp][0] = bnd[p], stack[sp][1] = bnd[p + 1], ++sp;
    }
  }
  free(thi);
  free(tlo);
  free(parts);
  free(tmp);
  return nn;
}

static int k2cmp(const void* a, const void* b) {
  const K2 *x = (const K2*)a, *y = (const K2*)b;
  if (x->h != y->h) return x->h < y->h ? -1 : 1;
  if (x->l != y->l) return x->l < y->l ? -1 : 1;
  return 0;
}

/* Rice encoding into a word array (recsplit.py:126-158). */
static void put_bits(uint64_t* w, int64_t pos, uint64_t v, int nb) {
  if (!nb) return;
  int64_t i = pos >> 6;
  int sh = (int)(pos & 63);
  w[i] |= v << sh;
  if (sh && sh + nb > 64) w[i + 1] |= v >> (64 - sh);
}

/* Full build from master codes (recsplit._build_hashed, recsplit.py:474-521)
 * except the ribbon.  Outputs: key_prefix[nb+1], bit_offsets[nb+1], stream
 * words (caller sizes them via max_words; returns bit length or -1 on
 * exhaustion, -2 if words too small), choice[N], sorted keys shi/slo,
 * stats[5] = evals, passes, checks, a_evals, split evals.  Buckets are built
 * in parallel (OpenMP) — the reference runs them one after another. */
int64_t o_build_hashed(const uint64_t* hi, const uint64_t* lo, int64_t N, int64_t nb, int n, int mode, int ck,
                       const int32_t* leaf_g, const int32_t* split_g, int64_t max_split_m, uint64_t* key_prefix,
                       uint64_t* bit_offsets, uint64_t* words, int64_t max_words, uint8_t* choice, uint64_t* shi,
                       uint64_t* slo, int64_t* stats) {
  int64_t* cnt = (int64_t*)calloc((size_t)nb + 1, 8);
  int64_t* bk = (int64_t*)malloc((size_t)N * 8);
  uint64_t xb = o_seed_mixer(0, T_BUCKET);
  for (int64_t i = 0; i < N; ++i) {
    bk[i] = (int64_t)o_hash_range(o_mix64(o_mix64(hi[i] ^ xb) ^ lo[i]), (uint64_t)nb);
    cnt[bk[i]]++;
  }
  key_prefix[0] = 0;
  for (int64_t b = 0; b < nb; ++b) key_prefix[b + 1] = key_prefix[b] + (uint64_t)cnt[b];
  K2* keys = (K2*)malloc((size_t)(N + 1) * sizeof(K2));
  int64_t* cur = (int64_t*)malloc((size_t)(nb + 1) * 8);
  for (int64_t b = 0; b < nb; ++b) cur[b] = (int64_t)key_prefix[b];
  for (int64_t i = 0; i < N; ++i) {
    K2 k = {hi[i], lo[i]};
    keys[cur[bk[i]]++] = k;
  }
  /* node capacity per bucket: a tree on m keys has < 2m nodes */
  int64_t** bseeds = (int64_t**)calloc((size_t)nb, sizeof(int64_t*));
  int32_t** bgs = (int32_t**)calloc((size_t)nb, sizeof(int32_t*));
  int64_t* bnn = (int64_t*)calloc((size_t)nb, 8);
  int64_t st[5] = {0, 0, 0, 0, 0};
  int bad = 0;
  (void)max_split_m;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : st[:5]) reduction(| : bad)
  for (int64_t b = 0; b < nb; ++b) {
    int64_t s0 = (int64_t)key_prefix[b], c = (int64_t)key_prefix[b + 1] - s0;
    if (!c) continue;
    qsort(keys + s0, (size_t)c, sizeof(K2), k2cmp);
    bseeds[b] = (int64_t*)malloc((size_t)(2 * c + 2) * 8);
    bgs[b] = (int32_t*)malloc((size_t)(2 * c + 2) * 4);
    int64_t lst[5] = {0, 0, 0, 0, 0};
    int64_t nn = o_build_bucket(keys + s0, c, n, mode, ck, leaf_g, split_g, bseeds[b], bgs[b], choice + s0, lst);
    if (nn < 0) bad |= 1;
    bnn[b] = nn;
    for (int j = 0; j < 5; ++j) st[j] += lst[j];
  }
  int64_t pos = 0;
  if (!bad) {
    memset(words, 0, (size_t)max_words * 8);
    for (int64_t b = 0; b < nb && pos >= 0; ++b) {
      bit_offsets[b] = (uint64_t)pos;
      for (int64_t j = 0; j < bnn[b]; ++j) {
        uint64_t x = (uint64_t)bseeds[b][j];
        int g = bgs[b][j];
        uint64_t q = x >> g;
        if ((pos + (int64_t)q + 1 + g + 63) / 64 + 1 > max_words) {
          pos = -2;
          break;
        }
        for (uint64_t k = 0; k < q; ++k) words[(pos + (int64_t)k) >> 6] |= 1ull << ((pos + (int64_t)k) & 63);
        pos += (int64_t)q + 1;
        if (g) put_bits(words, pos, x & ((1ull << g) - 1), g);
        pos += g;
      }
    }
    if (pos >= 0) bit_offsets[nb] = (uint64_t)pos;
  } else {
    pos = -1;
  }
  for (int64_t i = 0; i < N; ++i) shi[i] = keys[i].h, slo[i] = keys[i].l;
  for (int j = 0; j < 5; ++j) stats[j] = st[j];
  for (int64_t b = 0; b < nb; ++b) free(bseeds[b]), free(bgs[b]);
  free(bseeds);
  free(bgs);
  free(bnn);
  free(cnt);
  free(bk);
  free(keys);
  free(cur);
  (void)k2cmp_part;
  return pos;
}

/* Batched leaf search for the CPU baseline (OpenMP over leaves). */
void o_search_plain_batch(const uint64_t* hi, const uint64_t* lo, int64_t L, int n, int64_t* seeds) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < L; ++i) {
    int64_t t[5];
    o_search_plain(hi + i * n, lo + i * n, n, (int64_t)1 << 40, t);
    seeds[i] = t[0];
  }
}

/* query_stream, _pure.py:489-550 (reference-style: decodes the seeds of
 * skipped subtrees).  plan arrays per distinct bucket size are passed
 * flattened exactly as flatten_plan returns them: plan p = nodes
 * [poff[p], poff[p+1]) with sizes at sbase[p] + sizes_off[j]. */
int o_query(const uint64_t* hi, const uint64_t* lo, int64_t Q, int64_t nbk, const uint64_t* kp, const uint64_t* bo,
            const uint64_t* sw, int64_t bit_len, const int64_t* bucket_plan, const int64_t* poff,
            const int64_t* sbase, const int64_t* kind, const int64_t* g, const int64_t* sizes_off,
            const int64_t* subtree, const int64_t* m_node, const int64_t* sizes_flat, int mode, int64_t ck,
            uint64_t rseed, int64_t rm, const uint64_t* rw, int64_t rnw, uint64_t* out) {
  uint64_t xb = o_seed_mixer(0, T_BUCKET);
  for (int64_t t = 0; t < Q; ++t) {
    uint64_t h = hi[t], l = lo[t];
    int64_t b = (int64_t)o_hash_range(o_mix64(o_mix64(h ^ xb) ^ l), (uint64_t)nbk);
    int64_t msz = (int64_t)(kp[b + 1] - kp[b]), pos = (int64_t)bo[b], off = 0, v;
    if (msz > 0) {
      int64_t p = bucket_plan[b], base = poff[p], idx = 0;
      while (kind[base + idx] == 0) {
        if (o_rice_decode(sw, bit_len, &pos, (int)g[base + idx], &v)) return 1;
        int64_t mn = m_node[base + idx];
        int64_t r = (int64_t)o_hash_range(o_remix(h, l, (uint64_t)v, T_SPLIT), (uint64_t)mn);
        const int64_t* sz = sizes_flat + sbase[p] + sizes_off[base + idx];
        int part = 0;
        int64_t acc = sz[0];
        while (r >= acc) {
          off += sz[part];
          ++part;
          acc += sz[part];
        }
        int64_t j = idx + 1;
        for (int k = 0; k < part; ++k) {
          int64_t end = j + subtree[base + j];
          for (; j < end; ++j)
            if (o_rice_decode(sw, bit_len, &pos, (int)g[base + j], &v)) return 1;
        }
        idx = j;
      }
      int64_t q;
      if (o_rice_decode(sw, bit_len, &pos, (int)g[base + idx], &q)) return 1;
      int choice = 0;
      if (rm) {
        int64_t s = (int64_t)o_hash_range(o_remix(h, l, rseed, T_RSTART), (uint64_t)(rm - 127));
        choice = parity_window(rw, rnw, s, o_remix(h, l, rseed, T_RPAT0) | 1, o_remix(h, l, rseed, T_RPAT1));
      }
      off += o_leaf_cell(h, l, q, (int)m_node[base + idx], mode, ck, choice);
    }
    out[t] = kp[b] + (uint64_t)off;
  }
  return 0;
}

/* ---- analysis entry points of the kernel seam ---------------------------- */

/* search_bruteforce, _core.pyx:337-371 / _pure.py:273-296: out = (seed, evals) */
void o_search_bruteforce(const uint64_t* hi, const uint64_t* lo, int n, int64_t max_seed, int64_t* out) {
  uint64_t full = n < 64 ? (((uint64_t)1 << n) - 1) : ~(uint64_t)0;
  int64_t evals = 0;
  for (int64_t s = 0; s < max_seed; ++s) {
    uint64_t x = o_seed_mixer((uint64_t)s, T_LEAF), mask = 0;
    int ok = 1;
    for (int i = 0; i < n; ++i) {
      uint64_t bit = (uint64_t)1 << o_hash_range(o_mix64(o_mix64(hi[i] ^ x) ^ lo[i]), (uint64_t)n);
      if (mask & bit) {
        ok = 0;
        evals += i + 1;
        break;
      }
      mask |= bit;
    }
    if (ok) {
      evals += n;
      if (mask == full) {
        out[0] = s;
        out[1] = evals;
        return;
      }
    }
  }
  out[0] = -1;
  out[1] = evals;
}

/* mc_filter_pass_count, _core.pyx:832-860 / _pure.py:624-645 */
int64_t o_mc_filter_pass_count(int n, int64_t trials, uint64_t ent) {
  if (n == 1) return trials;
  uint64_t kh[64], kl[64];
  for (int i = 0; i < n; ++i) {
    kh[i] = o_mix64(ent + 2 * (uint64_t)i);
    kl[i] = o_mix64(ent + 2 * (uint64_t)i + 1);
  }
  uint64_t full = n < 64 ? (((uint64_t)1 << n) - 1) : ~(uint64_t)0;
  int64_t passes = 0;
  for (int64_t s = 0; s < trials; ++s) {
    uint64_t x = o_seed_mixer((uint64_t)s, T_LEAF), mask = 0;
    for (int i = 0; i < n; ++i) {
      int a, b;
      pair_x(kh[i], kl[i], x, n, &a, &b);
      mask |= ((uint64_t)1 << a) | ((uint64_t)1 << b);
    }
    passes += mask == full;
  }
  return passes;
}

/* enumerate_outcomes, _core.pyx:778-829 / _pure.py:576-621: odometer over
 * the n^(2n) tuples with the union-find check; out = (pf_count, sum 2^comps) */
void o_enumerate_outcomes(int n, uint64_t* out) {
  int edges[8] = {0};
  int total = n * n;
  uint64_t pf = 0, s2 = 0;
  for (;;) {
    UF u;
    for (int i = 0; i < n; ++i) {
      u.parent[i] = i;
      u.size[i] = 1;
      u.pseudo[i] = 0;
    }
    int comps = n, ok = 1;
    for (int i = 0; i < n && ok; ++i) {
      int a = uf_find(&u, edges[i] / n), b = uf_find(&u, edges[i] % n);
      if (a == b) {
        if (u.pseudo[a]) ok = 0;
        u.pseudo[a] = 1;
      } else {
        if (u.pseudo[a] && u.pseudo[b]) {
          ok = 0;
          break;
        }
        if (u.size[a] < u.size[b]) {
          int t = a;
          a = b;
          b = t;
        }
        u.parent[b] = a;
        u.size[a] += u.size[b];
        u.pseudo[a] |= u.pseudo[b];
        --comps;
      }
    }
    if (ok) {
      ++pf;
      s2 += (uint64_t)1 << comps;
    }
    int i = n - 1;
    while (i >= 0 && edges[i] == total - 1) edges[i--] = 0;
    if (i < 0) break;
    ++edges[i];
  }
  out[0] = pf;
  out[1] = s2;
}
