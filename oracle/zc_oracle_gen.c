/*
 * zc_oracle_gen.c -- host restatement of the product's counter-based R-MAT
 * generator (paper_2006_06890_b200/csrc/zc_gen.cu: mix64 / hash3, Feistel,
 * rmat_params, rmat_src, rmat_dst, k_rmat_count, k_rmat_fill).
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY.  The reference has no Kronecker
 * generator; this file exists so that bench.py's
 * `--impl reference` arm and the CPU baselines can build the bench's graphs
 * without loading the product library.  tests/test_gpu_parity.py pins it to
 * the GPU generator (identical offsets and lists, byte for byte).
 *
 * Same integer arithmetic as the device code: the arc multiset, every list
 * and its order are functions of (scale, edge_factor, a, b, c, seed) only.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static inline uint64_t hash3(uint64_t seed, uint64_t stream, uint64_t i) {
  return mix64(mix64(seed ^ (stream * 0xd1b54a32d192ed03ull)) + i);
}

typedef struct {
  uint32_t scale, thr_src, thr_dst0, thr_dst1;
  uint64_t seed;
  uint32_t half, bits;
  uint64_t key;
} rmat_t;

static rmat_t rmat_params(uint32_t scale, double a, double b, double c, uint64_t seed) {
  const double d = 1.0 - a - b - c;
  rmat_t p;
  p.scale = scale;
  p.thr_src = (uint32_t)((c + d) * 65536.0 + 0.5);
  p.thr_dst0 = (uint32_t)(b / (a + b) * 65536.0 + 0.5);
  p.thr_dst1 = (c + d) > 0 ? (uint32_t)(d / (c + d) * 65536.0 + 0.5) : 0;
  p.seed = seed;
  p.bits = scale;
  p.half = (scale + 1) / 2;
  p.key = mix64(seed ^ 0x5eedull);
  return p;
}

/* keyed 4-round Feistel on 2*half bits, cycle-walked into [0, 2^bits) */
static inline uint64_t feistel_f(const rmat_t *p, uint64_t x, int r) {
  return hash3(p->key, 100 + (uint64_t)r, x) & ((1ull << p->half) - 1);
}

static inline uint64_t perm_fwd(const rmat_t *p, uint64_t x) {
  const uint64_t m = (1ull << p->half) - 1;
  do {
    uint64_t l = x >> p->half, r = x & m;
    for (int k = 0; k < 4; ++k) {
      const uint64_t nl = r, nr = l ^ feistel_f(p, r, k);
      l = nl;
      r = nr;
    }
    x = (l << p->half) | r;
  } while (x >> p->bits);
  return x;
}

static inline uint64_t perm_inv(const rmat_t *p, uint64_t x) {
  const uint64_t m = (1ull << p->half) - 1;
  do {
    uint64_t l = x >> p->half, r = x & m;
    for (int k = 3; k >= 0; --k) {
      const uint64_t pr = l, pl = r ^ feistel_f(p, l, k);
      l = pl;
      r = pr;
    }
    x = (l << p->half) | r;
  } while (x >> p->bits);
  return x;
}

/* source (before the permutation) of arc i: bit l is Bernoulli(c + d) */
static inline uint64_t rmat_src(const rmat_t *p, uint64_t arc) {
  uint64_t s = 0, h = 0;
  for (uint32_t l = 0; l < p->scale; ++l) {
    if ((l & 3) == 0) h = hash3(p->seed, 1 + (l >> 2), arc);
    const uint32_t u = (uint32_t)(h >> ((l & 3) * 16)) & 0xffffu;
    s |= (uint64_t)(u < p->thr_src) << l;
  }
  return s;
}

/* destination (before the permutation) given the source's quadrant bits */
static inline uint64_t rmat_dst(const rmat_t *p, uint64_t src_old, uint64_t key) {
  uint64_t d = 0, h = 0;
  for (uint32_t l = 0; l < p->scale; ++l) {
    if ((l & 3) == 0) h = hash3(p->seed, 32 + (l >> 2), key);
    const uint32_t u = (uint32_t)(h >> ((l & 3) * 16)) & 0xffffu;
    const uint32_t thr = (src_old >> l) & 1 ? p->thr_dst1 : p->thr_dst0;
    d |= (uint64_t)(u < thr) << l;
  }
  return d;
}

/* out-degrees of the 2^scale (permuted) vertices: deg must hold 2^scale u32 */
int zco_rmat_degrees(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed,
                     uint32_t *deg, int threads) {
  if (scale < 1 || scale > 31 || ef < 1) return -1;
  const rmat_t p = rmat_params(scale, a, b, c, seed);
  const uint64_t nv = 1ull << scale, narcs = (uint64_t)ef << scale;
  memset(deg, 0, nv * sizeof(uint32_t));
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (uint64_t i = 0; i < narcs; ++i) {
    const uint64_t s = perm_fwd(&p, rmat_src(&p, i));
#pragma omp atomic
    deg[s] += 1u;
  }
  return 0;
}

/* lists in CSR order: element k of vertex v's list is the destination drawn
 * with key (v << 32) | k (k_rmat_fill); off = the exclusive degree scan */
int zco_rmat_fill(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed,
                  const int64_t *off, uint32_t *edges, int threads) {
  if (scale < 1 || scale > 31 || ef < 1) return -1;
  const rmat_t p = rmat_params(scale, a, b, c, seed);
  const uint64_t nv = 1ull << scale;
#pragma omp parallel for schedule(dynamic, 1024) num_threads(threads > 0 ? threads : 1)
  for (uint64_t v = 0; v < nv; ++v) {
    const uint64_t s = (uint64_t)off[v], e = (uint64_t)off[v + 1];
    if (s == e) continue;
    const uint64_t src_old = perm_inv(&p, v);
    for (uint64_t k = s; k < e; ++k)
      edges[k] = (uint32_t)perm_fwd(&p, rmat_dst(&p, src_old, (v << 32) | (k - s)));
  }
  return 0;
}
