/*
 * zc_oracle.c -- CPU ORACLE for the B200 zero-copy traversal path.
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this; the
 * product path (paper_2006_06890_b200) never does and has no CPU fallback.
 *
 * Plain-C restatement of the reference's level-synchronous drivers
 * (/root/reference/pkg/src/zcgraph/traversal.py), same results AND same
 * iteration counts / per-iteration traversed-edge counts:
 *   zco_bfs   <- bfs   traversal.py:98-120  (level[src]=0; each iteration
 *                the unvisited neighbours of the frontier get level =
 *                iteration; next frontier = them, ascending)
 *   zco_sssp  <- sssp  traversal.py:123-151 (Jacobi: cand = dist at the start
 *                of the iteration + w; dist = min; next = improved, ascending)
 *   zco_cc    <- cc    traversal.py:154-179 (Jacobi min-label propagation,
 *                all vertices active first)
 *   traversed[k] = sum of frontier degrees of iteration k (traversal.py:63-65)
 *   zco_pagerank <- pagerank traversal.py:191-249 (synchronous power
 *                iteration, dangling mass spread uniformly, L1 stopping
 *                rule, final normalisation) as a pull over in-lists -- the
 *                out-lists themselves for an undirected graph; float64 sums
 *                in a different order than the reference's bincount, so
 *                results agree to rounding, not bit for bit (the numpy
 *                restatement oracle.pagerank is the one pinned bit-close to
 *                the reference fixtures; tests check this one against it)
 *
 * Pinning: tests/test_oracle_golden.py checks this file against fixtures
 * produced by the reference itself (tests/golden/make_golden.py): 406 small
 * graphs (acceptance criteria 6 and 8 seeds, known-answer graphs) and the
 * config-1 crc32 goldens (BFS 171fbc8b, SSSP 2e5f7c3e, CC 1ad2bc45).
 *
 * Parallelism: OpenMP over the frontier with relaxed atomics (the fixpoints
 * and the Jacobi iterates are unique, so results do not depend on the
 * thread count); next frontiers are built by an ordered scan of a mark
 * array, so they are ascending like the reference's np.unique/flatnonzero.
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define INF64 INT64_MAX

static inline uint64_t ld_elem(const void *a, int w, uint64_t i) {
  return w == 8 ? ((const uint64_t *)a)[i] : ((const uint32_t *)a)[i];
}

static inline void atomic_min_i64(int64_t *p, int64_t v, uint8_t *mark) {
  int64_t cur = __atomic_load_n(p, __ATOMIC_RELAXED);
  while (v < cur) {
    if (__atomic_compare_exchange_n(p, &cur, v, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
      __atomic_store_n(mark, 1, __ATOMIC_RELAXED);
      return;
    }
  }
}

/* Collect marked vertices in ascending order into front (clearing the
 * marks); returns the count and adds the degree sum to *trav. */
static uint64_t collect(uint64_t nv, const int64_t *off, uint8_t *mark, uint64_t *front,
                        uint64_t *trav, int nthreads) {
  int nt = nthreads > 0 ? nthreads : 1;
  uint64_t *cnt = (uint64_t *)calloc((size_t)nt + 1, sizeof(uint64_t));
  uint64_t deg = 0;
  int team = 1;
#pragma omp parallel num_threads(nt) reduction(+ : deg)
  {
#ifdef _OPENMP
    int t = omp_get_thread_num();
    int T = omp_get_num_threads();
#else
    int t = 0, T = 1;
#endif
    uint64_t lo = nv * (uint64_t)t / T, hi = nv * (uint64_t)(t + 1) / T, c = 0;
    for (uint64_t v = lo; v < hi; ++v) c += mark[v];
    cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
    {
      team = T;
      for (int k = 0; k < T; ++k) cnt[k + 1] += cnt[k];
    }
    uint64_t pos = cnt[t];
    for (uint64_t v = lo; v < hi; ++v)
      if (mark[v]) {
        mark[v] = 0;
        front[pos++] = v;
        deg += (uint64_t)(off[v + 1] - off[v]);
      }
  }
  const uint64_t total = cnt[team];
  free(cnt);
  *trav = deg;
  return total;
}

typedef struct {
  uint64_t *front;
  int64_t *fval;
  uint8_t *mark;
} scratch;

static int alloc_scratch(scratch *s, uint64_t nv) {
  uint64_t n = nv ? nv : 1;
  s->front = (uint64_t *)malloc(n * sizeof(uint64_t));
  s->fval = (int64_t *)malloc(n * sizeof(int64_t));
  s->mark = (uint8_t *)calloc(n, 1);
  return s->front && s->fval && s->mark;
}
static void free_scratch(scratch *s) {
  free(s->front);
  free(s->fval);
  free(s->mark);
}

static void log_iter(uint64_t *trav, uint64_t cap, uint64_t it, uint64_t v) {
  if (trav && it < cap) trav[it] = v;
}

/* Returns the iteration count, or -1 on allocation failure. */
int64_t zco_bfs(uint64_t nv, const int64_t *off, const void *edges, int eb, uint64_t src,
                int64_t *level, uint64_t *trav, uint64_t cap, int nthreads) {
  scratch s;
  if (!alloc_scratch(&s, nv)) return -1;
  for (uint64_t v = 0; v < nv; ++v) level[v] = -1;
  level[src] = 0;
  s.front[0] = src;
  uint64_t n = 1, t = (uint64_t)(off[src + 1] - off[src]), it = 0;
  int nt = nthreads > 0 ? nthreads : 1;
  while (n) {
    log_iter(trav, cap, it, t);
    ++it;
    const int64_t lv = (int64_t)it;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 64)
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t v = s.front[i];
      for (int64_t k = off[v]; k < off[v + 1]; ++k) {
        const uint64_t w = ld_elem(edges, eb, (uint64_t)k);
        if (__atomic_load_n(&level[w], __ATOMIC_RELAXED) == -1) {
          __atomic_store_n(&level[w], lv, __ATOMIC_RELAXED);
          __atomic_store_n(&s.mark[w], 1, __ATOMIC_RELAXED);
        }
      }
    }
    n = collect(nv, off, s.mark, s.front, &t, nt);
  }
  free_scratch(&s);
  return (int64_t)it;
}

int64_t zco_sssp(uint64_t nv, const int64_t *off, const void *edges, int eb,
                 const void *weights, int wb, uint64_t src, int64_t *dist, uint64_t *trav,
                 uint64_t cap, int nthreads) {
  scratch s;
  if (!alloc_scratch(&s, nv)) return -1;
  for (uint64_t v = 0; v < nv; ++v) dist[v] = INF64;
  dist[src] = 0;
  s.front[0] = src;
  uint64_t n = 1, t = (uint64_t)(off[src + 1] - off[src]), it = 0;
  int nt = nthreads > 0 ? nthreads : 1;
  while (n) {
    log_iter(trav, cap, it, t);
    ++it;
    for (uint64_t i = 0; i < n; ++i) s.fval[i] = dist[s.front[i]]; /* Jacobi snapshot */
#pragma omp parallel for num_threads(nt) schedule(dynamic, 64)
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t v = s.front[i];
      const int64_t dv = s.fval[i];
      for (int64_t k = off[v]; k < off[v + 1]; ++k) {
        const uint64_t w = ld_elem(edges, eb, (uint64_t)k);
        const int64_t cand = dv + (int64_t)ld_elem(weights, wb, (uint64_t)k);
        atomic_min_i64(&dist[w], cand, &s.mark[w]);
      }
    }
    n = collect(nv, off, s.mark, s.front, &t, nt);
  }
  free_scratch(&s);
  return (int64_t)it;
}

int64_t zco_cc(uint64_t nv, const int64_t *off, const void *edges, int eb, int64_t *label,
               uint64_t *trav, uint64_t cap, int nthreads) {
  scratch s;
  if (!alloc_scratch(&s, nv)) return -1;
  for (uint64_t v = 0; v < nv; ++v) {
    label[v] = (int64_t)v;
    s.front[v] = v;
  }
  uint64_t n = nv, t = nv ? (uint64_t)off[nv] : 0, it = 0;
  int nt = nthreads > 0 ? nthreads : 1;
  while (n) {
    log_iter(trav, cap, it, t);
    ++it;
    for (uint64_t i = 0; i < n; ++i) s.fval[i] = label[s.front[i]];
#pragma omp parallel for num_threads(nt) schedule(dynamic, 64)
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t v = s.front[i];
      const int64_t lv = s.fval[i];
      for (int64_t k = off[v]; k < off[v + 1]; ++k)
        atomic_min_i64(&label[ld_elem(edges, eb, (uint64_t)k)], lv,
                       &s.mark[ld_elem(edges, eb, (uint64_t)k)]);
    }
    n = collect(nv, off, s.mark, s.front, &t, nt);
  }
  free_scratch(&s);
  return (int64_t)it;
}

/* ranks: float64[nv] out.  Returns the iteration count, -1 on allocation
 * failure.  symmetric != 0: the lists are their own transpose. */
int64_t zco_pagerank(uint64_t nv, const int64_t *off, const void *edges, int eb, int symmetric,
                     double damping, uint64_t max_iters, double tol, double *ranks,
                     int nthreads) {
  int nt = nthreads > 0 ? nthreads : 1;
  if (nv == 0) return 0;
  const int64_t *ioff = off;
  const uint32_t *iedges = NULL;
  int64_t *toff = NULL;
  uint32_t *tedges = NULL;
  if (!symmetric) {  /* counting transpose: in-list of v = the sources of arcs into v */
    const uint64_t ne = (uint64_t)off[nv];
    toff = calloc(nv + 1, sizeof(int64_t));
    tedges = malloc((ne ? ne : 1) * sizeof(uint32_t));
    uint64_t *cur = calloc(nv, sizeof(uint64_t));
    if (!toff || !tedges || !cur) {
      free(toff);
      free(tedges);
      free(cur);
      return -1;
    }
#pragma omp parallel for num_threads(nt) schedule(static)
    for (uint64_t k = 0; k < ne; ++k)
      __atomic_fetch_add(&toff[ld_elem(edges, eb, k) + 1], 1, __ATOMIC_RELAXED);
    for (uint64_t v = 0; v < nv; ++v) toff[v + 1] += toff[v];
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1024)
    for (uint64_t u = 0; u < nv; ++u)
      for (int64_t k = off[u]; k < off[u + 1]; ++k) {
        const uint64_t w = ld_elem(edges, eb, (uint64_t)k);
        tedges[toff[w] + __atomic_fetch_add(&cur[w], 1, __ATOMIC_RELAXED)] = (uint32_t)u;
      }
    free(cur);
    ioff = toff;
    iedges = tedges;
  }
  double *contrib = malloc(nv * sizeof(double)), *next = malloc(nv * sizeof(double));
  if (!contrib || !next) {
    free(contrib);
    free(next);
    free(toff);
    free(tedges);
    return -1;
  }
  for (uint64_t v = 0; v < nv; ++v) ranks[v] = 1.0 / (double)nv;
  uint64_t it = 0;
  while (it < max_iters) {
    ++it;
    double dang = 0;
#pragma omp parallel for num_threads(nt) schedule(static) reduction(+ : dang)
    for (uint64_t u = 0; u < nv; ++u) {
      const int64_t d = off[u + 1] - off[u];
      contrib[u] = d ? ranks[u] / (double)d : 0.0;
      if (!d) dang += ranks[u];
    }
    const double base = (1.0 - damping) / (double)nv + damping * dang / (double)nv;
    double delta = 0;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1024) reduction(+ : delta)
    for (uint64_t v = 0; v < nv; ++v) {
      double acc = 0;
      if (iedges)
        for (int64_t k = ioff[v]; k < ioff[v + 1]; ++k) acc += contrib[iedges[k]];
      else
        for (int64_t k = ioff[v]; k < ioff[v + 1]; ++k) acc += contrib[ld_elem(edges, eb, (uint64_t)k)];
      next[v] = base + damping * acc;
      delta += fabs(next[v] - ranks[v]);
    }
    memcpy(ranks, next, nv * sizeof(double));
    if (delta < tol) break;
  }
  double sum = 0;
  for (uint64_t v = 0; v < nv; ++v) sum += ranks[v];
  for (uint64_t v = 0; v < nv; ++v) ranks[v] /= sum;
  free(contrib);
  free(next);
  free(toff);
  free(tedges);
  return (int64_t)it;
}
