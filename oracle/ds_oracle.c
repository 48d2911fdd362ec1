/*
 * C restatement of the densescan hot path — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/ (and bench.py's CPU legs) load this library, as the checker for
 * sizes the numpy oracle (densescan_oracle.py) cannot reach in seconds. It is
 * the same algorithm, pinned by the same golden vectors through
 * tests/test_oracle_golden.py (numpy) and tests/test_c_oracle.py (this file vs
 * numpy and vs the reference fixtures).
 *
 * Arithmetic follows the reference exactly (see densescan_oracle.py header):
 * float32, one IEEE round-to-nearest per operation, left-to-right sums,
 * compiled with -ffp-contract=off (no FMA) and without -ffast-math:
 *   ALGEBRAIC d2 = (T_i + P_j) - ((X_i0*x_j0 + X_i1*x_j1) + ...)   kernels.py:383-417
 *   DIRECT    d2 = ((dx0*dx0 + dx1*dx1) + ...), dx = x_j - x_i      kernels.py:197-210
 * Counts include the point itself; core = counts >= min_pts (kernels.py:331-335).
 * Labels: connected components of core-core in-range pairs (merge_iterative,
 * merge.py:133-166), non-core points take their lowest-indexed in-range core
 * (merge.py:116-130), clusters numbered by first appearance (core.py:116-132).
 *
 * Parallelism: rows are split over pthreads; union-find uses C11 atomics with
 * the same "hook the larger root" rule as the device code, so the result is
 * independent of the schedule.
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BLK 2048

typedef struct {
  const float* p;     /* d x n narrowed coordinates (coordinate-major) */
  const float* norm;  /* n squared norms (algebraic) */
  int64_t n;
  int d;
  float thr;
  int formula;
  int64_t min_pts;
  int64_t* counts;
  const uint8_t* core;
  _Atomic int32_t* parent;
  int32_t* border;
  int64_t lo, hi;
  int phase;
} job_t;

/* d2 of row a against columns [b0, b1) into out[0 .. b1-b0); the loops run over
 * columns with the dimension loop outside, so every element sees the reference's
 * operation order while the compiler vectorises across columns. */
static void row_d2(const job_t* j, int64_t a, int64_t b0, int64_t b1, float* out) {
  const int64_t n = j->n, m = b1 - b0;
  if (j->formula == 1) {
    const float* x0 = j->p + b0;
    const float X0 = j->p[a] + j->p[a];
    for (int64_t b = 0; b < m; ++b) out[b] = X0 * x0[b];
    for (int k = 1; k < j->d; ++k) {
      const float* xk = j->p + (int64_t)k * n + b0;
      const float Xk = j->p[(int64_t)k * n + a] + j->p[(int64_t)k * n + a];
      for (int64_t b = 0; b < m; ++b) out[b] = out[b] + Xk * xk[b];
    }
    const float T = j->norm[a];
    const float* P = j->norm + b0;
    for (int64_t b = 0; b < m; ++b) out[b] = (T + P[b]) - out[b];
    return;
  }
  {
    const float* x0 = j->p + b0;
    const float c0 = j->p[a];
    for (int64_t b = 0; b < m; ++b) {
      const float dx = x0[b] - c0;
      out[b] = dx * dx;
    }
    for (int k = 1; k < j->d; ++k) {
      const float* xk = j->p + (int64_t)k * n + b0;
      const float ck = j->p[(int64_t)k * n + a];
      for (int64_t b = 0; b < m; ++b) {
        const float dx = xk[b] - ck;
        out[b] = out[b] + dx * dx;
      }
    }
  }
}

static int32_t find_root(_Atomic int32_t* parent, int32_t v) {
  int32_t p = atomic_load_explicit(&parent[v], memory_order_relaxed);
  while (p != v) {
    const int32_t g = atomic_load_explicit(&parent[p], memory_order_relaxed);
    if (g != p) atomic_store_explicit(&parent[v], g, memory_order_relaxed);
    v = p;
    p = g;
  }
  return v;
}

static void unite(_Atomic int32_t* parent, int32_t a, int32_t b) {
  for (;;) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    if (a < b) {
      const int32_t t = a;
      a = b;
      b = t;
    }
    int32_t expect = a;
    if (atomic_compare_exchange_strong(&parent[a], &expect, b)) return;
  }
}

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  float* buf = (float*)malloc(sizeof(float) * BLK);
  for (int64_t a = j->lo; a < j->hi; ++a) {
    if (j->phase == 0) {
      int64_t c = 0;
      for (int64_t b0 = 0; b0 < j->n; b0 += BLK) {
        const int64_t b1 = b0 + BLK < j->n ? b0 + BLK : j->n;
        row_d2(j, a, b0, b1, buf);
        for (int64_t b = 0; b < b1 - b0; ++b) c += buf[b] <= j->thr;
      }
      j->counts[a] = c;
    } else if (j->core[a]) {
      for (int64_t b0 = a + 1; b0 < j->n; b0 += BLK) {
        const int64_t b1 = b0 + BLK < j->n ? b0 + BLK : j->n;
        row_d2(j, a, b0, b1, buf);
        for (int64_t b = 0; b < b1 - b0; ++b)
          if (buf[b] <= j->thr && j->core[b0 + b]) unite(j->parent, (int32_t)a, (int32_t)(b0 + b));
      }
    } else {
      int32_t first = -1;
      for (int64_t b0 = 0; b0 < j->n && first < 0; b0 += BLK) {
        const int64_t b1 = b0 + BLK < j->n ? b0 + BLK : j->n;
        row_d2(j, a, b0, b1, buf);
        for (int64_t b = 0; b < b1 - b0; ++b)
          if (buf[b] <= j->thr && j->core[b0 + b]) {
            first = (int32_t)(b0 + b);
            break;
          }
      }
      j->border[a] = first;
    }
  }
  free(buf);
  return NULL;
}

static void run_phase(const job_t* base, int threads, int phase) {
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)threads);
  const int64_t n = base->n;
  for (int t = 0; t < threads; ++t) {
    jobs[t] = *base;
    jobs[t].phase = phase;
    /* phase 1 rows near 0 do the most work (b > a): split by equal triangle area */
    const double f0 = phase == 1 ? 1.0 - sqrt(1.0 - (double)t / threads) : (double)t / threads;
    const double f1 =
        phase == 1 ? 1.0 - sqrt(1.0 - (double)(t + 1) / threads) : (double)(t + 1) / threads;
    jobs[t].lo = (int64_t)(f0 * (double)n);
    jobs[t].hi = t == threads - 1 ? n : (int64_t)(f1 * (double)n);
  }
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, worker, &jobs[t]);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
  free(jobs);
}

static void prepare(const double* coords, int64_t n, int d, float* p, float* norm) {
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) p[(int64_t)k * n + i] = (float)coords[i * d + k]; /* RN */
  for (int64_t i = 0; i < n; ++i) {
    float acc = p[i] * p[i];
    for (int k = 1; k < d; ++k) acc = acc + p[(int64_t)k * n + i] * p[(int64_t)k * n + i];
    norm[i] = acc;
  }
}

/* Neighbour counts (int64, incl. self). Returns 0. */
int dso_counts(const double* coords, int64_t n, int d, double eps_sq, int formula, int threads,
               int64_t* counts_out) {
  float* p = (float*)malloc(sizeof(float) * (size_t)(n * d));
  float* norm = (float*)malloc(sizeof(float) * (size_t)n);
  prepare(coords, n, d, p, norm);
  job_t j;
  memset(&j, 0, sizeof(j));
  j.p = p;
  j.norm = norm;
  j.n = n;
  j.d = d;
  j.thr = (float)eps_sq;
  j.formula = formula;
  j.counts = counts_out;
  run_phase(&j, threads, 0);
  free(p);
  free(norm);
  return 0;
}

/* Full pipeline: canonical labels (int64) and counts (int64). Returns 0. */
int dso_dbscan(const double* coords, int64_t n, int d, double eps_sq, int64_t min_pts,
               int formula, int threads, int64_t* labels_out, int64_t* counts_out) {
  float* p = (float*)malloc(sizeof(float) * (size_t)(n * d));
  float* norm = (float*)malloc(sizeof(float) * (size_t)n);
  uint8_t* core = (uint8_t*)malloc((size_t)n);
  _Atomic int32_t* parent = (_Atomic int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* border = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* id = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  prepare(coords, n, d, p, norm);
  job_t j;
  memset(&j, 0, sizeof(j));
  j.p = p;
  j.norm = norm;
  j.n = n;
  j.d = d;
  j.thr = (float)eps_sq;
  j.formula = formula;
  j.min_pts = min_pts;
  j.counts = counts_out;
  run_phase(&j, threads, 0);
  for (int64_t i = 0; i < n; ++i) {
    core[i] = counts_out[i] >= min_pts;
    atomic_init(&parent[i], (int32_t)i);
    border[i] = -1;
    id[i] = -1;
  }
  j.core = core;
  j.parent = parent;
  j.border = border;
  run_phase(&j, threads, 1);
  int32_t next = 0;
  for (int64_t i = 0; i < n; ++i) {
    int32_t r = -1;
    if (core[i])
      r = find_root(parent, (int32_t)i);
    else if (border[i] >= 0)
      r = find_root(parent, border[i]);
    if (r < 0) {
      labels_out[i] = -1;
      continue;
    }
    if (id[r] < 0) id[r] = next++;
    labels_out[i] = id[r];
  }
  free(p);
  free(norm);
  free(core);
  free((void*)parent);
  free(border);
  free(id);
  return 0;
}
