/*
 * CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's sampling hot path
 * (pcsample, /root/reference/proj). It exists so the tests, smoke() and the
 * bench's cpu_baseline leg can CHECK the CUDA path; no product code links,
 * loads or calls it, and the product fails loudly when its CUDA extension is
 * missing instead of falling back to this file.
 *
 * Parity is pinned: tests/test_oracle.py checks this file against the golden
 * vectors in tests/golden/ (generated from the real reference compiled under
 * oracle/_ref by oracle/Makefile) and against the reference's own known-answer
 * tests (proj/tests/test_sampler.cpp, test_core.cpp, test_order.cpp).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no -march, so the
 * distance arithmetic is the same mul/add sequence as the reference's
 * default x86-64 build, which contains no FMA).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1

enum { OR_FPS = 1, OR_AFPS = 2, OR_NPDU_FPS = 3, OR_NPDU_AFPS = 4 };

/* ------------------------------------------------------------ SplitMix64
 * proj/include/pcs/rng.hpp:16-21 (next), :24-30 (below), :33-36 (unit). */
uint64_t or_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t or_splitmix_below(uint64_t* state, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound; /* 2^64 mod bound */
  for (;;) {
    const uint64_t r = or_splitmix_next(state);
    if (r >= threshold) return r % bound;
  }
}

double or_splitmix_unit(uint64_t* state) {
  return (double)(or_splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------ sectors
 * proj/src/sectors.cpp:9-24 partition_sectors, :26-36 allocate_samples,
 * :38-51 SectorPlan::make, :53-61 update_window. */
static void set_err(char* err, size_t errlen, const char* msg) {
  if (err && errlen) {
    strncpy(err, msg, errlen - 1);
    err[errlen - 1] = 0;
  }
}

int or_sector_plan(uint64_t n, uint64_t c, uint64_t m, uint64_t* begins,
                   uint64_t* ends, uint64_t* quotas, char* err, size_t errlen) {
  if (m < 1) { set_err(err, errlen, "partition_sectors: m must be >= 1"); return OR_EINVAL; }
  if (m > n) { set_err(err, errlen, "partition_sectors: m exceeds point count"); return OR_EINVAL; }
  if (m > c) { set_err(err, errlen, "allocate_samples: m exceeds sample count"); return OR_EINVAL; }
  uint64_t at = 0;
  for (uint64_t s = 0; s < m; ++s) {
    const uint64_t len = n / m + (s < n % m ? 1 : 0);
    begins[s] = at;
    ends[s] = at + len;
    at += len;
    quotas[s] = c / m + (s < c % m ? 1 : 0);
  }
  for (uint64_t s = 0; s < m; ++s) {
    if (quotas[s] > ends[s] - begins[s]) {
      char buf[160];
      snprintf(buf, sizeof buf, "sector %llu holds %llu points but owes %llu samples",
               (unsigned long long)s, (unsigned long long)(ends[s] - begins[s]),
               (unsigned long long)quotas[s]);
      set_err(err, errlen, buf);
      return OR_EINVAL;
    }
  }
  return OR_OK;
}

void or_update_window(uint64_t sb, uint64_t se, uint64_t idx, uint64_t k,
                      uint64_t* wb, uint64_t* we) {
  const uint64_t lo = idx >= k / 2 ? idx - k / 2 : 0;
  const uint64_t hi = idx + (k + 1) / 2;
  *wb = lo > sb ? lo : sb;
  *we = hi < se ? hi : se;
}

/* ------------------------------------------------------------ local_fps
 * proj/src/sampler.cpp:85-167. xyz is the whole cloud, AoS double[3].
 * k == 0 means "no window" (std::nullopt). trace, when non-null, receives
 * (quota-1) snapshots of the n-element distance array (sampler.cpp:130). */
int or_local_fps(const double* xyz, uint64_t n_total, uint64_t sb, uint64_t se,
                 uint64_t quota, int windowed, uint64_t k, int random_first,
                 uint64_t seed, int64_t* out_idx, uint64_t stats[4],
                 double* trace, char* err, size_t errlen) {
  if (se > n_total || sb >= se) { set_err(err, errlen, "local_fps: sector out of range"); return OR_EINVAL; }
  if (quota < 1 || quota > se - sb) { set_err(err, errlen, "local_fps: quota infeasible for sector"); return OR_EINVAL; }
  if (windowed && k < 1) { set_err(err, errlen, "local_fps: window size must be >= 1"); return OR_EINVAL; }

  const uint64_t n = se - sb;
  const double* pts = xyz + 3 * sb;
  double* d = (double*)malloc(n * sizeof(double));
  unsigned char* sampled = (unsigned char*)calloc(n, 1);
  for (uint64_t j = 0; j < n; ++j) d[j] = INFINITY;

  uint64_t state = seed;
  uint64_t cur = random_first ? sb + or_splitmix_below(&state, n) : sb;
  out_idx[0] = (int64_t)cur;
  sampled[cur - sb] = 1;

  uint64_t evals = 0, writes = 0, scans = 0, iters = 0;
  for (uint64_t i = 1; i < quota; ++i) {
    uint64_t wb = sb, we = se;
    if (windowed) or_update_window(sb, se, cur, k, &wb, &we);
    const double px = xyz[3 * cur], py = xyz[3 * cur + 1], pz = xyz[3 * cur + 2];
    for (uint64_t j = wb - sb; j < we - sb; ++j) {
      const double dx = pts[3 * j] - px;
      const double dy = pts[3 * j + 1] - py;
      const double dz = pts[3 * j + 2] - pz;
      const double dist = dx * dx + dy * dy + dz * dz;
      if (dist <= d[j]) { d[j] = dist; ++writes; }
    }
    evals += we - wb;
    if (trace) memcpy(trace + (i - 1) * n, d, n * sizeof(double));

    /* value max over the whole sector, then the first unsampled index that
     * holds it (sampler.cpp:137-154). */
    double best_dist = -INFINITY;
    for (uint64_t j = 0; j < n; ++j) if (d[j] > best_dist) best_dist = d[j];
    uint64_t best = 0;
    for (uint64_t j = 0; j < n; ++j) {
      if (d[j] == best_dist && !sampled[j]) { best = j; break; }
    }
    scans += n;
    ++iters;
    cur = sb + best;
    out_idx[i] = (int64_t)cur;
    sampled[best] = 1;
  }
  stats[0] = evals; stats[1] = writes; stats[2] = scans; stats[3] = iters;
  free(d);
  free(sampled);
  return OR_OK;
}

/* ------------------------------------------------------------ samplers
 * proj/src/sampler.cpp:20-23 check_sample_count, :48-79 sectored,
 * :171-204 fps/afps/npdu_fps/npdu_afps. */
int or_sample(int method, const double* xyz, uint64_t n, uint64_t c, uint64_t m,
              uint64_t k, int random_first, uint64_t seed, int64_t* out_idx,
              int64_t* out_sector, uint64_t stats[4], char* err, size_t errlen) {
  static const char* names[] = {"?", "fps", "afps", "npdu_fps", "npdu_afps"};
  if (method < OR_FPS || method > OR_NPDU_AFPS) { set_err(err, errlen, "run_sampler: unknown method"); return OR_EINVAL; }
  char buf[96];
  if (c < 1) { snprintf(buf, sizeof buf, "%s: c must be >= 1", names[method]); set_err(err, errlen, buf); return OR_EINVAL; }
  if (c > n) { snprintf(buf, sizeof buf, "%s: c exceeds point count", names[method]); set_err(err, errlen, buf); return OR_EINVAL; }
  const int windowed = method == OR_NPDU_FPS || method == OR_NPDU_AFPS;
  stats[0] = stats[1] = stats[2] = stats[3] = 0;
  if (method == OR_FPS || method == OR_NPDU_FPS) {
    int rc = or_local_fps(xyz, n, 0, n, c, windowed, k, random_first, seed, out_idx,
                          stats, NULL, err, errlen);
    if (rc) return rc;
    for (uint64_t i = 0; i < c; ++i) out_sector[i] = 0;
    return OR_OK;
  }
  uint64_t* plan = (uint64_t*)malloc(3 * m * sizeof(uint64_t) + 8);
  int rc = or_sector_plan(n, c, m, plan, plan + m, plan + 2 * m, err, errlen);
  uint64_t at = 0;
  for (uint64_t s = 0; rc == OR_OK && s < m; ++s) {
    uint64_t st[4];
    rc = or_local_fps(xyz, n, plan[s], plan[m + s], plan[2 * m + s], windowed, k,
                      random_first, seed ^ s, out_idx + at, st, NULL, err, errlen);
    if (rc) break;
    for (uint64_t i = 0; i < plan[2 * m + s]; ++i) out_sector[at + i] = (int64_t)s;
    at += plan[2 * m + s];
    for (int q = 0; q < 4; ++q) stats[q] += st[q];
  }
  free(plan);
  return rc;
}

/* ------------------------------------------------------------ exact_sort
 * proj/src/order.cpp:11-24: stable ascending sort of storage indices by
 * points[i][axis] with operator<, then a gather. A bottom-up merge sort is
 * stable by construction, so the permutation equals std::stable_sort's. */
void or_exact_sort(const double* xyz, uint64_t n, int axis, int64_t* perm, double* out) {
  int64_t* tmp = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
  for (uint64_t i = 0; i < n; ++i) perm[i] = (int64_t)i;
  for (uint64_t width = 1; width < n; width *= 2) {
    for (uint64_t lo = 0; lo < n; lo += 2 * width) {
      uint64_t mid = lo + width < n ? lo + width : n;
      uint64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
      uint64_t a = lo, b = mid, o = lo;
      while (a < mid && b < hi) {
        /* take from the right run only when strictly smaller: stability */
        if (xyz[3 * perm[b] + axis] < xyz[3 * perm[a] + axis]) tmp[o++] = perm[b++];
        else tmp[o++] = perm[a++];
      }
      while (a < mid) tmp[o++] = perm[a++];
      while (b < hi) tmp[o++] = perm[b++];
    }
    memcpy(perm, tmp, n * sizeof(int64_t));
  }
  free(tmp);
  if (out)
    for (uint64_t i = 0; i < n; ++i) {
      out[3 * i] = xyz[3 * perm[i]];
      out[3 * i + 1] = xyz[3 * perm[i] + 1];
      out[3 * i + 2] = xyz[3 * perm[i] + 2];
    }
}

/* Batched convenience for the bench's cpu_baseline leg and the tests: B
 * clouds of n fp32 points (the f32_bin layout, widened exactly to double as
 * proj/src/io.cpp:84-86 does), same (method, c, m, k) for every cloud.
 * Clouds [b0, b1) only, so callers can split work across threads. */
int or_sample_batch_f32(int method, const float* xyz, uint64_t batch_lo, uint64_t batch_hi,
                        uint64_t n, uint64_t c, uint64_t m, uint64_t k, int random_first,
                        uint64_t seed, int64_t* out_idx, uint64_t* stats, char* err,
                        size_t errlen) {
  double* buf = (double*)malloc(3 * n * sizeof(double));
  int64_t* sec = (int64_t*)malloc(c * sizeof(int64_t));
  int rc = OR_OK;
  for (uint64_t b = batch_lo; b < batch_hi && rc == OR_OK; ++b) {
    for (uint64_t i = 0; i < 3 * n; ++i) buf[i] = (double)xyz[b * 3 * n + i];
    rc = or_sample(method, buf, n, c, m, k, random_first, seed, out_idx + b * c, sec,
                   stats + 4 * b, err, errlen);
  }
  free(buf);
  free(sec);
  return rc;
}

/* ------------------------------------------------------------ metrics
 * proj/src/metrics.cpp:16-52: fill distance and minimum pairwise distance
 * over the samples, both fp64 squared_dist, sqrt at the end. */
double or_coverage_radius(const double* xyz, uint64_t n, const int64_t* s, uint64_t c) {
  double worst = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    double best = INFINITY;
    for (uint64_t q = 0; q < c; ++q) {
      const double dx = xyz[3 * i] - xyz[3 * s[q]];
      const double dy = xyz[3 * i + 1] - xyz[3 * s[q] + 1];
      const double dz = xyz[3 * i + 2] - xyz[3 * s[q] + 2];
      const double v = dx * dx + dy * dy + dz * dz;
      if (v < best) best = v;
    }
    if (best > worst) worst = best;
  }
  return sqrt(worst);
}

double or_separation(const double* xyz, const int64_t* s, uint64_t c) {
  double best = INFINITY;
  for (uint64_t i = 0; i < c; ++i)
    for (uint64_t j = i + 1; j < c; ++j) {
      const double dx = xyz[3 * s[i]] - xyz[3 * s[j]];
      const double dy = xyz[3 * s[i] + 1] - xyz[3 * s[j] + 1];
      const double dz = xyz[3 * s[i] + 2] - xyz[3 * s[j] + 2];
      const double v = dx * dx + dy * dy + dz * dz;
      if (v < best) best = v;
    }
  return sqrt(best);
}
