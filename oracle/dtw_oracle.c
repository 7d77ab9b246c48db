/*
 * oracle/dtw_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded CPU restatement of the reference's hot path
 * (arXiv 2307.04904, dtwclust reference under /root/reference/proj). It is the
 * parity CHECKER for the CUDA path: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product path
 * (paper_2307_04904_b200 + libdtwgpu.so) never links or calls it.
 *
 * Pinning: every function here is checked in tests/test_oracle.py against
 *   - the reference's own known-answer tests (test_dtw.cpp, test_kmedoids.cpp),
 *   - golden vectors produced by the reference itself (oracle/_ref, built from
 *     the reference headers by oracle/Makefile; fixtures in tests/golden/).
 *
 * Build: gcc -O2 -ffp-contract=off (no -march): the reference's Release flags
 * do not contract d*d + best into an FMA (SURVEY.md finding 4), so neither may we.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_INF (INFINITY)

/* dtw.hpp:16-19 square_diff: d = a - b; d * d (separate multiply, no FMA). */
static inline double sq_diff(double a, double b) {
  const double d = a - b;
  return d * d;
}

static inline double min2(double a, double b) { return b < a ? b : a; }

/*
 * dtw.hpp:40-75 dtw_distance. half_width < 0 means WarpWindow::unlimited()
 * (warp_window.hpp:33-35: effective = max(n, m)). The caller guarantees the
 * band is feasible (|n-m| <= hw), as require_valid_pair (dtw.hpp:21-27) does.
 * `work` must hold 2*(min(n,m)+1) doubles, or be NULL (allocated here).
 */
double oracle_dtw(const double* x, int64_t nx, const double* y, int64_t ny, int64_t half_width,
                  double* work) {
  /* dtw.hpp:45-47: longer series is the outer loop. */
  const int x_outer = nx >= ny;
  const double* outer = x_outer ? x : y;
  const double* inner = x_outer ? y : x;
  const int64_t n = x_outer ? nx : ny;
  const int64_t m = x_outer ? ny : nx;
  const int64_t hw = half_width < 0 ? n : half_width; /* max(n, m) == n */

  double* own = NULL;
  if (!work) {
    own = (double*)malloc(sizeof(double) * 2 * (size_t)(m + 1));
    work = own;
  }
  double* prev = work;
  double* cur = work + (m + 1);
  for (int64_t j = 0; j <= m; ++j) prev[j] = cur[j] = ORACLE_INF; /* dtw.hpp:55-56 */
  prev[0] = 0.0;                                                  /* dtw.hpp:57 */

  for (int64_t i = 1; i <= n; ++i) { /* dtw.hpp:59-73 */
    const double xi = outer[i - 1];
    const int64_t jb = (i - hw) > 1 ? (i - hw) : 1;
    const int64_t je = (i + hw) < m ? (i + hw) : m;
    cur[jb - 1] = ORACLE_INF; /* dtw.hpp:65 */
    for (int64_t j = jb; j <= je; ++j) {
      const double best = min2(min2(prev[j - 1], prev[j]), cur[j - 1]); /* dtw.hpp:68 */
      cur[j] = sq_diff(xi, inner[j - 1]) + best;                         /* dtw.hpp:69 */
    }
    if (je < m) cur[je + 1] = ORACLE_INF; /* dtw.hpp:71 */
    double* t = prev;
    prev = cur;
    cur = t;
  }
  const double r = prev[m]; /* dtw.hpp:74 */
  free(own);
  return r;
}

/* warp_window.hpp:26-30 feasible_for. */
static inline int feasible(int64_t n, int64_t m, int64_t hw) {
  if (hw < 0) return 1;
  const int64_t gap = n > m ? n - m : m - n;
  return hw >= gap;
}

/* pairwise.hpp:29-33 pair_window: auto-widen an infeasible band to |n-m|. */
int64_t oracle_pair_window(int64_t n, int64_t m, int64_t hw, int auto_widen) {
  if (!auto_widen || feasible(n, m, hw)) return hw;
  return n > m ? n - m : m - n;
}

/* pairwise.hpp:36-38 condensed_row_offset. */
int64_t oracle_row_offset(int64_t i, int64_t p) { return i * p - i * (i + 1) / 2; }

/* pairwise.hpp:41-53 condensed_pair (binary search for the row). */
void oracle_condensed_pair(int64_t slot, int64_t p, int64_t* out_i, int64_t* out_j) {
  int64_t lo = 0, hi = p - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (oracle_row_offset(mid, p) <= slot) lo = mid;
    else hi = mid - 1;
  }
  *out_i = lo;
  *out_j = lo + 1 + (slot - oracle_row_offset(lo, p));
}

/*
 * pairwise.hpp:70-79 first band-infeasible pair in row-major order, or -1.
 * Returns 1 and writes (i, j) when one exists.
 */
int oracle_first_infeasible(const int64_t* offsets, int64_t p, int64_t hw, int64_t* out_i,
                            int64_t* out_j) {
  if (hw < 0) return 0;
  for (int64_t i = 0; i < p; ++i) {
    const int64_t li = offsets[i + 1] - offsets[i];
    for (int64_t j = i + 1; j < p; ++j) {
      const int64_t lj = offsets[j + 1] - offsets[j];
      if (!feasible(li, lj, hw)) {
        *out_i = i;
        *out_j = j;
        return 1;
      }
    }
  }
  return 0;
}

/*
 * pairwise.hpp:81-100 compute_range for condensed slots [slot_begin, slot_end):
 * out[slot - slot_begin] = dtw(series i, series j, pair_window(...)).
 * Series are packed CSR: samples[offsets[i] .. offsets[i+1]).
 */
void oracle_build_condensed(const double* samples, const int64_t* offsets, int64_t p,
                            int64_t half_width, int auto_widen, int64_t slot_begin,
                            int64_t slot_end, double* out) {
  if (slot_begin >= slot_end) return;
  int64_t maxlen = 0;
  for (int64_t s = 0; s < p; ++s) {
    const int64_t l = offsets[s + 1] - offsets[s];
    if (l > maxlen) maxlen = l;
  }
  double* work = (double*)malloc(sizeof(double) * 2 * (size_t)(maxlen + 1));
  int64_t i, j;
  oracle_condensed_pair(slot_begin, p, &i, &j);
  for (int64_t slot = slot_begin; slot < slot_end; ++slot) {
    const int64_t ni = offsets[i + 1] - offsets[i];
    const int64_t nj = offsets[j + 1] - offsets[j];
    const int64_t hw = oracle_pair_window(ni, nj, half_width, auto_widen);
    out[slot - slot_begin] = oracle_dtw(samples + offsets[i], ni, samples + offsets[j], nj, hw, work);
    if (++j == p) {
      ++i;
      j = i + 1;
    }
  }
  free(work);
}

/* In-band cell count of one pair (the GCUPS unit). */
int64_t oracle_pair_cells(int64_t nx, int64_t ny, int64_t hw) {
  const int64_t n = nx >= ny ? nx : ny;
  const int64_t m = nx >= ny ? ny : nx;
  if (hw < 0) hw = n;
  int64_t cells = 0;
  for (int64_t i = 1; i <= n; ++i) {
    const int64_t jb = (i - hw) > 1 ? (i - hw) : 1;
    const int64_t je = (i + hw) < m ? (i + hw) : m;
    if (je >= jb) cells += je - jb + 1;
  }
  return cells;
}

/* Exhaustive path enumeration, tests/support/oracles.hpp:23-59 restated. */
static void enum_paths(const double* x, int64_t n, const double* y, int64_t m, int64_t hw, int64_t i,
                       int64_t j, double acc, double* best) {
  if (i - j > hw || j - i > hw) return;
  const double d = x[i - 1] - y[j - 1];
  acc += d * d;
  if (i == n && j == m) {
    if (acc < *best) *best = acc;
    return;
  }
  if (i < n && j < m) enum_paths(x, n, y, m, hw, i + 1, j + 1, acc, best);
  if (i < n) enum_paths(x, n, y, m, hw, i + 1, j, acc, best);
  if (j < m) enum_paths(x, n, y, m, hw, i, j + 1, acc, best);
}

double oracle_dtw_brute_force(const double* x, int64_t n, const double* y, int64_t m,
                              int64_t half_width) {
  double best = ORACLE_INF;
  const int64_t hw = half_width < 0 ? (n > m ? n : m) : half_width;
  enum_paths(x, n, y, m, hw, 1, 1, 0.0, &best);
  return best;
}

/* ------------------------------------------------------------------------- */
/* k-medoids (kmedoids.hpp, cluster_result.hpp, rng.hpp restated)            */
/* ------------------------------------------------------------------------- */

/* rng.hpp:10-33 SplitMix64. */
typedef struct {
  uint64_t state;
} oracle_rng;

static inline uint64_t rng_next(oracle_rng* r) {
  uint64_t z = (r->state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline double rng_next_double(oracle_rng* r) {
  return (double)(rng_next(r) >> 11) * 0x1.0p-53; /* rng.hpp:22 */
}
static inline uint64_t rng_next_below(oracle_rng* r, uint64_t n) { /* rng.hpp:26-29 */
  return (uint64_t)(((unsigned __int128)rng_next(r) * (unsigned __int128)n) >> 64);
}
/* rng.hpp:37-41 restart_stream. */
static inline oracle_rng restart_stream(uint64_t seed, uint64_t restart) {
  oracle_rng mixer = {seed};
  const uint64_t base = rng_next(&mixer);
  oracle_rng r = {base + (restart + 1) * 0xD1B54A32D192ED03ULL};
  return r;
}

uint64_t oracle_splitmix_next(uint64_t* state) {
  oracle_rng r = {*state};
  const uint64_t v = rng_next(&r);
  *state = r.state;
  return v;
}

/* distance_matrix.hpp:45-50,71-74 over condensed storage. */
static inline double dist(const double* D, int64_t p, int64_t i, int64_t j) {
  if (i == j) return 0.0;
  if (i > j) {
    const int64_t t = i;
    i = j;
    j = t;
  }
  return D[i * (2 * p - i - 1) / 2 + (j - i - 1)];
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* cluster_result.hpp:40-61 assign_to_medoids (medoids sorted ascending). */
void oracle_assign(const double* D, int64_t p, const int64_t* medoids, int64_t k, int64_t* assignment) {
  for (int64_t j = 0; j < p; ++j) {
    int is_medoid = 0;
    for (int64_t t = 0; t < k; ++t)
      if (medoids[t] == j) is_medoid = 1;
    if (is_medoid) {
      assignment[j] = j;
      continue;
    }
    int64_t best = medoids[0];
    double bd = dist(D, p, j, best);
    for (int64_t t = 1; t < k; ++t) {
      const double d = dist(D, p, j, medoids[t]);
      if (d < bd) {
        bd = d;
        best = medoids[t];
      }
    }
    assignment[j] = best;
  }
}

/* cluster_result.hpp:65-72 assignment_cost: ascending-j sequential sum. */
double oracle_assignment_cost(const double* D, int64_t p, const int64_t* assignment) {
  double total = 0.0;
  for (int64_t j = 0; j < p; ++j) total += dist(D, p, j, assignment[j]);
  return total;
}

/* kmedoids.hpp:33-79 spread_seeds. medoids_out holds k entries, sorted. */
static void spread_seeds(const double* D, int64_t p, int64_t k, oracle_rng* rng, int64_t* medoids) {
  char* chosen = (char*)calloc((size_t)p, 1);
  double* nearest = (double*)malloc(sizeof(double) * (size_t)p);
  for (int64_t j = 0; j < p; ++j) nearest[j] = ORACLE_INF;
  int64_t count = 0;
  int64_t current = (int64_t)rng_next_below(rng, (uint64_t)p);
  while (count < k) {
    medoids[count++] = current;
    chosen[current] = 1;
    if (count == k) break;
    double total = 0.0;
    for (int64_t j = 0; j < p; ++j) {
      if (chosen[j]) continue;
      nearest[j] = min2(nearest[j], dist(D, p, j, current)) ; /* std::min(a,b): b<a?b:a */
      total += nearest[j];
    }
    int64_t next = p;
    if (total > 0.0) {
      const double target = rng_next_double(rng) * total;
      double acc = 0.0;
      for (int64_t j = 0; j < p; ++j) {
        if (chosen[j]) continue;
        acc += nearest[j];
        if (acc > target) {
          next = j;
          break;
        }
      }
    }
    if (next == p) {
      for (int64_t j = 0; j < p; ++j)
        if (!chosen[j]) {
          next = j;
          break;
        }
    }
    current = next;
  }
  qsort(medoids, (size_t)k, sizeof(int64_t), cmp_i64);
  free(chosen);
  free(nearest);
}

/* kmedoids.hpp:84-139 update_medoids. updated holds k entries. */
void oracle_update(const double* D, int64_t p, const int64_t* medoids, int64_t k,
                   const int64_t* assignment, int64_t* updated) {
  /* kmedoids.hpp:88-92: stable bucket by the medoid's slot (lower_bound). */
  int64_t* count = (int64_t*)calloc((size_t)k + 1, sizeof(int64_t));
  int64_t* slot_of = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
  for (int64_t j = 0; j < p; ++j) {
    int64_t lo = 0, hi = k; /* lower_bound */
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (medoids[mid] < assignment[j]) lo = mid + 1;
      else hi = mid;
    }
    slot_of[j] = lo;
    count[lo + 1]++;
  }
  for (int64_t c = 0; c < k; ++c) count[c + 1] += count[c];
  int64_t* members = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  for (int64_t c = 0; c < k; ++c) fill[c] = count[c];
  for (int64_t j = 0; j < p; ++j) members[fill[slot_of[j]]++] = j;

  for (int64_t c = 0; c < k; ++c) {
    const int64_t b = count[c], e = count[c + 1];
    if (b == e) { /* kmedoids.hpp:97-109 empty-cluster repair */
      int64_t worst = medoids[c];
      double wd = -1.0;
      for (int64_t j = 0; j < p; ++j) {
        int is_medoid = 0;
        for (int64_t t = 0; t < k; ++t)
          if (medoids[t] == j) is_medoid = 1;
        if (is_medoid) continue;
        const double d = dist(D, p, j, assignment[j]);
        if (d > wd) {
          wd = d;
          worst = j;
        }
      }
      updated[c] = worst;
      continue;
    }
    int64_t best = members[b]; /* kmedoids.hpp:111-121 */
    double best_sum = ORACLE_INF;
    for (int64_t a = b; a < e; ++a) {
      double sum = 0.0;
      for (int64_t q = b; q < e; ++q) sum += dist(D, p, members[a], members[q]);
      if (sum < best_sum) {
        best_sum = sum;
        best = members[a];
      }
    }
    updated[c] = best;
  }
  /* kmedoids.hpp:123-137 sort, dedupe, refill from lowest unused. */
  qsort(updated, (size_t)k, sizeof(int64_t), cmp_i64);
  int64_t u = 0;
  for (int64_t c = 0; c < k; ++c)
    if (c == 0 || updated[c] != updated[u - 1]) updated[u++] = updated[c];
  if (u < k) {
    char* used = (char*)calloc((size_t)p, 1);
    for (int64_t c = 0; c < u; ++c) used[updated[c]] = 1;
    for (int64_t j = 0; j < p && u < k; ++j)
      if (!used[j]) {
        updated[u++] = j;
        used[j] = 1;
      }
    qsort(updated, (size_t)k, sizeof(int64_t), cmp_i64);
    free(used);
  }
  free(count);
  free(slot_of);
  free(members);
  free(fill);
}

typedef void (*oracle_observer_fn)(void* user, int64_t restart, int64_t iteration, double cost);

/*
 * kmedoids.hpp:148-189 kmedoids over a condensed matrix. Returns 0, or the
 * reference error code (KOutOfRange=10, InvalidArguments=2).
 */
int oracle_kmedoids_range(const double* D, int64_t p, int64_t k, int64_t restarts,
                          int64_t max_iter, uint64_t seed, int64_t rb, int64_t re,
                          oracle_observer_fn observer, void* user, int64_t* medoids_out,
                          int64_t* assignment_out, double* cost_out, int64_t* best_r_out);

int oracle_kmedoids(const double* D, int64_t p, int64_t k, int64_t restarts, int64_t max_iter,
                    uint64_t seed, oracle_observer_fn observer, void* user, int64_t* medoids_out,
                    int64_t* assignment_out, double* cost_out) {
  int64_t best_r = -1;
  return oracle_kmedoids_range(D, p, k, restarts, max_iter, seed, 0, restarts, observer, user,
                               medoids_out, assignment_out, cost_out, &best_r);
}

/* Restarts [rb, re) of a `restarts`-restart run (restart_stream(seed, r) per restart), so a
 * run can be split across workers and reduced in restart order. */
int oracle_kmedoids_range(const double* D, int64_t p, int64_t k, int64_t restarts,
                          int64_t max_iter, uint64_t seed, int64_t rb, int64_t re,
                          oracle_observer_fn observer, void* user, int64_t* medoids_out,
                          int64_t* assignment_out, double* cost_out, int64_t* best_r_out) {
  if (k < 1 || k > p) return 10;
  if (restarts < 1) return 2;
  if (max_iter < 1) return 2;
  if (re > restarts) re = restarts;
  int64_t* med = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  int64_t* upd = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  int64_t* asg = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
  int have_best = 0;
  double best_cost = 0.0;
  for (int64_t r = rb; r < re; ++r) {
    oracle_rng rng = restart_stream(seed, (uint64_t)r);
    spread_seeds(D, p, k, &rng, med);
    double cost = 0.0;
    int converged = 0;
    for (int64_t it = 0; it < max_iter && !converged; ++it) {
      oracle_assign(D, p, med, k, asg);
      cost = oracle_assignment_cost(D, p, asg);
      if (observer) observer(user, r, it, cost);
      oracle_update(D, p, med, k, asg, upd);
      if (memcmp(upd, med, sizeof(int64_t) * (size_t)k) == 0) converged = 1;
      else memcpy(med, upd, sizeof(int64_t) * (size_t)k);
    }
    if (!converged) {
      oracle_assign(D, p, med, k, asg);
      cost = oracle_assignment_cost(D, p, asg);
    }
    if (!have_best || cost < best_cost) {
      best_cost = cost;
      memcpy(medoids_out, med, sizeof(int64_t) * (size_t)k);
      memcpy(assignment_out, asg, sizeof(int64_t) * (size_t)p);
      have_best = 1;
      *best_r_out = r;
    }
  }
  *cost_out = best_cost;
  free(med);
  free(upd);
  free(asg);
  return 0;
}

/*
 * validation.hpp:30-79 silhouette_scores over a condensed matrix. Returns 0, or the
 * reference error code: 2 (size mismatch / non-medoid assignment), 13 (k < 2).
 */
int oracle_silhouette(const double* D, int64_t p, const int64_t* medoids, int64_t k,
                      const int64_t* assignment, int64_t p_assign, double* sil, double* mean) {
  if (p_assign != p) return 2;
  if (k < 2) return 13;
  int64_t* cls = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
  int64_t* cnt = (int64_t*)calloc((size_t)k + 1, sizeof(int64_t));
  for (int64_t j = 0; j < p; ++j) {
    int64_t lo = 0, hi = k;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (medoids[mid] < assignment[j]) lo = mid + 1;
      else hi = mid;
    }
    if (lo == k || medoids[lo] != assignment[j]) {
      free(cls);
      free(cnt);
      return 2;
    }
    cls[j] = lo;
    cnt[lo + 1]++;
  }
  for (int64_t c = 0; c < k; ++c) cnt[c + 1] += cnt[c];
  int64_t* mem = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  for (int64_t c = 0; c < k; ++c) fill[c] = cnt[c];
  for (int64_t j = 0; j < p; ++j) mem[fill[cls[j]]++] = j;
  for (int64_t j = 0; j < p; ++j) sil[j] = 0.0;
  double sum = 0.0;
  for (int64_t c = 0; c < k; ++c) {
    const int64_t nc = cnt[c + 1] - cnt[c];
    for (int64_t q = cnt[c]; q < cnt[c + 1]; ++q) {
      const int64_t t = mem[q];
      if (nc == 1) continue;
      double own = 0.0;
      for (int64_t u = cnt[c]; u < cnt[c + 1]; ++u)
        if (mem[u] != t) own += dist(D, p, t, mem[u]);
      const double a = own / (double)(nc - 1);
      double b = ORACLE_INF;
      for (int64_t o = 0; o < k; ++o) {
        const int64_t no = cnt[o + 1] - cnt[o];
        if (o == c || no == 0) continue;
        double across = 0.0;
        for (int64_t u = cnt[o]; u < cnt[o + 1]; ++u) across += dist(D, p, t, mem[u]);
        b = min2(b, across / (double)no);
      }
      const double denom = a < b ? b : a;
      const double s = denom > 0.0 ? (b - a) / denom : 0.0;
      sil[t] = s;
      sum += s;
    }
  }
  *mean = sum / (double)p;
  free(cls);
  free(cnt);
  free(mem);
  free(fill);
  return 0;
}
