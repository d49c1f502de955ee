/* TEST INFRASTRUCTURE — NOT PRODUCT CODE. See fsx_oracle.h.
 *
 * Plain-C restatement of the FreeScale reference hot path. Citations are
 * /root/reference/proj paths. Only tests/, __graft_entry__.smoke() and the
 * bench.py cpu_baseline leg load this library, and only as the checker.
 */
#include "fsx_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

const char* fso_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, unsigned long long a, unsigned long long b) {
  snprintf(g_err, sizeof g_err, fmt, a, b);
  return code;
}

/* ---- rng.hpp:11-17 (splitmix64) and :37-39 (rng_double) ---------------- */
static uint64_t splitmix_next(uint64_t* s) {
  *s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* embedding.cpp:59-64 */
double fso_initial_value(uint64_t seed, uint64_t row, uint32_t d) {
  uint64_t st = seed + row * 0x9e3779b97f4a7c15ULL + ((uint64_t)d + 1) * 0xbf58476d1ce4e5b9ULL;
  splitmix_next(&st);
  double u = (double)(splitmix_next(&st) >> 11) * 0x1.0p-53;
  return (u - 0.5) * 0.2;
}

/* embedding.hpp:22-25 */
uint64_t fso_local_rows(uint64_t total_rows, int num_shards, int shard) {
  uint64_t s = (uint64_t)shard;
  return total_rows > s ? (total_rows - 1 - s) / (uint64_t)num_shards + 1 : 0;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* embedding.cpp:12-16 (sorted_unique) */
uint64_t fso_sorted_unique(uint64_t* v, uint64_t n) {
  if (n == 0) return 0;
  qsort(v, n, 8, cmp_u64);
  uint64_t k = 1;
  for (uint64_t i = 1; i < n; ++i)
    if (v[i] != v[k - 1]) v[k++] = v[i];
  return k;
}

static int member(const uint64_t* sorted, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (sorted[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo < n && sorted[lo] == x;
}

/* index of x in sorted (must be present); lower_bound as embedding.cpp:162-164 */
static uint64_t lower_bound_u64(const uint64_t* sorted, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (sorted[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* embedding.cpp:82-93: inputs are raw shard-major id lists (IndexSet
 * shard_major sorts+uniques them, :74-80); outputs are sorted. */
int fso_compute_collision(const uint64_t* cur, uint64_t ncur, const uint64_t* next, uint64_t nnext,
                          uint64_t* co, uint64_t* nco, uint64_t* exc, uint64_t* nexc,
                          uint64_t* exn, uint64_t* nexn) {
  uint64_t* a = malloc((ncur + 1) * 8);
  uint64_t* b = malloc((nnext + 1) * 8);
  if (ncur) memcpy(a, cur, ncur * 8);
  if (nnext) memcpy(b, next, nnext * 8);
  uint64_t na = fso_sorted_unique(a, ncur), nb = fso_sorted_unique(b, nnext);
  uint64_t i = 0, j = 0, c = 0, x = 0, y = 0;
  /* std::set_intersection, then the two std::set_difference passes */
  while (i < na && j < nb) {
    if (a[i] < b[j]) exc[x++] = a[i++];
    else if (b[j] < a[i]) exn[y++] = b[j++];
    else { co[c++] = a[i]; ++i; ++j; }
  }
  while (i < na) exc[x++] = a[i++];
  while (j < nb) exn[y++] = b[j++];
  *nco = c; *nexc = x; *nexn = y;
  free(a); free(b);
  return FSO_OK;
}

/* ShardView ctor, embedding.cpp:108-119 */
int fso_init_shard(uint64_t total_rows, uint32_t dim, int num_shards, int shard, uint64_t seed,
                   double* values) {
  uint64_t rows = fso_local_rows(total_rows, num_shards, shard);
  for (uint64_t l = 0; l < rows; ++l) {
    uint64_t g = (uint64_t)shard + l * (uint64_t)num_shards;
    for (uint32_t d = 0; d < dim; ++d) values[l * dim + d] = fso_initial_value(seed, g, d);
  }
  return FSO_OK;
}

/* ShardView::local_of, embedding.cpp:121-132 */
static int local_of(uint64_t total_rows, int num_shards, int shard, uint64_t g, uint64_t* l) {
  if (g >= total_rows)
    return fail(FSO_DOMAIN, "embedding: row id %llu out of range (table has %llu rows)", g, total_rows);
  if ((int)(g % (uint64_t)num_shards) != shard)
    return fail(FSO_DOMAIN, "embedding: row id %llu is not owned by shard %llu", g, (unsigned long long)shard);
  *l = g / (uint64_t)num_shards;
  return FSO_OK;
}

/* ShardView::lookup, embedding.cpp:139-146 */
int fso_lookup(const double* values, uint64_t total_rows, uint32_t dim, int num_shards, int shard,
               const uint64_t* ids, uint64_t n, double* out) {
  for (uint64_t k = 0; k < n; ++k) {
    uint64_t l;
    int rc = local_of(total_rows, num_shards, shard, ids[k], &l);
    if (rc) return rc;
    memcpy(out + k * dim, values + l * dim, (size_t)dim * 8);
  }
  return FSO_OK;
}

/* ShardView::apply_gradients, embedding.cpp:148-181. Accumulates each row's
 * gradients in occurrence order starting from 0.0, then cell -= lr*acc. */
int fso_apply_gradients(double* values, uint64_t total_rows, uint32_t dim, int num_shards,
                        int shard, double lr, const uint64_t* ids, uint64_t n,
                        const double* grads, uint64_t* uniq, uint64_t* nuniq, double* rows) {
  if (n) memcpy(uniq, ids, n * 8);
  uint64_t u = fso_sorted_unique(uniq, n);
  double* acc = calloc(u * dim + 1, 8);
  for (uint64_t k = 0; k < n; ++k) {
    uint64_t slot = lower_bound_u64(uniq, u, ids[k]);
    for (uint32_t d = 0; d < dim; ++d) acc[slot * dim + d] += grads[k * dim + d];
  }
  for (uint64_t s = 0; s < u; ++s) {
    uint64_t l;
    int rc = local_of(total_rows, num_shards, shard, uniq[s], &l);
    if (rc) { free(acc); return rc; }
    for (uint32_t d = 0; d < dim; ++d) {
      double* cell = &values[l * dim + d];
      *cell -= lr * acc[s * dim + d];
      if (!isfinite(*cell)) {
        free(acc);
        return fail(FSO_DOMAIN, "embedding: non-finite value after update of row %llu%.0llu", uniq[s], 0);
      }
      if (rows) rows[s * dim + d] = *cell;
    }
  }
  *nuniq = u;
  free(acc);
  return FSO_OK;
}

/* route_to_shard_major, embedding.cpp:185-231, all ranks in one process:
 * occurrence j of rank r goes to shard id mod p; shard s receives segments
 * ordered by source rank, each in original position order. */
int fso_route(int world, uint64_t total_rows, const uint64_t* ids, const uint64_t* lens,
              int* occ_shard, uint64_t* recv_ids, uint64_t* recv_lens, uint64_t* uniq,
              uint64_t* nuniq) {
  uint64_t total = 0;
  uint64_t* start = malloc(((size_t)world + 1) * 8);
  for (int r = 0; r < world; ++r) { start[r] = total; total += lens[r]; }
  start[world] = total;
  for (uint64_t j = 0; j < total; ++j) {
    if (ids[j] >= total_rows) {
      free(start);
      return fail(FSO_DOMAIN, "embedding: row id %llu out of range (table has %llu rows)", ids[j], total_rows);
    }
    occ_shard[j] = (int)(ids[j] % (uint64_t)world);
  }
  uint64_t at = 0, uat = 0;
  for (int s = 0; s < world; ++s) {
    uint64_t base = at;
    for (int src = 0; src < world; ++src) {
      uint64_t n = 0;
      for (uint64_t j = start[src]; j < start[src + 1]; ++j)
        if (occ_shard[j] == s) { recv_ids[at++] = ids[j]; ++n; }
      recv_lens[s * world + src] = n;
    }
    memcpy(uniq + uat, recv_ids + base, (at - base) * 8);
    nuniq[s] = fso_sorted_unique(uniq + uat, at - base);
    uat += nuniq[s];
  }
  free(start);
  return FSO_OK;
}

/* ---- engine --------------------------------------------------------------
 * Dense single-process emulation of SynchronizedEmbedding (embedding.cpp:
 * 238-297): every rank looks up its occurrences from the table state after
 * iteration i-1; gradients g = scale*row + shift; each row's gradients are
 * summed in (source rank, position) order and applied once. The reference
 * proves PrioritizedEmbedding bitwise equal to this (test_embedding.cpp:
 * 237-282, acceptance.cpp:44-85), so it is the oracle for both modes.
 * stats_out (optional) restates PrioritizedEmbedding's IterationStats for
 * rank 0 (embedding.cpp:364-371, 498-593). */
typedef struct { uint64_t id, seq; } occ_t;
static int cmp_occ(const void* a, const void* b) {
  const occ_t *x = a, *y = b;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->seq < y->seq ? -1 : x->seq > y->seq;
}

/* unique ids with owner s over all ranks' batches of one iteration */
static uint64_t shard_unique(int world, const uint64_t* ids, uint64_t n, int s, uint64_t* out) {
  uint64_t k = 0;
  for (uint64_t j = 0; j < n; ++j)
    if ((int)(ids[j] % (uint64_t)world) == s) out[k++] = ids[j];
  return fso_sorted_unique(out, k);
}

/* store_f32 != 0 models an fp32 table: values are rounded to float after
 * init and after every update, and the caller's gradient fixture is evaluated
 * in float arithmetic (g = fl(fl(scale*row) + shift), as a float32 tensor op
 * would); sums and the update itself stay f64, exactly as the reference. */
int fso_run_engine(int world, int iters, const uint64_t* ids, const uint64_t* lens,
                   uint64_t total_rows, uint32_t dim, double lr, uint64_t seed, double grad_scale,
                   double grad_shift, double* table, uint64_t* stats_out) {
  return fso_run_engine_ex2(world, iters, ids, lens, total_rows, dim, lr, seed, grad_scale, grad_shift,
                            table, stats_out, 0, 0, 0);
}

int fso_run_engine_ex(int world, int iters, const uint64_t* ids, const uint64_t* lens,
                      uint64_t total_rows, uint32_t dim, double lr, uint64_t seed, double grad_scale,
                      double grad_shift, double* table, uint64_t* stats_out, int store_f32) {
  return fso_run_engine_ex2(world, iters, ids, lens, total_rows, dim, lr, seed, grad_scale, grad_shift,
                            table, stats_out, store_f32, 0, 0);
}

static double fixture(double row, double scale, double shift, int f32) {
  if (!f32) return scale * row + shift;
  float a = (float)row * (float)scale;
  float b = a + (float)shift;
  return (double)b;
}

/* The engine's fixed association of one row's gradient sum (the product's
 * SgdPlanOp / k_sgd_* kernels; not a reference choice — the reference's
 * embedding.cpp:165-168 is the chunk == 0 case): occurrences q[0..n) in their
 * given order are left-folded from 0.0 when chunk == 0 or n <= chunk;
 * otherwise each run of `chunk` consecutive occurrences is left-folded from
 * 0.0 and the chunk sums are left-folded from 0.0 in chunk order. */
static double chunk_fold(const occ_t* q, uint64_t n, uint32_t d, uint32_t dim, const double* served,
                         double scale, double shift, int f32, uint32_t chunk) {
  if (chunk == 0 || n <= chunk) {
    double acc = 0.0;
    for (uint64_t k = 0; k < n; ++k) acc += fixture(served[q[k].seq * dim + d], scale, shift, f32);
    return acc;
  }
  double acc = 0.0;
  for (uint64_t c0 = 0; c0 < n; c0 += chunk) {
    double part = 0.0;
    uint64_t c1 = c0 + chunk < n ? c0 + chunk : n;
    for (uint64_t k = c0; k < c1; ++k) part += fixture(served[q[k].seq * dim + d], scale, shift, f32);
    acc += part;
  }
  return acc;
}

/* reduce_chunk: see chunk_fold. presum (world > 1 only): a row of iteration
 * i (0 < i < iters-1) that iteration i+1 also touches — a collision row,
 * embedding.cpp:82-93 — is summed as the engine's PRESUM protocol does:
 * each source rank's occurrences of the row (position order) are chunk-folded
 * and rounded to the table type (the requester's pre-summed CO_G row), then
 * those per-source rows are left-folded from 0.0 in source-rank order (the
 * owner's k_co_apply). Every other row: one chunk_fold over all occurrences
 * in (source rank, position) order. */
int fso_run_engine_ex2(int world, int iters, const uint64_t* ids, const uint64_t* lens,
                       uint64_t total_rows, uint32_t dim, double lr, uint64_t seed, double grad_scale,
                       double grad_shift, double* table, uint64_t* stats_out, int store_f32,
                       uint32_t reduce_chunk, int presum) {
  for (uint64_t g = 0; g < total_rows; ++g)
    for (uint32_t d = 0; d < dim; ++d) {
      double v = fso_initial_value(seed, g, d);
      table[g * dim + d] = store_f32 ? (double)(float)v : v;
    }
  uint64_t* it_start = malloc(((size_t)iters + 1) * 8);
  uint64_t at = 0, maxn = 0;
  for (int i = 0; i < iters; ++i) {
    it_start[i] = at;
    uint64_t n = 0;
    for (int r = 0; r < world; ++r) n += lens[i * world + r];
    at += n;
    if (n > maxn) maxn = n;
  }
  it_start[iters] = at;
  for (uint64_t j = 0; j < at; ++j)
    if (ids[j] >= total_rows) {
      free(it_start);
      return fail(FSO_DOMAIN, "embedding: row id %llu out of range (table has %llu rows)", ids[j], total_rows);
    }

  /* stats first: they only depend on ids */
  if (stats_out) {
    uint64_t* ua = malloc((maxn + 1) * 8);
    uint64_t* ub = malloc((maxn + 1) * 8);
    uint64_t* co = malloc((maxn + 1) * 8);
    uint64_t* tmp = malloc((maxn + 1) * 8);
    uint64_t* cos_all = malloc(((size_t)world * maxn + 1) * 8);
    uint64_t* ncos = malloc((size_t)world * 8);
    for (int i = 0; i < iters; ++i) {
      const uint64_t* cur = ids + it_start[i];
      uint64_t ncur = it_start[i + 1] - it_start[i];
      uint64_t* st = stats_out + 3 * (size_t)i;
      st[0] = st[1] = st[2] = 0;
      int has_next = i + 1 < iters;
      if (!has_next) continue; /* final iteration: empty stats, no blocking traffic */
      const uint64_t* nxt = ids + it_start[i + 1];
      uint64_t nnxt = it_start[i + 2] - it_start[i + 1];
      /* collision set of every shard for the pair (i, i+1) */
      for (int s = 0; s < world; ++s) {
        uint64_t na = shard_unique(world, cur, ncur, s, ua);
        uint64_t nb = shard_unique(world, nxt, nnxt, s, ub);
        uint64_t c = 0, x = 0, y = 0;
        while (x < na && y < nb) {
          if (ua[x] < ub[y]) ++x; else if (ub[y] < ua[x]) ++y; else { co[c++] = ua[x]; ++x; ++y; }
        }
        memcpy(cos_all + (size_t)s * maxn, co, c * 8);
        ncos[s] = c;
        if (s == 0) { st[0] = c; st[1] = nb; }
      }
      uint64_t bytes = 0;
      const uint64_t rowb = 8ull * dim;
      if (i > 0) {
        /* co grads sent by rank 0 (embedding.cpp:526-545) */
        uint64_t off0 = 0;
        for (uint64_t j = 0; j < lens[i * world + 0]; ++j) {
          uint64_t id = cur[off0 + j];
          int s = (int)(id % (uint64_t)world);
          if (member(cos_all + (size_t)s * maxn, ncos[s], id)) bytes += rowb;
        }
        /* co grads received by shard 0 (:546-556) */
        for (uint64_t j = 0; j < ncur; ++j)
          if (cur[j] % (uint64_t)world == 0 && member(cos_all, ncos[0], cur[j])) bytes += rowb;
      }
      /* E_co sent by shard 0 to every src (:563-580) */
      uint64_t nb_at = 0;
      for (int src = 0; src < world; ++src) {
        uint64_t nl = lens[(i + 1) * world + src];
        uint64_t k = 0;
        for (uint64_t j = 0; j < nl; ++j)
          if (nxt[nb_at + j] % (uint64_t)world == 0) tmp[k++] = nxt[nb_at + j];
        k = fso_sorted_unique(tmp, k);
        uint64_t want = 0;
        for (uint64_t q = 0; q < k; ++q) want += member(cos_all, ncos[0], tmp[q]);
        bytes += 8 + want * (8 + rowb);
        nb_at += nl;
      }
      /* E_co received by rank 0 from every shard (:581-588) */
      {
        uint64_t nl = lens[(i + 1) * world + 0];
        for (int s = 0; s < world; ++s) {
          uint64_t k = 0;
          for (uint64_t j = 0; j < nl; ++j)
            if ((int)(nxt[j] % (uint64_t)world) == s) tmp[k++] = nxt[j];
          k = fso_sorted_unique(tmp, k);
          uint64_t want = 0;
          for (uint64_t q = 0; q < k; ++q) want += member(cos_all + (size_t)s * maxn, ncos[s], tmp[q]);
          bytes += 8 + want * (8 + rowb);
        }
      }
      st[2] = bytes;
    }
    free(ua); free(ub); free(co); free(tmp); free(cos_all); free(ncos);
  }

  occ_t* occ = malloc((maxn + 1) * sizeof(occ_t));
  double* served = malloc(((size_t)maxn * dim + 1) * 8);
  uint64_t* nxt_u = malloc((maxn + 1) * 8);
  uint64_t* src_end = malloc(((size_t)world + 1) * 8);
  for (int i = 0; i < iters; ++i) {
    const uint64_t* cur = ids + it_start[i];
    uint64_t n = it_start[i + 1] - it_start[i];
    /* collision rows of (i, i+1) for the PRESUM association */
    const int split_co = presum && world > 1 && i > 0 && i + 1 < iters;
    uint64_t nnu = 0;
    if (split_co) {
      nnu = it_start[i + 2] - it_start[i + 1];
      memcpy(nxt_u, ids + it_start[i + 1], nnu * 8);
      nnu = fso_sorted_unique(nxt_u, nnu);
    }
    uint64_t at2 = 0;
    for (int r = 0; r < world; ++r) { at2 += lens[i * world + r]; src_end[r] = at2; }
    /* forward: all lookups see the table after iteration i-1 */
    for (uint64_t j = 0; j < n; ++j) memcpy(served + j * dim, table + cur[j] * dim, (size_t)dim * 8);
    /* backward: seq = flat (rank, position) order; stable per-row sums */
    for (uint64_t j = 0; j < n; ++j) { occ[j].id = cur[j]; occ[j].seq = j; }
    qsort(occ, n, sizeof(occ_t), cmp_occ);
    uint64_t k = 0;
    while (k < n) {
      uint64_t e = k;
      while (e < n && occ[e].id == occ[k].id) ++e;
      double* row = table + occ[k].id * dim;
      const int co_row = split_co && member(nxt_u, nnu, occ[k].id);
      for (uint32_t d = 0; d < dim; ++d) {
        double acc = 0.0;
        if (!co_row) {
          acc = chunk_fold(occ + k, e - k, d, dim, served, grad_scale, grad_shift, store_f32, reduce_chunk);
        } else {
          /* occurrences are in seq order, so each source's run is contiguous */
          uint64_t q = k;
          for (int src = 0; src < world && q < e; ++src) {
            uint64_t q1 = q;
            while (q1 < e && occ[q1].seq < src_end[src]) ++q1;
            if (q1 == q) continue;
            double ps = chunk_fold(occ + q, q1 - q, d, dim, served, grad_scale, grad_shift, store_f32,
                                   reduce_chunk);
            if (store_f32) ps = (double)(float)ps;
            acc += ps;
            q = q1;
          }
        }
        row[d] -= lr * acc;
        if (store_f32) row[d] = (double)(float)row[d];
        if (!isfinite(row[d])) {
          free(occ); free(served); free(it_start); free(nxt_u); free(src_end);
          return fail(FSO_DOMAIN, "embedding: non-finite value after update of row %llu%.0llu", occ[k].id, 0);
        }
      }
      k = e;
    }
  }
  free(occ); free(served); free(it_start); free(nxt_u); free(src_end);
  return FSO_OK;
}

/* ---- pooled (bag) lookup + scatter -------------------------------------------
 * No reference operator exists (config 3's pooled lookup is an extension; the
 * reference's toy model mean-pools whole samples, pipeline.cpp:59-67). This is
 * the restatement of the product's fsx_pooled_* semantics, on a one-shard
 * table [total_rows x dim]:
 *   forward : out[b] = chunk_fold, in token order, of row(ids[k]) over the
 *             bag's tokens k in [offs[b], offs[b+1]) (f64; rounded to float when
 *             store_f32) — the product runs it as its update kernels' reduce,
 *             so the association is theirs
 *   backward: token k of bag b takes gradient row g[b]; each row's tokens in
 *             (row, token) order are chunk-folded (chunk_fold) and applied as
 *             ShardView::apply_gradients (embedding.cpp:148-181). */
int fso_pooled_forward(const double* table, uint64_t total_rows, uint32_t dim, const uint64_t* ids,
                       const uint64_t* offs, uint64_t n_bags, int store_f32, uint32_t reduce_chunk, double* out) {
  uint64_t n = offs[n_bags];
  occ_t* occ = malloc((n + 1) * sizeof(occ_t));
  for (uint64_t k = 0; k < n; ++k) {
    if (ids[k] >= total_rows) {
      free(occ);
      return fail(FSO_DOMAIN, "embedding: row id %llu out of range (table has %llu rows)", ids[k], total_rows);
    }
    occ[k].id = ids[k];
    occ[k].seq = ids[k]; /* chunk_fold reads served[seq * dim + d]: the table row itself */
  }
  for (uint64_t b = 0; b < n_bags; ++b)
    for (uint32_t d = 0; d < dim; ++d) {
      double acc = chunk_fold(occ + offs[b], offs[b + 1] - offs[b], d, dim, table, 1.0, 0.0, 0, reduce_chunk);
      out[b * dim + d] = store_f32 ? (double)(float)acc : acc;
    }
  free(occ);
  return FSO_OK;
}

int fso_pooled_backward(double* table, uint64_t total_rows, uint32_t dim, double lr, const uint64_t* ids,
                        const uint64_t* offs, uint64_t n_bags, const double* bag_grads, int store_f32,
                        uint32_t reduce_chunk) {
  uint64_t n = offs[n_bags];
  occ_t* occ = malloc((n + 1) * sizeof(occ_t));
  double* served = malloc(((size_t)n * dim + 1) * 8);  /* per-token gradient rows */
  for (uint64_t b = 0; b < n_bags; ++b)
    for (uint64_t k = offs[b]; k < offs[b + 1]; ++k) {
      if (ids[k] >= total_rows) {
        free(occ); free(served);
        return fail(FSO_DOMAIN, "embedding: row id %llu out of range (table has %llu rows)", ids[k], total_rows);
      }
      occ[k].id = ids[k];
      occ[k].seq = k;
      memcpy(served + k * dim, bag_grads + b * dim, (size_t)dim * 8);
    }
  qsort(occ, n, sizeof(occ_t), cmp_occ);
  uint64_t k = 0;
  while (k < n) {
    uint64_t e = k;
    while (e < n && occ[e].id == occ[k].id) ++e;
    double* row = table + occ[k].id * dim;
    for (uint32_t d = 0; d < dim; ++d) {
      /* the gradient rows are used as given (scale 1, shift 0: fixture()
       * returns them unchanged, in float when store_f32 — they are floats) */
      double acc = chunk_fold(occ + k, e - k, d, dim, served, 1.0, 0.0, 0, reduce_chunk);
      row[d] -= lr * acc;
      if (store_f32) row[d] = (double)(float)row[d];
    }
    k = e;
  }
  free(occ); free(served);
  return FSO_OK;
}

/* ---- partition.cpp --------------------------------------------------------- */
typedef struct { uint64_t len; int origin, local; uint64_t g; } meta_t;
static int cmp_meta(const void* a, const void* b) {
  const meta_t *x = a, *y = b;
  if (x->len != y->len) return x->len > y->len ? -1 : 1;         /* :18 */
  if (x->origin != y->origin) return x->origin < y->origin ? -1 : 1; /* :19-20 */
  return (x->local > y->local) - (x->local < y->local);           /* :21 */
}

/* sorted_indices, partition.cpp:14-24 */
static uint64_t* sorted_indices(const uint64_t* lens, const int* origin, const int* local, uint64_t m) {
  meta_t* v = malloc((m + 1) * sizeof(meta_t));
  for (uint64_t g = 0; g < m; ++g) { v[g].len = lens[g]; v[g].origin = origin[g]; v[g].local = local[g]; v[g].g = g; }
  qsort(v, m, sizeof(meta_t), cmp_meta);
  uint64_t* idx = malloc((m + 1) * 8);
  for (uint64_t k = 0; k < m; ++k) idx[k] = v[k].g;
  free(v);
  return idx;
}

/* fbs_partition, partition.cpp:157-176 (snake deal) */
int fso_fbs(const uint64_t* lens, const int* origin, const int* local, uint64_t m, int n,
            int* assignment, uint64_t* order, uint64_t* order_lens) {
  if (n < 1) return fail(FSO_INVALID_ARGUMENT, "fbs: num_ranks must be >= 1%.0llu%.0llu", 0, 0);
  if (m % (uint64_t)n != 0)
    return fail(FSO_INVALID_ARGUMENT, "fbs: %llu samples not divisible by %llu ranks", m, (unsigned long long)n);
  uint64_t* sorted = sorted_indices(lens, origin, local, m);
  uint64_t per = m / (uint64_t)n;
  for (uint64_t k = 0; k < m; ++k) {
    uint64_t pass = k / (uint64_t)n, pos = k % (uint64_t)n;
    uint64_t rank = (pass % 2 == 0) ? pos : (uint64_t)n - 1 - pos;
    order[rank * per + pass] = sorted[k];
    assignment[sorted[k]] = (int)rank;
  }
  for (int r = 0; r < n; ++r) order_lens[r] = per;
  free(sorted);
  return FSO_OK;
}

/* min_max_segment_sizes, partition.cpp:56-92 */
static void min_max_sizes(const double* w, uint64_t m, int n, int* sizes) {
  double* prefix = malloc((m + 1) * 8);
  prefix[0] = 0.0;
  for (uint64_t i = 0; i < m; ++i) prefix[i + 1] = prefix[i] + w[i];
  size_t cols = (size_t)n + 1;
  double* dp = malloc((m + 1) * cols * 8);
  uint64_t* cut = calloc((m + 1) * cols, 8);
  for (size_t q = 0; q < (m + 1) * cols; ++q) dp[q] = INFINITY;
  for (uint64_t j = 1; j <= m; ++j) dp[j * cols + 1] = prefix[j];
  for (int k = 2; k <= n; ++k) {
    for (uint64_t j = (uint64_t)k; j <= m; ++j) {
      double best = INFINITY;
      uint64_t best_x = j - 1;
      for (uint64_t x = j - 1; x + 1 >= (uint64_t)k; --x) {
        double seg = prefix[j] - prefix[x];
        if (seg >= best) break;
        double prev = dp[x * cols + (size_t)k - 1];
        double cost = prev > seg ? prev : seg; /* std::max(a,b) returns a unless a<b */
        if (cost < best) { best = cost; best_x = x; }
        if (x == 0) break;
      }
      dp[j * cols + (size_t)k] = best;
      cut[j * cols + (size_t)k] = best_x;
    }
  }
  uint64_t j = m;
  for (int k = n; k >= 1; --k) {
    uint64_t x = k == 1 ? 0 : cut[j * cols + (size_t)k];
    sizes[k - 1] = (int)(j - x);
    j = x;
  }
  free(prefix); free(dp); free(cut);
}

/* vbs_partition, partition.cpp:178-209. tuned_sizes (nullable) plays the
 * initialized AutoTuneState (:189-195); sizes_out (nullable) receives the
 * segment sizes used (the fresh-state seed at :202-207). */
int fso_vbs(const uint64_t* lens, const int* origin, const int* local, uint64_t m, int n,
            double alpha, const int* tuned_sizes, int* sizes_out, int* assignment,
            uint64_t* order, uint64_t* order_lens) {
  if (alpha <= 0) return fail(FSO_INVALID_ARGUMENT, "vbs: alpha must be > 0%.0llu%.0llu", 0, 0);
  if (m == 0) return fail(FSO_INVALID_ARGUMENT, "vbs: no samples%.0llu%.0llu", 0, 0);
  if ((uint64_t)n > m)
    return fail(FSO_INVALID_ARGUMENT, "vbs: %llu ranks but only %llu samples (cannot give every rank one)", (unsigned long long)n, m);
  uint64_t* sorted = sorted_indices(lens, origin, local, m);
  int* sizes = malloc(sizeof(int) * (size_t)n);
  int tuned = 0;
  if (tuned_sizes) {
    uint64_t tot = 0;
    for (int r = 0; r < n; ++r) tot += (uint64_t)tuned_sizes[r];
    tuned = tot == m;
  }
  if (tuned) {
    memcpy(sizes, tuned_sizes, sizeof(int) * (size_t)n);
  } else {
    double* w = malloc((m + 1) * 8);
    for (uint64_t k = 0; k < m; ++k) w[k] = pow((double)lens[sorted[k]], alpha);
    min_max_sizes(w, m, n, sizes);
    free(w);
  }
  uint64_t cursor = 0;
  for (int r = 0; r < n; ++r) {
    order_lens[r] = (uint64_t)sizes[r];
    for (int q = 0; q < sizes[r]; ++q) {
      order[cursor] = sorted[cursor];
      assignment[sorted[cursor]] = r;
      ++cursor;
    }
  }
  if (sizes_out) memcpy(sizes_out, sizes, sizeof(int) * (size_t)n);
  free(sizes); free(sorted);
  return FSO_OK;
}

/* autotune_update, partition.cpp:211-269, `rounds` consecutive calls */
int fso_autotune(int n, int* sizes, double* ema_local, double* ema_global, int step, double delta,
                 double decay, const double* times, int rounds) {
  for (int round = 0; round < rounds; ++round) {
    const double* t = times + (size_t)round * (size_t)n;
    double mean = 0;
    for (int r = 0; r < n; ++r) {
      if (t[r] <= 0) return fail(FSO_INVALID_ARGUMENT, "autotune: execution times must be > 0%.0llu%.0llu", 0, 0);
      mean += t[r];
    }
    mean /= (double)n;
    int first = *ema_global == 0.0;
    *ema_global = first ? mean : decay * *ema_global + (1 - decay) * mean;
    for (int r = 0; r < n; ++r) ema_local[r] = first ? t[r] : decay * ema_local[r] + (1 - decay) * t[r];
    int total = 0;
    for (int r = 0; r < n; ++r) total += sizes[r];
    for (int r = 0; r < n; ++r) {
      if (ema_local[r] > (1 + delta) * *ema_global) {
        int v = sizes[r] - step;
        sizes[r] = v > 1 ? v : 1;
      } else if (ema_local[r] < (1 - delta) * *ema_global) {
        sizes[r] += step;
      }
    }
    int diff = -total;
    for (int r = 0; r < n; ++r) diff += sizes[r];
    while (diff > 0) {
      int donor = 0;
      for (int r = 1; r < n; ++r)
        if (sizes[r] > sizes[donor] || (sizes[r] == sizes[donor] && ema_local[r] > ema_local[donor])) donor = r;
      if (sizes[donor] <= 1) break;
      --sizes[donor];
      --diff;
    }
    while (diff < 0) {
      int recv = 0;
      for (int r = 1; r < n; ++r)
        if (sizes[r] < sizes[recv] || (sizes[r] == sizes[recv] && ema_local[r] < ema_local[recv])) recv = r;
      ++sizes[recv];
      ++diff;
    }
  }
  return FSO_OK;
}

/* CostModel::compute_time_for_lengths, sim.hpp:24-35 */
double fso_cost(double c0, double c1, double c2, const uint64_t* lens, uint64_t n) {
  uint64_t tokens = 0;
  double sq = 0;
  for (uint64_t i = 0; i < n; ++i) {
    tokens += lens[i];
    sq += (double)lens[i] * (double)lens[i];
  }
  return c0 + c1 * (double)tokens + c2 * sq;
}

/* min_max_contiguous_bruteforce, partition.cpp:292-319 */
static double bf_rec(const double* prefix, uint64_t m, uint64_t* cuts, int ncuts, int k, uint64_t lo, double best) {
  if (k == ncuts) {
    double mx = 0;
    uint64_t prev = 0;
    for (int c = 0; c < ncuts; ++c) {
      double s = prefix[cuts[c]] - prefix[prev];
      if (mx < s) mx = s;
      prev = cuts[c];
    }
    double s = prefix[m] - prefix[prev];
    if (mx < s) mx = s;
    return mx < best ? mx : best;
  }
  for (uint64_t c = lo; c + (uint64_t)(ncuts - k) <= m; ++c) {
    cuts[k] = c;
    best = bf_rec(prefix, m, cuts, ncuts, k + 1, c + 1, best);
  }
  return best;
}

double fso_bruteforce(const double* w, uint64_t m, int segments) {
  double* prefix = malloc((m + 1) * 8);
  prefix[0] = 0;
  for (uint64_t i = 0; i < m; ++i) prefix[i + 1] = prefix[i] + w[i];
  double r;
  if (segments == 1) {
    r = prefix[m];
  } else {
    uint64_t* cuts = malloc(sizeof(uint64_t) * (size_t)segments);
    r = bf_rec(prefix, m, cuts, segments - 1, 0, 1, INFINITY);
    free(cuts);
  }
  free(prefix);
  return r;
}
