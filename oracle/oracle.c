/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference hot path
 * (see oracle.h for who may call it and how it is pinned).  Every function
 * cites the reference file:line it restates; paths are relative to
 * /root/reference/proj.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ rng.hpp */

/* rng.hpp:16-21 (SplitMix64 finalizer) */
uint64_t orc_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.hpp:25-27 (Rng constructor) */
uint64_t orc_rng_base(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return orc_mix64(orc_mix64(orc_mix64(seed) ^ a) ^ b) ^ orc_mix64(c);
}

/* rng.hpp:29-34 (at + uniform_i32: 64-bit modulo of the mixed counter) */
int32_t orc_uniform_i32(uint64_t base, uint64_t index, int32_t lo, int32_t hi) {
  uint64_t range = (uint64_t)(int64_t)hi - (uint64_t)(int64_t)lo + 1;
  return (int32_t)((int64_t)lo + (int64_t)(orc_mix64(base + index) % range));
}

/* rng.hpp:36-39 */
float orc_uniform_float(uint64_t base, uint64_t index, float lo, float hi) {
  double u = (double)(orc_mix64(base + index) >> 11) * 0x1.0p-53;
  return (float)((double)lo + u * ((double)hi - (double)lo));
}

/* tools/tq_main.cpp:147-152 */
void orc_random_i32(int32_t* out, int64_t n, uint64_t seed, uint64_t stream, int32_t lo,
                    int32_t hi) {
  uint64_t base = orc_rng_base(seed, stream, 0, 0);
  for (int64_t i = 0; i < n; ++i) out[i] = orc_uniform_i32(base, (uint64_t)i, lo, hi);
}

/* tools/tq_main.cpp:335-340 */
void orc_project_inputs(float* x1, float* x2, int64_t n, uint64_t seed) {
  uint64_t base = orc_rng_base(seed, 2, 0, 0);
  for (int64_t i = 0; i < n; ++i) {
    x1[i] = orc_uniform_float(base, (uint64_t)(2 * i), -4.0f, 4.0f);
    x2[i] = orc_uniform_float(base, (uint64_t)(2 * i + 1), -4.0f, 4.0f);
  }
}

/* -------------------------------------------------------- ssb_gen.cpp */

enum { kLineorder = 1, kDate, kSupplier, kCustomer, kPart }; /* ssb_gen.cpp:11 */

/* ssb_gen.cpp:179-186 */
int64_t orc_lineorder_rows(int64_t sf) { return 6000000LL * sf; }
int64_t orc_supplier_rows(int64_t sf) { return 2000LL * sf; }
int64_t orc_customer_rows(int64_t sf) { return 30000LL * sf; }
int64_t orc_part_rows(int64_t sf) {
  int w = 0;
  for (uint64_t v = (uint64_t)sf; v; v >>= 1) ++w; /* std::bit_width */
  return 200000LL * w;
}

static int is_leap(int y) { return y % 4 == 0 && (y % 100 != 0 || y % 400 == 0); }
static int days_in_month(int y, int m) {
  static const int kDays[12] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  return (m == 2 && is_leap(y)) ? 29 : kDays[m - 1];
}

/* ssb_gen.cpp:60-90 */
void orc_gen_date(int32_t* c) {
  const int64_t R = 2556;
  int y = 1992, m = 1, d = 1, doy = 1;
  for (int64_t i = 0; i < R; ++i) {
    c[0 * R + i] = y * 10000 + m * 100 + d;
    c[1 * R + i] = y;
    c[2 * R + i] = y * 100 + m;
    c[3 * R + i] = (y - 1992) * 12 + (m - 1);
    c[4 * R + i] = (doy - 1) / 7 + 1;
    ++d;
    ++doy;
    if (d > days_in_month(y, m)) {
      d = 1;
      if (++m > 12) {
        m = 1;
        ++y;
        doy = 1;
      }
    }
  }
}

/* ssb_gen.cpp:94-112 */
void orc_gen_geo(int table_id, int64_t sf, uint64_t seed, int64_t rows, int32_t* c) {
  uint64_t base = orc_rng_base(seed, (uint64_t)sf, (uint64_t)table_id, 0);
  for (int64_t i = 0; i < rows; ++i) {
    int32_t city = orc_uniform_i32(base, (uint64_t)i, 0, 249);
    c[0 * rows + i] = (int32_t)(i + 1);
    c[1 * rows + i] = city;
    c[2 * rows + i] = city / 10;
    c[3 * rows + i] = city / 10 / 5;
  }
}

/* ssb_gen.cpp:114-129 */
void orc_gen_part(int64_t sf, uint64_t seed, int64_t rows, int32_t* c) {
  uint64_t base = orc_rng_base(seed, (uint64_t)sf, kPart, 0);
  for (int64_t i = 0; i < rows; ++i) {
    int32_t brand = orc_uniform_i32(base, (uint64_t)i, 0, 999);
    c[0 * rows + i] = (int32_t)(i + 1);
    c[1 * rows + i] = brand;
    c[2 * rows + i] = brand / 40;
    c[3 * rows + i] = brand / 40 / 5;
  }
}

typedef struct {
  uint64_t base;
  int32_t lo, hi;
  const int32_t* date_keys;
  int64_t begin, end;
  int32_t* out;
} gen_job;

static void* gen_worker(void* arg) {
  gen_job* j = (gen_job*)arg;
  for (int64_t i = j->begin; i < j->end; ++i) {
    int32_t v = orc_uniform_i32(j->base, (uint64_t)i, j->lo, j->hi);
    j->out[i] = j->date_keys ? j->date_keys[v] : v;
  }
  return NULL;
}

/* ssb_gen.cpp:131-157: column_id 0 is lo_orderdate (a date-key index), 1..8
 * are uniform columns over the ranges below. */
void orc_gen_lineorder_col(int64_t sf, uint64_t seed, int column_id, int64_t begin, int64_t end,
                           int32_t* out, int nthreads) {
  int32_t date_keys[2556];
  int32_t dates[5 * 2556];
  int32_t lo = 0, hi = 0;
  const int32_t* dk = NULL;
  switch (column_id) {
    case 0:
      orc_gen_date(dates);
      memcpy(date_keys, dates, sizeof(date_keys));
      dk = date_keys;
      lo = 0;
      hi = 2555;
      break;
    case 1: lo = 1; hi = (int32_t)orc_customer_rows(sf); break;
    case 2: lo = 1; hi = (int32_t)orc_supplier_rows(sf); break;
    case 3: lo = 1; hi = (int32_t)orc_part_rows(sf); break;
    case 4: lo = 1; hi = 50; break;
    case 5: lo = 0; hi = 10; break;
    case 6: lo = 1; hi = 100000; break;
    case 7: lo = 1; hi = 1000000; break;
    case 8: lo = 1; hi = 100000; break;
    default: return;
  }
  uint64_t base = orc_rng_base(seed, (uint64_t)sf, kLineorder, (uint64_t)column_id);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 64) nthreads = 64;
  pthread_t th[64];
  gen_job jobs[64];
  int64_t n = end - begin, chunk = (n + nthreads - 1) / nthreads;
  int started = 0;
  for (int t = 0; t < nthreads; ++t) {
    int64_t b = begin + t * chunk, e = b + chunk > end ? end : b + chunk;
    if (b >= e) break;
    jobs[t] = (gen_job){base, lo, hi, dk, b, e, out - begin};
    if (nthreads == 1) {
      gen_worker(&jobs[t]);
    } else {
      pthread_create(&th[t], NULL, gen_worker, &jobs[t]);
      ++started;
    }
  }
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------ SSB plans + semantics */

/* Restatement of ssb_plans.cpp:21-253 (probe order, filters, payloads, group
 * parts) with dictionary literals resolved through the canonical
 * dictionaries of ssb_gen.cpp:196-241 (codes pinned by test_storage.cpp:186-229:
 * AMERICA=1 ASIA=2 EUROPE=3, UNITED STATES=9, UNITED KI1=191 KI5=195,
 * MFGR#1=0 MFGR#2=1, MFGR#12=1 MFGR#14=3, MFGR#2221=260 MFGR#2228=267
 * MFGR#2239=278, Dec1997=71). */
enum { D_SUPP = 0, D_CUST = 1, D_PART = 2, D_DATE = 3 };
enum { AGG_REV = 0, AGG_EXT_DISC = 1, AGG_REV_COST = 2 };

typedef struct {
  int dim, filter_col, nranges;
  int32_t r[2][2];
  int payload_col; /* -1: join carries no payload (payload 0, ssb_queries.cpp:116) */
} orc_join;

typedef struct {
  int nfact; /* flight 1 */
  int fcol[3], fop[3];
  int32_t flo[3], fhi[3];
  int njoins;
  orc_join j[4];
  int ngroup;
  int gjoin[3];
  int32_t glo[3], ghi[3];
  int agg;
} orc_plan;

#define J(dim, fc, nr, a0, b0, a1, b1, pc) {dim, fc, nr, {{a0, b0}, {a1, b1}}, pc}
#define NOJ {0, -1, 0, {{0, 0}, {0, 0}}, -1}

static const orc_plan kPlans[13] = {
    /* q11 ssb_plans.cpp:21-35 */
    {3, {0, 5, 4}, {5, 5, 0}, {19930101, 1, 25}, {19940101, 3, 25}, 0, {NOJ, NOJ, NOJ, NOJ}, 0, {0}, {0}, {0}, AGG_EXT_DISC},
    /* q12 :37-51 */
    {3, {0, 5, 4}, {5, 5, 5}, {19940101, 4, 26}, {19940131, 6, 35}, 0, {NOJ, NOJ, NOJ, NOJ}, 0, {0}, {0}, {0}, AGG_EXT_DISC},
    /* q13 :53-68 */
    {3, {0, 5, 4}, {5, 5, 5}, {19940205, 5, 26}, {19940211, 7, 35}, 0, {NOJ, NOJ, NOJ, NOJ}, 0, {0}, {0}, {0}, AGG_EXT_DISC},
    /* q21 :110-131 (q2x) supplier(s_region) -> part(filter, brand1) -> date(year) */
    {0, {0}, {0}, {0}, {0}, 3,
     {J(D_SUPP, 3, 1, 1, 1, 0, 0, -1), J(D_PART, 2, 1, 1, 1, 0, 0, 1), J(D_DATE, -1, 0, 0, 0, 0, 0, 1), NOJ},
     2, {2, 1}, {1992, 0}, {1998, 999}, AGG_REV},
    /* q22 :133-138 */
    {0, {0}, {0}, {0}, {0}, 3,
     {J(D_SUPP, 3, 1, 2, 2, 0, 0, -1), J(D_PART, 1, 1, 260, 267, 0, 0, 1), J(D_DATE, -1, 0, 0, 0, 0, 0, 1), NOJ},
     2, {2, 1}, {1992, 0}, {1998, 999}, AGG_REV},
    /* q23 :140-144 */
    {0, {0}, {0}, {0}, {0}, 3,
     {J(D_SUPP, 3, 1, 3, 3, 0, 0, -1), J(D_PART, 1, 1, 278, 278, 0, 0, 1), J(D_DATE, -1, 0, 0, 0, 0, 0, 1), NOJ},
     2, {2, 1}, {1992, 0}, {1998, 999}, AGG_REV},
    /* q31 :148-176 (q3x) supplier -> customer -> date; group (c_geo, s_geo, year) */
    {0, {0}, {0}, {0}, {0}, 3,
     {J(D_SUPP, 3, 1, 2, 2, 0, 0, 2), J(D_CUST, 3, 1, 2, 2, 0, 0, 2), J(D_DATE, 1, 1, 1992, 1997, 0, 0, 1), NOJ},
     3, {1, 0, 2}, {0, 0, 1992}, {24, 24, 1998}, AGG_REV},
    /* q32 :178-186 */
    {0, {0}, {0}, {0}, {0}, 3,
     {J(D_SUPP, 2, 1, 9, 9, 0, 0, 1), J(D_CUST, 2, 1, 9, 9, 0, 0, 1), J(D_DATE, 1, 1, 1992, 1997, 0, 0, 1), NOJ},
     3, {1, 0, 2}, {0, 0, 1992}, {249, 249, 1998}, AGG_REV},
    /* q33 :195-201 */
    {0, {0}, {0}, {0}, {0}, 3,
     {J(D_SUPP, 1, 2, 191, 191, 195, 195, 1), J(D_CUST, 1, 2, 191, 191, 195, 195, 1), J(D_DATE, 1, 1, 1992, 1997, 0, 0, 1), NOJ},
     3, {1, 0, 2}, {0, 0, 1992}, {249, 249, 1998}, AGG_REV},
    /* q34 :203-210 */
    {0, {0}, {0}, {0}, {0}, 3,
     {J(D_SUPP, 1, 2, 191, 191, 195, 195, 1), J(D_CUST, 1, 2, 191, 191, 195, 195, 1), J(D_DATE, 3, 1, 71, 71, 0, 0, 1), NOJ},
     3, {1, 0, 2}, {0, 0, 1992}, {249, 249, 1998}, AGG_REV},
    /* q41 :215-233 supplier -> customer(c_nation) -> part -> date(year) */
    {0, {0}, {0}, {0}, {0}, 4,
     {J(D_SUPP, 3, 1, 1, 1, 0, 0, -1), J(D_CUST, 3, 1, 1, 1, 0, 0, 2), J(D_PART, 3, 1, 0, 1, 0, 0, -1), J(D_DATE, -1, 0, 0, 0, 0, 0, 1)},
     2, {3, 1}, {1992, 0}, {1998, 24}, AGG_REV_COST},
    /* q42 :235-253 supplier(s_nation) -> customer -> part(category) -> date(year 97-98) */
    {0, {0}, {0}, {0}, {0}, 4,
     {J(D_SUPP, 3, 1, 1, 1, 0, 0, 2), J(D_CUST, 3, 1, 1, 1, 0, 0, -1), J(D_PART, 3, 1, 0, 1, 0, 0, 2), J(D_DATE, 1, 1, 1997, 1998, 0, 0, 1)},
     3, {3, 0, 2}, {1992, 0, 0}, {1998, 24, 24}, AGG_REV_COST},
    /* q43 :255-275 supplier(s_city) -> part(brand1) -> customer -> date */
    {0, {0}, {0}, {0}, {0}, 4,
     {J(D_SUPP, 2, 1, 9, 9, 0, 0, 1), J(D_PART, 2, 1, 3, 3, 0, 0, 1), J(D_CUST, 3, 1, 1, 1, 0, 0, -1), J(D_DATE, 1, 1, 1997, 1998, 0, 0, 1)},
     3, {3, 0, 1}, {1992, 0, 0}, {1998, 249, 999}, AGG_REV_COST},
};

/* ssb_queries.cpp:17-27 (AggregateTable strides, last part fastest) */
static int64_t plan_cells(const orc_plan* p, int64_t* strides) {
  int64_t cells = 1;
  for (int g = p->ngroup - 1; g >= 0; --g) {
    if (strides) strides[g] = cells;
    cells *= (int64_t)(p->ghi[g] - p->glo[g] + 1);
  }
  return cells;
}

int64_t orc_query_cells(int qid) {
  if (qid < 0 || qid >= 13) return -1;
  return plan_cells(&kPlans[qid], NULL);
}

int orc_query_ngroup(int qid) { return (qid < 0 || qid >= 13) ? -1 : kPlans[qid].ngroup; }

/* tile.hpp:122-132 */
static int eval_pred(int op, int32_t y, int32_t lo, int32_t hi) {
  switch (op) {
    case 0: return y < lo;
    case 1: return y <= lo;
    case 2: return y > lo;
    case 3: return y >= lo;
    case 4: return y == lo;
    case 5: return y >= lo && y <= hi;
  }
  return 0;
}

/* positional date lookup: ssb_reference.cpp:16-21, 30 (datekey -> row) */
typedef struct {
  int32_t* keys;
  int32_t* rows;
  int64_t n;
} date_index;

static int cmp_pair(const void* a, const void* b) {
  const int32_t* x = (const int32_t*)a;
  const int32_t* y = (const int32_t*)b;
  return (x[0] > y[0]) - (x[0] < y[0]);
}

static int64_t date_row(const date_index* ix, int32_t key) {
  int64_t lo = 0, hi = ix->n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    int32_t k = ix->keys[2 * mid];
    if (k == key) return ix->keys[2 * mid + 1];
    if (k < key) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

/* Row-at-a-time interpreter following ssb_reference.cpp:138-261 for the
 * arithmetic (positional dimension rows: key-1, date via index) and
 * ssb_queries.cpp:212-273 for probe order, survivors and dense-cell
 * accumulation with occupancy (ssb_queries.cpp:32-35). */
int orc_query_partial(const orc_db* db, int qid, int64_t begin, int64_t end, int64_t* sums,
                      int64_t* counts, int64_t* survivors) {
  if (qid < 0 || qid >= 13) return -2;
  const orc_plan* p = &kPlans[qid];
  if (p->njoins == 0) {
    /* flight 1: ssb_reference.cpp:46-63 / ssb_queries.cpp:157-210 */
    const int32_t* ext = db->lo[6];
    const int32_t* disc = db->lo[5];
    int64_t s = 0, c = 0;
    for (int64_t i = begin; i < end; ++i) {
      int pass = 1;
      for (int f = 0; f < p->nfact && pass; ++f)
        pass = eval_pred(p->fop[f], db->lo[p->fcol[f]][i], p->flo[f], p->fhi[f]);
      if (!pass) continue;
      s += (int64_t)ext[i] * (int64_t)disc[i];
      ++c;
    }
    sums[0] += s;
    counts[0] += c;
    survivors[0] += c;
    return 0;
  }

  date_index ix = {0};
  ix.n = db->date_rows;
  ix.keys = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)(ix.n ? ix.n : 1));
  for (int64_t r = 0; r < ix.n; ++r) {
    ix.keys[2 * r] = db->date[0][r];
    ix.keys[2 * r + 1] = (int32_t)r;
  }
  qsort(ix.keys, (size_t)ix.n, 2 * sizeof(int32_t), cmp_pair);

  static const int fact_key_col[4] = {2, 1, 3, 0}; /* supp cust part date */
  int64_t strides[3];
  plan_cells(p, strides);
  int rc = 0;
  for (int64_t i = begin; i < end; ++i) {
    int32_t payload[4] = {0, 0, 0, 0};
    int ok = 1;
    for (int j = 0; j < p->njoins && ok; ++j) {
      const orc_join* jn = &p->j[j];
      int32_t key = db->lo[fact_key_col[jn->dim]][i];
      int64_t row;
      const int32_t* const* cols;
      switch (jn->dim) {
        case D_SUPP: row = key - 1; cols = db->supp; ok = row >= 0 && row < db->supp_rows; break;
        case D_CUST: row = key - 1; cols = db->cust; ok = row >= 0 && row < db->cust_rows; break;
        case D_PART: row = key - 1; cols = db->part; ok = row >= 0 && row < db->part_rows; break;
        default: row = date_row(&ix, key); cols = db->date; ok = row >= 0; break;
      }
      if (!ok) break;
      if (jn->filter_col >= 0) {
        int32_t v = cols[jn->filter_col][row];
        int hit = 0;
        for (int r = 0; r < jn->nranges; ++r) hit |= v >= jn->r[r][0] && v <= jn->r[r][1];
        ok = hit;
      }
      if (!ok) break;
      survivors[j] += 1;
      payload[j] = jn->payload_col >= 0 ? cols[jn->payload_col][row] : 0;
    }
    if (!ok) continue;
    int64_t idx = 0;
    for (int g = 0; g < p->ngroup; ++g) {
      int32_t v = payload[p->gjoin[g]];
      if (v < p->glo[g] || v > p->ghi[g]) rc = -1; /* ssb_queries.cpp:32-33 */
      idx += (int64_t)(v - p->glo[g]) * strides[g];
    }
    if (rc) break;
    int64_t value;
    if (p->agg == AGG_REV)
      value = db->lo[7][i];
    else
      value = (int64_t)db->lo[7][i] - (int64_t)db->lo[8][i];
    sums[idx] += value;
    counts[idx] += 1;
  }
  free(ix.keys);
  return rc;
}

/* ssb_queries.cpp:49-56 (key_of) */
void orc_cell_key(int qid, int64_t cell, int32_t* values) {
  const orc_plan* p = &kPlans[qid];
  int64_t strides[3];
  plan_cells(p, strides);
  for (int g = 0; g < p->ngroup; ++g) {
    values[g] = p->glo[g] + (int32_t)(cell / strides[g]);
    cell %= strides[g];
  }
}

/* ssb_queries.cpp:145-155 (grouped_result) and :207-209 (flight 1 always
 * emits one row). */
int64_t orc_query(const orc_db* db, int qid, int32_t* groups, int64_t* sums, int64_t max_rows,
                  int64_t* survivors) {
  if (qid < 0 || qid >= 13) return -2;
  const orc_plan* p = &kPlans[qid];
  int64_t cells = plan_cells(p, NULL);
  int64_t* s = (int64_t*)calloc((size_t)cells, sizeof(int64_t));
  int64_t* c = (int64_t*)calloc((size_t)cells, sizeof(int64_t));
  for (int j = 0; j < 4; ++j) survivors[j] = 0;
  int rc = orc_query_partial(db, qid, 0, db->lo_rows, s, c, survivors);
  int64_t n = 0;
  if (rc == 0) {
    if (p->njoins == 0) {
      if (max_rows >= 1) sums[0] = s[0];
      n = 1;
    } else {
      for (int64_t i = 0; i < cells; ++i) {
        if (!c[i]) continue;
        if (n < max_rows) {
          orc_cell_key(qid, i, groups + 3 * n);
          sums[n] = s[i];
        }
        ++n;
      }
    }
  }
  free(s);
  free(c);
  return rc ? rc : n;
}

/* ------------------------------------------------------- hash table */

static int shift_for(int64_t capacity) { /* hash_table.cpp:12-16 */
  int tz = 0;
  while (((uint64_t)capacity >> tz & 1) == 0) ++tz;
  return 32 - tz;
}

/* hash_table.cpp:20-48 (serial build; workers <= 1) */
int orc_ht_build(const int32_t* keys, const int32_t* payloads, int64_t n, int64_t capacity,
                 int32_t* slot_keys, int32_t* slot_payloads) {
  if (capacity < 2 || (capacity & (capacity - 1))) return 1;
  if (n * 2 > capacity) return 3;
  int shift = shift_for(capacity);
  uint32_t mask = (uint32_t)(capacity - 1);
  for (int64_t s = 0; s < capacity; ++s) {
    slot_keys[s] = INT32_MIN;
    slot_payloads[s] = 0;
  }
  for (int64_t i = 0; i < n; ++i) {
    int32_t key = keys[i];
    if (key == INT32_MIN) return 3;
    uint32_t s = (uint32_t)(((uint32_t)key * 2654435769u) >> shift);
    for (;;) {
      if (slot_keys[s] == INT32_MIN) {
        slot_keys[s] = key;
        slot_payloads[s] = payloads[i];
        break;
      }
      if (slot_keys[s] == key) return 3;
      s = (s + 1) & mask;
    }
  }
  return 0;
}

/* hash_table.hpp:35-51 */
int orc_ht_probe(const int32_t* slot_keys, const int32_t* slot_payloads, int64_t capacity,
                 int32_t key, int32_t* payload) {
  if (key == INT32_MIN) return 0;
  int shift = shift_for(capacity);
  uint32_t mask = (uint32_t)(capacity - 1);
  uint32_t s = (uint32_t)(((uint32_t)key * 2654435769u) >> shift);
  for (int64_t step = 0; step <= mask; ++step, s = (s + 1) & mask) {
    int32_t k = slot_keys[s];
    if (k == key) {
      *payload = slot_payloads[s];
      return 1;
    }
    if (k == INT32_MIN) return 0;
  }
  return 0;
}

/* join.cpp:11-18 */
int64_t orc_join_checksum(const int32_t* pk, const int32_t* pp, int64_t n,
                          const int32_t* slot_keys, const int32_t* slot_payloads,
                          int64_t capacity) {
  int64_t sum = 0;
  for (int64_t i = 0; i < n; ++i) {
    int32_t v;
    if (orc_ht_probe(slot_keys, slot_payloads, capacity, pk[i], &v)) sum += (int64_t)v + pp[i];
  }
  return sum;
}

/* ------------------------------------------------------------ select */

/* select.hpp:56-73 with workers = 1: output in input order */
int64_t orc_select_input_order(const int32_t* in, int64_t n, int op, int32_t lo, int32_t hi,
                               int32_t* out) {
  int64_t d = 0;
  for (int64_t i = 0; i < n; ++i)
    if (eval_pred(op, in[i], lo, hi)) out[d++] = in[i];
  return d;
}

/* select.hpp:107-135 in deterministic mode: blocks in order; inside a block
 * thread t owns slots t, t+bt, ... and writes its matches (stride order) at
 * its exclusive prefix (block_ops.hpp:85-122). */
int64_t orc_select_crystal_order(const int32_t* in, int64_t n, int op, int32_t lo, int32_t hi,
                                 int bt, int ipt, int32_t* out) {
  int64_t tile = (int64_t)bt * ipt, d = 0;
  for (int64_t off = 0; off < n; off += tile) {
    int64_t valid = n - off < tile ? n - off : tile;
    for (int t = 0; t < bt; ++t)
      for (int64_t i = t; i < valid; i += bt)
        if (eval_pred(op, in[off + i], lo, hi)) out[d++] = in[off + i];
  }
  return d;
}

/* ----------------------------------------------------------- project */

/* project.hpp:49-54 (float mul, float mul, float add; built with
 * -ffp-contract=off so no FMA contraction, matching x86-64 baseline codegen) */
void orc_project_linear(const float* x1, const float* x2, int64_t n, float a, float b,
                        float* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = a * x1[i] + b * x2[i];
}

/* project.hpp:56-64 */
void orc_project_sigmoid(const float* x1, const float* x2, int64_t n, float a, float b,
                         float* out) {
  const double ad = a, bd = b;
  for (int64_t i = 0; i < n; ++i) {
    double z = ad * x1[i] + bd * x2[i];
    out[i] = (float)(1.0 / (1.0 + exp(-z)));
  }
}

/* ------------------------------------------------------------- radix */

/* radix.hpp:44-47 */
uint32_t orc_radix_digit(int32_t key, int start_bit, int num_bits) {
  uint32_t biased = (uint32_t)key ^ 0x80000000u;
  return (biased >> start_bit) & ((1u << num_bits) - 1);
}

/* radix.cpp:138-163 with one owner: stable counting-sort passes low to high */
void orc_lsb_sort(int32_t* keys, int32_t* payloads, int64_t n, int bits_per_pass) {
  if (n <= 1) return;
  int32_t* tk = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* tp = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *sk = keys, *sp = payloads, *dk = tk, *dp = tp;
  int64_t count[256];
  for (int start = 0; start < 32; start += bits_per_pass) {
    int bits = bits_per_pass < 32 - start ? bits_per_pass : 32 - start;
    int digits = 1 << bits;
    memset(count, 0, sizeof(count));
    for (int64_t i = 0; i < n; ++i) ++count[orc_radix_digit(sk[i], start, bits)];
    int64_t run = 0;
    for (int d = 0; d < digits; ++d) {
      int64_t c = count[d];
      count[d] = run;
      run += c;
    }
    for (int64_t i = 0; i < n; ++i) {
      int64_t pos = count[orc_radix_digit(sk[i], start, bits)]++;
      dk[pos] = sk[i];
      dp[pos] = sp[i];
    }
    int32_t* t;
    t = sk; sk = dk; dk = t;
    t = sp; sp = dp; dp = t;
  }
  if (sk != keys) {
    memcpy(keys, sk, sizeof(int32_t) * (size_t)n);
    memcpy(payloads, sp, sizeof(int32_t) * (size_t)n);
  }
  free(tk);
  free(tp);
}
