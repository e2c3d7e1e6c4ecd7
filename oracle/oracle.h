/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this (through oracle/oracle.py).  The product library never links,
 * calls or falls back to it.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function here against
 * the golden vectors in tests/golden/ (produced by the reference itself,
 * compiled from /root/reference/proj by oracle/Makefile, see
 * tests/golden/make_golden.py) and against the reference's own hand-checked
 * fixtures (test_ssb.cpp:17-227, test_tile_engine.cpp:18-79,
 * test_radix.cpp:112-142).
 */
#ifndef CRYSTAL_ORACLE_H
#define CRYSTAL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:16-45 ---- */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_rng_base(uint64_t seed, uint64_t a, uint64_t b, uint64_t c);
int32_t orc_uniform_i32(uint64_t base, uint64_t index, int32_t lo, int32_t hi);
float orc_uniform_float(uint64_t base, uint64_t index, float lo, float hi);
/* tq_main.cpp:147-152: Rng(seed, stream).uniform_i32(i, lo, hi) for i < n */
void orc_random_i32(int32_t* out, int64_t n, uint64_t seed, uint64_t stream, int32_t lo,
                    int32_t hi);
/* tq_main.cpp:335-340: x1 = Rng(seed,2).uniform_float(2i,-4,4), x2 at 2i+1 */
void orc_project_inputs(float* x1, float* x2, int64_t n, uint64_t seed);

/* ---- ssb_gen.cpp ---- */
int64_t orc_lineorder_rows(int64_t sf);
int64_t orc_supplier_rows(int64_t sf);
int64_t orc_customer_rows(int64_t sf);
int64_t orc_part_rows(int64_t sf);
/* date table, 2556 rows: datekey, year, yearmonthnum, yearmonth, weeknum */
void orc_gen_date(int32_t* cols5);
/* geography table (table_id 3 supplier, 4 customer): key, city, nation, region */
void orc_gen_geo(int table_id, int64_t sf, uint64_t seed, int64_t rows, int32_t* cols4);
/* part table: key, brand1, category, mfgr */
void orc_gen_part(int64_t sf, uint64_t seed, int64_t rows, int32_t* cols4);
/* one lineorder column (column_id 0..8) for rows [begin, end) */
void orc_gen_lineorder_col(int64_t sf, uint64_t seed, int column_id, int64_t begin, int64_t end,
                           int32_t* out, int nthreads);

/* ---- SSB query semantics (ssb_reference.cpp + plan order ssb_plans.cpp) ---- */
typedef struct {
  int64_t lo_rows, date_rows, supp_rows, cust_rows, part_rows;
  const int32_t* lo[9];   /* orderdate custkey suppkey partkey quantity discount extprice revenue supplycost */
  const int32_t* date[5]; /* datekey year yearmonthnum yearmonth weeknum */
  const int32_t* supp[4]; /* suppkey city nation region */
  const int32_t* cust[4]; /* custkey city nation region */
  const int32_t* part[4]; /* partkey brand1 category mfgr */
} orc_db;

/* Number of dense aggregate cells of query qid (0..12). */
int64_t orc_query_cells(int qid);
/* Group arity of qid (0 for flight 1). */
int orc_query_ngroup(int qid);
/* Dense partial aggregation over lineorder rows [begin, end): sums[cells],
 * counts[cells] are ACCUMULATED into; survivors[4] accumulated per join stage
 * in plan order.  Returns 0, or -1 when a group value leaves its domain. */
int orc_query_partial(const orc_db* db, int qid, int64_t begin, int64_t end, int64_t* sums,
                      int64_t* counts, int64_t* survivors);
/* Full query: rows in lexicographic order.  groups: max_rows*3, sums: max_rows.
 * Returns nrows (or <0 on error). */
int64_t orc_query(const orc_db* db, int qid, int32_t* groups, int64_t* sums, int64_t max_rows,
                  int64_t* survivors);
/* Decode a dense cell index into group values (AggregateTable::key_of). */
void orc_cell_key(int qid, int64_t cell, int32_t* values);

/* ---- hash table (hash_table.hpp:21-63, hash_table.cpp:20-48) ---- */
/* returns 0 ok, 1 config (capacity), 3 build (dup / sentinel / overflow) */
int orc_ht_build(const int32_t* keys, const int32_t* payloads, int64_t n, int64_t capacity,
                 int32_t* slot_keys, int32_t* slot_payloads);
int orc_ht_probe(const int32_t* slot_keys, const int32_t* slot_payloads, int64_t capacity,
                 int32_t key, int32_t* payload);
/* join.cpp:11-18: sum over hits of (build payload + probe payload) */
int64_t orc_join_checksum(const int32_t* pk, const int32_t* pp, int64_t n,
                          const int32_t* slot_keys, const int32_t* slot_payloads,
                          int64_t capacity);

/* ---- select (select.hpp), op: 0 LT 1 LE 2 GT 3 GE 4 EQ 5 BETWEEN ---- */
int64_t orc_select_input_order(const int32_t* in, int64_t n, int op, int32_t lo, int32_t hi,
                               int32_t* out);
int64_t orc_select_crystal_order(const int32_t* in, int64_t n, int op, int32_t lo, int32_t hi,
                                 int bt, int ipt, int32_t* out);

/* ---- project (project.hpp:49-64) ---- */
void orc_project_linear(const float* x1, const float* x2, int64_t n, float a, float b,
                        float* out);
void orc_project_sigmoid(const float* x1, const float* x2, int64_t n, float a, float b,
                         float* out);

/* ---- radix (radix.hpp:44-47, radix.cpp:138-163) ---- */
uint32_t orc_radix_digit(int32_t key, int start_bit, int num_bits);
void orc_lsb_sort(int32_t* keys, int32_t* payloads, int64_t n, int bits_per_pass);

#ifdef __cplusplus
}
#endif
#endif
