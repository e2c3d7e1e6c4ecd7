// TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the reference's own C++ hot path, compiled together
// with the reference translation units from /root/reference/proj/src (see
// oracle/Makefile; the namespace is renamed tq -> tq_ref at compile time).
// Used by tests/golden/make_golden.py to pin golden vectors, by the parity
// tests as a second checker, and by bench.py's `--impl reference` arm as the
// reference's CPU implementation timed on the host cores.  Never linked into
// or called by the product library.
//
// Entry points wrap, one to one:
//   generate_ssb                    ssb_gen.cpp:243-270
//   run_reference                   ssb_reference.cpp:138-261
//   run_query (+QueryStats)         ssb_queries.cpp:277-286
//   select_*_into                   select.hpp:56-135
//   project_{linear,sigmoid}_into   project.hpp:49-64
//   HashTable::build / probe        hash_table.cpp:20-94, hash_table.hpp:41-51
//   join_probe_{scalar,prefetch,tile} join.cpp:53-96
//   lsb/msb_radix_sort              radix.cpp:138-216
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tq/common.hpp"
#include "tq/hash_table.hpp"
#include "tq/join.hpp"
#include "tq/project.hpp"
#include "tq/radix.hpp"
#include "tq/select.hpp"
#include "tq/ssb_gen.hpp"
#include "tq/ssb_plans.hpp"
#include "tq/ssb_queries.hpp"
#include "tq/ssb_reference.hpp"

using namespace tq_ref;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 2;
  } catch (const BuildError& e) {
    g_err = e.what();
    return 3;
  } catch (const IoError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

SsbTable* table_of(SsbDatabase* db, const std::string& name) {
  for (SsbTable* t : {&db->lineorder, &db->date, &db->supplier, &db->customer, &db->part})
    if (t->name == name) return t;
  throw ContractError("no table named " + name);
}

PredicateSpec<i32> make_pred(int op, i32 lo, i32 hi) {
  switch (op) {
    case 0: return PredicateSpec<i32>::lt(lo);
    case 1: return PredicateSpec<i32>::le(lo);
    case 2: return PredicateSpec<i32>::gt(lo);
    case 3: return PredicateSpec<i32>::ge(lo);
    case 4: return PredicateSpec<i32>::eq(lo);
    case 5: return PredicateSpec<i32>::between(lo, hi);
  }
  throw ConfigError("unknown predicate op");
}
}  // namespace

extern "C" {

const char* tqref_last_error() { return g_err.c_str(); }

void* tqref_generate(int64_t sf, uint64_t seed) {
  SsbDatabase* db = nullptr;
  if (guarded([&] { db = new SsbDatabase(generate_ssb(sf, seed)); }) != 0) return nullptr;
  return db;
}

// An empty database carrying the canonical dictionaries (the fixture in
// test_ssb.cpp:17-81 is assembled this way, column by column).
void* tqref_db_empty() {
  auto* db = new SsbDatabase();
  db->scale_factor = 1;
  db->lineorder.name = "lineorder";
  db->date.name = "date";
  db->supplier.name = "supplier";
  db->customer.name = "customer";
  db->part.name = "part";
  db->dictionaries = {ssb_region_dict("s_region"), ssb_nation_dict("s_nation"),
                      ssb_city_dict("s_city"),     ssb_region_dict("c_region"),
                      ssb_nation_dict("c_nation"), ssb_city_dict("c_city"),
                      ssb_mfgr_dict(),             ssb_category_dict(),
                      ssb_brand_dict(),            ssb_yearmonth_dict()};
  return db;
}

int tqref_db_set_column(void* h, const char* table, const char* column,
                        const int32_t* data, int64_t rows) {
  return guarded([&] {
    SsbTable* t = table_of(static_cast<SsbDatabase*>(h), table);
    std::vector<i32> v(data, data + rows);
    for (Column& c : t->columns)
      if (c.name == column) {
        c = Column::int32(column, std::move(v));
        return;
      }
    t->columns.push_back(Column::int32(column, std::move(v)));
  });
}

void tqref_db_free(void* h) { delete static_cast<SsbDatabase*>(h); }

int tqref_db_column(void* h, const char* table, const char* column, const int32_t** ptr,
                    int64_t* rows) {
  return guarded([&] {
    const SsbTable* t = table_of(static_cast<SsbDatabase*>(h), table);
    auto s = t->ints(column);
    *ptr = s.data();
    *rows = static_cast<int64_t>(s.size());
  });
}

// qid: 0..12 in all_query_ids() order.  use_reference != 0 runs the row-at-a-
// time interpreter, otherwise the tile pipeline with the given config/workers.
// groups: max_rows*3 int32 (row-major, ngroup used per row); sums: max_rows.
int tqref_query(void* h, int qid, int use_reference, int bt, int ipt, int workers,
                int32_t* groups, int64_t* sums, int64_t max_rows, int64_t* nrows,
                int32_t* ngroup, int64_t* survivors, int32_t* nsurv, double* ms) {
  return guarded([&] {
    const SsbDatabase& db = *static_cast<SsbDatabase*>(h);
    auto ids = all_query_ids();
    TQ_CONFIG_CHECK(qid >= 0 && qid < static_cast<int>(ids.size()), "bad qid");
    QueryStats stats;
    auto t0 = std::chrono::steady_clock::now();
    QueryResult r = use_reference ? run_reference(db, ids[qid])
                                  : run_query(db, ids[qid], TileConfig{bt, ipt}, workers, &stats);
    if (ms) *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *nrows = static_cast<int64_t>(r.rows.size());
    *ngroup = static_cast<int32_t>(r.group_labels.size());
    if (nsurv) {
      *nsurv = static_cast<int32_t>(stats.survivors.size());
      for (size_t j = 0; j < stats.survivors.size() && j < 4; ++j) survivors[j] = stats.survivors[j];
    }
    TQ_CHECK(*nrows <= max_rows, "result larger than caller buffer");
    for (size_t i = 0; i < r.rows.size(); ++i) {
      for (size_t g = 0; g < r.rows[i].group.size(); ++g) groups[i * 3 + g] = r.rows[i].group[g];
      sums[i] = r.rows[i].sum;
    }
  });
}

// variant: 0 branching, 1 predicated, 2 per-element, 3 tile (mode 0 det, 1 arrival)
int64_t tqref_select(int variant, const int32_t* in, int64_t n, int op, int32_t lo, int32_t hi,
                     int32_t* out, int bt, int ipt, int mode, int workers) {
  int64_t count = -1;
  int st = guarded([&] {
    std::span<const i32> s_in(in, static_cast<size_t>(n));
    std::span<i32> s_out(out, static_cast<size_t>(n));
    auto pred = make_pred(op, lo, hi);
    switch (variant) {
      case 0: count = select_branching_into(s_in, pred, s_out, workers); break;
      case 1: count = select_predicated_into(s_in, pred, s_out, workers); break;
      case 2: count = select_per_element_into(s_in, pred, s_out, workers); break;
      case 3:
        count = select_tile_into(s_in, pred, s_out, TileConfig{bt, ipt},
                                 mode ? ScheduleMode::kArrivalOrder : ScheduleMode::kDeterministic,
                                 workers);
        break;
      default: throw ConfigError("unknown select variant");
    }
  });
  return st == 0 ? count : -st;
}

int tqref_project(int sigmoid, const float* x1, const float* x2, int64_t n, float a, float b,
                  float* out, int bt, int ipt, int workers) {
  return guarded([&] {
    std::span<const float> s1(x1, static_cast<size_t>(n)), s2(x2, static_cast<size_t>(n));
    std::span<float> so(out, static_cast<size_t>(n));
    if (sigmoid)
      project_sigmoid_into(s1, s2, a, b, so, TileConfig{bt, ipt}, workers);
    else
      project_linear_into(s1, s2, a, b, so, TileConfig{bt, ipt}, workers);
  });
}

void* tqref_ht_build(const int32_t* keys, const int32_t* payloads, int64_t n, int64_t cap,
                     int workers, int* status) {
  HashTable* ht = nullptr;
  *status = guarded([&] {
    ht = new HashTable(HashTable::build(std::span<const i32>(keys, static_cast<size_t>(n)),
                                        std::span<const i32>(payloads, static_cast<size_t>(n)),
                                        cap, workers));
  });
  return ht;
}

void tqref_ht_slots(void* h, const int32_t** keys, const int32_t** payloads, int64_t* cap) {
  auto* ht = static_cast<HashTable*>(h);
  *keys = ht->slot_keys();
  *payloads = ht->slot_payloads();
  *cap = ht->capacity();
}

void tqref_ht_free(void* h) { delete static_cast<HashTable*>(h); }

// variant: 0 scalar, 1 prefetch, 2 tile.  Returns the Q4 checksum.
int tqref_join_probe(int variant, const int32_t* pk, const int32_t* pp, int64_t n, void* h,
                     int bt, int ipt, int workers, int64_t* checksum) {
  return guarded([&] {
    const HashTable& ht = *static_cast<HashTable*>(h);
    std::span<const i32> k(pk, static_cast<size_t>(n)), p(pp, static_cast<size_t>(n));
    if (variant == 0)
      *checksum = join_probe_scalar(k, p, ht, workers);
    else if (variant == 1)
      *checksum = join_probe_prefetch(k, p, ht, workers);
    else
      *checksum = join_probe_tile(k, p, ht, TileConfig{bt, ipt}, workers);
  });
}

int tqref_sort(int msb, int32_t* keys, int32_t* payloads, int64_t n, int workers, int bits) {
  return guarded([&] {
    std::span<i32> k(keys, static_cast<size_t>(n)), p(payloads, static_cast<size_t>(n));
    if (msb)
      msb_radix_sort(k, p, workers);
    else
      lsb_radix_sort(k, p, workers, bits);
  });
}

}  // extern "C"
