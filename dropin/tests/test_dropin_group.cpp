// test_dropin_group.cpp -- the drop-in's device-group and upload-cache
// behaviour, through the reference's own tq:: API (built by dropin/Makefile
// against the reference headers + libcrystal_b200.so; run by
// tests/test_gpu_dropin.py).
//
//  * run_query(db, id, config, workers) with workers in {1, 2, 8}: every
//    result equals run_reference (ssb_reference.cpp) -- workers maps to a
//    device group (CRYS_GROUP_EMULATE=1 keeps `workers` shards on one GPU);
//  * the host database is uploaded ONCE per (group, database): repeated
//    queries do no H2D (b200::upload_count);
//  * results follow changed data after b200::invalidate, and a reallocated
//    column (new data pointer) re-uploads by itself;
//  * a duplicate dimension key raises BuildError on the sharded path.
#include <cstdlib>

#include "doctest.h"
#include "tq/b200_runtime.hpp"
#include "tq/ssb_gen.hpp"
#include "tq/ssb_queries.hpp"
#include "tq/ssb_reference.hpp"

using namespace tq;

namespace {
const SsbDatabase& sf1() {
  static const SsbDatabase db = generate_ssb(1, 42);
  return db;
}
std::vector<i32>& column(SsbTable& t, const std::string& name) {
  for (Column& c : t.columns)
    if (c.name == name) return c.ints;
  throw std::runtime_error("no column " + name);
}
}  // namespace

TEST_CASE("workers map to a device group: SF=1 suite equals the reference for workers 1, 2, 8") {
  setenv("CRYS_GROUP_EMULATE", "1", 1);
  const SsbDatabase& db = sf1();
  for (int workers : {1, 2, 8}) {
    for (QueryId id : all_query_ids()) {
      QueryStats st;
      CHECK(diff_results(run_query(db, id, {}, workers, &st), run_reference(db, id)) == "");
      CHECK(!st.survivors.empty());
    }
  }
}

TEST_CASE("the host database is uploaded once per group") {
  setenv("CRYS_GROUP_EMULATE", "1", 1);
  const SsbDatabase& db = sf1();
  run_query(db, QueryId::kQ21, {}, 2);
  const long long before = b200::upload_count();
  for (int rep = 0; rep < 3; ++rep)
    for (QueryId id : all_query_ids()) run_query(db, id, {}, 2);
  CHECK(b200::upload_count() == before);
}

TEST_CASE("results follow changed data: invalidate and reallocation") {
  setenv("CRYS_GROUP_EMULATE", "1", 1);
  SsbDatabase db = generate_ssb(1, 7);
  const QueryResult a = run_query(db, QueryId::kQ11, {}, 2);
  CHECK(diff_results(a, run_reference(db, QueryId::kQ11)) == "");
  // in place, same pointers: the fingerprint of a 1 GB-class table is sampled,
  // so the caller says so explicitly
  std::vector<i32>& price = column(db.lineorder, "lo_extendedprice");
  for (size_t i = 0; i < price.size(); i += 3) price[i] = price[i] / 2 + 1;
  b200::invalidate(&db);
  const long long n0 = b200::upload_count();
  const QueryResult b = run_query(db, QueryId::kQ11, {}, 2);
  CHECK(b200::upload_count() == n0 + 1);
  CHECK(diff_results(b, run_reference(db, QueryId::kQ11)) == "");
  CHECK(diff_results(b, a) != "");
  // a reallocated column changes the signature: re-upload without invalidate
  std::vector<i32> fresh(price.size(), 7);
  price.swap(fresh);
  const QueryResult c = run_query(db, QueryId::kQ11, {}, 2);
  CHECK(b200::upload_count() == n0 + 2);
  CHECK(diff_results(c, run_reference(db, QueryId::kQ11)) == "");
  b200::invalidate(&db);
}

TEST_CASE("a duplicate dimension key raises BuildError on the sharded path") {
  setenv("CRYS_GROUP_EMULATE", "1", 1);
  SsbDatabase db = generate_ssb(1, 42);
  std::vector<i32>& key = column(db.supplier, "s_suppkey");
  key[10] = key[11];
  for (int workers : {1, 4}) CHECK_THROWS_AS(run_query(db, QueryId::kQ21, {}, workers), BuildError);
  b200::invalidate(&db);
}
