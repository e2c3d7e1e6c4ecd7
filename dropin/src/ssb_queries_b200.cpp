// ssb_queries_b200.cpp -- B200 drop-in for P:src/ssb_queries.cpp.
//
// Defines everything P:include/tq/ssb_queries.hpp declares.  run_query maps
// `workers` to a device group (b200::group_context: lineorder row-range
// shards, one per GPU, one NCCL reduce per query), uploads the host database
// ONCE into that group's HBM (b200::cached_database, keyed by identity +
// content fingerprint) and runs crys_run_query: dimension builds, ONE fused
// lineorder pass per shard and the group compaction on the GPUs; the
// AggregateTable / sort_result / diff_results helpers are host utilities with
// the reference's semantics (ssb_queries.cpp:15-88).
#include <algorithm>
#include <sstream>
#include <vector>

#include "tq/b200_runtime.hpp"
#include "tq/ssb_queries.hpp"

namespace tq {

// ------------------------------------------------------- aggregate table

AggregateTable::AggregateTable(std::vector<GroupPart> parts) : parts_(std::move(parts)) {
  strides_.assign(parts_.size(), 1);
  i64 cells = 1;
  for (size_t j = parts_.size(); j-- > 0;) {  // mixed radix, last part fastest
    TQ_CHECK(parts_[j].hi >= parts_[j].lo, "group part with empty domain");
    strides_[j] = cells;
    cells *= parts_[j].cardinality();
  }
  sums_.assign(static_cast<size_t>(cells), 0);
  used_.assign(static_cast<size_t>(cells), 0);
}

i64 AggregateTable::index_of(const i32* values) const {
  i64 idx = 0;
  for (size_t j = 0; j < parts_.size(); ++j) {
    TQ_CHECK(values[j] >= parts_[j].lo && values[j] <= parts_[j].hi,
             "group value outside its declared domain: " + parts_[j].label);
    idx += static_cast<i64>(values[j] - parts_[j].lo) * strides_[j];
  }
  return idx;
}

void AggregateTable::merge(const AggregateTable& other) {
  TQ_CHECK(cells() == other.cells(), "merging aggregate tables of different shape");
  for (i64 i = 0; i < cells(); ++i) {
    const size_t k = static_cast<size_t>(i);
    if (!other.used_[k]) continue;
    sums_[k] += other.sums_[k];
    used_[k] = 1;
  }
}

std::vector<i32> AggregateTable::key_of(i64 index) const {
  std::vector<i32> v(parts_.size());
  for (size_t j = 0; j < parts_.size(); ++j) {
    v[j] = parts_[j].lo + static_cast<i32>(index / strides_[j]);
    index %= strides_[j];
  }
  return v;
}

// --------------------------------------------------------------- results

void sort_result(QueryResult& result) {
  std::sort(result.rows.begin(), result.rows.end(),
            [](const ResultRow& a, const ResultRow& b) { return a.group < b.group; });
}

std::string diff_results(const QueryResult& got, const QueryResult& expected) {
  std::ostringstream out;
  if (got.rows.size() != expected.rows.size())
    out << "row count " << got.rows.size() << " vs " << expected.rows.size() << "; ";
  auto group = [&out](const ResultRow& r) {
    out << "(";
    for (size_t j = 0; j < r.group.size(); ++j) out << (j ? "," : "") << r.group[j];
    out << ")=" << r.sum;
  };
  int reported = 0;
  const size_t n = std::min(got.rows.size(), expected.rows.size());
  for (size_t i = 0; i < n && reported < 5; ++i) {
    const ResultRow& g = got.rows[i];
    const ResultRow& e = expected.rows[i];
    if (g.group == e.group && g.sum == e.sum) continue;
    ++reported;
    out << "row " << i << ": ";
    group(g);
    out << " vs ";
    group(e);
    out << "; ";
  }
  return out.str();
}

// -------------------------------------------------------------- executor

QueryResult run_query(const SsbDatabase& db, QueryId id, const TileConfig& config, int workers,
                      QueryStats* stats) {
  config.validate();
  TQ_CONFIG_CHECK(workers >= 1, "run_query: workers must be >= 1");
  const QueryPlan& plan = plan_for(id);  // ConfigError for an unknown id

  // every int32 column of every table, by (table, column) name
  std::vector<crys_host_column> cols;
  for (const SsbTable* t : {&db.lineorder, &db.date, &db.supplier, &db.customer, &db.part}) {
    for (const Column& c : t->columns) {
      if (c.kind != ElemKind::kInt32) continue;
      cols.push_back({t->name.c_str(), c.name.c_str(), c.ints.data(), c.length()});
    }
  }
  TQ_CHECK(!cols.empty(), "run_query: empty database");

  // `workers` -> a device group of lineorder shards (one NCCL reduce per
  // query); the host database is uploaded once and cached by identity
  crys_ctx* group = b200::group_context(workers);
  crys_db* hbm = b200::cached_database(group, &db, cols);

  int64_t cells = 0;
  int32_t ngroup = 0, njoins = 0;
  b200::check(crys_query_shape(static_cast<int>(id), &cells, &ngroup, &njoins));
  const int64_t max_rows = std::max<int64_t>(cells, 1);
  thread_local std::vector<int32_t> groups;
  thread_local std::vector<int64_t> sums;
  if ((int64_t)sums.size() < max_rows) {
    groups.resize(static_cast<size_t>(3 * max_rows));
    sums.resize(static_cast<size_t>(max_rows));
  }
  int64_t survivors[4] = {0, 0, 0, 0};
  int64_t nrows = 0;
  b200::check(crys_run_query(group, hbm, static_cast<int>(id), config.block_threads, config.items_per_thread,
                             groups.data(), sums.data(), max_rows, &nrows, survivors));

  QueryResult result;
  for (const GroupPart& g : plan.group) result.group_labels.push_back(g.label);
  result.rows.resize(static_cast<size_t>(nrows));
  for (int64_t i = 0; i < nrows; ++i) {
    ResultRow& r = result.rows[static_cast<size_t>(i)];
    r.group.assign(groups.begin() + 3 * i, groups.begin() + 3 * i + ngroup);
    r.sum = sums[static_cast<size_t>(i)];
  }
  if (stats) {
    stats->survivors.clear();
    for (int j = 0; j < std::max<int32_t>(njoins, 1); ++j) stats->survivors.push_back(survivors[j]);
  }
  return result;
}

}  // namespace tq
