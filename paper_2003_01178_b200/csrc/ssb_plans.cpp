// ssb_plans.cpp -- the 13 SSB query plans and the canonical dictionaries.
//
// Plans restate ssb_plans.cpp:21-275 of the reference (same probe order, the
// same filters/payloads/group parts and aggregate).  Filter literals are
// resolved through the same fixed dictionaries the generator defines
// (ssb_gen.cpp:13-52, :188-241), so a plan reads like the reference's.
#include <climits>
#include <map>

#include "internal.hpp"

namespace crys {
namespace {

const char* const kRegions[5] = {"AFRICA", "AMERICA", "ASIA", "EUROPE", "MIDDLE EAST"};
const char* const kNations[25] = {
    "ALGERIA",   "ETHIOPIA", "KENYA",   "MOROCCO",   "MOZAMBIQUE", "ARGENTINA", "BRAZIL",
    "CANADA",    "PERU",     "UNITED STATES", "CHINA", "INDIA",    "INDONESIA", "JAPAN",
    "VIETNAM",   "FRANCE",   "GERMANY", "ROMANIA",   "RUSSIA",     "UNITED KINGDOM",
    "EGYPT",     "IRAN",     "IRAQ",    "JORDAN",    "SAUDI ARABIA"};
const char* const kMonths[12] = {"Jan", "Feb", "Mar", "Apr", "May", "Jun",
                                 "Jul", "Aug", "Sep", "Oct", "Nov", "Dec"};

std::vector<std::string> dict_entries(const std::string& d) {
  std::vector<std::string> e;
  if (d == "s_region" || d == "c_region") {
    e.assign(kRegions, kRegions + 5);
  } else if (d == "s_nation" || d == "c_nation") {
    e.assign(kNations, kNations + 25);
  } else if (d == "s_city" || d == "c_city") {  // ssb_gen.cpp:40-45
    for (int c = 0; c < 250; ++c) {
      std::string base = kNations[c / 10];
      base.resize(9, ' ');
      base.push_back(char('0' + c % 10));
      e.push_back(base);
    }
  } else if (d == "p_mfgr") {
    for (int m = 1; m <= 5; ++m) e.push_back("MFGR#" + std::to_string(m));
  } else if (d == "p_category") {
    for (int m = 1; m <= 5; ++m)
      for (int c = 1; c <= 5; ++c) e.push_back("MFGR#" + std::to_string(m) + std::to_string(c));
  } else if (d == "p_brand1") {
    for (auto& c : dict_entries("p_category"))
      for (int b = 1; b <= 40; ++b) e.push_back(c + std::to_string(b));
  } else if (d == "d_yearmonth") {
    for (int y = 1992; y <= 1998; ++y)
      for (int m = 0; m < 12; ++m) e.push_back(std::string(kMonths[m]) + std::to_string(y));
  } else {
    fail(CRYS_ECONTRACT, "no dictionary named " + d);
  }
  return e;
}

DimJoin supplier_join(std::vector<RangeFilter> f, std::string payload = "") {
  return {kSupplier, "supplier", "s_suppkey", "lo_suppkey", std::move(f), std::move(payload)};
}
DimJoin customer_join(std::vector<RangeFilter> f, std::string payload = "") {
  return {kCustomer, "customer", "c_custkey", "lo_custkey", std::move(f), std::move(payload)};
}
DimJoin part_join(std::vector<RangeFilter> f, std::string payload = "") {
  return {kPart, "part", "p_partkey", "lo_partkey", std::move(f), std::move(payload)};
}
DimJoin date_join(std::vector<RangeFilter> f, std::string payload = "") {
  return {kDate, "date", "d_datekey", "lo_orderdate", std::move(f), std::move(payload)};
}
GroupPart year_part(int j) { return {j, 1992, 1998, "d_year"}; }
RangeFilter eq_filter(const std::string& col, int32_t v) { return {col, {{v, v}}}; }

QueryPlan flight1(int qid, const char* name, int32_t d0, int32_t d1, int32_t disc0, int32_t disc1,
                  int32_t q0, int32_t q1) {
  QueryPlan p;
  p.qid = qid;
  p.name = name;
  p.fact_filters = {{"lo_orderdate", d0, d1}, {"lo_discount", disc0, disc1},
                    {"lo_quantity", q0, q1}};
  p.agg = kAggExtPriceTimesDiscount;
  return p;
}

QueryPlan q2x(int qid, const char* name, RangeFilter part_filter, const char* region) {
  QueryPlan p;
  p.qid = qid;
  p.name = name;
  p.joins = {supplier_join({eq_filter("s_region", dict_code("s_region", region))}),
             part_join({std::move(part_filter)}, "p_brand1"), date_join({}, "d_year")};
  p.group = {year_part(2), {1, 0, 999, "p_brand1"}};
  p.agg = kAggRevenue;
  return p;
}

QueryPlan q3x(int qid, const char* name, RangeFilter c_filter, RangeFilter s_filter,
              const char* c_group, const char* s_group, int32_t geo_hi, RangeFilter d_filter) {
  QueryPlan p;
  p.qid = qid;
  p.name = name;
  p.joins = {supplier_join({std::move(s_filter)}, s_group),
             customer_join({std::move(c_filter)}, c_group), date_join({std::move(d_filter)}, "d_year")};
  p.group = {{1, 0, geo_hi, c_group}, {0, 0, geo_hi, s_group}, year_part(2)};
  p.agg = kAggRevenue;
  return p;
}

std::vector<QueryPlan> make_plans() {
  std::vector<QueryPlan> v;
  // flight 1 (ssb_plans.cpp:21-68); PredicateSpec::lt(25) lowered to [INT_MIN, 24]
  v.push_back(flight1(0, "q11", 19930101, 19940101, 1, 3, INT32_MIN, 24));
  v.push_back(flight1(1, "q12", 19940101, 19940131, 4, 6, 26, 35));
  v.push_back(flight1(2, "q13", 19940205, 19940211, 5, 7, 26, 35));
  // flight 2 (ssb_plans.cpp:110-144)
  const int32_t cat12 = dict_code("p_category", "MFGR#12");
  v.push_back(q2x(3, "q21", eq_filter("p_category", cat12), "AMERICA"));
  v.push_back(q2x(4, "q22",
                  {"p_brand1", {{dict_code("p_brand1", "MFGR#2221"), dict_code("p_brand1", "MFGR#2228")}}},
                  "ASIA"));
  v.push_back(q2x(5, "q23", eq_filter("p_brand1", dict_code("p_brand1", "MFGR#2239")), "EUROPE"));
  // flight 3 (ssb_plans.cpp:148-210)
  const int32_t asia_c = dict_code("c_region", "ASIA"), asia_s = dict_code("s_region", "ASIA");
  v.push_back(q3x(6, "q31", eq_filter("c_region", asia_c), eq_filter("s_region", asia_s), "c_nation",
                  "s_nation", 24, {"d_year", {{1992, 1997}}}));
  const int32_t us_c = dict_code("c_nation", "UNITED STATES"), us_s = dict_code("s_nation", "UNITED STATES");
  v.push_back(q3x(7, "q32", eq_filter("c_nation", us_c), eq_filter("s_nation", us_s), "c_city", "s_city",
                  249, {"d_year", {{1992, 1997}}}));
  const int32_t ki1 = dict_code("c_city", "UNITED KI1"), ki5 = dict_code("c_city", "UNITED KI5");
  RangeFilter c_cities{"c_city", {{ki1, ki1}, {ki5, ki5}}};
  RangeFilter s_cities{"s_city", {{ki1, ki1}, {ki5, ki5}}};
  v.push_back(q3x(8, "q33", c_cities, s_cities, "c_city", "s_city", 249, {"d_year", {{1992, 1997}}}));
  const int32_t dec97 = dict_code("d_yearmonth", "Dec1997");
  v.push_back(q3x(9, "q34", c_cities, s_cities, "c_city", "s_city", 249, eq_filter("d_yearmonth", dec97)));
  // flight 4 (ssb_plans.cpp:215-275)
  const int32_t america_s = dict_code("s_region", "AMERICA"), america_c = dict_code("c_region", "AMERICA");
  const int32_t m1 = dict_code("p_mfgr", "MFGR#1"), m2 = dict_code("p_mfgr", "MFGR#2");
  {
    QueryPlan p;
    p.qid = 10;
    p.name = "q41";
    p.joins = {supplier_join({eq_filter("s_region", america_s)}),
               customer_join({eq_filter("c_region", america_c)}, "c_nation"),
               part_join({{"p_mfgr", {{m1, m2}}}}), date_join({}, "d_year")};
    p.group = {year_part(3), {1, 0, 24, "c_nation"}};
    p.agg = kAggRevenueMinusSupplyCost;
    v.push_back(p);
  }
  {
    QueryPlan p;
    p.qid = 11;
    p.name = "q42";
    p.joins = {supplier_join({eq_filter("s_region", america_s)}, "s_nation"),
               customer_join({eq_filter("c_region", america_c)}),
               part_join({{"p_mfgr", {{m1, m2}}}}, "p_category"),
               date_join({{"d_year", {{1997, 1998}}}}, "d_year")};
    p.group = {year_part(3), {0, 0, 24, "s_nation"}, {2, 0, 24, "p_category"}};
    p.agg = kAggRevenueMinusSupplyCost;
    v.push_back(p);
  }
  {
    QueryPlan p;
    p.qid = 12;
    p.name = "q43";
    p.joins = {supplier_join({eq_filter("s_nation", us_s)}, "s_city"),
               part_join({eq_filter("p_category", dict_code("p_category", "MFGR#14"))}, "p_brand1"),
               customer_join({eq_filter("c_region", america_c)}),
               date_join({{"d_year", {{1997, 1998}}}}, "d_year")};
    p.group = {year_part(3), {0, 0, 249, "s_city"}, {1, 0, 999, "p_brand1"}};
    p.agg = kAggRevenueMinusSupplyCost;
    v.push_back(p);
  }
  return v;
}

}  // namespace

int dict_code(const std::string& dict, const std::string& value) {
  auto e = dict_entries(dict);
  for (size_t i = 0; i < e.size(); ++i)
    if (e[i] == value) return (int)i;
  fail(CRYS_ECONTRACT, "dictionary " + dict + ": no entry '" + value + "'");
}

const QueryPlan& plan_for(int qid) {
  static const std::vector<QueryPlan> plans = make_plans();
  CRYS_CHECK(qid >= 0 && qid < (int)plans.size(), CRYS_ECONFIG,
             "unknown query id " + std::to_string(qid));
  return plans[qid];
}

void lower_pred(const crys_pred& p, int32_t* lo, int32_t* hi) {
  switch (p.op) {
    case CRYS_LT:
      if (p.lo == INT32_MIN) { *lo = 1; *hi = 0; } else { *lo = INT32_MIN; *hi = p.lo - 1; }
      return;
    case CRYS_LE: *lo = INT32_MIN; *hi = p.lo; return;
    case CRYS_GT:
      if (p.lo == INT32_MAX) { *lo = 1; *hi = 0; } else { *lo = p.lo + 1; *hi = INT32_MAX; }
      return;
    case CRYS_GE: *lo = p.lo; *hi = INT32_MAX; return;
    case CRYS_EQ: *lo = p.lo; *hi = p.lo; return;
    case CRYS_BETWEEN:
      // PredicateSpec::between requires lo <= hi (tile.hpp:112-114)
      CRYS_CHECK(!(p.hi < p.lo), CRYS_ECONFIG, "PredicateSpec: BETWEEN requires lo <= hi");
      *lo = p.lo; *hi = p.hi;
      return;
  }
  fail(CRYS_ECONFIG, "unknown predicate op");
}

}  // namespace crys

namespace crys {

// The plan as JSON (introspection for tools / tests; the same contract the
// fused kernels implement).
std::string plan_json(int qid) {
  const QueryPlan& p = plan_for(qid);
  std::string s = "{\"qid\":" + std::to_string(p.qid) + ",\"name\":\"" + p.name + "\",\"fact_filters\":[";
  for (size_t i = 0; i < p.fact_filters.size(); ++i)
    s += std::string(i ? "," : "") + "{\"column\":\"" + p.fact_filters[i].column + "\",\"lo\":" +
         std::to_string(p.fact_filters[i].lo) + ",\"hi\":" + std::to_string(p.fact_filters[i].hi) + "}";
  s += "],\"joins\":[";
  for (size_t j = 0; j < p.joins.size(); ++j) {
    const DimJoin& d = p.joins[j];
    s += std::string(j ? "," : "") + "{\"dim_table\":\"" + d.dim_table + "\",\"dim_key\":\"" + d.dim_key +
         "\",\"fact_key\":\"" + d.fact_key + "\",\"payload\":\"" + d.payload + "\",\"filters\":[";
    for (size_t f = 0; f < d.filters.size(); ++f) {
      s += std::string(f ? "," : "") + "{\"column\":\"" + d.filters[f].column + "\",\"ranges\":[";
      for (size_t r = 0; r < d.filters[f].ranges.size(); ++r)
        s += std::string(r ? "," : "") + "[" + std::to_string(d.filters[f].ranges[r].first) + "," +
             std::to_string(d.filters[f].ranges[r].second) + "]";
      s += "]}";
    }
    s += "]}";
  }
  s += "],\"group\":[";
  for (size_t g = 0; g < p.group.size(); ++g)
    s += std::string(g ? "," : "") + "{\"join\":" + std::to_string(p.group[g].join_index) + ",\"lo\":" +
         std::to_string(p.group[g].lo) + ",\"hi\":" + std::to_string(p.group[g].hi) + ",\"label\":\"" +
         p.group[g].label + "\"}";
  static const char* kAgg[3] = {"revenue", "extendedprice*discount", "revenue-supplycost"};
  s += std::string("],\"agg\":\"") + kAgg[p.agg] + "\"}";
  return s;
}

}  // namespace crys
