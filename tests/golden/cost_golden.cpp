// TEST INFRASTRUCTURE: prints the reference's own cost models
// (/root/reference/proj/src/cost_models.cpp, compiled in place by
// make_cost_golden.sh) for a fixed set of inputs as JSON; the output is
// committed as tests/golden/cost_models.json and pins
// paper_2003_01178_b200/cost_models.py.
#include <cstdio>
#include <string>
#include <vector>

#include "tq/cost_models.hpp"

using namespace tq;

static void emit(const char* name, const std::string& args, const CostEstimate& e, bool& first) {
  std::printf("%s  {\"model\": \"%s\", \"args\": %s, \"total_seconds\": %.17g, \"terms\": [", first ? "" : ",\n",
              name, args.c_str(), e.total_seconds);
  for (size_t i = 0; i < e.terms.size(); ++i)
    std::printf("%s[\"%s\", %.17g]", i ? ", " : "", e.terms[i].label.c_str(), e.terms[i].seconds);
  std::printf("]}");
  first = false;
}

int main() {
  HardwareProfile b200;
  b200.label = "b200";
  b200.read_bw = 6539.9e9;
  b200.write_bw = 6539.9e9;
  b200.cache_line_bytes = 32;
  b200.cache_levels = {{126e6, 12e12}};
  std::vector<std::pair<std::string, HardwareProfile>> profiles = {
      {"table2-cpu", HardwareProfile::table2_cpu()}, {"table2-gpu", HardwareProfile::table2_gpu()}, {"b200", b200}};
  bool first = true;
  std::printf("[\n");
  for (auto& [pn, p] : profiles) {
    char a[256];
    for (long long n : {0LL, 1000LL, 1LL << 29}) {
      std::snprintf(a, sizeof a, "{\"profile\": \"%s\", \"n\": %lld}", pn.c_str(), n);
      emit("project", a, model_project(n, p), first);
      for (double s : {0.0, 0.1, 0.5, 1.0}) {
        std::snprintf(a, sizeof a, "{\"profile\": \"%s\", \"n\": %lld, \"sigma\": %g}", pn.c_str(), n, s);
        emit("select", a, model_select(n, s, p), first);
      }
      for (int k : {1, 4}) {
        std::snprintf(a, sizeof a, "{\"profile\": \"%s\", \"n\": %lld, \"passes\": %d}", pn.c_str(), n, k);
        emit("sort", a, model_sort(n, k, p), first);
      }
    }
    for (double h = 8192; h <= 1073741824.0; h *= 2) {
      std::snprintf(a, sizeof a, "{\"profile\": \"%s\", \"p\": %lld, \"ht_bytes\": %.17g}", pn.c_str(), 1LL << 28, h);
      emit("join_probe", a, model_join_probe(1LL << 28, h, p), first);
    }
    for (int t = 0; t < 2; ++t) {
      std::snprintf(a, sizeof a, "{\"profile\": \"%s\", \"params\": \"ssb_sf20\", \"target\": \"%s\"}", pn.c_str(),
                    t ? "gpu_like" : "cpu_like");
      emit("q21", a, model_q21(Q21Params::ssb_sf20(), p, t ? Q21Target::kGpuLike : Q21Target::kCpuLike), first);
    }
  }
  std::printf("\n]\n");
  return 0;
}
