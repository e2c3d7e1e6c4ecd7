// runtime.cpp -- per-thread contexts, device groups, the host-database upload
// cache and status mapping for the C++ drop-in (dropin/include/tq/b200_runtime.hpp).
#include "tq/b200_runtime.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace tq::b200 {

namespace {

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

std::vector<int> visible_devices() {
  std::vector<int> devs;
  if (const char* e = std::getenv("CRYS_DEVICES")) {
    std::stringstream ss(e);
    std::string tok;
    while (std::getline(ss, tok, ','))
      if (!tok.empty()) devs.push_back(std::atoi(tok.c_str()));
  } else {
    const int n = crys_device_count();
    for (int d = 0; d < n; ++d) devs.push_back(d);
  }
  if (devs.empty()) throw std::runtime_error("crystal_b200: no CUDA device visible");
  return devs;
}

}  // namespace

// ------------------------------------------------------------ upload cache

struct CacheEntry {
  std::vector<uint64_t> sig;
  crys_db* db = nullptr;
};
struct SsbDatabaseCache {
  std::map<std::pair<const crys_ctx*, const void*>, CacheEntry> entries;
  long long uploads = 0;
};

namespace {
// Everything one host thread owns, torn down in dependency order: cached
// databases before the groups / context they live on.
struct ThreadContext {
  crys_ctx* ctx = nullptr;
  std::map<int, crys_ctx*> groups;  // shard count -> group
  SsbDatabaseCache cache;
  ~ThreadContext() {
    for (auto& kv : cache.entries) crys_db_free(kv.second.db);
    cache.entries.clear();
    for (auto& kv : groups) crys_destroy(kv.second);
    if (ctx) crys_destroy(ctx);
  }
};

ThreadContext& tc() {
  thread_local ThreadContext t;
  return t;
}
SsbDatabaseCache& cache() { return tc().cache; }
}  // namespace

crys_ctx* context() {
  ThreadContext& t = tc();
  if (!t.ctx) check(crys_init(env_int("CRYS_DEVICE", 0), &t.ctx));
  return t.ctx;
}

crys_ctx* group_context(int workers) {
  TQ_CONFIG_CHECK(workers >= 1, "run_query: workers must be >= 1");
  const std::vector<int> devs = visible_devices();
  const bool emulate = env_int("CRYS_GROUP_EMULATE", 0) != 0;
  const int shards = emulate ? workers : std::min<int>(workers, (int)devs.size());
  ThreadContext& t = tc();
  auto it = t.groups.find(shards);
  if (it != t.groups.end()) return it->second;
  std::vector<int> place((size_t)shards);
  for (int s = 0; s < shards; ++s) place[(size_t)s] = devs[(size_t)s % devs.size()];
  crys_ctx* g = nullptr;
  check(crys_init_group(shards, place.data(), &g));
  t.groups[shards] = g;
  return g;
}

void invalidate(const void* db) {
  auto& c = cache();
  for (auto it = c.entries.begin(); it != c.entries.end();) {
    if (it->first.second == db) {
      crys_db_free(it->second.db);
      it = c.entries.erase(it);
    } else {
      ++it;
    }
  }
}

void invalidate_all() {
  auto& c = cache();
  for (auto& kv : c.entries) crys_db_free(kv.second.db);
  c.entries.clear();
}

long long upload_count() { return cache().uploads; }

namespace detail {
uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  return h * 0xff51afd7ed558ccdULL;
}
uint64_t fingerprint(const int32_t* p, int64_t n, bool full) {
  uint64_t h = 0xcbf29ce484222325ULL ^ (uint64_t)n;
  if (n <= 0) return h;
  const unsigned char* b = reinterpret_cast<const unsigned char*>(p);
  const size_t bytes = sizeof(int32_t) * (size_t)n;
  auto block = [&](size_t off, size_t len) {
    for (size_t i = off; i + 8 <= off + len; i += 8) {
      uint64_t w;
      std::memcpy(&w, b + i, 8);
      h = mix(h, w);
    }
    for (size_t i = off + (len & ~size_t(7)); i < off + len; ++i) h = mix(h, b[i]);
  };
  if (full) {
    block(0, bytes);
  } else {  // first/last 4 KB + 4096 evenly spaced 64-byte blocks
    block(0, std::min<size_t>(bytes, 4096));
    block(bytes - std::min<size_t>(bytes, 4096), std::min<size_t>(bytes, 4096));
    const size_t step = bytes / 4096;
    for (size_t k = 0; step >= 64 && k < 4096; ++k) block(k * step, 64);
  }
  return h;
}
}  // namespace detail

crys_db* cached_database(crys_ctx* g, const void* key, const std::vector<crys_host_column>& cols) {
  size_t total = 0;
  for (const auto& c : cols) total += sizeof(int32_t) * (size_t)c.rows;
  const bool full = total <= (size_t(64) << 20);
  std::vector<uint64_t> sig;
  for (const auto& c : cols) {
    sig.push_back(reinterpret_cast<uint64_t>(c.h_data));
    sig.push_back((uint64_t)c.rows);
    sig.push_back(detail::fingerprint(c.h_data, c.rows, full));
  }
  auto& ent = cache().entries[{g, key}];
  if (ent.db && ent.sig == sig) return ent.db;
  if (ent.db) crys_db_free(ent.db);
  ent.db = nullptr;
  crys_db* db = nullptr;
  check(crys_db_create(g, 0, 0, &db));
  const crys_status s = crys_db_upload_host(db, cols.data(), (int)cols.size());
  if (s != CRYS_OK) {
    crys_db_free(db);
    cache().entries.erase({g, key});
    raise(s);
  }
  ent.db = db;
  ent.sig = std::move(sig);
  ++cache().uploads;
  return db;
}

void raise(crys_status s) {
  const std::string msg = crys_last_error();
  switch (s) {
    case CRYS_ECONFIG: throw ConfigError(msg);
    case CRYS_ECONTRACT: throw ContractError(msg);
    case CRYS_EBUILD: throw BuildError(msg);
    case CRYS_EIO: throw IoError(msg);
    default: throw std::runtime_error("crystal_b200: " + msg);
  }
}

}  // namespace tq::b200
