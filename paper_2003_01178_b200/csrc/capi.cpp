// capi.cpp -- the extern "C" boundary (include/crystal_b200.h).
//
// Every entry point catches internal errors and maps them to crys_status, the
// C-ABI image of the reference's exception taxonomy (include/tq/common.hpp:
// 16-34).  No C++ exception crosses this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "internal.hpp"

namespace {
thread_local std::string g_last_error;

template <class F>
crys_status guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return CRYS_OK;
  } catch (const crys::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return CRYS_ECUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CRYS_ECONTRACT;
  }
}

void bind(crys_ctx* ctx) {
  CRYS_CHECK(ctx != nullptr, CRYS_ECONFIG, "null context");
  CUDA_TRY(cudaSetDevice(ctx->device));
}
}  // namespace

crys_ctx::~crys_ctx() {
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  qws.reset();
  sws.reset();
  delete staging;
  for (auto& e : io_ev)
    if (e) cudaEventDestroy(e);
  if (graph_fence) cudaEventDestroy(graph_fence);
  if (graph_stream) cudaStreamDestroy(graph_stream);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (own_stream) cudaStreamDestroy(own_stream);
}

crys_db::crys_db() {
  static std::atomic<uint64_t> next{1};
  uid = next.fetch_add(1);
}

crys_db::~crys_db() {
  for (auto& kv : cols)
    if (kv.second.ready) cudaEventDestroy(kv.second.ready);
  for (crys_db* s : shards) delete s;
}

const int32_t* crys_db::col(const std::string& table, const std::string& column, int64_t* rows) const {
  auto it = cols.find(table + "." + column);
  CRYS_CHECK(it != cols.end(), CRYS_ECONTRACT, "table " + table + ": no column " + column);
  if (rows) *rows = it->second.rows;
  const Col& c = it->second;
  if (c.pending) {  // column still in flight from crys_db_upload_host
    if (cudaEventQuery(c.ready) == cudaSuccess)
      c.pending = false;
    else
      CUDA_TRY(cudaStreamWaitEvent(ctx->stream, c.ready, 0));
  }
  return c.buf->as<int32_t>();
}

bool crys_db::col_range(const std::string& table, const std::string& column, int32_t* lo,
                        int32_t* hi) const {
  auto it = cols.find(table + "." + column);
  if (it == cols.end() || !it->second.stats) return false;
  *lo = it->second.vmin;
  *hi = it->second.vmax;
  return true;
}

// Dimension columns get value-range statistics on upload (they are small;
// lineorder columns are not scanned on the host).
static void host_stats(crys_db::Col& c, const std::string& table, const int32_t* h, int64_t rows) {
  c.stats = false;
  if (table == "lineorder" || rows <= 0) return;
  int32_t lo = h[0], hi = h[0];
  for (int64_t i = 1; i < rows; ++i) {
    lo = h[i] < lo ? h[i] : lo;
    hi = h[i] > hi ? h[i] : hi;
  }
  c.stats = true;
  c.vmin = lo;
  c.vmax = hi;
}

int64_t crys_db::table_rows(const std::string& table) const {
  for (auto& kv : cols)
    if (kv.first.compare(0, table.size() + 1, table + ".") == 0) return kv.second.rows;
  return 0;
}

namespace crys {

void ensure_dyn_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set_to;
  if (bytes == 0) return;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = set_to[{dev, fn}];
  if (bytes <= cur) return;
  if (cur == 0) {  // the default limit is 48 KB of static + dynamic shared memory
    cudaFuncAttributes fa;
    CUDA_TRY(cudaFuncGetAttributes(&fa, fn));
    if (bytes + fa.sharedSizeBytes <= 48 * 1024) return;
  }
  CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  cur = bytes;
}

void timing_begin(crys_ctx* c) {
  if (c->timing) CUDA_TRY(cudaEventRecord(c->ev[0], c->stream));
}
void timing_kernel_begin(crys_ctx* c) {
  if (c->timing) CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
}
void timing_kernel_end(crys_ctx* c) {
  if (c->timing) CUDA_TRY(cudaEventRecord(c->ev[2], c->stream));
}
void timing_end(crys_ctx* c) {
  if (!c->timing) return;
  CUDA_TRY(cudaEventRecord(c->ev[3], c->stream));
  CUDA_TRY(cudaEventSynchronize(c->ev[3]));
  float k = 0, t = 0;
  CUDA_TRY(cudaEventElapsedTime(&k, c->ev[1], c->ev[2]));
  CUDA_TRY(cudaEventElapsedTime(&t, c->ev[0], c->ev[3]));
  c->kernel_ms = k;
  c->total_ms = t;
}

// Result rows -> (groups, sums) in lexicographic order.
void emit_rows(int qid, const std::vector<int64_t>& cell, const std::vector<int64_t>& sums,
               int32_t* h_groups, int64_t* h_sums, int64_t max_rows, int64_t* nrows) {
  const QueryPlan& plan = plan_for(qid);
  const int64_t n = (int64_t)cell.size();
  *nrows = n;
  CRYS_CHECK(n <= max_rows, CRYS_ECONTRACT, "result has more rows than the caller's buffer");
  std::vector<int64_t> strides(plan.group.size(), 1);
  int64_t s = 1;
  for (int g = (int)plan.group.size() - 1; g >= 0; --g) {
    strides[g] = s;
    s *= (int64_t)(plan.group[g].hi - plan.group[g].lo + 1);
  }
  for (int64_t i = 0; i < n; ++i) {
    int64_t idx = cell[(size_t)i];
    for (size_t g = 0; g < plan.group.size(); ++g) {  // AggregateTable::key_of (ssb_queries.cpp:49-56)
      if (h_groups) h_groups[i * 3 + (int64_t)g] = plan.group[g].lo + (int32_t)(idx / strides[g]);
      idx %= strides[g];
    }
    if (h_sums) h_sums[i] = sums[(size_t)i];
  }
}

}  // namespace crys

namespace crys {
crys_ctx* new_context(int device) {
  int n = 0;
  CUDA_TRY(cudaGetDeviceCount(&n));
  CRYS_CHECK(device >= 0 && device < n, CRYS_ECONFIG, "no such CUDA device");
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  CRYS_CHECK(prop.major == 10, CRYS_ENOTBUILT,
             std::string("library is compiled for sm_100a only; device is ") + prop.name);
  auto* ctx = new crys_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    crys::fail(CRYS_ECUDA, cudaGetErrorString(e));
  }
  ctx->stream = ctx->own_stream;
  for (auto& ev : ctx->ev) {
    e = cudaEventCreate(&ev);
    if (e != cudaSuccess) {
      delete ctx;
      crys::fail(CRYS_ECUDA, cudaGetErrorString(e));
    }
  }
  return ctx;
}
}  // namespace crys

namespace crys {
// Header words of a reduced partial -> the reference's exceptions (the same
// messages as the device finalize, ssb_query.cu finalize_host_part).
void raise_partial_errors(int qid, const int64_t* h_hdr) {
  if (!h_hdr) return;
  for (int j = 0; j < 4; ++j)
    for (int c = 1; c <= 4; ++c)
      if (h_hdr[8 + 4 * j + (c - 1)]) {
        static const char* kMsg[5] = {"", "HashTable: key equals empty sentinel", "HashTable: duplicate key",
                                      "HashTable: capacity overflow", "dimension key outside its column statistics"};
        fail(c == 4 ? CRYS_ECONTRACT : CRYS_EBUILD,
             std::string(kMsg[c]) + " (join " + std::to_string(j) + " of " + plan_for(qid).name + ")");
      }
  if (h_hdr[4]) fail(CRYS_ECONTRACT, "group value outside its declared domain");
}
}  // namespace crys

extern "C" {

const char* crys_last_error(void) { return g_last_error.c_str(); }

const char* crys_version(void) {
  return "crystal_b200 2.0 (sm_100a; fused SSB q1.1-q4.3, device groups + NCCL reduce, select/project, "
         "hash join, radix sort)";
}

const char* crys_nccl_version(void) { return crys::nccl_status(); }

int crys_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}


crys_status crys_init(int device, crys_ctx** out) {
  return guarded([&] {
    CRYS_CHECK(out != nullptr, CRYS_ECONFIG, "null output handle");
    *out = crys::new_context(device);
  });
}

crys_status crys_init_group(int nshards, const int* devices, crys_ctx** out) {
  return guarded([&] {
    CRYS_CHECK(out != nullptr, CRYS_ECONFIG, "null output handle");
    *out = crys::new_group(nshards, devices);
  });
}

int crys_group_shards(const crys_ctx* ctx) { return ctx ? crys::group_shards(ctx) : 0; }
int crys_group_devices(const crys_ctx* ctx) { return ctx ? crys::group_devices(ctx) : 0; }
int crys_group_uses_nccl(const crys_ctx* ctx) { return ctx && crys::group_nccl(ctx) ? 1 : 0; }

void crys_destroy(crys_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete ctx;
}

crys_status crys_set_stream(crys_ctx* ctx, void* s) {
  return guarded([&] {
    bind(ctx);
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
  });
}

crys_status crys_synchronize(crys_ctx* ctx) {
  return guarded([&] {
    bind(ctx);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  });
}

int64_t crys_kernel_launches(const crys_ctx* ctx) { return ctx ? ctx->launches : 0; }

crys_status crys_enable_timing(crys_ctx* ctx, int enable) {
  return guarded([&] {
    bind(ctx);
    ctx->timing = enable != 0;
  });
}

crys_status crys_radix_histogram(crys_ctx* ctx, const int32_t* d_keys, int64_t n, int start_bit,
                                 int num_bits, int64_t num_owners, int64_t* h_counts) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(h_counts && n >= 0 && (n == 0 || d_keys), CRYS_ECONFIG, "bad argument");
    crys::radix_owner_histogram(ctx, d_keys, n, start_bit, num_bits, num_owners, h_counts);
  });
}

crys_status crys_radix_partition(crys_ctx* ctx, const int32_t* d_keys, const int32_t* d_payloads,
                                 int64_t n, int start_bit, int num_bits, int32_t* d_out_keys,
                                 int32_t* d_out_payloads) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(n >= 0 && (n == 0 || (d_keys && d_payloads && d_out_keys && d_out_payloads)),
               CRYS_ECONFIG, "bad argument");
    crys::timing_begin(ctx);
    crys::radix_partition_pass(ctx, d_keys, d_payloads, d_out_keys, d_out_payloads, n, start_bit, num_bits);
    crys::timing_end(ctx);
  });
}

crys_status crys_last_timing(const crys_ctx* ctx, double* kernel_ms, double* total_ms) {
  return guarded([&] {
    CRYS_CHECK(ctx != nullptr, CRYS_ECONFIG, "null context");
    if (kernel_ms) *kernel_ms = ctx->kernel_ms;
    if (total_ms) *total_ms = ctx->total_ms;
  });
}

// ---------------------------------------------------------------- device memory

crys_status crys_device_alloc(crys_ctx* ctx, size_t bytes, void** d_out) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(d_out != nullptr, CRYS_ECONFIG, "null output");
    void* p = nullptr;
    CUDA_TRY(cudaMalloc(&p, bytes + 256));
    *d_out = p;
  });
}

void crys_device_free(crys_ctx* ctx, void* d_ptr) {
  if (!ctx || !d_ptr) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaFree(d_ptr);
}

crys_status crys_copy_to_device(crys_ctx* ctx, void* d_dst, const void* h_src, size_t bytes) {
  return guarded([&] {
    bind(ctx);
    if (bytes == 0) return;
    CRYS_CHECK(d_dst && h_src, CRYS_ECONFIG, "null argument");
    CUDA_TRY(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  });
}

crys_status crys_copy_to_host(crys_ctx* ctx, void* h_dst, const void* d_src, size_t bytes) {
  return guarded([&] {
    bind(ctx);
    if (bytes == 0) return;
    CRYS_CHECK(h_dst && d_src, CRYS_ECONFIG, "null argument");
    CUDA_TRY(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  });
}

// ---------------------------------------------------------------- database

crys_status crys_db_generate(crys_ctx* ctx, int64_t sf, uint64_t seed, int64_t lo_begin,
                             int64_t lo_end, crys_db** out) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(out != nullptr, CRYS_ECONFIG, "null output handle");
    CRYS_CHECK(sf >= 1, CRYS_ECONFIG, "scale factor must be >= 1");
    auto* db = new crys_db();
    db->ctx = ctx;
    db->sf = sf;
    db->seed = seed;
    db->lo_begin = lo_begin;
    db->lo_end = lo_end;
    try {
      if (ctx->group) {  // every shard generates its row range + the dimensions on its device
        const int64_t rows = 6000000LL * sf;  // ssb_gen.cpp:179
        if (db->lo_end < 0 || db->lo_end > rows) db->lo_end = rows;
        CRYS_CHECK(db->lo_begin >= 0 && db->lo_begin <= db->lo_end, CRYS_ECONFIG, "bad lineorder shard range");
        const int S = crys::group_shards(ctx);
        for (int sh = 0; sh < S; ++sh) {
          crys_ctx* m = crys::group_member_of_shard(ctx, sh);
          CUDA_TRY(cudaSetDevice(m->device));
          auto* part = new crys_db();
          db->shards.push_back(part);
          part->ctx = m;
          part->sf = sf;
          part->seed = seed;
          crys::shard_range(db->lo_begin, db->lo_end, sh, S, &part->lo_begin, &part->lo_end);
          crys::ssb_generate(m, part);
        }
        CUDA_TRY(cudaSetDevice(ctx->device));
      } else {
        crys::ssb_generate(ctx, db);
      }
    } catch (...) {
      delete db;
      throw;
    }
    *out = db;
  });
}

crys_status crys_fill_uniform_i32(crys_ctx* ctx, int32_t* d_out, int64_t n, uint64_t seed,
                                  uint64_t stream, int64_t index0, int32_t lo, int32_t hi) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(n == 0 || d_out, CRYS_ECONFIG, "null output");
    crys::fill_uniform_i32(ctx, d_out, n, seed, stream, index0, lo, hi);
  });
}

crys_status crys_fill_float_pairs(crys_ctx* ctx, float* d_x1, float* d_x2, int64_t n, uint64_t seed,
                                  uint64_t stream, float lo, float hi) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(n == 0 || (d_x1 && d_x2), CRYS_ECONFIG, "null output");
    crys::fill_float_pairs(ctx, d_x1, d_x2, n, seed, stream, lo, hi);
  });
}

crys_status crys_db_create(crys_ctx* ctx, int64_t sf, uint64_t seed, crys_db** out) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(out != nullptr, CRYS_ECONFIG, "null output handle");
    auto* db = new crys_db();
    db->ctx = ctx;
    db->sf = sf;
    db->seed = seed;
    for (int sh = 0; ctx->group && sh < crys::group_shards(ctx); ++sh) {
      auto* part = new crys_db();
      db->shards.push_back(part);
      part->ctx = crys::group_member_of_shard(ctx, sh);
      part->sf = sf;
      part->seed = seed;
    }
    *out = db;
  });
}

crys_status crys_db_upload_column(crys_db* db, const char* table, const char* column,
                                  const int32_t* h_data, int64_t rows) {
  if (db && db->is_group()) {  // lineorder: row-range slices; dimensions: every shard
    const bool fact = table && std::string(table) == "lineorder";
    const int S = (int)db->shards.size();
    for (int sh = 0; sh < S; ++sh) {
      int64_t b = 0, e = rows;
      if (fact) crys::shard_range(0, rows, sh, S, &b, &e);
      const crys_status st = crys_db_upload_column(db->shards[(size_t)sh], table, column,
                                                   h_data ? h_data + b : nullptr, e - b);
      if (st != CRYS_OK) return st;
      if (fact) {
        db->shards[(size_t)sh]->lo_begin = b;
        db->shards[(size_t)sh]->lo_end = e;
      }
    }
    if (fact) {
      db->lo_begin = 0;
      db->lo_end = rows;
    }
    cudaSetDevice(db->ctx->device);
    return CRYS_OK;
  }
  return guarded([&] {
    CRYS_CHECK(db && table && column, CRYS_ECONFIG, "null argument");
    bind(db->ctx);
    CRYS_CHECK(rows >= 0 && (rows == 0 || h_data), CRYS_ECONFIG, "bad column data");
    auto& c = db->cols[std::string(table) + "." + column];
    if (!c.buf) c.buf.reset(new crys::DevBuf());
    c.buf->reserve(sizeof(int32_t) * (size_t)std::max<int64_t>(rows, 1));
    c.rows = rows;
    host_stats(c, table, h_data, rows);
    if (rows)
      CUDA_TRY(cudaMemcpyAsync(c.buf->p, h_data, sizeof(int32_t) * (size_t)rows,
                               cudaMemcpyHostToDevice, db->ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(db->ctx->stream));
    if (std::string(table) == "lineorder") {
      db->lo_begin = 0;
      db->lo_end = rows;
    }
  });
}

crys_status crys_db_upload_host(crys_db* db, const crys_host_column* cols, int ncols) {
  if (db && db->is_group()) {
    // lineorder columns are cut into the shards' row ranges; dimension columns
    // go to the first shard of every device (the one that builds its tables)
    int64_t lo_rows = -1;
    for (int i = 0; i < ncols && cols; ++i)
      if (cols[i].table && std::string(cols[i].table) == "lineorder") {
        if (lo_rows >= 0 && cols[i].rows != lo_rows) {
          g_last_error = "lineorder columns of different length";
          return CRYS_ECONTRACT;
        }
        lo_rows = cols[i].rows;
      }
    const int S = (int)db->shards.size();
    for (int sh = 0; sh < S; ++sh) {
      crys_db* part = db->shards[(size_t)sh];
      const bool dims = crys::shard_holds_dims(db->ctx, sh);
      int64_t b = 0, e = 0;
      if (lo_rows >= 0) crys::shard_range(0, lo_rows, sh, S, &b, &e);
      std::vector<crys_host_column> mine;
      for (int i = 0; i < ncols; ++i) {
        crys_host_column c = cols[i];
        if (c.table && std::string(c.table) == "lineorder") {
          c.h_data = c.h_data ? c.h_data + b : nullptr;
          c.rows = e - b;
        } else if (!dims) {
          continue;
        }
        mine.push_back(c);
      }
      const crys_status st = crys_db_upload_host(part, mine.data(), (int)mine.size());
      if (st != CRYS_OK) return st;
      if (lo_rows >= 0) {
        part->lo_begin = b;
        part->lo_end = e;
      }
    }
    if (lo_rows >= 0) {
      db->lo_begin = 0;
      db->lo_end = lo_rows;
    }
    cudaSetDevice(db->ctx->device);
    return CRYS_OK;
  }
  return guarded([&] {
    CRYS_CHECK(db && (ncols == 0 || cols), CRYS_ECONFIG, "null argument");
    crys_ctx* ctx = db->ctx;
    bind(ctx);
    if (!ctx->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    // WAR: work already queued on the compute stream may still read the
    // previous contents of these buffers
    cudaEvent_t fence;
    CUDA_TRY(cudaEventCreateWithFlags(&fence, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(fence, ctx->stream));
    CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, fence, 0));
    CUDA_TRY(cudaEventDestroy(fence));
    std::vector<crys_db::Col*> issued((size_t)ncols, nullptr);
    for (int i = 0; i < ncols; ++i) {  // issue every copy first, in the caller's order
      const crys_host_column& hc = cols[i];
      CRYS_CHECK(hc.table && hc.column, CRYS_ECONFIG, "null column name");
      CRYS_CHECK(hc.rows >= 0 && (hc.rows == 0 || hc.h_data), CRYS_ECONFIG, "bad column data");
      auto& c = db->cols[std::string(hc.table) + "." + hc.column];
      if (!c.buf) c.buf.reset(new crys::DevBuf());
      if (sizeof(int32_t) * (size_t)std::max<int64_t>(hc.rows, 1) > c.buf->bytes) {
        CUDA_TRY(cudaStreamSynchronize(ctx->copy_stream));
        c.buf->reserve(sizeof(int32_t) * (size_t)std::max<int64_t>(hc.rows, 1));
      }
      c.rows = hc.rows;
      if (!c.ready) CUDA_TRY(cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming));
      if (hc.rows)
        CUDA_TRY(cudaMemcpyAsync(c.buf->p, hc.h_data, sizeof(int32_t) * (size_t)hc.rows,
                                 cudaMemcpyHostToDevice, ctx->copy_stream));
      CUDA_TRY(cudaEventRecord(c.ready, ctx->copy_stream));
      c.pending = true;
      issued[(size_t)i] = &c;
      if (std::string(hc.table) == "lineorder") {
        db->lo_begin = 0;
        db->lo_end = hc.rows;
      }
    }
    // dimension statistics on the host while the DMA runs
    for (int i = 0; i < ncols; ++i) host_stats(*issued[(size_t)i], cols[i].table, cols[i].h_data, cols[i].rows);
  });
}

// ---------------------------------------------------------------- CRYS column files
// The reference's on-disk column format (column_io.hpp:3-13, column_io.cpp:
// 50-100): "CRYS", u16 version 1, u8 kind (0 int32, 1 float32), u8 0, u64
// count, then raw little-endian 4-byte elements.  Loading streams the payload
// through two pinned staging buffers: the file read of chunk i+1 overlaps the
// DMA of chunk i on the copy stream; the column's ready event then gates the
// queries that read it (as crys_db_upload_host).
namespace {
constexpr size_t kIoChunk = size_t(32) << 20;  // bytes per staging buffer

struct FileCloser {
  void operator()(FILE* f) const {
    if (f) fclose(f);
  }
};

void io_ready(crys_ctx* ctx) {
  if (!ctx->copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    ctx->io[i].reserve(kIoChunk);
    if (!ctx->io_ev[i]) CUDA_TRY(cudaEventCreateWithFlags(&ctx->io_ev[i], cudaEventDisableTiming));
  }
}
}  // namespace

crys_status crys_db_load_column_file(crys_db* db, const char* table, const char* column, const char* path) {
  return guarded([&] {
    CRYS_CHECK(!(db && db->is_group()), CRYS_ECONFIG,
               "a device-group database has one column per shard (use a shard's context)");
    CRYS_CHECK(db && table && column && path, CRYS_ECONFIG, "null argument");
    crys_ctx* ctx = db->ctx;
    bind(ctx);
    std::unique_ptr<FILE, FileCloser> f(fopen(path, "rb"));
    CRYS_CHECK(f != nullptr, CRYS_EIO, std::string("cannot open for reading: ") + path);
    unsigned char h[16];
    CRYS_CHECK(fread(h, 1, 16, f.get()) == 16, CRYS_EIO, std::string("truncated header: ") + path);
    CRYS_CHECK(std::memcmp(h, "CRYS", 4) == 0, CRYS_EIO, std::string("bad magic: ") + path);
    CRYS_CHECK((h[4] | (h[5] << 8)) == 1, CRYS_EIO, std::string("unsupported format version: ") + path);
    CRYS_CHECK(h[6] <= 1, CRYS_EIO, std::string("unknown element kind byte: ") + path);
    CRYS_CHECK(h[6] == 0, CRYS_EIO,
               std::string("element kind mismatch: ") + path + " holds float32, expected int32");
    uint64_t n = 0;
    for (int i = 0; i < 8; ++i) n |= (uint64_t)h[8 + i] << (8 * i);
    CRYS_CHECK(n < (uint64_t(1) << 40), CRYS_EIO, std::string("implausible element count: ") + path);
    io_ready(ctx);
    // WAR against queued work that may still read the previous buffer
    cudaEvent_t fence;
    CUDA_TRY(cudaEventCreateWithFlags(&fence, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(fence, ctx->stream));
    CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, fence, 0));
    CUDA_TRY(cudaEventDestroy(fence));
    auto& c = db->cols[std::string(table) + "." + column];
    if (!c.buf) c.buf.reset(new crys::DevBuf());
    if (sizeof(int32_t) * (size_t)std::max<uint64_t>(n, 1) > c.buf->bytes) {
      CUDA_TRY(cudaStreamSynchronize(ctx->copy_stream));
      c.buf->reserve(sizeof(int32_t) * (size_t)std::max<uint64_t>(n, 1));
    }
    c.rows = (int64_t)n;
    const bool stats = std::string(table) != "lineorder" && n > 0;
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    const size_t total = 4 * (size_t)n;
    for (size_t off = 0, i = 0; off < total; off += kIoChunk, ++i) {
      const int b = (int)(i & 1);
      CUDA_TRY(cudaEventSynchronize(ctx->io_ev[b]));  // staging buffer b free again
      const size_t len = std::min(kIoChunk, total - off);
      CRYS_CHECK(fread(ctx->io[b].p, 1, len, f.get()) == len, CRYS_EIO, std::string("truncated payload: ") + path);
      if (stats) {
        const int32_t* v = ctx->io[b].as<int32_t>();
        for (size_t k = 0; k < len / 4; ++k) {
          lo = v[k] < lo ? v[k] : lo;
          hi = v[k] > hi ? v[k] : hi;
        }
      }
      CUDA_TRY(cudaMemcpyAsync(c.buf->as<char>() + off, ctx->io[b].p, len, cudaMemcpyHostToDevice,
                               ctx->copy_stream));
      CUDA_TRY(cudaEventRecord(ctx->io_ev[b], ctx->copy_stream));
    }
    if (!c.ready) CUDA_TRY(cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(c.ready, ctx->copy_stream));
    c.pending = true;
    c.stats = stats;
    c.vmin = stats ? lo : 0;
    c.vmax = stats ? hi : -1;
    if (std::string(table) == "lineorder") {
      db->lo_begin = 0;
      db->lo_end = (int64_t)n;
    }
  });
}

crys_status crys_db_save_column_file(const crys_db* db, const char* table, const char* column, const char* path) {
  return guarded([&] {
    CRYS_CHECK(!(db && db->is_group()), CRYS_ECONFIG,
               "a device-group database has one column per shard (use a shard's context)");
    CRYS_CHECK(db && table && column && path, CRYS_ECONFIG, "null argument");
    crys_ctx* ctx = db->ctx;
    bind(ctx);
    int64_t n = 0;
    const int32_t* d = db->col(table, column, &n);  // orders after a pending upload
    io_ready(ctx);
    std::unique_ptr<FILE, FileCloser> f(fopen(path, "wb"));
    CRYS_CHECK(f != nullptr, CRYS_EIO, std::string("cannot open for writing: ") + path);
    unsigned char h[16] = {'C', 'R', 'Y', 'S', 1, 0, 0, 0};
    for (int i = 0; i < 8; ++i) h[8 + i] = (unsigned char)((uint64_t)n >> (8 * i));
    CRYS_CHECK(fwrite(h, 1, 16, f.get()) == 16, CRYS_EIO, std::string("write failed: ") + path);
    const size_t total = 4 * (size_t)n;
    for (size_t off = 0; off < total; off += kIoChunk) {
      const size_t len = std::min(kIoChunk, total - off);
      CUDA_TRY(cudaMemcpyAsync(ctx->io[0].p, reinterpret_cast<const char*>(d) + off, len,
                               cudaMemcpyDeviceToHost, ctx->stream));
      CUDA_TRY(cudaStreamSynchronize(ctx->stream));
      CRYS_CHECK(fwrite(ctx->io[0].p, 1, len, f.get()) == len, CRYS_EIO, std::string("write failed: ") + path);
    }
    CRYS_CHECK(fflush(f.get()) == 0, CRYS_EIO, std::string("write failed: ") + path);
  });
}

crys_status crys_db_column(const crys_db* db, const char* table, const char* column,
                           const int32_t** d_data, int64_t* rows) {
  return guarded([&] {
    CRYS_CHECK(!(db && db->is_group()), CRYS_ECONFIG,
               "a device-group database has one column per shard (use a shard's context)");
    CRYS_CHECK(db && table && column && d_data, CRYS_ECONFIG, "null argument");
    *d_data = db->col(table, column, rows);
  });
}

crys_status crys_db_column_rows(const crys_db* db, const char* table, const char* column, int64_t* rows) {
  return guarded([&] {
    CRYS_CHECK(db && table && column && rows, CRYS_ECONFIG, "null argument");
    const bool fact = std::string(table) == "lineorder";
    int64_t total = 0;
    if (!db->is_group()) {
      auto it = db->cols.find(std::string(table) + "." + column);
      CRYS_CHECK(it != db->cols.end(), CRYS_ECONTRACT, std::string("table ") + table + ": no column " + column);
      total = it->second.rows;
    }
    for (const crys_db* part : db->shards) {
      auto it = part->cols.find(std::string(table) + "." + column);
      CRYS_CHECK(it != part->cols.end(), CRYS_ECONTRACT, std::string("table ") + table + ": no column " + column);
      total += it->second.rows;
      if (!fact) break;
    }
    *rows = total;
  });
}

crys_status crys_db_download_column(const crys_db* db, const char* table, const char* column,
                                    int32_t* h_out, int64_t rows) {
  if (db && db->is_group()) {  // lineorder: the shards in row order; dimensions: shard 0
    const bool fact = table && std::string(table) == "lineorder";
    int64_t off = 0;
    for (const crys_db* part : db->shards) {
      int64_t n = 0;
      const int32_t* d = nullptr;
      const crys_status st0 = crys_db_column(part, table, column, &d, &n);
      if (st0 != CRYS_OK) return st0;
      if (!fact) return crys_db_download_column(part, table, column, h_out, rows);
      if (off + n > rows) {
        g_last_error = "row count mismatch";
        return CRYS_ECONTRACT;
      }
      const crys_status st = crys_db_download_column(part, table, column, h_out + off, n);
      if (st != CRYS_OK) return st;
      off += n;
    }
    cudaSetDevice(db->ctx->device);
    if (off != rows) {
      g_last_error = "row count mismatch";
      return CRYS_ECONTRACT;
    }
    return CRYS_OK;
  }
  return guarded([&] {
    CRYS_CHECK(db && table && column && h_out, CRYS_ECONFIG, "null argument");
    bind(db->ctx);
    int64_t n = 0;
    const int32_t* d = db->col(table, column, &n);
    CRYS_CHECK(rows == n, CRYS_ECONTRACT, "row count mismatch");
    if (n)
      CUDA_TRY(cudaMemcpyAsync(h_out, d, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToHost,
                               db->ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(db->ctx->stream));
  });
}

void crys_db_free(crys_db* db) {
  if (!db) return;
  for (crys_db* part : db->shards) {
    cudaSetDevice(part->ctx->device);
    cudaStreamSynchronize(part->ctx->stream);
    crys::forget_db(part->ctx, part->uid);
  }
  cudaSetDevice(db->ctx->device);
  cudaStreamSynchronize(db->ctx->stream);
  crys::forget_db(db->ctx, db->uid);
  delete db;
}

// ---------------------------------------------------------------- queries

crys_status crys_query_shape(int qid, int64_t* cells, int32_t* ngroup, int32_t* njoins) {
  return guarded([&] {
    const crys::QueryPlan& p = crys::plan_for(qid);
    if (cells) *cells = p.cells();
    if (ngroup) *ngroup = (int32_t)p.group.size();
    if (njoins) *njoins = (int32_t)p.joins.size();
  });
}

crys_status crys_query_plan_json(int qid, char* out, size_t cap, size_t* len) {
  return guarded([&] {
    const std::string j = crys::plan_json(qid);
    if (len) *len = j.size();
    if (out && cap) {
      const size_t n = std::min(cap - 1, j.size());
      std::memcpy(out, j.data(), n);
      out[n] = 0;
    }
  });
}

static void fill_survivors(int qid, const crys::ResultRows& r, int64_t* h_survivors) {
  if (!h_survivors) return;
  const crys::QueryPlan& p = crys::plan_for(qid);
  const int ns = p.joins.empty() ? 1 : (int)p.joins.size();
  for (int j = 0; j < 4; ++j) h_survivors[j] = j < ns ? r.survivors[j] : 0;
}

crys_status crys_run_query(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt,
                           int32_t* h_groups, int64_t* h_sums, int64_t max_rows, int64_t* nrows,
                           int64_t* h_survivors) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(db != nullptr && nrows != nullptr, CRYS_ECONFIG, "null argument");
    CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
    crys::plan_for(qid);  // ConfigError for an unknown id
    crys::ResultRows r;
    if (db->is_group()) {
      CRYS_CHECK(db->ctx == ctx, CRYS_ECONFIG, "device-group database belongs to another context");
      crys::ssb_run_group(ctx, db, qid, bt, ipt, &r);
    } else {
      CRYS_CHECK(db->ctx->device == ctx->device, CRYS_ECONFIG, "database lives on another device");
      crys::ssb_run_query(ctx, db, qid, bt, ipt, &r);
    }
    fill_survivors(qid, r, h_survivors);
    crys::emit_rows(qid, r.cell, r.sum, h_groups, h_sums, max_rows, nrows);
  });
}

crys_status crys_run_query_host(crys_ctx* ctx, const crys_host_column* cols, int ncols, int qid,
                                int bt, int ipt, int32_t* h_groups, int64_t* h_sums,
                                int64_t max_rows, int64_t* nrows, int64_t* h_survivors) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(cols != nullptr && ncols > 0 && nrows != nullptr, CRYS_ECONFIG, "null argument");
    CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
    const crys::QueryPlan& plan = crys::plan_for(qid);
    // The columns the plan references: fact keys / filters / aggregates and
    // each joined dimension's key, filter and payload columns.
    std::vector<std::pair<std::string, std::string>> need;
    for (auto& f : plan.fact_filters) need.push_back({"lineorder", f.column});
    for (auto& j : plan.joins) {
      need.push_back({"lineorder", j.fact_key});
      need.push_back({j.dim_table, j.dim_key});
      for (auto& f : j.filters) need.push_back({j.dim_table, f.column});
      if (!j.payload.empty()) need.push_back({j.dim_table, j.payload});
    }
    if (plan.agg == crys::kAggExtPriceTimesDiscount) {
      need.push_back({"lineorder", "lo_extendedprice"});
      need.push_back({"lineorder", "lo_discount"});
    } else {
      need.push_back({"lineorder", "lo_revenue"});
      if (plan.agg == crys::kAggRevenueMinusSupplyCost) need.push_back({"lineorder", "lo_supplycost"});
    }
    // Staging database owned by the context: device buffers are reused across
    // calls, but every call copies its inputs H2D (the reference takes a host
    // `const SsbDatabase&`).
    if (!ctx->staging) {
      ctx->staging = new crys_db();
      ctx->staging->ctx = ctx;
    }
    crys_db* staging = ctx->staging;
    for (auto& tc : need) {
      const crys_host_column* hc = nullptr;
      for (int i = 0; i < ncols; ++i)
        if (tc.first == cols[i].table && tc.second == cols[i].column) hc = &cols[i];
      CRYS_CHECK(hc != nullptr, CRYS_ECONTRACT, "table " + tc.first + ": no column " + tc.second);
      auto& c = staging->cols[tc.first + "." + tc.second];
      if (!c.buf) c.buf.reset(new crys::DevBuf());
      c.buf->reserve(sizeof(int32_t) * (size_t)std::max<int64_t>(hc->rows, 1));
      c.rows = hc->rows;
      host_stats(c, tc.first, hc->h_data, hc->rows);
      if (hc->rows)
        CUDA_TRY(cudaMemcpyAsync(c.buf->p, hc->h_data, sizeof(int32_t) * (size_t)hc->rows,
                                 cudaMemcpyHostToDevice, ctx->stream));
    }
    crys::ResultRows r;
    crys::ssb_run_query(ctx, staging, qid, bt, ipt, &r);
    fill_survivors(qid, r, h_survivors);
    crys::emit_rows(qid, r.cell, r.sum, h_groups, h_sums, max_rows, nrows);
  });
}

crys_status crys_query_partial(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt,
                               int64_t* d_agg, int64_t* d_hdr) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(db && d_agg && d_hdr, CRYS_ECONFIG, "null argument");
    CRYS_CHECK(!db->is_group() && db->ctx->device == ctx->device, CRYS_ECONFIG,
               "partial: a single-device database on this context's device");
    crys::ssb_query_partial(ctx, db, qid, bt, ipt, reinterpret_cast<unsigned long long*>(d_agg),
                            reinterpret_cast<long long*>(d_hdr));
  });
}

crys_status crys_query_partial_box(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt,
                                   int64_t* d_buf, int64_t cap, int64_t* len, crys_group_box* box) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(db && d_buf && len && box, CRYS_ECONFIG, "null argument");
    CRYS_CHECK(!db->is_group() && db->ctx->device == ctx->device, CRYS_ECONFIG,
               "partial: a single-device database on this context's device");
    crys::ssb_partial_box(ctx, {db}, qid, bt, ipt, reinterpret_cast<long long*>(d_buf), cap, box, len, false);
  });
}

crys_status crys_query_finalize_box(crys_ctx* ctx, int qid, const crys_group_box* box, const int64_t* d_buf,
                                    int32_t* h_groups, int64_t* h_sums, int64_t max_rows, int64_t* nrows,
                                    int64_t* h_survivors) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(box && d_buf && nrows, CRYS_ECONFIG, "null argument");
    crys::ResultRows r;
    crys::ssb_finalize_packed(ctx, qid, *box, reinterpret_cast<const long long*>(d_buf), &r);
    fill_survivors(qid, r, h_survivors);
    crys::emit_rows(qid, r.cell, r.sum, h_groups, h_sums, max_rows, nrows);
  });
}

crys_status crys_query_finalize(crys_ctx* ctx, int qid, const int64_t* d_agg, const int64_t* d_hdr,
                                int32_t* h_groups, int64_t* h_sums, int64_t max_rows, int64_t* nrows,
                                int64_t* h_survivors) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(d_agg && nrows, CRYS_ECONFIG, "null argument");
    crys::ResultRows r;
    crys::ssb_finalize_device(ctx, qid, reinterpret_cast<const unsigned long long*>(d_agg),
                              reinterpret_cast<const long long*>(d_hdr), &r);
    fill_survivors(qid, r, h_survivors);
    crys::emit_rows(qid, r.cell, r.sum, h_groups, h_sums, max_rows, nrows);
  });
}


crys_status crys_query_finalize_host(int qid, const int64_t* h_agg, const int64_t* h_hdr, int32_t* h_groups,
                                     int64_t* h_sums, int64_t max_rows, int64_t* nrows, int64_t* h_survivors) {
  return guarded([&] {
    CRYS_CHECK(h_agg && nrows, CRYS_ECONFIG, "null argument");
    const crys::QueryPlan& plan = crys::plan_for(qid);
    const int64_t cells = plan.cells();
    std::vector<int64_t> cell, sums;
    for (int64_t c = 0; c < cells; ++c) {
      if (h_agg[cells + c] != 0 || (plan.joins.empty() && c == 0)) {
        cell.push_back(c);
        sums.push_back(h_agg[c]);
      }
    }
    if (h_survivors) {
      const int ns = plan.joins.empty() ? 1 : (int)plan.joins.size();
      for (int j = 0; j < 4; ++j) h_survivors[j] = (h_hdr && j < ns) ? h_hdr[j] : 0;
    }
    crys::emit_rows(qid, cell, sums, h_groups, h_sums, max_rows, nrows);
    crys::raise_partial_errors(qid, h_hdr);
  });
}

// ---------------------------------------------------------------- operators

crys_status crys_select_i32(crys_ctx* ctx, const int32_t* d_in, int64_t n, crys_pred pred,
                            int32_t* d_out, int64_t* count, int order, int bt, int ipt) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(count != nullptr, CRYS_ECONFIG, "null argument");
    CRYS_CHECK(n == 0 || (d_in && d_out), CRYS_ECONFIG, "null argument");
    int32_t lo, hi;
    crys::lower_pred(pred, &lo, &hi);
    crys::timing_begin(ctx);
    *count = crys::select_i32(ctx, d_in, n, lo, hi, d_out, order, bt, ipt);
    crys::timing_end(ctx);
  });
}

crys_status crys_block_ops_run(crys_ctx* ctx, const int32_t* d_in, int64_t n, int bt, int ipt, crys_pred pred,
                               int32_t* d_out, int64_t* d_counts, int64_t* d_prefix, int64_t* d_totals,
                               int64_t* d_aggs) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
    CRYS_CHECK(d_in && d_out && d_counts && d_prefix && d_totals && d_aggs, CRYS_ECONFIG, "null argument");
    int32_t lo, hi;
    crys::lower_pred(pred, &lo, &hi);
    crys::block_ops_run(ctx, d_in, n, bt, ipt, lo, hi, d_out, d_counts, d_prefix, d_totals, d_aggs);
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  });
}

crys_status crys_stream_read_gbs(crys_ctx* ctx, const void* d_buf, size_t bytes, int reps, double* gbs) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(gbs != nullptr, CRYS_ECONFIG, "null argument");
    *gbs = crys::stream_read(ctx, d_buf, bytes, reps);
  });
}

crys_status crys_project_f32(crys_ctx* ctx, const float* d_x1, const float* d_x2, int64_t n,
                             float a, float b, float* d_out, int sigmoid, int bt, int ipt) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
    CRYS_CHECK(n == 0 || (d_x1 && d_x2 && d_out), CRYS_ECONFIG, "null argument");
    crys::timing_begin(ctx);
    crys::project_f32(ctx, d_x1, d_x2, n, a, b, d_out, sigmoid);
    crys::timing_end(ctx);
  });
}

crys_status crys_ht_build(crys_ctx* ctx, const int32_t* d_keys, const int32_t* d_payloads,
                          int64_t n, int64_t capacity, crys_ht** out) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(out != nullptr, CRYS_ECONFIG, "null output handle");
    // shift_for_capacity (hash_table.cpp:12-16) and the 50% fill rule (:24-26)
    CRYS_CHECK(capacity >= 2 && (capacity & (capacity - 1)) == 0 && capacity <= (1LL << 31),
               CRYS_ECONFIG, "HashTable: capacity must be a power of two >= 2");
    CRYS_CHECK(n >= 0, CRYS_ECONFIG, "HashTable: negative build size");
    if (n * 2 > capacity) crys::fail(CRYS_EBUILD, "HashTable: capacity overflow (fill would exceed 50%)");
    CRYS_CHECK(n == 0 || (d_keys && d_payloads), CRYS_ECONFIG, "null argument");
    auto* ht = new crys_ht();
    ht->ctx = ctx;
    ht->capacity = capacity;
    int lg = 0;
    while ((1LL << lg) < capacity) ++lg;
    ht->shift = 32 - lg;
    try {
      ht->slots.reserve(sizeof(int2) * (size_t)capacity);
      crys::ht_build(ctx, ht, d_keys, d_payloads, n);
    } catch (...) {
      delete ht;
      throw;
    }
    *out = ht;
  });
}

crys_status crys_ht_upload(crys_ctx* ctx, const int32_t* h_keys, const int32_t* h_payloads,
                           int64_t capacity, crys_ht** out) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(out != nullptr, CRYS_ECONFIG, "null output handle");
    CRYS_CHECK(capacity >= 2 && (capacity & (capacity - 1)) == 0 && capacity <= (1LL << 31),
               CRYS_ECONFIG, "HashTable: capacity must be a power of two >= 2");
    CRYS_CHECK(h_keys && h_payloads, CRYS_ECONFIG, "null argument");
    std::vector<int2> v((size_t)capacity);
    int64_t size = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      v[i] = make_int2(h_keys[i], h_payloads[i]);
      size += h_keys[i] != crys::kEmptyKey;
    }
    auto* ht = new crys_ht();
    ht->ctx = ctx;
    ht->capacity = capacity;
    int lg = 0;
    while ((1LL << lg) < capacity) ++lg;
    ht->shift = 32 - lg;
    ht->size = size;
    try {
      ht->slots.reserve(sizeof(int2) * (size_t)capacity);
      CUDA_TRY(cudaMemcpyAsync(ht->slots.p, v.data(), sizeof(int2) * v.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
      CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      delete ht;
      throw;
    }
    *out = ht;
  });
}

crys_status crys_ht_download(const crys_ht* ht, int32_t* h_keys, int32_t* h_payloads) {
  return guarded([&] {
    CRYS_CHECK(ht != nullptr, CRYS_ECONFIG, "null hash table");
    bind(ht->ctx);
    std::vector<int2> v((size_t)ht->capacity);
    CUDA_TRY(cudaMemcpy(v.data(), ht->slots.p, sizeof(int2) * v.size(), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < v.size(); ++i) {
      if (h_keys) h_keys[i] = v[i].x;
      if (h_payloads) h_payloads[i] = v[i].y;
    }
  });
}

int64_t crys_ht_capacity(const crys_ht* ht) { return ht ? ht->capacity : 0; }

void crys_ht_free(crys_ht* ht) {
  if (!ht) return;
  cudaSetDevice(ht->ctx->device);
  cudaStreamSynchronize(ht->ctx->stream);
  delete ht;
}

crys_status crys_join_probe_sum(crys_ctx* ctx, const int32_t* d_keys, const int32_t* d_payloads,
                                int64_t n, const crys_ht* ht, int bt, int ipt, int64_t* checksum) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(ht && checksum, CRYS_ECONFIG, "null argument");
    CRYS_CHECK(bt > 0 && ipt > 0, CRYS_ECONFIG, "TileConfig: block_threads/items_per_thread must be positive");
    CRYS_CHECK(n >= 0 && (n == 0 || (d_keys && d_payloads)), CRYS_ECONFIG, "bad probe input");
    crys::timing_begin(ctx);
    *checksum = crys::join_probe_sum(ctx, d_keys, d_payloads, n, ht);
    crys::timing_end(ctx);
  });
}

crys_status crys_sort_pairs(crys_ctx* ctx, int32_t* d_keys, int32_t* d_payloads, int64_t n,
                            int algo, int bits_per_pass) {
  return guarded([&] {
    bind(ctx);
    CRYS_CHECK(n >= 0 && (n == 0 || (d_keys && d_payloads)), CRYS_ECONFIG, "bad sort input");
    CRYS_CHECK(algo == CRYS_SORT_LSB || algo == CRYS_SORT_MSB, CRYS_ECONFIG, "unknown sort algorithm");
    if (algo == CRYS_SORT_LSB)
      CRYS_CHECK(bits_per_pass >= 1 && bits_per_pass <= 8, CRYS_ECONFIG,
                 "lsb_radix_sort: bits_per_pass must be in [1,8]");
    crys::timing_begin(ctx);
    crys::sort_pairs(ctx, d_keys, d_payloads, n, algo, bits_per_pass);
    crys::timing_end(ctx);
  });
}

}  // extern "C"
