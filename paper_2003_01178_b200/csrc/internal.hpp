// internal.hpp -- host-side runtime objects behind the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace crys {

// ------------------------------------------------------------ device memory
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  // Grow-only reservation (contents not preserved).
  // 256 B of slack past `n` lets bulk copies round a column tail up to 16 B.
  void reserve(size_t n) {
    if (n <= bytes) return;
    release();
    CUDA_TRY(cudaMalloc(&p, n + 256));
    bytes = n;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void reserve(size_t n) {
    if (n <= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    CUDA_TRY(cudaMallocHost(&p, n));
    bytes = n;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// ------------------------------------------------------------ SSB plans
// Restatement of the reference's hand-built plans (ssb_plans.hpp:19-87,
// ssb_plans.cpp:21-275): this is the contract each fused kernel implements.
enum Dim { kSupplier = 0, kCustomer = 1, kPart = 2, kDate = 3 };
enum AggKind { kAggRevenue = 0, kAggExtPriceTimesDiscount = 1, kAggRevenueMinusSupplyCost = 2 };

struct RangeFilter {  // DimFilter (ssb_plans.hpp:39-48): union of inclusive ranges
  std::string column;
  std::vector<std::pair<int32_t, int32_t>> ranges;
};

struct FactFilter {  // FactFilter (ssb_plans.hpp:31-34), op lowered to [lo, hi]
  std::string column;
  int32_t lo, hi;
};

struct DimJoin {  // DimJoin (ssb_plans.hpp:50-56)
  Dim dim;
  std::string dim_table, dim_key, fact_key;
  std::vector<RangeFilter> filters;
  std::string payload;  // empty: no payload (0)
};

struct GroupPart {  // GroupPart (ssb_plans.hpp:60-67)
  int join_index;
  int32_t lo, hi;
  std::string label;
};

struct QueryPlan {  // QueryPlan (ssb_plans.hpp:78-85)
  int qid;
  std::string name;
  std::vector<FactFilter> fact_filters;
  std::vector<DimJoin> joins;
  std::vector<GroupPart> group;
  AggKind agg;
  int64_t cells() const {
    int64_t c = 1;
    for (auto& g : group) c *= (int64_t)(g.hi - g.lo + 1);
    return c;
  }
};

const QueryPlan& plan_for(int qid);  // ConfigError for an unknown id
std::string plan_json(int qid);
int dict_code(const std::string& dict, const std::string& value);

// Lowers PredicateSpec (tile.hpp:92-133) to an inclusive range.
void lower_pred(const crys_pred& p, int32_t* lo, int32_t* hi);

// ------------------------------------------------------------ runtime
struct QueryWorkspace;
struct SortWorkspace;
struct Group;
// Workspaces are complete only in their own .cu file.
struct WsDeleter {
  void operator()(QueryWorkspace* p) const;
  void operator()(SortWorkspace* p) const;
  void operator()(Group* p) const;
};

}  // namespace crys

struct crys_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double kernel_ms = 0, total_ms = 0;
  // generic scratch
  crys::DevBuf scratch, scratch2, status;
  crys::DevBuf part;  // radix-partitioned join probe: the probe pairs by hash bucket
  crys::PinnedBuf pinned;
  std::unique_ptr<crys::QueryWorkspace, crys::WsDeleter> qws;
  std::unique_ptr<crys::SortWorkspace, crys::WsDeleter> sws;
  crys_db* staging = nullptr;  // device copies for crys_run_query_host
  cudaStream_t copy_stream = nullptr;  // H2D of crys_db_upload_host (lazy)
  crys::PinnedBuf io[2];               // CRYS column file staging (double-buffered)
  cudaStream_t graph_stream = nullptr; // query graphs are captured/replayed here (lazy)
  cudaEvent_t graph_fence = nullptr;
  cudaEvent_t io_ev[2] = {nullptr, nullptr};
  // non-null: a device group (crys_init_group); this ctx then acts on the
  // root device and the members do the per-device work
  std::unique_ptr<crys::Group, crys::WsDeleter> group;
  ~crys_ctx();
};

struct crys_db {
  crys_ctx* ctx = nullptr;
  uint64_t uid = 0;  // unique for the process lifetime (graph / tuning cache keys)
  // a database on a device group: one complete database per shard (its
  // lineorder row range + replicated dimensions) on the shard's member ctx
  std::vector<crys_db*> shards;
  bool is_group() const { return !shards.empty(); }
  crys_db();
  int64_t sf = 0;
  uint64_t seed = 0;
  int64_t lo_begin = 0, lo_end = 0;  // shard of the full lineorder
  struct Col {
    std::unique_ptr<crys::DevBuf> buf;
    int64_t rows = 0;
    // value range (catalog statistics, kept for dimension columns): sizes the
    // exact key-range membership bitmaps of the SSB dimension builds
    bool stats = false;
    int32_t vmin = 0, vmax = -1;
    // asynchronous host upload (crys_db_upload_host): the copy stream records
    // `ready` after this column's H2D; consumers on the compute stream wait on
    // it per column, so a query starts as soon as ITS columns have landed
    mutable cudaEvent_t ready = nullptr;
    mutable bool pending = false;
  };
  std::map<std::string, Col> cols;  // "table.column"
  const int32_t* col(const std::string& table, const std::string& column, int64_t* rows) const;
  // false when the column carries no statistics
  bool col_range(const std::string& table, const std::string& column, int32_t* lo, int32_t* hi) const;
  int64_t table_rows(const std::string& table) const;
  ~crys_db();
};

struct crys_ht {
  crys_ctx* ctx = nullptr;
  crys::DevBuf slots;  // int2[capacity]
  int64_t capacity = 0;
  int32_t shift = 0;
  int64_t size = 0;
};

namespace crys {

// Contexts and device groups (capi.cpp, group.cpp).
crys_ctx* new_context(int device);
crys_ctx* new_group(int nshards, const int* devices);
int group_shards(const crys_ctx* ctx);
int group_devices(const crys_ctx* ctx);
bool group_nccl(const crys_ctx* ctx);
crys_ctx* group_member_of_shard(const crys_ctx* gctx, int shard);
bool shard_holds_dims(const crys_ctx* gctx, int shard);
void shard_range(int64_t lo, int64_t hi, int s, int S, int64_t* b, int64_t* e);
const char* nccl_status();

// Raise (never lower) a kernel's dynamic shared-memory limit; the attribute
// is per function, so one kernel shared by plans of different sizes must keep
// the largest value it has ever been launched with.  The attribute is also per
// device, so the bookkeeping is keyed by (current device, function).
void ensure_dyn_smem(const void* fn, size_t bytes);

// Launch accounting + event timing helpers.
inline void count_launch(crys_ctx* c, int n = 1) { c->launches += n; }

// CRYS_PDL=0 turns off the programmatic dependent launch of launch_k.
bool pdl_enabled();

// A kernel launch that may overlap its stream predecessor's tail (programmatic
// stream serialization): the kernel must pdl_wait() before it reads anything
// the predecessor wrote (common.cuh).  Captured into CUDA graphs as a
// programmatic edge.
template <typename... KArgs, typename... Args>
void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl_enabled() ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&lc, k, std::forward<Args>(args)...));
}
void timing_begin(crys_ctx* c);
void timing_kernel_begin(crys_ctx* c);
void timing_kernel_end(crys_ctx* c);
void timing_end(crys_ctx* c);  // synchronises and fills kernel_ms/total_ms when enabled

// Entry points implemented in the .cu files.
void ssb_generate(crys_ctx* ctx, crys_db* db);
void fill_uniform_i32(crys_ctx* ctx, int32_t* out, int64_t n, uint64_t seed, uint64_t stream,
                      int64_t index0, int32_t lo, int32_t hi);
void fill_float_pairs(crys_ctx* ctx, float* x1, float* x2, int64_t n, uint64_t seed, uint64_t stream,
                      float lo, float hi);
void ssb_query_partial(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt,
                       unsigned long long* d_agg, long long* d_hdr);
struct ResultRows {
  std::vector<int64_t> cell;
  std::vector<int64_t> sum;
  int64_t survivors[4] = {0, 0, 0, 0};
  int32_t err = 0;
};
void ssb_run_query(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt, ResultRows* out);
void ssb_finalize_device(crys_ctx* ctx, int qid, const unsigned long long* d_agg, const long long* d_hdr,
                         ResultRows* out);
void ssb_finalize_packed(crys_ctx* ctx, int qid, const crys_group_box& box, const long long* d_buf,
                         ResultRows* out);
// One device's packed partial over its fact shards (dimensions from facts[0]).
void ssb_partial_box(crys_ctx* ctx, const std::vector<const crys_db*>& facts, int qid, int bt, int ipt,
                     long long* d_out, int64_t cap, crys_group_box* box, int64_t* len, bool defer_tune);
void ssb_tune_done(crys_ctx* ctx);               // completes a deferred autotuning measurement
long long* ssb_group_buffer(crys_ctx* ctx, int64_t n);  // member workspace for the packed partial
void forget_db(crys_ctx* ctx, uint64_t uid);     // drop a freed database's graphs / tuning
void ssb_run_group(crys_ctx* gctx, const crys_db* gdb, int qid, int bt, int ipt, ResultRows* out);
void emit_rows(int qid, const std::vector<int64_t>& cell, const std::vector<int64_t>& sums,
               int32_t* h_groups, int64_t* h_sums, int64_t max_rows, int64_t* nrows);

double stream_read(crys_ctx* ctx, const void* d, size_t bytes, int reps);
void block_ops_run(crys_ctx* ctx, const int32_t* in, int64_t n, int bt, int ipt, int32_t lo, int32_t hi,
                   int32_t* out, int64_t* counts, int64_t* prefix, int64_t* totals, int64_t* aggs);
int64_t select_i32(crys_ctx* ctx, const int32_t* d_in, int64_t n, int32_t lo, int32_t hi,
                   int32_t* d_out, int order, int bt, int ipt);
void project_f32(crys_ctx* ctx, const float* x1, const float* x2, int64_t n, float a, float b,
                 float* out, int sigmoid);
void ht_build(crys_ctx* ctx, crys_ht* ht, const int32_t* d_keys, const int32_t* d_payloads,
              int64_t n);
int64_t join_probe_sum(crys_ctx* ctx, const int32_t* d_keys, const int32_t* d_payloads, int64_t n,
                       const crys_ht* ht);
void sort_pairs(crys_ctx* ctx, int32_t* d_keys, int32_t* d_payloads, int64_t n, int algo,
                int bits_per_pass);
void radix_owner_histogram(crys_ctx* ctx, const int32_t* d_keys, int64_t n, int start, int bits,
                           int64_t num_owners, int64_t* h_counts);
void radix_partition_pass(crys_ctx* ctx, const int32_t* sk, const int32_t* sp, int32_t* dk, int32_t* dp,
                          int64_t n, int start, int bits);

}  // namespace crys
