/*
 * crystal_b200.h -- the drop-in C ABI of the B200-native Crystal hot path.
 *
 * Plain C: raw pointers, sizes and status codes; no torch or C++ types.  One
 * shared library (paper_2003_01178_b200/libcrystal_b200.so) exports every
 * symbol below.  Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).
 *
 * Memory: "d_" pointers are DEVICE pointers owned by the caller; "h_"
 * pointers are host pointers.  Contexts, databases and hash tables are opaque
 * handles with explicit free.  All calls are synchronous with respect to the
 * host unless stated (they run on the context's stream and synchronise before
 * returning when a host-visible result is produced).
 *
 * Errors: no C++ exception crosses this boundary.  The reference throws
 * ConfigError / ContractError / BuildError / IoError (include/tq/common.hpp:16-34);
 * these map to CRYS_ECONFIG / CRYS_ECONTRACT / CRYS_EBUILD / CRYS_EIO.  The
 * message is available from crys_last_error().
 */
#ifndef CRYSTAL_B200_H
#define CRYSTAL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CRYS_OK = 0,
  CRYS_ECONFIG = 1,   /* tq::ConfigError   (common.hpp:17)  */
  CRYS_ECONTRACT = 2, /* tq::ContractError (common.hpp:22)  */
  CRYS_EBUILD = 3,    /* tq::BuildError    (common.hpp:27)  */
  CRYS_EIO = 4,       /* tq::IoError       (common.hpp:32)  */
  CRYS_ECUDA = 5,     /* CUDA runtime failure (no reference analogue) */
  CRYS_ENOTBUILT = 6, /* kernel shape not compiled for sm_100a */
  CRYS_ENCCL = 7      /* NCCL missing or failed (device groups, SURVEY 8(b) C ABI) */
} crys_status;

/* PredOp (tile.hpp:92): comparison against lo (or inclusive [lo,hi]). */
typedef enum { CRYS_LT = 0, CRYS_LE, CRYS_GT, CRYS_GE, CRYS_EQ, CRYS_BETWEEN } crys_pred_op;

typedef struct {
  int32_t op; /* crys_pred_op */
  int32_t lo;
  int32_t hi;
} crys_pred;

/* Output order of a selection (select.hpp:1-17):
 *   CRYS_ORDER_INPUT   = select_branching/predicated_into(workers=1): input order
 *   CRYS_ORDER_CRYSTAL = select_tile_into(kDeterministic): blocks in order, each
 *                        block thread-major over strided items (block_ops.hpp:98-122) */
typedef enum { CRYS_ORDER_INPUT = 0, CRYS_ORDER_CRYSTAL = 1 } crys_order;

typedef enum { CRYS_SORT_LSB = 0, CRYS_SORT_MSB = 1 } crys_sort_algo;

typedef struct crys_ctx crys_ctx;
typedef struct crys_db crys_db;
typedef struct crys_ht crys_ht;

/* ------------------------------------------------------------ context */

/* Thread-local message of the last failing call (any handle). */
const char* crys_last_error(void);
/* Library / build identification ("sm_100a ..."). */
const char* crys_version(void);
/* Visible CUDA devices (0 when there is no usable driver/device). */
int crys_device_count(void);

/* Bind to CUDA device `device`, create a stream and scratch.  Replaces the
 * per-call std::thread pool of parallel_for_blocks (kernel.cpp:60-103). */
crys_status crys_init(int device, crys_ctx** out);
void crys_destroy(crys_ctx* ctx);
/* A DEVICE GROUP: one host thread drives `nshards` lineorder row-range shards
 * placed on devices[0..nshards) (the reference's `workers`
 * fan-out, kernel.cpp:60-103, ssb_queries.cpp:265-266).  Every distinct device
 * gets a member context; the members share one NCCL communicator
 * (ncclCommInitAll, libnccl.so.2 loaded on first use) and each query ends in
 * ONE ncclReduce(int64, sum) of the members' packed partial aggregates to
 * devices[0], grouped with ncclGroupStart/End.  Several shards on one device
 * (devices[] repeating an ordinal: the emulation of an N-GPU box on fewer GPUs)
 * accumulate into that device's aggregate before the reduce.  Dimension tables
 * are replicated and built once per device.  ENCCL when NCCL cannot be loaded
 * and the group spans more than one device (a one-device group does not need
 * it; CRYS_GROUP_NCCL=1 forces the NCCL path anyway, =0 disables it).
 * Databases created on a group (crys_db_generate / crys_db_create +
 * crys_db_upload_host / crys_db_upload_column) are sharded; crys_run_query
 * on them runs the whole group.  Every other entry point treats a group
 * context as a context on devices[0]. */
crys_status crys_init_group(int nshards, const int* devices, crys_ctx** out);
/* Shards / distinct devices of a context (1 / 1 for crys_init). */
int crys_group_shards(const crys_ctx* ctx);
int crys_group_devices(const crys_ctx* ctx);
/* 1 when the group reduces through NCCL. */
int crys_group_uses_nccl(const crys_ctx* ctx);
/* "libnccl <version code>" once libnccl.so.2 loads (dlopen), else why not. */
const char* crys_nccl_version(void);

/* Run subsequent work on `cuda_stream` (a cudaStream_t; NULL = the ctx's own
 * stream).  The legacy default stream (handle 0, e.g. torch's default stream)
 * is CRYS_STREAM_LEGACY -- passing 0 would select the ctx's own non-blocking
 * stream, which does NOT order with work on the legacy stream. */
#define CRYS_STREAM_LEGACY ((void*)0x1) /* == cudaStreamLegacy */
crys_status crys_set_stream(crys_ctx* ctx, void* cuda_stream);
crys_status crys_synchronize(crys_ctx* ctx);
/* Number of kernels this ctx launched since creation (telemetry for bench). */
int64_t crys_kernel_launches(const crys_ctx* ctx);

/* Device memory for host code that has no CUDA headers (the C++ drop-in layer
 * under dropin/): allocations are 256 B aligned with 256 B of slack. Copies are
 * synchronous with respect to the host. */
crys_status crys_device_alloc(crys_ctx* ctx, size_t bytes, void** d_out);
void crys_device_free(crys_ctx* ctx, void* d_ptr);
crys_status crys_copy_to_device(crys_ctx* ctx, void* d_dst, const void* h_src, size_t bytes);
crys_status crys_copy_to_host(crys_ctx* ctx, void* h_dst, const void* d_src, size_t bytes);

/* ------------------------------------------------------------ database
 * An HBM-resident SSB database (columnar int32).  Lineorder may be a row-range
 * SHARD [lo_begin, lo_end) of the full fact table; dimensions are always whole
 * (replicated per GPU). Table names: "lineorder","date","supplier","customer",
 * "part"; column names as ssb_gen.cpp:60-157. */

/* Generate generate_ssb(sf, seed) (ssb_gen.cpp:243-270) directly in HBM,
 * bit-identical to the host generator; lineorder rows [lo_begin, lo_end) only
 * (lo_end < 0 means the whole table). */
crys_status crys_db_generate(crys_ctx* ctx, int64_t sf, uint64_t seed, int64_t lo_begin,
                             int64_t lo_end, crys_db** out);
/* Empty database; columns then come from crys_db_upload_column. */
crys_status crys_db_create(crys_ctx* ctx, int64_t sf, uint64_t seed, crys_db** out);
/* Copy one host column into HBM (replacing any previous one of that name). */
crys_status crys_db_upload_column(crys_db* db, const char* table, const char* column,
                                  const int32_t* h_data, int64_t rows);
typedef struct {
  const char* table;
  const char* column;
  const int32_t* h_data;
  int64_t rows;
} crys_host_column;
/* Asynchronous bulk upload of HOST columns (the reference's host-resident
 * `const SsbDatabase&`, ssb_gen.hpp): every copy is issued in array order on
 * the context's copy stream (pinned host memory makes it a true DMA), each
 * column gets a ready event, and work enqueued later on the compute stream
 * waits only for the columns it reads -- so a query suite overlaps its first
 * queries with the upload of the columns later queries need.  Dimension
 * statistics are computed on the host while the DMA runs.  The host arrays
 * must stay alive until the queries that read them have completed. */
crys_status crys_db_upload_host(crys_db* db, const crys_host_column* cols, int ncols);
/* One column from a file in the reference's CRYS format (column_io.hpp:3-13;
 * replaces load_column, column_io.cpp:65-100) straight into HBM: the payload
 * streams through double-buffered pinned staging on the copy stream and later
 * queries wait on the column's ready event.  int32 only; EIO on a missing
 * file, bad magic, unsupported version, float32 kind or short payload
 * (BadMagicError / KindMismatchError / TruncatedFileError, column_io.hpp:24-32). */
crys_status crys_db_load_column_file(crys_db* db, const char* table, const char* column, const char* path);
/* Writes a column in the CRYS format (replaces save_column, column_io.cpp:50-63). */
crys_status crys_db_save_column_file(const crys_db* db, const char* table, const char* column, const char* path);
/* Device pointer + rows of a column (borrowed; valid until the db is freed). */
crys_status crys_db_column(const crys_db* db, const char* table, const char* column,
                           const int32_t** d_data, int64_t* rows);
/* Rows of a column (a device-group database: lineorder summed over its
 * shards, a dimension as replicated). */
crys_status crys_db_column_rows(const crys_db* db, const char* table, const char* column, int64_t* rows);
/* Copy a column back to the host (h_out must hold `rows` values; a group's
 * lineorder comes back whole, shards in row order). */
crys_status crys_db_download_column(const crys_db* db, const char* table, const char* column,
                                    int32_t* h_out, int64_t rows);
void crys_db_free(crys_db* db);

/* Microbenchmark inputs generated in HBM, bit-identical to the reference CLI's
 * host generators: d_out[i] = Rng(seed, stream).uniform_i32(index0 + i, lo, hi)
 * (random_i32, tools/tq_main.cpp:147-152; rng.hpp:23-35).  Asynchronous. */
crys_status crys_fill_uniform_i32(crys_ctx* ctx, int32_t* d_out, int64_t n, uint64_t seed,
                                  uint64_t stream, int64_t index0, int32_t lo, int32_t hi);
/* d_x1[i] = uniform_float(2i, lo, hi), d_x2[i] = uniform_float(2i+1, lo, hi) of
 * Rng(seed, stream) (the project inputs, tools/tq_main.cpp:335-340). Asynchronous. */
crys_status crys_fill_float_pairs(crys_ctx* ctx, float* d_x1, float* d_x2, int64_t n, uint64_t seed,
                                  uint64_t stream, float lo, float hi);

/* ------------------------------------------------------------ SSB queries
 * qid: 0..12 = q11 q12 q13 q21 q22 q23 q31 q32 q33 q34 q41 q42 q43 (all_query_ids,
 * ssb_plans.cpp:301-306).  bt/ipt: TileConfig (tile.hpp:24-36). */

/* Number of dense aggregate cells (AggregateTable::cells, ssb_queries.cpp:17-27)
 * and group arity of qid. */
crys_status crys_query_shape(int qid, int64_t* cells, int32_t* ngroup, int32_t* njoins);

/* The query's plan (plan_for, ssb_plans.cpp:21-322) as JSON: fact filters,
 * ordered joins (dimension table / key / fact key / filters as inclusive
 * ranges / payload), group parts and the aggregate.  Writes at most cap bytes
 * (NUL-terminated); *len = the full length. */
crys_status crys_query_plan_json(int qid, char* out, size_t cap, size_t* len);

/* Replaces tq::run_query(db, id, config, workers, stats) (ssb_queries.hpp:76-78,
 * ssb_queries.cpp:277-286) on one GPU: dimension hash builds, one fused
 * lineorder pass, group compaction.  Rows come back lexicographically ordered
 * (grouped_result, ssb_queries.cpp:145-155): groups row-major [max_rows][3]
 * (ngroup used), sums [max_rows].  survivors[4] = QueryStats.survivors
 * (ssb_queries.hpp:70-74).  ECONTRACT (with *nrows set) if max_rows is short. */
crys_status crys_run_query(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt,
                           int32_t* h_groups, int64_t* h_sums, int64_t max_rows,
                           int64_t* nrows, int64_t* h_survivors);

/* End-to-end variant over HOST columns (the reference's `const SsbDatabase&`):
 * the query's referenced columns are copied H2D inside the call, then as
 * crys_run_query.  Tables are described by parallel arrays of names/pointers. */
crys_status crys_run_query_host(crys_ctx* ctx, const crys_host_column* cols, int ncols, int qid,
                                int bt, int ipt, int32_t* h_groups, int64_t* h_sums,
                                int64_t max_rows, int64_t* nrows, int64_t* h_survivors);

/* Multi-GPU building blocks (lineorder row-range shards), dense
 * form: the shard's partial aggregate ADDS into d_agg = int64[2*cells] laid
 * out as [sums | counts], and its survivors and error words add into d_hdr =
 * int64[CRYS_PARTIAL_HEADER] (layout below) -- both caller-zeroed, so several
 * shards can accumulate into one buffer.  Asynchronous on the ctx stream. */
crys_status crys_query_partial(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt,
                               int64_t* d_agg, int64_t* d_hdr);
/* The packed partial (the payload of the ONE collective per query): the
 * dense sub-box of the group-by domain the query can occupy, computed on the
 * device from the dimension builds (identical on every shard because the
 * dimensions are replicated).  Layout, int64:
 *   [0..3]    survivors per join (QueryStats.survivors)
 *   [4]       shards whose rows hit a group value outside its domain
 *             (ContractError, ssb_queries.cpp:32-33)
 *   [8+4j+c-1] shards whose build of join j failed with code c: 1 sentinel
 *             key, 2 duplicate key, 3 capacity (BuildError,
 *             hash_table.cpp:51-93), 4 key outside the column statistics
 *   [32 .. 32+cells)          sums of the box cells
 *   [32+cells .. 32+2*cells)  occupancy counts
 * Element-wise SUM over shards is the merge (AggregateTable::merge,
 * ssb_queries.cpp:38-47). */
#define CRYS_PARTIAL_HEADER 32
typedef struct {
  int32_t nparts;  /* group parts of the plan (0..3) */
  int32_t lo[3];   /* first group VALUE of the box per part */
  int32_t card[3]; /* extent per part */
  int32_t pad;
  int64_t cells;   /* product of card (1 for flight 1; 0: nothing can match) */
} crys_group_box;
/* Enqueue the shard's query and pack its partial into d_buf (capacity
 * `cap` int64); *len = CRYS_PARTIAL_HEADER + 2*box->cells.  Returns once the
 * dimension builds have fixed the box (the fused pass is still running on
 * the ctx stream), so the caller can size the collective right away. */
crys_status crys_query_partial_box(crys_ctx* ctx, const crys_db* db, int qid, int bt, int ipt,
                                   int64_t* d_buf, int64_t cap, int64_t* len, crys_group_box* box);
/* Rows of a (reduced) packed partial; raises the errors its header carries. */
crys_status crys_query_finalize_box(crys_ctx* ctx, int qid, const crys_group_box* box,
                                    const int64_t* d_buf, int32_t* h_groups, int64_t* h_sums,
                                    int64_t max_rows, int64_t* nrows, int64_t* h_survivors);

/* Compact a (reduced) dense aggregate [sums | counts] on the device into
 * result rows; d_hdr (nullable) is the matching reduced header: its survivors
 * go to h_survivors[4] (nullable) and its error words raise EBUILD /
 * ECONTRACT exactly as crys_run_query does. */
crys_status crys_query_finalize(crys_ctx* ctx, int qid, const int64_t* d_agg, const int64_t* d_hdr,
                                int32_t* h_groups, int64_t* h_sums, int64_t max_rows,
                                int64_t* nrows, int64_t* h_survivors);
/* Same compaction on the host (pure CPU; no device needed). */
crys_status crys_query_finalize_host(int qid, const int64_t* h_agg, const int64_t* h_hdr,
                                     int32_t* h_groups, int64_t* h_sums, int64_t max_rows,
                                     int64_t* nrows, int64_t* h_survivors);

/* ------------------------------------------------------------ operators */

/* Replaces select_{branching,predicated}_into(workers=1) (order INPUT) and
 * select_tile_into(config, kDeterministic) (order CRYSTAL), select.hpp:56-135.
 * d_out must hold n values; *count = matches. */
crys_status crys_select_i32(crys_ctx* ctx, const int32_t* d_in, int64_t n, crys_pred pred,
                            int32_t* d_out, int64_t* count, int order, int bt, int ipt);

/* Replaces project_linear_into / project_sigmoid_into (project.hpp:49-64). */
crys_status crys_project_f32(crys_ctx* ctx, const float* d_x1, const float* d_x2, int64_t n,
                             float a, float b, float* d_out, int sigmoid, int bt, int ipt);

/* Replaces HashTable::build (hash_table.hpp:29-30, hash_table.cpp:20-94):
 * capacity a power of two >= 2 (ECONFIG), n*2 <= capacity, no INT32_MIN or
 * duplicate keys (EBUILD).  Slots are interleaved {key, payload} int2. */
crys_status crys_ht_build(crys_ctx* ctx, const int32_t* d_keys, const int32_t* d_payloads,
                          int64_t n, int64_t capacity, crys_ht** out);
/* Slot arrays back to the host (for layout checks): capacity keys/payloads. */
crys_status crys_ht_download(const crys_ht* ht, int32_t* h_keys, int32_t* h_payloads);
int64_t crys_ht_capacity(const crys_ht* ht);
void crys_ht_free(crys_ht* ht);

/* A device table from existing slot arrays (a host-built tq::HashTable, whose
 * slot_keys()/slot_payloads() are exposed at hash_table.hpp:53-54): capacity
 * a power of two >= 2, empty slots hold INT32_MIN. */
crys_status crys_ht_upload(crys_ctx* ctx, const int32_t* h_keys, const int32_t* h_payloads,
                           int64_t capacity, crys_ht** out);

/* Replaces join_probe_{scalar,prefetch,tile} (join.hpp:17-32, join.cpp:53-96):
 * *checksum = sum over hits of (build payload + probe payload), int64. */
crys_status crys_join_probe_sum(crys_ctx* ctx, const int32_t* d_keys, const int32_t* d_payloads,
                                int64_t n, const crys_ht* ht, int bt, int ipt, int64_t* checksum);

/* Replaces lsb_radix_sort / msb_radix_sort (radix.hpp:90-93, radix.cpp:138-216),
 * in place on device key/payload arrays.  LSB: stable, bits_per_pass in [1,8]
 * (== std::stable_sort by key).  MSB: keys ascending, pairs preserved. */
crys_status crys_sort_pairs(crys_ctx* ctx, int32_t* d_keys, int32_t* d_payloads, int64_t n,
                            int algo, int bits_per_pass);

/* Replaces radix_histogram (radix.hpp:77-78, radix.cpp:33-53): h_counts =
 * int64[num_owners][2^num_bits], owner o = input chunk [o*chunk, (o+1)*chunk),
 * chunk = max(1, ceil(n / num_owners)); digit = radix_digit (radix.hpp:44-47). */
crys_status crys_radix_histogram(crys_ctx* ctx, const int32_t* d_keys, int64_t n, int start_bit,
                                 int num_bits, int64_t num_owners, int64_t* h_counts);
/* Replaces radix_shuffle with a stable pass (radix.hpp:80-83, radix.cpp:75-136):
 * d_out_* = the input stably partitioned by digit (what per-owner cursors over
 * column-major offsets produce for ANY owner count).  Out-of-place. */
crys_status crys_radix_partition(crys_ctx* ctx, const int32_t* d_keys, const int32_t* d_payloads,
                                 int64_t n, int start_bit, int num_bits, int32_t* d_out_keys,
                                 int32_t* d_out_payloads);

/* The Crystal device primitives (PAPER Table 1; block_ops.hpp:23-173), one
 * logical tile of bt*ipt slots per CTA with the reference's striped ownership
 * (slot t + k*bt): BlockLoad -> BlockPred(pred) -> per-thread counts ->
 * BlockScan -> BlockShuffle -> BlockStore, plus BlockAggregate.  Per tile b:
 * d_out[b*bt*ipt ..) = the compacted tile (thread-major, block_shuffle order),
 * d_counts / d_prefix[b*bt + t] = block_thread_counts / block_scan prefix,
 * d_totals[b] = matches, d_aggs[b*8 + 0..3] = SUM, COUNT, MIN, MAX over the
 * matches and [4..7] over all valid slots (identities 0, 0, INT32_MAX,
 * INT32_MIN on empty input).  1 <= bt <= 1024, 1 <= ipt <= 16.  Synchronous. */
crys_status crys_block_ops_run(crys_ctx* ctx, const int32_t* d_in, int64_t n, int bt, int ipt,
                               crys_pred pred, int32_t* d_out, int64_t* d_counts, int64_t* d_prefix,
                               int64_t* d_totals, int64_t* d_aggs);

/* Read-only HBM bandwidth of this device, measured: a 128-bit streaming read
 * of [d_buf, d_buf + bytes) (use >> L2, e.g. 4 GB), best of `reps`, in GB/s.
 * The fused query kernels only read; this is the read-side reference beside
 * the copy bandwidth of MEASURED_PEAKS.json. */
crys_status crys_stream_read_gbs(crys_ctx* ctx, const void* d_buf, size_t bytes, int reps, double* gbs);

/* ------------------------------------------------------------ timing hooks
 * Device-timed (CUDA events on the ctx stream) duration of the last call's
 * dominant kernel (the fused lineorder pass / select / probe / sort passes)
 * and of the whole call, in milliseconds. */
crys_status crys_last_timing(const crys_ctx* ctx, double* kernel_ms, double* total_ms);
/* Enable per-call event timing (adds two event records per call). */
crys_status crys_enable_timing(crys_ctx* ctx, int enable);

#ifdef __cplusplus
}
#endif
#endif /* CRYSTAL_B200_H */
