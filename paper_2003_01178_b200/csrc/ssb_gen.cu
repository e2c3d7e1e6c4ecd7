// ssb_gen.cu -- bit-exact SSB generator running in HBM.
//
// The reference generator (ssb_gen.cpp:54-157) draws every value from a
// counter-based SplitMix64 stream Rng(seed, sf, table, column).at(index)
// (rng.hpp:16-45), i.e. a pure function of (stream, row).  That lets each GPU
// generate exactly its lineorder row range [lo_begin, lo_end) in parallel with
// no host involvement and no H2D traffic; dimensions are generated whole
// (replicated per GPU).
#include <vector>

#include "internal.hpp"

namespace crys {
namespace {

enum TableId : uint64_t { kTLineorder = 1, kTDate, kTSupplier, kTCustomer, kTPart };  // ssb_gen.cpp:11

__host__ __device__ inline uint64_t mix64(uint64_t x) {  // rng.hpp:16-21
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t rng_base(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {  // rng.hpp:25-27
  return mix64(mix64(mix64(seed) ^ a) ^ b) ^ mix64(c);
}

// uniform_i32 (rng.hpp:31-34): lo + (at(index) % range), range = hi - lo + 1.
__device__ __forceinline__ int32_t uniform_i32(uint64_t base, uint64_t index, int32_t lo,
                                               uint64_t range) {
  return (int32_t)((int64_t)lo + (int64_t)(mix64(base + index) % range));
}

__global__ void gen_uniform_kernel(int32_t* __restrict__ out, int64_t begin, int64_t n,
                                   uint64_t base, int32_t lo, uint64_t range,
                                   const int32_t* __restrict__ lut) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = uniform_i32(base, (uint64_t)(begin + i), lo, range);
    out[i] = lut ? __ldg(lut + v) : v;
  }
}

// make_geo_table (ssb_gen.cpp:94-112): key, city, nation = city/10, region = nation/5.
__global__ void gen_geo_kernel(int32_t* key, int32_t* city, int32_t* nation, int32_t* region,
                               int64_t rows, uint64_t base) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = uniform_i32(base, (uint64_t)i, 0, 250);
    key[i] = (int32_t)(i + 1);
    city[i] = c;
    nation[i] = c / 10;
    region[i] = c / 10 / 5;
  }
}

// make_part_table (ssb_gen.cpp:114-129): key, brand1, category = brand/40, mfgr = category/5.
__global__ void gen_part_kernel(int32_t* key, int32_t* brand, int32_t* cat, int32_t* mfgr,
                                int64_t rows, uint64_t base) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = uniform_i32(base, (uint64_t)i, 0, 1000);
    key[i] = (int32_t)(i + 1);
    brand[i] = b;
    cat[i] = b / 40;
    mfgr[i] = b / 40 / 5;
  }
}

// uniform_float (rng.hpp:37-40): x1[i] = at(2i), x2[i] = at(2i+1) of one stream
// (the project microbenchmark inputs, tools/tq_main.cpp:335-340).
__global__ void gen_float_pairs_kernel(float* __restrict__ x1, float* __restrict__ x2, int64_t n,
                                       uint64_t base, float lo, float hi) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double u1 = (double)(mix64(base + (uint64_t)(2 * i)) >> 11) * 0x1.0p-53;
    const double u2 = (double)(mix64(base + (uint64_t)(2 * i + 1)) >> 11) * 0x1.0p-53;
    x1[i] = (float)((double)lo + u1 * ((double)hi - (double)lo));
    x2[i] = (float)((double)lo + u2 * ((double)hi - (double)lo));
  }
}

bool is_leap(int y) { return y % 4 == 0 && (y % 100 != 0 || y % 400 == 0); }

// make_date_table (ssb_gen.cpp:60-90): a 2556-day calendar from 1992-01-01.
void date_columns(std::vector<int32_t> (&c)[5]) {
  static const int kDays[12] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  int y = 1992, m = 1, d = 1, doy = 1;
  for (int i = 0; i < 2556; ++i) {
    c[0].push_back(y * 10000 + m * 100 + d);
    c[1].push_back(y);
    c[2].push_back(y * 100 + m);
    c[3].push_back((y - 1992) * 12 + (m - 1));
    c[4].push_back((doy - 1) / 7 + 1);
    ++d;
    ++doy;
    const int dim = (m == 2 && is_leap(y)) ? 29 : kDays[m - 1];
    if (d > dim) {
      d = 1;
      if (++m > 12) {
        m = 1;
        ++y;
        doy = 1;
      }
    }
  }
}

int32_t* new_col(crys_db* db, const std::string& table, const std::string& col, int64_t rows,
                 int32_t vmin = 0, int32_t vmax = -1) {
  auto& c = db->cols[table + "." + col];
  c.buf.reset(new DevBuf());
  c.buf->reserve(sizeof(int32_t) * (size_t)std::max<int64_t>(rows, 1));
  c.rows = rows;
  c.stats = vmin <= vmax;  // value ranges are closed forms of the generator
  c.vmin = vmin;
  c.vmax = vmax;
  return c.buf->as<int32_t>();
}

int grid_for(crys_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16));
}

}  // namespace

// random_i32 of the reference CLI (tools/tq_main.cpp:147-152):
// out[i] = Rng(seed, stream).uniform_i32(index0 + i, lo, hi).
void fill_uniform_i32(crys_ctx* ctx, int32_t* out, int64_t n, uint64_t seed, uint64_t stream,
                      int64_t index0, int32_t lo, int32_t hi) {
  CRYS_CHECK(n >= 0 && index0 >= 0, CRYS_ECONFIG, "bad length");
  CRYS_CHECK(lo <= hi, CRYS_ECONFIG, "uniform_i32 requires lo <= hi");
  if (n == 0) return;
  const uint64_t range = (uint64_t)((int64_t)hi - (int64_t)lo + 1);
  gen_uniform_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(out, index0, n, rng_base(seed, stream, 0, 0),
                                                                lo, range, nullptr);
  CRYS_LAUNCHED("gen_uniform_kernel");
  count_launch(ctx);
}

void fill_float_pairs(crys_ctx* ctx, float* x1, float* x2, int64_t n, uint64_t seed, uint64_t stream,
                      float lo, float hi) {
  CRYS_CHECK(n >= 0, CRYS_ECONFIG, "bad length");
  if (n == 0) return;
  gen_float_pairs_kernel<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(x1, x2, n, rng_base(seed, stream, 0, 0),
                                                                    lo, hi);
  CRYS_LAUNCHED("gen_float_pairs_kernel");
  count_launch(ctx);
}

void ssb_generate(crys_ctx* ctx, crys_db* db) {
  const int64_t sf = db->sf;
  const uint64_t seed = db->seed;
  CRYS_CHECK(sf >= 1, CRYS_ECONFIG, "scale factor must be >= 1");
  cudaStream_t st = ctx->stream;
  // cardinalities, ssb_gen.cpp:179-186
  const int64_t lo_rows = 6000000LL * sf, supp = 2000LL * sf, cust = 30000LL * sf;
  int bw = 0;
  for (uint64_t v = (uint64_t)sf; v; v >>= 1) ++bw;
  const int64_t part = 200000LL * bw;
  if (db->lo_end < 0 || db->lo_end > lo_rows) db->lo_end = lo_rows;
  CRYS_CHECK(db->lo_begin >= 0 && db->lo_begin <= db->lo_end, CRYS_ECONFIG, "bad lineorder shard range");

  std::vector<int32_t> date[5];
  date_columns(date);
  static const char* kDateCols[5] = {"d_datekey", "d_year", "d_yearmonthnum", "d_yearmonth",
                                     "d_weeknuminyear"};
  for (int i = 0; i < 5; ++i) {
    int32_t* d = i == 0 ? new_col(db, "date", kDateCols[i], 2556, date[0].front(), date[0].back())
                        : new_col(db, "date", kDateCols[i], 2556);
    CUDA_TRY(cudaMemcpyAsync(d, date[i].data(), sizeof(int32_t) * 2556, cudaMemcpyHostToDevice, st));
  }
  int32_t* s[4] = {new_col(db, "supplier", "s_suppkey", supp, 1, (int32_t)supp), new_col(db, "supplier", "s_city", supp),
                   new_col(db, "supplier", "s_nation", supp), new_col(db, "supplier", "s_region", supp)};
  gen_geo_kernel<<<grid_for(ctx, supp), 256, 0, st>>>(s[0], s[1], s[2], s[3], supp,
                                                       rng_base(seed, (uint64_t)sf, kTSupplier, 0));
  int32_t* c[4] = {new_col(db, "customer", "c_custkey", cust, 1, (int32_t)cust), new_col(db, "customer", "c_city", cust),
                   new_col(db, "customer", "c_nation", cust), new_col(db, "customer", "c_region", cust)};
  gen_geo_kernel<<<grid_for(ctx, cust), 256, 0, st>>>(c[0], c[1], c[2], c[3], cust,
                                                       rng_base(seed, (uint64_t)sf, kTCustomer, 0));
  int32_t* p[4] = {new_col(db, "part", "p_partkey", part, 1, (int32_t)part), new_col(db, "part", "p_brand1", part),
                   new_col(db, "part", "p_category", part), new_col(db, "part", "p_mfgr", part)};
  gen_part_kernel<<<grid_for(ctx, part), 256, 0, st>>>(p[0], p[1], p[2], p[3], part,
                                                        rng_base(seed, (uint64_t)sf, kTPart, 0));
  count_launch(ctx, 3);

  // make_lineorder_table (ssb_gen.cpp:131-157)
  struct ColSpec {
    const char* name;
    int32_t lo;
    int64_t hi;
  };
  const ColSpec specs[9] = {{"lo_orderdate", 0, 2555},   {"lo_custkey", 1, cust},
                            {"lo_suppkey", 1, supp},     {"lo_partkey", 1, part},
                            {"lo_quantity", 1, 50},      {"lo_discount", 0, 10},
                            {"lo_extendedprice", 1, 100000}, {"lo_revenue", 1, 1000000},
                            {"lo_supplycost", 1, 100000}};
  const int64_t n = db->lo_end - db->lo_begin;
  const int32_t* datekeys = db->col("date", "d_datekey", nullptr);
  for (int cid = 0; cid < 9; ++cid) {
    int32_t* out = new_col(db, "lineorder", specs[cid].name, n);
    if (n == 0) continue;
    const uint64_t range = (uint64_t)(specs[cid].hi - specs[cid].lo + 1);
    gen_uniform_kernel<<<grid_for(ctx, n), 256, 0, st>>>(
        out, db->lo_begin, n, rng_base(seed, (uint64_t)sf, kTLineorder, (uint64_t)cid), specs[cid].lo,
        range, cid == 0 ? datekeys : nullptr);
    count_launch(ctx);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(st));
}

}  // namespace crys
