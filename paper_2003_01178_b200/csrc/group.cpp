// group.cpp -- device groups: ONE host thread drives every lineorder shard of
// an SSB database over the distinct devices of the group, and each query ends
// in ONE NCCL reduce of the members' packed partial aggregates (SURVEY 8(b)
// "Threading" and 8(e); the reference's workers fan-out + merge,
// kernel.cpp:60-103 and ssb_queries.cpp:265-266).
//
//   per member device m (stream-ordered, graph-replayed per query):
//     prologue + dimension builds (once per device, from its first shard)
//     box_publish_kernel   -> host learns the payload size right away
//     fused lineorder pass  x (shards placed on m; they ADD into one aggregate)
//     pack_partial_kernel  -> [header | box sums | box counts]
//   host: ncclGroupStart; ncclReduce(int64, sum, root 0) per member; ncclGroupEnd
//   root: finalize over the reduced box -> rows, survivors, errors
//
// libnccl.so.2 is resolved with dlopen on first use (the process may already
// hold torch's copy; loading a second, different NCCL next to it would
// clash), so single-device users never need NCCL at all.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.hpp"

namespace crys {

namespace {

struct NcclApi {
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  std::string why;  // empty: loaded
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // 1. an explicit library (the Python package points this at the NCCL
    //    torch ships, so torch and this library share ONE libnccl);
    // 2. a libnccl.so.2 the process already holds;  3. the system one
    void* h = nullptr;
    if (const char* path = getenv("CRYS_NCCL_LIBRARY")) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p && api.why.empty()) api.why = std::string("libnccl.so.2 lacks ") + n;
      return p;
    };
    api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(sym("ncclCommInitAll"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.reduce = reinterpret_cast<decltype(api.reduce)>(sym("ncclReduce"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(sym("ncclGetVersion"));
  });
  return api;
}

void nccl_try(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(CRYS_ENCCL, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "error"));
}

}  // namespace

struct Group {
  std::vector<crys_ctx*> members;  // one per distinct device, owned
  std::vector<int> shard_member;   // member index of every shard
  std::vector<ncclComm_t> comms;   // one per member when the group reduces through NCCL
  std::vector<cudaEvent_t> fence;  // per member: orders it after the caller's stream
  ~Group() {
    for (ncclComm_t c : comms)
      if (c && nccl().comm_destroy) nccl().comm_destroy(c);
    for (size_t m = 0; m < members.size(); ++m) {
      if (m < fence.size() && fence[m]) {
        cudaSetDevice(members[m]->device);
        cudaEventDestroy(fence[m]);
      }
      crys_destroy(members[m]);
    }
  }
};

void WsDeleter::operator()(Group* p) const { delete p; }

crys_ctx* new_group(int nshards, const int* devices) {
  CRYS_CHECK(nshards >= 1 && devices, CRYS_ECONFIG, "device group: need at least one shard");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  std::vector<int> devs;  // distinct devices in first-use order; devs[0] is the root
  std::vector<int> shard_member((size_t)nshards);
  for (int s = 0; s < nshards; ++s) {
    CRYS_CHECK(devices[s] >= 0 && devices[s] < ndev, CRYS_ECONFIG, "device group: no such CUDA device");
    auto it = std::find(devs.begin(), devs.end(), devices[s]);
    if (it == devs.end()) {
      devs.push_back(devices[s]);
      it = devs.end() - 1;
    }
    shard_member[(size_t)s] = (int)(it - devs.begin());
  }
  crys_ctx* g = new_context(devs[0]);
  try {
    g->group.reset(new Group());
    Group& G = *g->group;
    G.shard_member = shard_member;
    for (int d : devs) G.members.push_back(new_context(d));
    for (crys_ctx* m : G.members) {
      CUDA_TRY(cudaSetDevice(m->device));
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      G.fence.push_back(e);
    }
    // NCCL: required across devices; a one-device group reduces in place
    const char* env = getenv("CRYS_GROUP_NCCL");
    const int want = env ? atoi(env) : -1;  // -1 auto
    bool use = devs.size() > 1 ? want != 0 : want == 1;
    if (devs.size() > 1 && want == 0)
      fail(CRYS_ECONFIG, "device group over several devices needs NCCL (CRYS_GROUP_NCCL=0)");
    if (use) {
      const NcclApi& api = nccl();
      if (!api.why.empty()) fail(CRYS_ENCCL, api.why);
      G.comms.assign(devs.size(), nullptr);
      nccl_try(api.comm_init_all(G.comms.data(), (int)devs.size(), devs.data()), "ncclCommInitAll");
    }
    CUDA_TRY(cudaSetDevice(devs[0]));
  } catch (...) {
    crys_destroy(g);
    throw;
  }
  return g;
}

int group_shards(const crys_ctx* ctx) { return ctx->group ? (int)ctx->group->shard_member.size() : 1; }
int group_devices(const crys_ctx* ctx) { return ctx->group ? (int)ctx->group->members.size() : 1; }
bool group_nccl(const crys_ctx* ctx) { return ctx->group && !ctx->group->comms.empty(); }

crys_ctx* group_member_of_shard(const crys_ctx* gctx, int shard) {
  const Group& G = *gctx->group;
  return G.members[(size_t)G.shard_member[(size_t)shard]];
}

// Row range of shard s of S over [lo, hi): contiguous, covering, sizes differ
// by at most one (dist.shard_range).
void shard_range(int64_t lo, int64_t hi, int s, int S, int64_t* b, int64_t* e) {
  const int64_t n = hi - lo;
  *b = lo + (n * s) / S;
  *e = lo + (n * (s + 1)) / S;
}

bool shard_holds_dims(const crys_ctx* gctx, int shard) {
  const Group& G = *gctx->group;
  for (int s = 0; s < shard; ++s)
    if (G.shard_member[(size_t)s] == G.shard_member[(size_t)shard]) return false;
  return true;  // the first shard of its member builds that device's dimension tables
}

void ssb_run_group(crys_ctx* gctx, const crys_db* gdb, int qid, int bt, int ipt, ResultRows* out) {
  Group& G = *gctx->group;
  const QueryPlan& plan = plan_for(qid);
  const size_t M = G.members.size();
  std::vector<std::vector<const crys_db*>> facts(M);
  for (size_t s = 0; s < gdb->shards.size(); ++s) facts[(size_t)G.shard_member[s]].push_back(gdb->shards[s]);
  const int64_t cap = CRYS_PARTIAL_HEADER + 2 * plan.cells();
  // every member orders after the caller's earlier work on the group stream
  CUDA_TRY(cudaSetDevice(gctx->device));
  CUDA_TRY(cudaEventRecord(G.fence[0], gctx->stream));
  for (size_t m = 0; m < M; ++m) {
    CUDA_TRY(cudaSetDevice(G.members[m]->device));
    CUDA_TRY(cudaStreamWaitEvent(G.members[m]->stream, G.fence[0], 0));
  }
  crys_ctx* root = G.members[0];
  const bool timing = gctx->timing;
  root->timing = timing;
  std::vector<long long*> buf(M);
  std::vector<crys_group_box> box(M);
  std::vector<int64_t> len(M);
  for (size_t m = 0; m < M; ++m) {
    crys_ctx* mc = G.members[m];
    CUDA_TRY(cudaSetDevice(mc->device));
    buf[m] = ssb_group_buffer(mc, cap);
    ssb_partial_box(mc, facts[m], qid, bt, ipt, buf[m], cap, &box[m], &len[m], true);
  }
  for (size_t m = 1; m < M; ++m)  // the replicated dimensions must agree
    CRYS_CHECK(len[m] == len[0] && std::memcmp(&box[m], &box[0], sizeof(crys_group_box)) == 0, CRYS_ECONTRACT,
               "device group: dimension replicas disagree (group box differs across devices)");
  if (!G.comms.empty()) {  // ONE collective per query: SUM of the packed partials into the root
    const NcclApi& api = nccl();
    nccl_try(api.group_start(), "ncclGroupStart");
    ncclResult_t r = ncclSuccess;
    for (size_t m = 0; m < M && r == ncclSuccess; ++m)
      r = api.reduce(buf[m], buf[m], (size_t)len[0], ncclInt64, ncclSum, 0, G.comms[m], G.members[m]->stream);
    nccl_try(api.group_end(), "ncclGroupEnd");
    nccl_try(r, "ncclReduce");
  }
  CUDA_TRY(cudaSetDevice(root->device));
  ssb_finalize_packed(root, qid, box[0], buf[0], out);  // synchronises the root stream
  if (timing) {
    timing_end(root);
    gctx->kernel_ms = root->kernel_ms;
    gctx->total_ms = root->total_ms;
  }
  root->timing = false;
  for (size_t m = 0; m < M; ++m) {
    CUDA_TRY(cudaSetDevice(G.members[m]->device));
    CUDA_TRY(cudaStreamSynchronize(G.members[m]->stream));
    ssb_tune_done(G.members[m]);
  }
  CUDA_TRY(cudaSetDevice(gctx->device));
  // the group stream orders after the result (and the caller's stream after it)
  CUDA_TRY(cudaEventRecord(G.fence[0], root->stream));
  CUDA_TRY(cudaStreamWaitEvent(gctx->stream, G.fence[0], 0));
}

const char* nccl_status() {
  static std::string s;
  const NcclApi& api = nccl();
  if (!api.why.empty()) return api.why.c_str();
  int v = 0;
  if (api.get_version) api.get_version(&v);
  s = "libnccl " + std::to_string(v);
  return s.c_str();
}

}  // namespace crys
