// dist.cu — multi-GPU SpMM over NCCL (north_star / SURVEY.md §8e): the path
// is partitioned by destination rows; the one real exchange is the source
// features, which every rank holds in equal row shards.
//
//   exact   (chunks = 0): one ncclAllGather of the shards into a full X, then
//           one gm_spmm over the rank's rows (bit-identical to one GPU);
//   blocked (chunks = G): G ncclAllGathers of shard row chunks are issued on
//           comm_stream; block 0 (sources in the rank's own shard) aggregates
//           on `stream` meanwhile; block 1+c continues the rows as soon as
//           chunk c has landed (cudaStreamWaitEvent, no host sync);
//   halo:   ncclSend / ncclRecv of only the referenced remote rows (packed
//           per peer by gm_gather_rows) inside one NCCL group, the own-shard
//           block overlapping it.
// NCCL is resolved at run time (dlopen of libnccl.so.2; a process that already
// loaded NCCL, e.g. through torch, shares that copy), so single-GPU users of
// the library never load it.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "gm_common.cuh"
#include <nccl.h>

namespace gm {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) api.why += std::string(" missing ") + name;
    };
    sym(api.get_unique_id, "ncclGetUniqueId");
    sym(api.comm_init_rank, "ncclCommInitRank");
    sym(api.comm_destroy, "ncclCommDestroy");
    sym(api.all_gather, "ncclAllGather");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.group_start, "ncclGroupStart");
    sym(api.group_end, "ncclGroupEnd");
    sym(api.error_string, "ncclGetErrorString");
    api.ok = api.why.empty();
  });
  return api;
}

gm_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return GM_OK;
  return fail(GM_ERR_NCCL, std::string(what) + ": " + nccl().error_string(r));
}

#define GM_TRY_NCCL(expr)                                       \
  do {                                                          \
    ncclResult_t gm_r_ = (expr);                                \
    if (gm_r_ != ncclSuccess) return nccl_status(gm_r_, #expr); \
  } while (0)

// Per host thread: events that gate the blocks on their exchange chunks.
struct DistEvents {
  std::vector<cudaEvent_t> ev;
  int device = -1;
};
thread_local DistEvents t_events;

gm_status events(int n, cudaEvent_t** out) {
  int dev = 0;
  GM_TRY_CUDA(cudaGetDevice(&dev));
  if (t_events.device != dev) {
    t_events.ev.clear();  // events of another device are not reusable here
    t_events.device = dev;
  }
  while (static_cast<int>(t_events.ev.size()) < n) {
    cudaEvent_t e;
    GM_TRY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    t_events.ev.push_back(e);
  }
  *out = t_events.ev.data();
  return GM_OK;
}

size_t esize(gm_dtype d) { return d == GM_F64 ? 8 : d == GM_F32 ? 4 : 2; }

}  // namespace
}  // namespace gm

using namespace gm;

extern "C" {

GM_API gm_status gm_nccl_unique_id(void* id_out) {
  GM_REQUIRE(id_out, GM_ERR_INVALID_ARGUMENT, "gm_nccl_unique_id: null output");
  GM_REQUIRE(nccl().ok, GM_ERR_NCCL, "gm_nccl_unique_id: " + nccl().why);
  ncclUniqueId id;
  GM_TRY_NCCL(nccl().get_unique_id(&id));
  memcpy(id_out, &id, sizeof(id));
  return GM_OK;
}

GM_API gm_status gm_nccl_comm_init(int32_t world, const void* id, int32_t rank, ncclComm_t* comm) {
  GM_REQUIRE(id && comm && world >= 1 && rank >= 0 && rank < world, GM_ERR_INVALID_ARGUMENT,
             "gm_nccl_comm_init: bad arguments");
  GM_REQUIRE(nccl().ok, GM_ERR_NCCL, "gm_nccl_comm_init: " + nccl().why);
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  GM_TRY_NCCL(nccl().comm_init_rank(comm, world, u, rank));
  return GM_OK;
}

GM_API gm_status gm_nccl_comm_destroy(ncclComm_t comm) {
  if (!comm) return GM_OK;
  GM_REQUIRE(nccl().ok, GM_ERR_NCCL, "gm_nccl_comm_destroy: " + nccl().why);
  GM_TRY_NCCL(nccl().comm_destroy(comm));
  return GM_OK;
}

// ---- peer memory (the push epilogue's targets) -------------------------------
// A CUDA IPC handle covers a whole allocation; the importer adds the offset of
// the exported pointer inside it (caching allocators sub-allocate), found with
// the driver's cuMemGetAddressRange (libcuda is resolved at run time).
namespace {
using cuMemGetAddressRange_t = int (*)(unsigned long long*, size_t*, unsigned long long);
cuMemGetAddressRange_t address_range() {
  static cuMemGetAddressRange_t fn = [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
    return h ? reinterpret_cast<cuMemGetAddressRange_t>(dlsym(h, "cuMemGetAddressRange_v2")) : nullptr;
  }();
  return fn;
}
}  // namespace

GM_API size_t gm_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t) + sizeof(int64_t); }

GM_API gm_status gm_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  GM_REQUIRE(dev_ptr && handle_out, GM_ERR_INVALID_ARGUMENT, "gm_ipc_get_handle: null argument");
  auto range = address_range();
  GM_REQUIRE(range, GM_ERR_CUDA, "gm_ipc_get_handle: cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  GM_REQUIRE(range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) == 0, GM_ERR_CUDA,
             "gm_ipc_get_handle: pointer is not device memory");
  cudaIpcMemHandle_t h;
  GM_TRY_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  const int64_t off = static_cast<int64_t>(reinterpret_cast<unsigned long long>(dev_ptr) - base);
  memcpy(handle_out, &h, sizeof(h));
  memcpy(static_cast<unsigned char*>(handle_out) + sizeof(h), &off, sizeof(off));
  return GM_OK;
}

GM_API gm_status gm_ipc_open_handle(const void* handle, void** dev_ptr_out, void** base_out) {
  GM_REQUIRE(handle && dev_ptr_out && base_out, GM_ERR_INVALID_ARGUMENT, "gm_ipc_open_handle: null argument");
  cudaIpcMemHandle_t h;
  int64_t off = 0;
  memcpy(&h, handle, sizeof(h));
  memcpy(&off, static_cast<const unsigned char*>(handle) + sizeof(h), sizeof(off));
  void* base = nullptr;
  GM_TRY_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *base_out = base;
  *dev_ptr_out = static_cast<unsigned char*>(base) + off;
  return GM_OK;
}

GM_API gm_status gm_ipc_close_handle(void* base) {
  GM_REQUIRE(base, GM_ERR_INVALID_ARGUMENT, "gm_ipc_close_handle: null base");
  GM_TRY_CUDA(cudaIpcCloseMemHandle(base));
  return GM_OK;
}

namespace {
// bf16 sums in the blocked / halo modes carry fp32 rows between the blocks
size_t carry_bytes(const gm_dist_layout* L, gm_dtype dtype, int64_t f) {
  if (dtype != GM_BF16 || L->mode == GM_DIST_EXACT || !L->blocks) return 0;
  return align_up(static_cast<size_t>(L->blocks[0].num_rows) * static_cast<size_t>(f) * sizeof(float), 256);
}
size_t exchange_bytes(const gm_dist_layout* L, gm_dtype dtype, int64_t f);
}  // namespace

GM_API size_t gm_dist_spmm_workspace(const gm_dist_layout* L, gm_dtype dtype, int64_t f) {
  if (!L || f < 0 || L->world < 1) return 0;
  return exchange_bytes(L, dtype, f) + carry_bytes(L, dtype, f);
}

namespace {
size_t exchange_bytes(const gm_dist_layout* L, gm_dtype dtype, int64_t f) {
  const size_t row = static_cast<size_t>(f) * esize(dtype);
  if (L->mode == GM_DIST_EXACT) return align_up(static_cast<size_t>(L->world) * L->shard_rows * row, 256);
  if (L->mode == GM_DIST_BLOCKED)
    return static_cast<size_t>(L->chunks) * align_up(static_cast<size_t>(L->world) * L->chunk_rows * row, 256);
  // halo: send pack + receive buffer
  int64_t send = 0, recv = 0;
  for (int q = 0; q < L->world; ++q) {
    send += L->halo_send_counts_host ? L->halo_send_counts_host[q] : 0;
    recv += L->halo_recv_counts_host ? L->halo_recv_counts_host[q] : 0;
  }
  return align_up(static_cast<size_t>(send) * row, 256) + align_up(static_cast<size_t>(recv) * row, 256);
}
}  // namespace

GM_API gm_status gm_dist_spmm(const gm_dist_layout* L, gm_dtype dtype, const void* x_shard, int64_t f,
                              gm_reduce reduce, void* out, int32_t* arg_out, void* workspace, size_t workspace_bytes,
                              ncclComm_t comm, gm_stream_t comm_stream, gm_stream_t stream) {
  GM_REQUIRE(L && L->blocks && L->plans, GM_ERR_INVALID_ARGUMENT, "gm_dist_spmm: null layout");
  GM_REQUIRE(L->world >= 1 && L->rank >= 0 && L->rank < L->world, GM_ERR_INVALID_ARGUMENT,
             "gm_dist_spmm: bad rank/world");
  GM_REQUIRE(f >= 0 && x_shard && out, GM_ERR_INVALID_ARGUMENT, "gm_dist_spmm: null x_shard/out");
  const bool maxmin = reduce == GM_MAX || reduce == GM_MIN;
  GM_REQUIRE(!maxmin || L->mode == GM_DIST_EXACT || arg_out, GM_ERR_INVALID_ARGUMENT,
             "gm_dist_spmm: blocked/halo max/min need arg_out (ties across blocks break on COO id)");
  GM_REQUIRE(workspace_bytes >= gm_dist_spmm_workspace(L, dtype, f) && (workspace || workspace_bytes == 0),
             GM_ERR_INVALID_ARGUMENT, "gm_dist_spmm: workspace too small");
  GM_REQUIRE(comm, GM_ERR_INVALID_ARGUMENT, "gm_dist_spmm: null communicator");
  GM_REQUIRE(nccl().ok, GM_ERR_NCCL, "gm_dist_spmm: " + nccl().why);
  cudaStream_t st = as_stream(stream);
  cudaStream_t cst = as_stream(comm_stream);
  const size_t row = static_cast<size_t>(f) * esize(dtype);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  const int nev = 2 + (L->mode == GM_DIST_BLOCKED ? L->chunks : 0);
  cudaEvent_t* ev = nullptr;
  gm_status s = events(nev, &ev);
  if (s != GM_OK) return s;
  // the exchange may only read x_shard (and overwrite the receive buffers of
  // the previous call) once `stream` has reached this point
  GM_TRY_CUDA(cudaEventRecord(ev[0], st));
  GM_TRY_CUDA(cudaStreamWaitEvent(cst, ev[0], 0));

  if (L->mode == GM_DIST_EXACT) {
    GM_TRY_NCCL(nccl().all_gather(x_shard, ws, static_cast<size_t>(L->shard_rows) * row, ncclUint8, comm, cst));
    GM_TRY_CUDA(cudaEventRecord(ev[1], cst));
    GM_TRY_CUDA(cudaStreamWaitEvent(st, ev[1], 0));
    return gm_spmm(&L->blocks[0], &L->plans[0], dtype, ws, f, nullptr, nullptr, reduce, out, arg_out, stream);
  }

  const gm_reduce first = reduce == GM_MEAN ? GM_SUM : reduce;
  // bf16 sum/mean: fp32 running rows in the workspace tail, one rounding at the end
  gm_spmm_epilogue ep{};
  const bool carry = carry_bytes(L, dtype, f) > 0 && !maxmin;
  if (carry) ep.carry = reinterpret_cast<float*>(ws + exchange_bytes(L, dtype, f));
  auto run_block = [&](int b, const void* xb, gm_reduce k, bool cont, bool last) -> gm_status {
    if (carry) {
      ep.carry_mode = !cont ? GM_CARRY_START : last ? GM_CARRY_FINISH : GM_CARRY_CONTINUE;
      return gm_spmm_ex(&L->blocks[b], &L->plans[b], dtype, xb, f, nullptr, k, cont ? 1 : 0,
                        k == GM_MEAN ? L->mean_deg : nullptr, &ep, out, nullptr, stream);
    }
    if (!cont) return gm_spmm(&L->blocks[b], &L->plans[b], dtype, xb, f, nullptr, nullptr, k, out, arg_out, stream);
    return gm_spmm_accumulate(&L->blocks[b], &L->plans[b], dtype, xb, f, nullptr, k,
                              k == GM_MEAN ? L->mean_deg : nullptr, out, arg_out, stream);
  };
  if (L->mode == GM_DIST_BLOCKED) {
    GM_REQUIRE(L->chunks >= 1 && L->chunk_rows >= 1, GM_ERR_INVALID_ARGUMENT, "gm_dist_spmm: bad chunk layout");
    const size_t chunk_bytes = align_up(static_cast<size_t>(L->world) * L->chunk_rows * row, 256);
    // every chunk's all-gather is queued before the local block starts
    for (int c = 0; c < L->chunks; ++c) {
      GM_TRY_NCCL(nccl().all_gather(static_cast<const unsigned char*>(x_shard) + static_cast<size_t>(c) * L->chunk_rows * row,
                                    ws + c * chunk_bytes, static_cast<size_t>(L->chunk_rows) * row, ncclUint8, comm, cst));
      GM_TRY_CUDA(cudaEventRecord(ev[2 + c], cst));
    }
    s = run_block(0, x_shard, first, false, false);
    if (s != GM_OK) return s;
    for (int c = 0; c < L->chunks; ++c) {
      GM_TRY_CUDA(cudaStreamWaitEvent(st, ev[2 + c], 0));
      const bool last = c == L->chunks - 1;
      const gm_reduce k = (last || reduce != GM_MEAN) ? reduce : GM_SUM;
      s = run_block(1 + c, ws + c * chunk_bytes, k, true, last);
      if (s != GM_OK) return s;
    }
    return GM_OK;
  }

  // halo: pack the rows each peer needs from my shard, exchange in one group
  GM_REQUIRE(L->mode == GM_DIST_HALO && L->halo_send_counts_host && L->halo_recv_counts_host,
             GM_ERR_INVALID_ARGUMENT, "gm_dist_spmm: halo mode needs per-peer counts");
  int64_t n_send = 0, n_recv = 0;
  for (int q = 0; q < L->world; ++q) {
    n_send += L->halo_send_counts_host[q];
    n_recv += L->halo_recv_counts_host[q];
  }
  unsigned char* send_buf = ws;
  unsigned char* recv_buf = ws + align_up(static_cast<size_t>(n_send) * row, 256);
  if (n_send > 0) {
    s = gm_gather_rows(dtype, x_shard, f, L->halo_send_idx, n_send, send_buf, comm_stream);
    if (s != GM_OK) return s;
  }
  GM_TRY_NCCL(nccl().group_start());
  int64_t so = 0, ro = 0;
  for (int q = 0; q < L->world; ++q) {
    const int64_t ns = L->halo_send_counts_host[q], nr = L->halo_recv_counts_host[q];
    if (q != L->rank && ns > 0)
      GM_TRY_NCCL(nccl().send(send_buf + so * row, static_cast<size_t>(ns) * row, ncclUint8, q, comm, cst));
    if (q != L->rank && nr > 0)
      GM_TRY_NCCL(nccl().recv(recv_buf + ro * row, static_cast<size_t>(nr) * row, ncclUint8, q, comm, cst));
    so += ns;
    ro += nr;
  }
  GM_TRY_NCCL(nccl().group_end());
  GM_TRY_CUDA(cudaEventRecord(ev[1], cst));
  s = run_block(0, x_shard, first, false, false);
  if (s != GM_OK) return s;
  GM_TRY_CUDA(cudaStreamWaitEvent(st, ev[1], 0));
  return run_block(1, recv_buf, reduce, true, true);
}

}  // extern "C"
