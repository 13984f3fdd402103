// comm.cu -- transports of the node-sharded solve (comm.hpp) and the Engine's
// node-exchange staging (pool records in HBM).
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "comm.hpp"
#include "engine.hpp"
#include "pool_kernels.cuh"

namespace bnbg {

#define CK(call)                                          \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
  } while (0)

#define NK(call)                                                               \
  do {                                                                         \
    ncclResult_t r_ = (call);                                                  \
    if (r_ != ncclSuccess)                                                     \
      return fail(4, std::string("NCCL error in " #call ": ") + ncclGetErrorString(r_)); \
  } while (0)

static PoolDev pool_view2(void* const* mem, int p, int k, int cap) {
  PoolDev P;
  P.p = p;
  P.k = std::max(k, 1);
  P.cap = cap;
  P.state = static_cast<uint8_t*>(mem[0]);
  P.warm = static_cast<double*>(mem[1]);
  P.j0 = static_cast<int*>(mem[2]);
  P.j1 = static_cast<int*>(mem[3]);
  P.n0 = static_cast<int*>(mem[4]);
  P.n1 = static_cast<int*>(mem[5]);
  P.depth = static_cast<int*>(mem[6]);
  return P;
}

size_t Engine::node_record_bytes() const { return node_rec_bytes(p, std::max(k, 1)); }

static int grow(void** ptr, size_t* cap, size_t want, cudaStream_t st) {
  if (want <= *cap) return 0;
  if (*ptr) cudaFreeAsync(*ptr, st);
  *ptr = nullptr;
  const size_t c = std::max(want, *cap * 2);
  if (cudaMallocAsync(ptr, c, st) != cudaSuccess) return 1;
  *cap = c;
  return 0;
}

int Engine::pool_pack(int cnt, const int* slots, const double* lbs, uint8_t** d_send) {
  const size_t rb = node_record_bytes();
  if (grow(reinterpret_cast<void**>(&dXSend_), &xsend_bytes_, std::max<size_t>(rb * cnt, 64), stream_))
    return fail(4, "node exchange: out of device memory");
  if (cnt > xslots_cap_) {
    dfree(dXSlots_);
    dfree(dXLb_);
    xslots_cap_ = std::max(cnt, 2 * xslots_cap_);
    CK(cudaMallocAsync(&dXSlots_, sizeof(int) * xslots_cap_, stream_));
    CK(cudaMallocAsync(&dXLb_, sizeof(double) * xslots_cap_, stream_));
  }
  *d_send = dXSend_;
  if (cnt <= 0) return 0;
  if (int rc = h2d(dXSlots_, slots, sizeof(int) * cnt)) return rc;
  if (int rc = h2d(dXLb_, lbs, sizeof(double) * cnt)) return rc;
  k_pool_pack<<<cnt, 128, 0, stream_>>>(pool_view2(pool_mem_, p, k, pool_cap_), cnt, dXSlots_,
                                         dXLb_, dXSend_);
  ++launches;
  CK(cudaGetLastError());
  return 0;
}

int Engine::pool_recv_buffer(int cnt, uint8_t** d_recv) {
  const size_t rb = node_record_bytes();
  if (grow(reinterpret_cast<void**>(&dXRecv_), &xrecv_bytes_, std::max<size_t>(rb * cnt, 64), stream_))
    return fail(4, "node exchange: out of device memory");
  *d_recv = dXRecv_;
  return 0;
}

int Engine::pool_unpack(int cnt, const int* slots, double* lbs) {
  if (cnt <= 0) return 0;
  if (cnt > xslots_cap_) {
    dfree(dXSlots_);
    dfree(dXLb_);
    xslots_cap_ = std::max(cnt, 2 * xslots_cap_);
    CK(cudaMallocAsync(&dXSlots_, sizeof(int) * xslots_cap_, stream_));
    CK(cudaMallocAsync(&dXLb_, sizeof(double) * xslots_cap_, stream_));
  }
  if (int rc = h2d(dXSlots_, slots, sizeof(int) * cnt)) return rc;
  k_pool_unpack<<<cnt, 128, 0, stream_>>>(pool_view2(pool_mem_, p, k, pool_cap_), cnt, dXRecv_,
                                           dXSlots_, dXLb_);
  ++launches;
  CK(cudaGetLastError());
  if (int rc = d2h(lbs, dXLb_, sizeof(double) * cnt)) return rc;
  CK(cudaStreamSynchronize(stream_));
  return 0;
}

// Process-wide communicator cache: an engine created later in the same process
// (same device, rank, world and unique id) reuses the communicator instead of
// paying ncclCommInitRank / ncclCommDestroy again.  Cached communicators live
// until the process exits.
static std::mutex g_comm_mu;
static std::map<std::string, ncclComm_t>& comm_cache() {
  static std::map<std::string, ncclComm_t> m;
  return m;
}

void Engine::comm_release() {
  dfree(dXSend_);
  dfree(dXRecv_);
  dfree(dXSlots_);
  dfree(dXLb_);
  dfree(dGather_);
  dXSend_ = dXRecv_ = nullptr;
  dXSlots_ = nullptr;
  dXLb_ = nullptr;
  dGather_ = nullptr;
  nccl_comm = nullptr;  // owned by the process-wide cache
}

int Engine::nccl_init(const uint8_t* uid, int rank, int world) {
  CK(cudaSetDevice(device));
  std::string key(reinterpret_cast<const char*>(uid), sizeof(ncclUniqueId));
  key += ":" + std::to_string(device) + ":" + std::to_string(rank) + ":" + std::to_string(world);
  std::lock_guard<std::mutex> lk(g_comm_mu);
  auto it = comm_cache().find(key);
  if (it == comm_cache().end()) {
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    ncclComm_t c = nullptr;
    NK(ncclCommInitRank(&c, world, id, rank));
    it = comm_cache().emplace(key, c).first;
  }
  nccl_comm = it->second;
  nccl_rank = rank;
  nccl_world = world;
  return 0;
}

int Engine::comm_allgather_nccl(const void* send, size_t bytes, void* recv) {
  if (!nccl_comm) return fail(1, "solve_sharded: no NCCL communicator (bnbg_nccl_init)");
  const size_t need = bytes * (nccl_world + 1);
  if (grow(&dGather_, &gather_bytes_, need, stream_)) return fail(4, "allgather: out of device memory");
  uint8_t* d_in = static_cast<uint8_t*>(dGather_);
  uint8_t* d_out = d_in + bytes;
  if (int rc = h2d(d_in, send, bytes)) return rc;
  NK(ncclAllGather(d_in, d_out, bytes, ncclUint8, static_cast<ncclComm_t>(nccl_comm), stream_));
  if (int rc = d2h(recv, d_out, bytes * nccl_world)) return rc;
  CK(cudaStreamSynchronize(stream_));
  return 0;
}

int Engine::comm_exchange_nccl(int world, const int64_t* send_nodes, const uint8_t* d_send,
                               const int64_t* recv_nodes, uint8_t* d_recv, size_t rb) {
  if (!nccl_comm) return fail(1, "solve_sharded: no NCCL communicator (bnbg_nccl_init)");
  ncclComm_t c = static_cast<ncclComm_t>(nccl_comm);
  size_t so = 0, ro = 0;
  NK(ncclGroupStart());
  for (int peer = 0; peer < world; ++peer) {
    if (send_nodes[peer] > 0) {
      NK(ncclSend(d_send + so, rb * send_nodes[peer], ncclUint8, peer, c, stream_));
      so += rb * send_nodes[peer];
    }
    if (recv_nodes[peer] > 0) {
      NK(ncclRecv(d_recv + ro, rb * recv_nodes[peer], ncclUint8, peer, c, stream_));
      ro += rb * recv_nodes[peer];
    }
  }
  NK(ncclGroupEnd());
  CK(cudaStreamSynchronize(stream_));
  return 0;
}

int Engine::comm_exchange_host(const bnbg_comm_ops* ops, const int64_t* send_nodes,
                               const uint8_t* d_send, const int64_t* recv_nodes, uint8_t* d_recv,
                               size_t rb) {
  const int world = ops->world;
  std::vector<int64_t> sb(world), rbs(world);
  size_t st = 0, rt = 0;
  for (int q = 0; q < world; ++q) {
    sb[q] = (int64_t)rb * send_nodes[q];
    rbs[q] = (int64_t)rb * recv_nodes[q];
    st += sb[q];
    rt += rbs[q];
  }
  std::vector<uint8_t> hs(std::max<size_t>(st, 1)), hr(std::max<size_t>(rt, 1));
  if (st) {
    if (int rc = d2h(hs.data(), d_send, st)) return rc;
    CK(cudaStreamSynchronize(stream_));
  }
  if (ops->alltoallv(ops->ctx, hs.data(), sb.data(), hr.data(), rbs.data()) != 0)
    return fail(4, "solve_sharded: alltoallv callback failed");
  if (rt) {
    if (int rc = h2d(d_recv, hr.data(), rt)) return rc;
    CK(cudaStreamSynchronize(stream_));
  }
  return 0;
}

int CallbackComm::allgather(Engine& eng, const void* send, size_t bytes, void* recv) {
  if (ops->allgather(ops->ctx, send, (int64_t)bytes, recv) != 0) {
    eng.err = "solve_sharded: allgather callback failed";
    return BNBG_CUDA_ERROR;
  }
  return 0;
}

int CallbackComm::exchange(Engine& eng, const std::vector<int64_t>& send_nodes,
                           const uint8_t* d_send, const std::vector<int64_t>& recv_nodes,
                           uint8_t* d_recv, size_t rec_bytes) {
  return eng.comm_exchange_host(ops, send_nodes.data(), d_send, recv_nodes.data(), d_recv,
                                rec_bytes);
}

int NcclComm::allgather(Engine& eng, const void* send, size_t bytes, void* recv) {
  return eng.comm_allgather_nccl(send, bytes, recv);
}

int NcclComm::exchange(Engine& eng, const std::vector<int64_t>& send_nodes, const uint8_t* d_send,
                       const std::vector<int64_t>& recv_nodes, uint8_t* d_recv,
                       size_t rec_bytes) {
  return eng.comm_exchange_nccl(world, send_nodes.data(), d_send, recv_nodes.data(), d_recv,
                                rec_bytes);
}

bool balance_plan(int world, const int64_t* counts, int64_t* moves) {
  std::fill(moves, moves + (size_t)world * world, 0);
  int64_t total = 0, mx = 0, mn = INT64_MAX;
  for (int r = 0; r < world; ++r) {
    total += counts[r];
    mx = std::max(mx, counts[r]);
    mn = std::min(mn, counts[r]);
  }
  // skew rule max > factor * min + slack; BNBG_BALANCE_SKEW="factor,slack"
  // (default "2,8"; "1,0" rebalances whenever the queues differ -- tests use
  // it to push many node records through the exchange)
  int64_t factor = 2, slack = 8;
  if (const char* e = getenv("BNBG_BALANCE_SKEW")) {
    long long f = 2, s = 8;
    if (sscanf(e, "%lld,%lld", &f, &s) == 2 && f >= 1 && s >= 0) {
      factor = f;
      slack = s;
    }
  }
  const bool starving = mn == 0 && mx >= 2;
  const bool skewed = mx > factor * mn + slack;
  if (world < 2 || !(starving || skewed)) return false;
  std::vector<int64_t> surplus(world), deficit(world);
  for (int r = 0; r < world; ++r) {
    const int64_t target = total / world + (r < total % world ? 1 : 0);
    surplus[r] = std::max<int64_t>(0, counts[r] - target);
    deficit[r] = std::max<int64_t>(0, target - counts[r]);
  }
  bool any = false;
  int d = 0;
  for (int r = 0; r < world; ++r) {
    while (deficit[r] > 0) {
      while (d < world && surplus[d] == 0) ++d;
      if (d >= world) break;
      const int64_t t = std::min(deficit[r], surplus[d]);
      moves[(size_t)d * world + r] += t;
      deficit[r] -= t;
      surplus[d] -= t;
      any = true;
    }
  }
  return any;
}

}  // namespace bnbg

extern "C" int bnbg_nccl_unique_id(uint8_t* out) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return BNBG_CUDA_ERROR;
  std::memcpy(out, &id, sizeof(id));
  return BNBG_OK;
}

extern "C" int bnbg_balance_plan(int world, const int64_t* counts, int64_t* moves) {
  return bnbg::balance_plan(world, counts, moves) ? 1 : 0;
}
