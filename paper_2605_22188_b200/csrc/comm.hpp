// comm.hpp -- the per-pass exchange of the node-sharded multi-GPU solve
// (SURVEY 8(e)): X and y are replicated, every rank runs the node-processing
// pipeline on its own queue and pool, and only three things cross between
// ranks once per pass:
//   1. the incumbent: an allgather of (objective, support, coefficients); the
//      lowest objective wins, ties to the lowest rank (deterministic);
//   2. termination / time-limit state: an allgather of (queue size, pending
//      leaves, local lower bound, stop flag);
//   3. load balancing: when some rank starves, the deterministic plan
//      (balance_plan) moves queue nodes; a node travels as one fixed-size
//      record straight out of the sender's HBM pool into the receiver's.
//
// Two transports implement it:
//   NcclComm      NCCL over NVLink / NVSwitch: allgather of small host records
//                 through a device scratch, node records ncclSend/ncclRecv
//                 device-to-device (grouped), on the engine's stream.
//   CallbackComm  caller-supplied host callbacks (bnbg_comm_ops), e.g.
//                 torch.distributed over gloo: node records staged through
//                 host memory.  Used by the CPU-driven multi-process tests and
//                 to run several ranks on one GPU.
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/bnbg.h"

namespace bnbg {

class Engine;

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // recv = world blocks of `bytes` in rank order (host buffers)
  virtual int allgather(Engine& eng, const void* send, size_t bytes, void* recv) = 0;
  // node records: send_nodes[peer] records leave d_send (grouped by peer in
  // rank order), recv_nodes[peer] arrive into d_recv (same grouping)
  virtual int exchange(Engine& eng, const std::vector<int64_t>& send_nodes, const uint8_t* d_send,
                       const std::vector<int64_t>& recv_nodes, uint8_t* d_recv,
                       size_t rec_bytes) = 0;
};

struct CallbackComm : Comm {
  const bnbg_comm_ops* ops;
  explicit CallbackComm(const bnbg_comm_ops* o) : ops(o) {
    rank = o->rank;
    world = o->world;
  }
  int allgather(Engine& eng, const void* send, size_t bytes, void* recv) override;
  int exchange(Engine& eng, const std::vector<int64_t>& send_nodes, const uint8_t* d_send,
               const std::vector<int64_t>& recv_nodes, uint8_t* d_recv, size_t rec_bytes) override;
};

struct NcclComm : Comm {
  void* comm = nullptr;  // ncclComm_t owned by the engine
  int allgather(Engine& eng, const void* send, size_t bytes, void* recv) override;
  int exchange(Engine& eng, const std::vector<int64_t>& send_nodes, const uint8_t* d_send,
               const std::vector<int64_t>& recv_nodes, uint8_t* d_recv, size_t rec_bytes) override;
};

// Deterministic load-balancing plan from every rank's queue size.  Returns
// false when no move is needed; otherwise moves[d * world + r] = nodes donor d
// sends to receiver r.  Rebalances when a rank is idle while another holds >= 2
// queued nodes, or when the largest queue exceeds twice the smallest plus 8.
bool balance_plan(int world, const int64_t* counts, int64_t* moves);

}  // namespace bnbg
