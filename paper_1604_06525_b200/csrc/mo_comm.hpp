// mo_comm.hpp — communication for strip-sharded grids: halo
// exchange of axis-0 rows between neighbouring strips and a fixed-order
// all-gather of scalar partials.  Two transports:
//   * NcclComm  — one process per GPU; NCCL send/recv + all-gather on the
//                 session stream (libnccl is dlopen'ed: the process may
//                 already hold torch's copy).
//   * LocalComm — N shard sessions in ONE process (one GPU): peer copies
//                 ordered with events and host barriers.  Exercises the same
//                 partition / halo / reduction schedule on a single device.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <vector>

namespace mo {

// One contiguous segment laid out as [top halo rows][owned rows][bottom halo rows].
struct HaloSeg {
  char* base = nullptr;  // first byte of the top halo
  size_t row_bytes = 0;
  int top = 0, owned = 0, bottom = 0;  // rows held by this rank
  int send_up = 0, send_down = 0;      // rows the neighbours above/below hold as halo
};

// One-shot deterministic all-gather of the reductions' rank partials through
// peer-mapped device memory: every rank owns a small
// exchange block; a single-block kernel (k_peer_fin, mo_kernels.cuh) stores
// this rank's pair into slot `rank` of EVERY rank's block, raises a flag
// there, waits for all flags in its own block and sums the slots in rank
// order - one kernel over NVLink instead of an NCCL all-gather plus a
// finalisation kernel, and kernel-only (capturable).
//   block layout: double val[2][kPeerMax][2] | u64 flag[2][kPeerMax] | u64 epoch
// (two parities: a rank can be at most one reduction ahead of any peer).
constexpr int kPeerMax = 64;
constexpr size_t kPeerBlock = 4096;
struct PeerTable {
  char* block[kPeerMax] = {};  // every rank's block, in this process's address space
};

class Comm {
 public:
  virtual ~Comm() = default;
  int rank = 0, world = 1, device = 0;
  // Exchange halo rows of every segment with the neighbouring ranks.
  virtual void halo(const std::vector<HaloSeg>& segs, cudaStream_t st) = 0;
  // recv[r*n + i] = rank r's send[i], identical on every rank.
  virtual void allgather(const double* send, double* recv, int n, cudaStream_t st) = 0;
  // Pure stream operations (no host synchronisation): CUDA-graph capturable.
  virtual bool capturable() const { return false; }
  // Peer-mapped exchange blocks for k_peer_fin, or nullptr if the transport
  // has none (then reductions use allgather + k_global_fin).
  virtual const PeerTable* peers() { return nullptr; }
};

class LocalWorld;  // shared state of the single-process fake
std::shared_ptr<LocalWorld> make_local_world(int world, int device);
std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalWorld> w, int rank);

// NCCL: `id` is the 128-byte ncclUniqueId produced by nccl_unique_id on rank 0.
void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(const void* id128, int rank, int world, int device);

}  // namespace mo
