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
};

class LocalWorld;  // shared state of the single-process fake
std::shared_ptr<LocalWorld> make_local_world(int world, int device);
std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalWorld> w, int rank);

// NCCL: `id` is the 128-byte ncclUniqueId produced by nccl_unique_id on rank 0.
void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(const void* id128, int rank, int world, int device);

}  // namespace mo
