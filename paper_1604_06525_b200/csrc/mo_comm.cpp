// mo_comm.cpp — see mo_comm.hpp.
#include "mo_comm.hpp"

#include <dlfcn.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "mo_plan.hpp"

namespace mo {

#define CKC(x)                                                                              \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) fail(Err::kCuda, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------ local (1 process)
class LocalWorld {
 public:
  LocalWorld(int world, int device) : n(world), dev(device), posted(size_t(world)), ev(size_t(world)), cev(size_t(world)) {
    CKC(cudaSetDevice(dev));
    for (int r = 0; r < n; ++r) {
      CKC(cudaEventCreateWithFlags(&ev[size_t(r)], cudaEventDisableTiming));
      CKC(cudaEventCreateWithFlags(&cev[size_t(r)], cudaEventDisableTiming));
    }
    CKC(cudaMalloc(&gbuf, sizeof(double) * size_t(n) * 64));
    CKC(cudaMalloc(&pblk, kPeerBlock * size_t(n)));
    CKC(cudaMemset(pblk, 0, kPeerBlock * size_t(n)));
    for (int r = 0; r < n; ++r) table.block[r] = pblk + kPeerBlock * size_t(r);
  }
  ~LocalWorld() {
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : cev) cudaEventDestroy(e);
    cudaFree(gbuf);
    cudaFree(pblk);
  }
  // Reusable generation barrier.
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++count == n) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
  int n, dev;
  std::vector<std::vector<HaloSeg>> posted;  // per rank, current exchange
  std::vector<cudaEvent_t> ev, cev;          // produced / consumed per rank
  double* gbuf = nullptr;
  char* pblk = nullptr;  // the ranks' peer-exchange blocks (one device: plain pointers)
  PeerTable table;

 private:
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  long gen = 0;
};

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalWorld> w, int r) : W(std::move(w)) {
    rank = r;
    world = W->n;
    device = W->dev;
  }
  // Each rank PULLS its halos from the neighbours' owned rows, then waits
  // until the neighbours have pulled from it before overwriting anything.
  void halo(const std::vector<HaloSeg>& segs, cudaStream_t st) override {
    W->posted[size_t(rank)] = segs;
    CKC(cudaEventRecord(W->ev[size_t(rank)], st));
    W->barrier();
    for (int nb : {rank - 1, rank + 1}) {
      if (nb < 0 || nb >= world) continue;
      CKC(cudaStreamWaitEvent(st, W->ev[size_t(nb)], 0));
      const auto& theirs = W->posted[size_t(nb)];
      check(theirs.size() == segs.size(), Err::kInternal, "halo exchange: segment mismatch");
      for (size_t k = 0; k < segs.size(); ++k) {
        const HaloSeg& m = segs[k];
        const HaloSeg& o = theirs[k];
        if (nb == rank - 1 && m.top) {  // my top halo = their last `top` owned rows
          const char* src = o.base + (size_t(o.top) + size_t(o.owned - m.top)) * o.row_bytes;
          CKC(cudaMemcpyAsync(m.base, src, size_t(m.top) * m.row_bytes, cudaMemcpyDeviceToDevice, st));
        }
        if (nb == rank + 1 && m.bottom) {  // my bottom halo = their first `bottom` owned rows
          const char* src = o.base + size_t(o.top) * o.row_bytes;
          char* dst = m.base + (size_t(m.top) + size_t(m.owned)) * m.row_bytes;
          CKC(cudaMemcpyAsync(dst, src, size_t(m.bottom) * m.row_bytes, cudaMemcpyDeviceToDevice, st));
        }
      }
    }
    CKC(cudaEventRecord(W->cev[size_t(rank)], st));
    W->barrier();
    for (int nb : {rank - 1, rank + 1})
      if (nb >= 0 && nb < world) CKC(cudaStreamWaitEvent(st, W->cev[size_t(nb)], 0));
    W->barrier();  // posted[] may be reused by the next exchange
  }
  void allgather(const double* send, double* recv, int n, cudaStream_t st) override {
    check(n <= 64, Err::kInternal, "allgather: too many values");
    CKC(cudaMemcpyAsync(W->gbuf + size_t(rank) * size_t(n), send, sizeof(double) * size_t(n),
                        cudaMemcpyDeviceToDevice, st));
    CKC(cudaEventRecord(W->ev[size_t(rank)], st));
    W->barrier();
    for (int r = 0; r < world; ++r) CKC(cudaStreamWaitEvent(st, W->ev[size_t(r)], 0));
    CKC(cudaMemcpyAsync(recv, W->gbuf, sizeof(double) * size_t(n) * size_t(world), cudaMemcpyDeviceToDevice, st));
    CKC(cudaEventRecord(W->cev[size_t(rank)], st));
    W->barrier();
    for (int r = 0; r < world; ++r) CKC(cudaStreamWaitEvent(st, W->cev[size_t(r)], 0));
    W->barrier();
  }
  // Opt-in (MO_B200_LOCAL_P2P=1): the ranks share one device, so a host
  // call that waits for the whole device (cudaFree, graph re-upload) on one
  // rank would wait for another rank's k_peer_fin spinning on its flag.
  // One process per GPU (NcclComm) has no such coupling.
  const PeerTable* peers() override { return std::getenv("MO_B200_LOCAL_P2P") ? &W->table : nullptr; }

 private:
  std::shared_ptr<LocalWorld> W;
};

std::shared_ptr<LocalWorld> make_local_world(int world, int device) {
  check(world >= 1 && world <= 64, Err::kBindError, "local world size out of range");
  return std::make_shared<LocalWorld>(world, device);
}
std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalWorld> w, int rank) {
  check(rank >= 0 && rank < w->n, Err::kBindError, "rank out of range");
  return std::make_unique<LocalComm>(std::move(w), rank);
}

// ------------------------------------------------------------ NCCL
namespace nccl {
// Minimal ABI-stable subset of nccl.h (NCCL 2.x).
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclChar = 0, ncclFloat64 = 8 };
struct Api {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
Api& api() {
  static Api a;
  if (!a.h) {
    // Prefer a copy already loaded into the process (e.g. torch's).
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    check(a.h != nullptr, Err::kCuda, "libnccl.so.2 not found");
    auto sym = [&](const char* n) {
      void* p = dlsym(a.h, n);
      check(p != nullptr, Err::kCuda, std::string("NCCL symbol missing: ") + n);
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  }
  return a;
}
void ok(ncclResult_t r, const char* what) {
  if (r != 0) fail(Err::kCuda, std::string(what) + ": " + api().GetErrorString(r));
}
}  // namespace nccl

class NcclComm final : public Comm {
 public:
  NcclComm(const void* id128, int r, int w, int dev) {
    rank = r;
    world = w;
    device = dev;
    nccl::ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    CKC(cudaSetDevice(dev));
    nccl::ok(nccl::api().CommInitRank(&comm_, w, id, r), "ncclCommInitRank");
  }
  void halo(const std::vector<HaloSeg>& segs, cudaStream_t st) override {
    auto& A = nccl::api();
    nccl::ok(A.GroupStart(), "ncclGroupStart");
    for (const HaloSeg& m : segs) {
      char* owned = m.base + size_t(m.top) * m.row_bytes;
      if (rank > 0) {
        if (m.send_up) nccl::ok(A.Send(owned, size_t(m.send_up) * m.row_bytes, nccl::ncclChar, rank - 1, comm_, st), "ncclSend");
        if (m.top) nccl::ok(A.Recv(m.base, size_t(m.top) * m.row_bytes, nccl::ncclChar, rank - 1, comm_, st), "ncclRecv");
      }
      if (rank < world - 1) {
        if (m.send_down)
          nccl::ok(A.Send(owned + size_t(m.owned - m.send_down) * m.row_bytes, size_t(m.send_down) * m.row_bytes,
                          nccl::ncclChar, rank + 1, comm_, st),
                   "ncclSend");
        if (m.bottom)
          nccl::ok(A.Recv(owned + size_t(m.owned) * m.row_bytes, size_t(m.bottom) * m.row_bytes, nccl::ncclChar,
                          rank + 1, comm_, st),
                   "ncclRecv");
      }
    }
    nccl::ok(A.GroupEnd(), "ncclGroupEnd");
  }
  void allgather(const double* send, double* recv, int n, cudaStream_t st) override {
    nccl::ok(nccl::api().AllGather(send, recv, size_t(n), nccl::ncclFloat64, comm_, st), "ncclAllGather");
  }
  bool capturable() const override { return true; }
  // Exchange blocks mapped with CUDA IPC (each rank allocates its own; the
  // handles travel by one NCCL all-gather; peers open them with lazy peer
  // access over NVLink).  Any failure leaves the NCCL reductions in place.
  const PeerTable* peers() override {
    if (peer_state_ == 0) {
      peer_state_ = -1;
      if (world <= kPeerMax && !std::getenv("MO_B200_NO_P2P")) try_map_peers();
    }
    return peer_state_ > 0 ? &table_ : nullptr;
  }
  ~NcclComm() override;

 private:
  void try_map_peers() {
    if (cudaMalloc(&mine_, kPeerBlock) != cudaSuccess) return;
    CKC(cudaMemset(mine_, 0, kPeerBlock));
    cudaIpcMemHandle_t h;
    std::memset(&h, 0, sizeof h);
    const bool can = world == 1 || cudaIpcGetMemHandle(&h, mine_) == cudaSuccess;
    // every rank learns every rank's handle and whether it could export one
    struct Msg {
      cudaIpcMemHandle_t h;
      int ok;
      char pad[60];
    };
    static_assert(sizeof(Msg) == 128, "handle message is 128 bytes");
    Msg m;
    std::memset(&m, 0, sizeof m);
    m.h = h;
    m.ok = can ? 1 : 0;
    char* d = nullptr;
    CKC(cudaMalloc(&d, sizeof(Msg) * size_t(world + 1)));
    CKC(cudaMemcpy(d, &m, sizeof m, cudaMemcpyHostToDevice));
    cudaStream_t s;
    CKC(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    nccl::ok(nccl::api().AllGather(d, d + sizeof(Msg), sizeof(Msg), nccl::ncclChar, comm_, s), "ncclAllGather");
    CKC(cudaStreamSynchronize(s));
    CKC(cudaStreamDestroy(s));
    std::vector<Msg> all(static_cast<size_t>(world));
    CKC(cudaMemcpy(all.data(), d + sizeof(Msg), sizeof(Msg) * size_t(world), cudaMemcpyDeviceToHost));
    cudaFree(d);
    bool every = true;
    for (const Msg& x : all) every = every && x.ok;
    bool opened = every;
    for (int r = 0; r < world && opened; ++r) {
      if (r == rank) {
        table_.block[r] = mine_;
        continue;
      }
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, all[size_t(r)].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        opened = false;
        break;
      }
      table_.block[r] = static_cast<char*>(p);
    }
    // all ranks must agree (a rank that could not map every peer would stall
    // the others): one more all-gather of the outcome
    int* f = nullptr;
    CKC(cudaMalloc(&f, sizeof(int) * size_t(world + 1)));
    const int mineok = opened ? 1 : 0;
    CKC(cudaMemcpy(f, &mineok, sizeof(int), cudaMemcpyHostToDevice));
    CKC(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    nccl::ok(nccl::api().AllGather(f, f + 1, sizeof(int), nccl::ncclChar, comm_, s), "ncclAllGather");
    CKC(cudaStreamSynchronize(s));
    CKC(cudaStreamDestroy(s));
    std::vector<int> oks(static_cast<size_t>(world));
    CKC(cudaMemcpy(oks.data(), f + 1, sizeof(int) * size_t(world), cudaMemcpyDeviceToHost));
    cudaFree(f);
    bool all_ok = true;
    for (int x : oks) all_ok = all_ok && x;
    peer_state_ = all_ok ? 1 : -1;
  }
  nccl::ncclComm_t comm_ = nullptr;
  char* mine_ = nullptr;
  PeerTable table_;
  int peer_state_ = 0;  // 0 not tried, 1 mapped, -1 unavailable
};

NcclComm::~NcclComm() {
  for (int r = 0; r < world && r < kPeerMax; ++r)
    if (r != rank && table_.block[r]) cudaIpcCloseMemHandle(table_.block[r]);
  if (mine_) cudaFree(mine_);
  if (comm_) nccl::api().CommDestroy(comm_);
}

void nccl_unique_id(void* out128) {
  nccl::ncclUniqueId id;
  nccl::ok(nccl::api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof id);
}

std::unique_ptr<Comm> make_nccl_comm(const void* id128, int rank, int world, int device) {
  check(world >= 1 && rank >= 0 && rank < world, Err::kBindError, "bad NCCL rank/world");
  return std::make_unique<NcclComm>(id128, rank, world, device);
}

}  // namespace mo
