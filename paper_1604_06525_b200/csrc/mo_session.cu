// mo_session.cu — device-resident solver session: the B200 replacement of
// minopt::Solver<Real> (solver.hpp:80-635) and its executor/PCG layers
// (exec.hpp, pcg.hpp).  One session = one device, one stream, all vectors in
// HBM in the reference column layout.
//
// Per nonlinear iteration (solver.hpp:415-509) the host issues:
//   refresh    computed arrays + exclusion masks            (125-168)
//   cost       generated cost kernels, deterministic reduce (174-193)
//   normal     generated b/m gather (+ graph gather, patch) (220-251)
//   PCG        init + linear_iters x {apply+p'Ap, update+r'z, p} (pcg.hpp:63-130),
//              captured once into a CUDA graph, device-side scalars/stop flags
//   step       x_trial / in-place GN step, trial cost, LM predicted decrease
// and synchronises once to read the scalar state for the trace row.
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <limits>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "mo_codegen.hpp"
#include "mo_jit.hpp"
#include "mo_kernels.cuh"
#include "mo_comm.hpp"
#include "mo_session.hpp"

namespace mo {

// NVTX range per reference routine (SURVEY.md §5 tracing): visible in nsys /
// ncu timelines, no cost without an attached tool (NVTX v3 is header-only).
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};

const char* device_prelude();

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) fail(Err::kCuda, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace {

constexpr int kPartCap = 1 << 18;
enum { SLOT_COST = 0, SLOT_PRED = 2 };

template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc(&p, n * sizeof(T)));
  return static_cast<T*>(p);
}

int vgrid(long long n, int nsm, int per_sm = 4) {
  long long g = (n + MO_THREADS - 1) / MO_THREADS;
  long long cap = (long long)nsm * per_sm;  // one wave (4 x 256 threads at <= 64 regs)
  if (g > cap) g = cap;
  return int(std::max<long long>(g, 1));
}

}  // namespace

template <class Real>
class Session final : public SessionBase {
 public:
  // comm != nullptr: strip shard owning axis-0 rows [row0, row1) of the
  // plan's single grid domain.  Fields are stored for rows
  // [lo, hi) = owned rows plus halo_rows(P) on each side (clipped); kernels
  // keep GLOBAL coordinates, so InBounds / index() / OOB semantics are those
  // of the unsharded problem.
  Session(const Plan& plan, int device, Comm* comm = nullptr, int64_t row0 = 0, int64_t row1 = -1, int halo = 0)
      : P_(plan), dev_(device), comm_(comm) {
    if (comm_) setup_shard(row0, row1, halo);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      fail(Err::kNoDevice, "no CUDA device available (the B200 path has no CPU fallback)");
    check(device >= 0 && device < ndev, Err::kNoDevice, "device index out of range");
    CK(cudaSetDevice(dev_));
    CK(cudaDeviceGetAttribute(&nsm_, cudaDevAttrMultiProcessorCount, dev_));
    CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sd_, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev_p_, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_h_, cudaEventDisableTiming));
    cfg_ = P_.cfg;
    if (cfg_.pcg_rel_tol < 0) cfg_.pcg_rel_tol = cfg_.precision == 0 ? 1e-4 : 1e-8;
    mat_ = P_.cfg.materialize;
    check(!mat_ || !comm_, Err::kBindError, "materialized plans cannot be strip-sharded");

    // JIT the plan's per-element kernels (plan time; cached on disk).
    std::string src = generate_module(P_, sizeof(Real) == 8, device_prelude(), &minfo_);
    module_key_ = std::to_string(std::hash<std::string>()(src)) + (P_.exact ? "/exact" : "/fma");
    mod_.load(compile_cubin(src, "mo_plan.cu", P_.exact));

    const size_t n = size_t(P_.num_cols);
    x_ = dalloc<Real>(n);
    xt_ = dalloc<Real>(n);
    b_ = dalloc<Real>(n);
    damp_ = dalloc<Real>(n);
    // The PCG working set (every vector the inner loop touches 20x per
    // nonlinear iteration) lives in one arena.  (An L2 access-policy window
    // over it was measured to make no difference on B200.)
    {
      const size_t vn = (n * sizeof(Real) + 255) / 256 * 256;
      char* base = static_cast<char*>(static_cast<void*>(dalloc<unsigned char>(6 * vn)));
      arena_ = base;
      arena_bytes_ = 6 * vn;
      p_ = reinterpret_cast<Real*>(base);
      ap_ = reinterpret_cast<Real*>(base + vn);
      r_ = reinterpret_cast<Real*>(base + 2 * vn);
      delta_ = reinterpret_cast<Real*>(base + 3 * vn);
      m_ = reinterpret_cast<Real*>(base + 4 * vn);
      md_ = reinterpret_cast<Real*>(base + 5 * vn);
    }
    vtmp_ = dalloc<Real>(n);
    otmp_ = dalloc<Real>(n);
    bd_ = dalloc<double>(n);
    CK(cudaMemsetAsync(damp_, 0, n * sizeof(Real), st_));
    CK(cudaMemsetAsync(x_, 0, n * sizeof(Real), st_));
    arr_.resize(P_.arrays.size(), nullptr);
    arr_n_.assign(P_.arrays.size(), -1);
    for (size_t i = 0; i < P_.arrays.size(); ++i)
      arr_[i] = dalloc<Real>(size_t(lext(P_.arrays[i].dom) * P_.arrays[i].channels));
    comp_.resize(P_.computed.size(), nullptr);
    for (size_t i = 0; i < P_.computed.size(); ++i)
      comp_[i] = dalloc<Real>(size_t(lext(P_.computed[i].dom) * P_.computed[i].channels));
    masks_.resize(P_.exclude_kernels.size(), nullptr);
    for (size_t i = 0; i < P_.exclude_kernels.size(); ++i)
    {
      masks_[i] = dalloc<unsigned char>(size_t(lext(P_.exclude_kernels[i].dom)));
      CK(cudaMemsetAsync(masks_[i], 0, size_t(lext(P_.exclude_kernels[i].dom)), st_));
    }
    if (!P_.exclude_kernels.empty() || comm_) {
      colmask_ = dalloc<unsigned char>(n);
      CK(cudaMemsetAsync(colmask_, 0, n, st_));
    }
    if (comm_) {
      rankbuf_ = dalloc<double>(size_t(comm_->world) * 64);
      chob_ = dalloc<double>(64);
    }
    if (comm_ && !std::getenv("MO_B200_NO_P2P")) {  // one-shot peer reductions (mo_comm.hpp)
      if (const PeerTable* t = comm_->peers()) {
        for (int r = 0; r < comm_->world; ++r) peer_.block[r] = t->block[r];
        peer_.rank = comm_->rank;
        peer_.world = comm_->world;
        const char* to = std::getenv("MO_B200_P2P_TIMEOUT_S");
        peer_.timeout_ns = (unsigned long long)((to ? std::atof(to) : 60.0) * 1e9);
        peer_on_ = true;
      }
    }
    params_d_ = dalloc<double>(std::max<size_t>(P_.params.size(), 1));
    state_ = dalloc<mo_state>(1);
    CK(cudaMallocHost(&state_h_, sizeof(mo_state)));
    CK(cudaMallocHost(&mu_h_, sizeof(double)));
    std::memset(state_h_, 0, sizeof(mo_state));
    state_h_->tol_rel = cfg_.pcg_rel_tol;
    state_h_->tol_abs = cfg_.pcg_abs_tol;
    state_h_->use_precond = cfg_.use_preconditioner;
    CK(cudaMemcpyAsync(state_, state_h_, sizeof(mo_state), cudaMemcpyHostToDevice, st_));
    partials_ = dalloc<double>(2 * size_t(kPartCap));
    partials2_ = dalloc<double>(2 * size_t(kPartCap));
    graphs_.resize(P_.graphs.size());
    gsets_.resize(P_.graph_sets.size());
    grid_rowbase_.resize(P_.grid_sets.size(), nullptr);
    for (size_t i = 0; i < P_.grid_sets.size(); ++i)
      grid_rowbase_[i] = dalloc<long long>(P_.grid_sets[i].templates.size());
    for (size_t i = 0; i < P_.graph_sets.size(); ++i) setup_graph_set(int(i));
    jl_grid_.assign(P_.grid_sets.size(), nullptr);
    jl_rb_grid_.assign(P_.grid_sets.size(), nullptr);
    jl_graph_.assign(P_.graph_sets.size(), nullptr);
    jl_rb_graph_.assign(P_.graph_sets.size(), nullptr);
    jl_graph_cap_.assign(P_.graph_sets.size(), 0);
    mat_vptr_.assign(P_.graphs.size(), nullptr);
    mat_vedge_.assign(P_.graphs.size(), nullptr);
    mat_nverts_.assign(P_.graphs.size(), 0);
    CK(cudaStreamSynchronize(st_));
  }

  ~Session() override {
    cudaSetDevice(dev_);
    cudaStreamSynchronize(st_);
    for (auto& kv : stage_exec_) cudaGraphExecDestroy(kv.second);
    for (void* p : owned_) cudaFree(p);
    for (Real* p : {x_, xt_, b_, damp_, vtmp_, otmp_, resid_}) cudaFree(p);
    cudaFree(arena_);
    cudaFree(bd_);
    for (Real* p : lcache_) cudaFree(p);
    cudaFree(anyflag_);
    for (Real* p : arr_) cudaFree(p);
    for (Real* p : comp_) cudaFree(p);
    for (unsigned char* p : masks_) cudaFree(p);
    cudaFree(colmask_);
    cudaFree(params_d_);
    cudaFree(state_);
    cudaFree(partials_);
    cudaFree(partials2_);
    cudaFree(rankbuf_);
    cudaFree(chob_);
    if (tl_temp_) cudaFree(tl_temp_);
    for (void* q : {(void*)glist_, (void*)gvals_, (void*)gflags_, gl_temp_}) cudaFree(q);
    for (int* t : tiles_) cudaFree(t);
    for (unsigned char* f : tflags_) cudaFree(f);
    cudaFreeHost(state_h_);
    for (auto& g : graphs_) cudaFree(g.d_verts);
    for (auto& gs : gsets_) {
      cudaFree(gs.contrib);
      cudaFree(gs.rowbase);
      for (auto& d : gs.doms) {
        cudaFree(d.vptr);
        cudaFree(d.vedge);
        cudaFree(d.outs_bm);
        cudaFree(d.outs_jtj);
      }
    }
    for (Real* p : jl_grid_) cudaFree(p);
    for (Real* p : jl_graph_) cudaFree(p);
    for (long long* p : jl_rb_grid_) cudaFree(p);
    for (long long* p : jl_rb_graph_) cudaFree(p);
    for (int* p : mat_vptr_) cudaFree(p);
    for (int* p : mat_vedge_) cudaFree(p);
    for (void* p : mt_bufs_) cudaFree(p);
    cudaFree(jtmp_);
    cudaFree(hcol_);
    cudaFree(hval_);
    cudaFree(hcnt_);
    cudaFree(ecol_);
    cudaFree(eval_);
    cudaFree(ecnt_);
    for (auto& kv : stage_ev_)
      for (auto& ev : kv.second) {
        cudaEventDestroy(ev.a);
        cudaEventDestroy(ev.b);
      }
    cudaFreeHost(mu_h_);
    cudaStreamDestroy(st_);
    cudaStreamDestroy(sd_);
    cudaEventDestroy(ev_p_);
    cudaEventDestroy(ev_h_);
  }

  // ------------------------------------------------------------ binding
  void bind_x(const void* x, int64_t n, bool device) override {
    check(n == P_.num_cols, Err::kBindError, "unknown vector size does not match the plan layout");
    CK(cudaSetDevice(dev_));
    CK(cudaMemcpyAsync(x_, x, size_t(n) * sizeof(Real), device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st_));
    CK(cudaStreamSynchronize(st_));
    x_bound_ = true;
  }
  void bind_array(int i, const void* d, int64_t n, bool device) override {
    check(i >= 0 && size_t(i) < P_.arrays.size(), Err::kBindError, "array count does not match the declaration");
    const ArrayFieldSize want = array_size(i);
    check(n == want, Err::kBindError, "array '" + P_.arrays[size_t(i)].name + "' has the wrong size");
    CK(cudaSetDevice(dev_));
    CK(cudaMemcpyAsync(arr_[size_t(i)], d, size_t(n) * sizeof(Real), device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st_));
    CK(cudaStreamSynchronize(st_));
    arr_n_[size_t(i)] = n;
  }
  void bind_params(const double* p, int64_t n) override {
    check(size_t(n) == P_.params.size(), Err::kBindError, "parameter count does not match the declaration");
    CK(cudaSetDevice(dev_));
    if (n) CK(cudaMemcpyAsync(params_d_, p, size_t(n) * sizeof(double), cudaMemcpyHostToDevice, st_));
    CK(cudaStreamSynchronize(st_));
    // Kernels read parameters from their (graph-captured) launch arguments:
    // new values invalidate the captured stage graphs.
    std::vector<double> nv(p, p + n);
    if (params_bound_ && nv != params_h_) invalidate_graphs();
    params_h_ = nv;
    params_bound_ = true;
  }
  void bind_graph(int i, const uint64_t* verts, int64_t n, int arity) override {
    check(i >= 0 && size_t(i) < P_.graphs.size(), Err::kBindError, "graph count does not match the declaration");
    GraphData& g = graphs_[size_t(i)];
    g.arity = arity;
    g.verts.assign(verts, verts + n);
    g.bound = true;
    g.dirty = true;
  }

  // refresh(): solver.hpp:125-168
  // refresh(): solver.hpp:125-168.  Host half (bind validation, graph upload,
  // residual rows) + device half (computed arrays, masks), the latter
  // captured into the per-iteration CUDA graphs.
  void refresh() override {
    Range nv("minopt::refresh");
    refresh_host();
    refresh_device();
    refreshed_ = true;
    jvalid_ = false;  // solver.hpp:167
    // Does any column carry a mask bit?  The PCG vector kernels then test
    // the column mask (and skip fully excluded groups); otherwise they get no
    // mask at all (1 B per column and a load dependency less).  Masks that
    // follow x (exclude programs reading unknowns) and strips (halo bits)
    // always keep it.
    bool any = colmask_ != nullptr;
    if (colmask_ && !sh_.on && !exclude_reads_x()) {
      if (!anyflag_) anyflag_ = dalloc<int>(1);
      CK(cudaMemsetAsync(anyflag_, 0, sizeof(int), st_));
      kl(k_any_byte, dim3(vgrid(P_.num_cols, nsm_)), dim3(MO_THREADS), colmask_, (long long)P_.num_cols, anyflag_);
      int h = 0;
      CK(cudaMemcpyAsync(&h, anyflag_, sizeof(int), cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
      any = h != 0;
    }
    if (any != cm_any_) invalidate_graphs();
    const bool was = cm_any_;
    cm_any_ = any;
    if (any && !was) {  // (refresh_device skipped the lists under the old value)
      build_tile_lists();
      build_group_list();
    }
    // Active counts on the host (masks that do not follow x change only
    // here): the apply and PCG vector grids are sized to the active work,
    // so small problems launch and reduce over fewer blocks (grid-stride
    // loops stay correct for any grid, so a stale count costs speed only).
    gl_count_ = -1;
    tl_count_.assign(P_.gather_sets.size(), -1);
    if (cm_any_ && !exclude_reads_x() && !sh_.on) {
      int gc = -1;
      if (glist_) CK(cudaMemcpyAsync(&gc, glist_, sizeof(int), cudaMemcpyDeviceToHost, st_));
      std::vector<int> tc(P_.gather_sets.size(), -1);
      for (size_t i = 0; i < tiles_.size(); ++i)
        if (tiles_[i]) CK(cudaMemcpyAsync(&tc[i], tiles_[i], sizeof(int), cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
      gl_count_ = gc;
      for (size_t i = 0; i < tc.size(); ++i) tl_count_[i] = tc[i];
    }
  }
  // The column mask the PCG vector kernels read (null: no column is masked).
  const unsigned char* cmv() const { return cm_any_ ? colmask_ : nullptr; }

  // Do the exclusion programs read the unknowns (or computed arrays)?  If
  // not, the masks only change when arrays are re-bound.
  bool exclude_reads_x() const {
    for (const ExcludeKernel& ek : P_.exclude_kernels)
      for (const Instr& in : ek.prog.instrs)
        if (in.op == kLoadU || in.op == kLoadC || in.op == kLoadP) return true;
    return false;
  }
  void refresh_device(bool masks = true) {
    for (const ComputedKernel& ck : P_.computed_kernels) {
      mo_kparams kp = kp_grid(ck.dom, x_, nullptr);
      kp.out0 = comp_[size_t(ck.index)];
      launch_grid("mo_computed_" + std::to_string(&ck - P_.computed_kernels.data()), ck.dom, kp);
    }
    exchange_computed();
    if (!masks) return;
    for (size_t i = 0; i < P_.exclude_kernels.size(); ++i) {
      const ExcludeKernel& ek = P_.exclude_kernels[i];
      mo_kparams kp = kp_grid(ek.dom, x_, nullptr);
      kp.out0 = masks_[i];
      launch_grid("mo_exclude_" + std::to_string(i), ek.dom, kp);
    }
    if (colmask_) {
      CK(cudaMemsetAsync(colmask_, 0, size_t(P_.num_cols), st_));
      for (size_t i = 0; i < P_.exclude_kernels.size(); ++i)
        for (size_t f = 0; f < P_.unknowns.size(); ++f) {
          if (!(P_.unknowns[f].dom == P_.exclude_kernels[i].dom)) continue;
          long long ne = lext(P_.unknowns[f].dom);
          kl(k_colmask, dim3(vgrid(ne, nsm_)), dim3(MO_THREADS), ne, P_.unknowns[f].channels, masks_[i],
                                                           colmask_ + P_.ubase[f]);
          ++launches_;
        }
      if (sh_.on) mark_halo_cols();  // bit 1: halo column, skipped by vector kernels
    }
    build_tile_lists();
    build_group_list();
  }
  // Active 4-column groups of an unsharded problem with excluded columns
  // (mo_for_groups, mo_kernels.cuh): the PCG vector kernels walk this list
  // instead of streaming the column mask over every group.
  void build_group_list() {
    if (sh_.on || !colmask_ || !cm_any_ || std::getenv("MO_B200_NO_GROUP_LIST")) return;
    const long long n4 = P_.num_cols >> 2;
    if (n4 <= 0 || n4 >= (1LL << 31)) return;
    if (!glist_) {
      glist_ = dalloc<int>(size_t(n4) + 1);
      gvals_ = dalloc<int>(size_t(n4));
      gflags_ = dalloc<unsigned char>(size_t(n4));
      CK(cub::DeviceSelect::Flagged(nullptr, gl_temp_bytes_, gvals_, gflags_, glist_ + 1, glist_, int(n4), st_));
      CK(cudaMalloc(&gl_temp_, gl_temp_bytes_));
    }
    kl(k_group_flags, dim3(vgrid(n4, nsm_, 8)), dim3(MO_THREADS), (const unsigned char*)colmask_, n4, gvals_, gflags_);
    size_t bytes = gl_temp_bytes_;
    CK(cub::DeviceSelect::Flagged(gl_temp_, bytes, gvals_, gflags_, glist_ + 1, glist_, int(n4), st_));
    launches_ += 2;
  }
  // The active-group list the PCG vector kernels walk (null: stream the mask).
  const int* gl() const { return cm_any_ && !sh_.on ? glist_ : nullptr; }
  // Tiles (mo_tile_at numbering of the strip / domain rows) with at least
  // one non-excluded element, per gather set on a masked domain:
  // tiles_[i] = [count, ids ascending].  Rebuilt whenever the masks are.
  static int host_tiles(const mo_kparams& k) {
    const int rows = k.row1 - k.row0;
    if (rows <= 0) return 0;
    if (k.dnd == 1) return (rows + MO_THREADS - 1) / MO_THREADS;
    const int fx = k.dnd == 2 ? k.d1 : k.d2;
    const int ntx = (fx + MO_TILE_X - 1) / MO_TILE_X;
    return ntx * (k.dnd == 2 ? (rows + MO_TILE_Y - 1) / MO_TILE_Y : rows * ((k.d1 + MO_TILE_Y - 1) / MO_TILE_Y));
  }
  void build_tile_lists() {
    if (std::getenv("MO_B200_NO_TILE_LIST") || !cm_any_) return;  // (nothing excluded: every tile active)
    tiles_.resize(P_.gather_sets.size(), nullptr);
    tflags_.resize(P_.gather_sets.size(), nullptr);
    for (size_t i = 0; i < P_.gather_sets.size(); ++i) {
      const mo_kparams kp = kp_grid(P_.gather_sets[i].dom, x_, nullptr);
      if (!kp.mask) continue;
      const int nt = host_tiles(kp);
      if (nt <= 0) continue;
      if (!tiles_[i]) {
        tiles_[i] = dalloc<int>(size_t(nt) + 1);
        tflags_[i] = dalloc<unsigned char>(size_t(nt));
        size_t need = 0;
        CK(cub::DeviceSelect::Flagged(nullptr, need, thrust::counting_iterator<int>(0), tflags_[i], tiles_[i] + 1,
                                      tiles_[i], nt, st_));
        if (need > tl_temp_bytes_) {
          if (tl_temp_) cudaFree(tl_temp_);
          CK(cudaMalloc(&tl_temp_, need));
          tl_temp_bytes_ = need;
        }
      }
      kl(k_tile_active, dim3(std::min(nt, nsm_ * 8)), dim3(MO_TILE_X, MO_TILE_Y), kp, tflags_[i], nt);
      size_t bytes = tl_temp_bytes_;
      CK(cub::DeviceSelect::Flagged(tl_temp_, bytes, thrust::counting_iterator<int>(0), tflags_[i], tiles_[i] + 1,
                                    tiles_[i], nt, st_));
      launches_ += 2;
    }
  }

  void refresh_host() {
    CK(cudaSetDevice(dev_));
    validate();
    upload_graphs();
    // Residual row offsets (graph sizes may change through callbacks).
    rowbase_.assign(P_.residuals.size(), 0);
    int64_t row = 0;
    for (size_t t = 0; t < P_.residuals.size(); ++t) {
      rowbase_[t] = row;
      const Residual& r = P_.residuals[t];
      row += r.graph ? graphs_[size_t(r.graph_idx)].E : P_.extent_of(r.dom);
    }
    rows_ = row;
    if (mat_) mat_prepare();
    if (rowbase_ == rowbase_dev_) {  // unchanged since the last upload
      refreshed_ = true;
      return;
    }
    rowbase_dev_ = rowbase_;
    for (size_t i = 0; i < P_.grid_sets.size(); ++i) {
      std::vector<long long> rb;
      for (int t : P_.grid_sets[i].templates) rb.push_back(rowbase_[size_t(t)]);
      CK(cudaMemcpyAsync(grid_rowbase_[i], rb.data(), rb.size() * sizeof(long long), cudaMemcpyHostToDevice, st_));
      CK(cudaStreamSynchronize(st_));
    }
    for (size_t i = 0; i < P_.graph_sets.size(); ++i) {
      std::vector<long long> rb;
      for (int t : P_.graph_sets[i].templates) rb.push_back(rowbase_[size_t(t)]);
      CK(cudaMemcpyAsync(gsets_[i].rowbase, rb.data(), rb.size() * sizeof(long long), cudaMemcpyHostToDevice, st_));
      CK(cudaStreamSynchronize(st_));
    }
    refreshed_ = true;
  }

  int64_t num_cols() const override { return P_.num_cols; }
  int64_t num_rows() override {
    ensure_refreshed();
    return rows_;
  }
  void excluded(uint8_t* out, int64_t n) override {
    ensure_refreshed();
    check(n == P_.num_cols, Err::kShapeMismatch, "excluded(): size mismatch");
    if (!colmask_) {
      std::memset(out, 0, size_t(n));
      return;
    }
    CK(cudaMemcpyAsync(out, colmask_, size_t(n), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    // bit 1 marks strip halo columns (internal); the reference's excluded()
    // is 0/1 (solver.hpp:619)
    for (int64_t i = 0; i < n; ++i) out[i] &= 1u;
  }

  // ------------------------------------------------------------ routines
  double cost() override {
    Range nv("minopt::cost");
    ensure_refreshed();
    cost_at(x_, SLOT_COST);
    sync_state();
    return state_h_->sums[SLOT_COST];
  }

  void residuals(void* out, int64_t n) override {
    ensure_refreshed();
    check(n == rows_, Err::kShapeMismatch, "residual vector size does not match the instance count");
    if (size_t(n) > resid_cap_) {
      cudaFree(resid_);
      resid_ = dalloc<Real>(size_t(n));
      resid_cap_ = size_t(n);
    }
    for (size_t i = 0; i < P_.grid_sets.size(); ++i) {
      mo_kparams kp = kp_grid(P_.grid_sets[i].dom, x_, nullptr);
      kp.out0 = resid_;
      kp.rowbase = grid_rowbase_[i];
      launch_grid("mo_grid_evalf_" + std::to_string(i), P_.grid_sets[i].dom, kp);
    }
    for (size_t i = 0; i < P_.graph_sets.size(); ++i) {
      mo_kparams kp = kp_graph(int(i), x_, nullptr);
      kp.out0 = resid_;
      kp.rowbase = gsets_[i].rowbase;
      launch_edges("mo_graph_evalf_" + std::to_string(i), int(i), kp);
    }
    if (n) CK(cudaMemcpyAsync(out, resid_, size_t(n) * sizeof(Real), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
  }

  void build_normal() override {
    Range nv("minopt::build_normal");
    ensure_refreshed();
    cur_stage_ = -1;
    normal_device();
    sync_state();
    unconstrained_ = state_h_->unconstrained;
  }
  void get_rhs(void* out, int64_t n) override { download(b_, out, n); }
  void get_precond(void* out, int64_t n) override { download(m_, out, n); }

  void apply_jtj(const void* v, void* out, int64_t n, bool device) override {
    Range nv("minopt::apply_jtj");
    ensure_refreshed();
    tune_apply();
    check(n == P_.num_cols, Err::kShapeMismatch, "apply_jtj(): vector size mismatch");
    lanecache_fill();  // (x may have changed since the last linearisation)
    if (device) {
      apply(static_cast<const Real*>(v), static_cast<Real*>(out), 0);
      CK(cudaStreamSynchronize(st_));
      return;
    }
    if (n) CK(cudaMemcpyAsync(vtmp_, v, size_t(n) * sizeof(Real), cudaMemcpyHostToDevice, st_));
    apply(vtmp_, otmp_, 0);
    download(otmp_, out, n);
  }

  void get_x(void* out, int64_t n) override { download(x_, out, n); }
  bool saw_nonfinite() override {
    sync_state();
    return state_h_->nonfinite_kernel != 0;
  }

  // ------------------------------------------------------------ solve
  SolveResult solve(IterCallback cb, void* user) override {
    Range nv("minopt::solve");
    // Peer reductions spin on the device until every rank has joined: they
    // start with the second solve, once every rank is past the one-time
    // host work of the first (JIT compiles, kernel timing, allocations that
    // wait for the device), which keeps ranks apart for seconds, unevenly.
    struct PeerReady {
      bool& ready;
      bool on;
      ~PeerReady() {
        if (on) ready = true;
      }
    } peer_ready_at_exit{peer_ready_, peer_on_};
    using clock = std::chrono::steady_clock;
    CK(cudaSetDevice(dev_));
    const bool lm = cfg_.method == 1;
    const long long n = P_.num_cols;
    const int vg = vgrid(n, nsm_);
    SolveResult res;
    double mu = cfg_.lm_radius0, nu = 2.0;
    auto t_prev = clock::now();
    auto take_ms = [&] {
      auto now = clock::now();
      double ms = std::chrono::duration<double, std::milli>(now - t_prev).count();
      t_prev = now;
      return ms;
    };
    auto finish = [&] {
      reduce_flags();
      sync_state();
      res.nonfinite_kernels = state_h_->nonfinite_kernel != 0;
      res.unconstrained = unconstrained_;
    };

    refresh_host();
    if (!tuned_) {
      refresh_device();  // bound data in place for the timing runs
      tune_apply();
    }
    for (int it = 0; it < cfg_.nonlinear_iters; ++it) {
      Range nv_it(lm ? "LM iteration" : "GN iteration");
      refresh_host();
      if (!lm) {
        // One GN iteration = one graph, one host sync (solver.hpp:415-464).
        // build_normal/PCG/step run even when cost_old turns out non-finite;
        // the step kernel then leaves x untouched and the host stops exactly
        // where the reference would.
        // cost_old of iteration it > 0 is cost_new of iteration it - 1 (same
        // x, same arrays, no computed arrays to refresh, no callback that
        // could rebind data): reuse it instead of re-evaluating the cost.
        const bool reuse_cost = it > 0 && !cb && P_.computed.empty() && !std::getenv("MO_B200_NO_COST_REUSE");
        run_stage(reuse_cost ? kStageGNNext : kStageGN, [&] {
          // (with reuse_cost no array can have changed since iteration 0, so
          // masks that do not depend on x are still current)
          refresh_device(!reuse_cost || exclude_reads_x());
          if (reuse_cost)
            CK(cudaMemcpyAsync(&state_->sums[SLOT_COST], &state_->sums[SLOT_COST + 1], sizeof(double),
                               cudaMemcpyDeviceToDevice, st_));
          else
            cost_at(x_, SLOT_COST);
          const bool fi = bm_init_ok();
          normal_device(fi);
          if (mat_) linearize_device();  // solver.hpp:426
          pcg_body(false, fi);
          CK(cudaMemsetAsync(&state_->any_nonzero, 0, sizeof(int), st_));
          kl(k_xtrial<Real>, dim3(vg), dim3(MO_THREADS), state_, n, cmv(), x_, delta_, xt_, 1, SLOT_COST);
          ++launches_;
          exchange_cols(x_);
          cost_at(x_, SLOT_COST + 1);
          reduce_flags();
        });
        sync_state();
        if (mat_) {  // (the replayed stage ran linearize)
          check_mat_bad();
          jvalid_ = true;
        }
        collect_profile(reuse_cost ? kStageGNNext : kStageGN);
        const mo_state S = *state_h_;
        const double cost_old = S.sums[SLOT_COST];
        if (!std::isfinite(cost_old)) {
          res.trace.push_back({it, cost_old, false, 0.0, 0, take_ms()});
          res.reason = 3;
          res.final_cost = cost_old;
          finish();
          return res;
        }
        unconstrained_ = S.unconstrained;
        res.indefinite_operator |= S.indefinite != 0;
        if (S.nonfinite) {
          res.reason = 3;
          res.final_cost = cost_old;
          res.trace.push_back({it, cost_old, false, 0.0, S.iters, take_ms()});
          finish();
          return res;
        }
        const double cost_new = S.sums[SLOT_COST + 1];
        res.trace.push_back({it, cost_new, true, 0.0, S.iters, take_ms()});
        if (!std::isfinite(cost_new)) {
          res.reason = 3;
          res.final_cost = cost_new;
          finish();
          return res;
        }
        if (cb) cb(it, user);
        double rel = (cost_old - cost_new) / std::max(cost_old, 1e-300);
        if (rel >= 0 && rel < cfg_.cost_stop_tol) {
          res.reason = 1;
          break;
        }
        continue;
      }

      // LM (solver.hpp:427-501): linearise once, then damped trials.
      run_stage(kStageLMLin, [&] {
        refresh_device();
        cost_at(x_, SLOT_COST);
        normal_device();
        if (mat_) linearize_device();  // solver.hpp:426
        kl(k_lm_base_diag<Real>, dim3(vg), dim3(MO_THREADS), n, m_, bd_, cfg_.lm_diag_min, cfg_.lm_diag_max);
        ++launches_;
      });
      sync_state();
      if (mat_) {
        check_mat_bad();
        jvalid_ = true;
      }
      collect_profile(kStageLMLin);
      const double cost_old = state_h_->sums[SLOT_COST];
      if (!std::isfinite(cost_old)) {
        res.trace.push_back({it, cost_old, false, mu, 0, take_ms()});
        res.reason = 3;
        res.final_cost = cost_old;
        finish();
        return res;
      }
      unconstrained_ = state_h_->unconstrained;
      double cost_after = cost_old;
      bool stepped = false;
      while (!stepped) {
        *mu_h_ = mu;
        CK(cudaMemcpyAsync(&state_->mu, mu_h_, sizeof(double), cudaMemcpyHostToDevice, st_));
        run_stage(kStageLMTrial, [&] {
          kl(k_lm_damp<Real>, dim3(vg), dim3(MO_THREADS), state_, n, colmask_, m_, bd_, damp_, md_);
          ++launches_;
          pcg_body(true);
          CK(cudaMemsetAsync(&state_->any_nonzero, 0, sizeof(int), st_));
          kl(k_xtrial<Real>, dim3(vg), dim3(MO_THREADS), state_, n, colmask_, x_, delta_, xt_, 0, SLOT_COST);
          ++launches_;
          exchange_cols(xt_);
          cost_at(xt_, SLOT_COST + 1);
          exchange_cols(delta_);
          apply(delta_, ap_, 0);  // undamped model curvature (solver.hpp:467)
          kl(k_lm_predicted<Real>, dim3(vg), dim3(MO_THREADS), red(0, vg, MO_FIN_STORE2, SLOT_PRED), n, colmask_, b_,
                                                           delta_, ap_);
          ++launches_;
          reduce_done(MO_FIN_STORE2, SLOT_PRED);
          reduce_flags();
        });
        sync_state();
        collect_profile(kStageLMTrial);
        const mo_state S = *state_h_;
        res.indefinite_operator |= S.indefinite != 0;
        const double cost_new = S.nonfinite ? std::numeric_limits<double>::infinity() : S.sums[SLOT_COST + 1];
        double predicted = 0.0 - S.sums[SLOT_PRED + 1];
        predicted += S.sums[SLOT_PRED];
        double rho = predicted > 0 ? (cost_old - cost_new) / predicted : -1.0;
        if (std::isfinite(cost_new) && predicted > 0 && rho > cfg_.lm_min_decrease) {
          CK(cudaMemcpyAsync(x_, xt_, size_t(n) * sizeof(Real), cudaMemcpyDeviceToDevice, st_));
          double shrink = std::max(1.0 / 3.0, 1.0 - std::pow(2.0 * rho - 1.0, 3));
          res.trace.push_back({it, cost_new, true, mu, S.iters, take_ms()});
          mu = std::clamp(mu / shrink, cfg_.lm_radius_min, cfg_.lm_radius_max);
          nu = 2.0;
          cost_after = cost_new;
          stepped = true;
        } else {
          res.trace.push_back({it, cost_new, false, mu, S.iters, take_ms()});
          const bool zero_step = S.any_nonzero == 0;
          mu /= nu;
          nu *= 2.0;
          if (zero_step || mu < cfg_.lm_radius_min) {
            res.reason = 2;
            res.final_cost = cost_old;
            finish();
            return res;
          }
        }
      }
      if (cb) {
        CK(cudaStreamSynchronize(st_));
        cb(it, user);
      }
      double rel = (cost_old - cost_after) / std::max(cost_old, 1e-300);
      if (rel >= 0 && rel < cfg_.cost_stop_tol) {
        res.reason = 1;
        break;
      }
    }
    refresh();
    res.final_cost = cost();
    if (!std::isfinite(res.final_cost)) res.reason = 3;
    finish();
    return res;
  }

  // ------------------------------------------------------------ profiling
  void set_profiling(bool on) override {
    profiling_ = on;
    invalidate_graphs();
  }
  void profile_read(int kind, double* ms, int64_t* n) override {
    check(kind >= 0 && kind < 4, Err::kBindError, "profile kind out of range");
    *ms = prof_[size_t(kind)].total_ms;
    *n = prof_[size_t(kind)].count;
  }
  void profile_reset() override {
    for (auto& p : prof_) {
      p.total_ms = 0;
      p.count = 0;
    }
  }
  // Unperturbed kernel timing for the roofline (bench.py): `reps` launches
  // of the J^T J p apply (which = 0, on the session's p, as a PCG iteration
  // launches it) or of build_normal (which = 1) captured as one CUDA graph,
  // best of 3 replays; ms per launch.  Clobbers the PCG scratch vectors.
  double bench_kernel(int which, int reps) override {
    check(which == 0 || which == 1, Err::kBindError, "bench_kernel: which must be 0 (apply) or 1 (build_normal)");
    check(reps >= 1 && reps <= 1000, Err::kBindError, "bench_kernel: reps out of range");
    ensure_refreshed();
    tune_apply();
    const int stage = cur_stage_;
    cur_stage_ = -1;  // no profiling events
    const int64_t launched = launches_;
    const bool cons = !sh_.on && !mat_ && (P_.graph_sets.empty() || vertex_apply_one_pass());
    float ms = 0;
    if (which == 0) {
      lanecache_fill();
      auto body = [&] {
        for (int r = 0; r < reps; ++r) {
          consumer_ = cons;
          apply(p_, ap_, MO_F_REDUCE | MO_F_ZEROEXCL | MO_F_EXSKIP);
          consumer_ = false;
        }
      };
      body();  // warm-up (tensor maps, module load)
      ms = time_graph(body);
    } else {
      normal_device();
      ms = time_graph([&] {
        for (int r = 0; r < reps; ++r) normal_device();
      });
    }
    CK(cudaStreamSynchronize(st_));
    launches_ = launched;
    cur_stage_ = stage;
    return double(ms) / reps;
  }
  void* stream() override { return st_; }
  int64_t launches() const override { return launches_; }
  std::string apply_kernel(int i) override {
    check(i >= 0 && size_t(i) < P_.gather_sets.size(), Err::kIndexOutOfRange, "no such gather set");
    ensure_refreshed();
    tune_apply();
    if (mat_) return "k_mat_cols";
    if (vertex_apply_one_pass()) return "mo_graph_vjtjf_0";
    return jtj_kernel(size_t(i));
  }
  std::string normal_kernel(int i) override {
    check(i >= 0 && size_t(i) < P_.gather_sets.size(), Err::kIndexOutOfRange, "no such gather set");
    ensure_refreshed();
    tune_apply();
    if (!P_.graph_sets.empty() && vertex_path(0)) return "mo_graph_vbm_0";
    const int bc = bm_choice_.size() > size_t(i) ? bm_choice_[size_t(i)] : 0;
    if (bc == 2 && bm8c_fuses(size_t(i))) return "mo_gather_bm8c_" + std::to_string(i);
    return (bc == 2 ? "mo_gather_bm8_" : bc == 1 ? "mo_gather_bm4_" : "mo_gather_bm_") +
           std::to_string(i);
  }

 private:
  using ArrayFieldSize = int64_t;
  struct GraphData {
    int arity = -1;
    std::vector<uint64_t> verts;
    int64_t E = 0;      // edges stored (a strip: every edge touching its rows)
    int64_t E_own = 0;  // of which this strip evaluates for cost (slot-0 vertex owned; stored first)
    bool bound = false, dirty = true;
    int* d_verts = nullptr;
    size_t cap = 0;
  };
  struct GatherDom {
    Domain dom;
    int64_t nverts = 0;
    std::vector<int> slots;  // slots whose outputs target this domain
    int* vptr = nullptr;
    int* vedge = nullptr;
    size_t vedge_cap = 0;
    mo_gather_out* outs_bm = nullptr;
    mo_gather_out* outs_jtj = nullptr;
  };
  struct GSet {
    Real* contrib = nullptr;
    size_t cap = 0;
    long long* rowbase = nullptr;
    std::vector<GatherDom> doms;
    std::vector<int64_t> slot_bound;
  };
  struct Prof {
    double total_ms = 0;
    int64_t count = 0;
  };
  struct ProfEv {
    int kind = 0;
    cudaEvent_t a = nullptr, b = nullptr;
  };
  enum { kStageGN = 0, kStageLMLin = 1, kStageLMTrial = 2, kStageGNNext = 3 };

  // ------------------------------------------------------------ sharding
  struct Shard {
    bool on = false;
    Domain dom;
    int64_t d0 = 0, S = 1;  // axis-0 extent, elements per row
    int64_t row0 = 0, row1 = 0, lo = 0, hi = 0;
    int R = 0;
  };

  // Graph energies shard too when their vertices are the elements of the one
  // domain: a strip holds every edge with an endpoint in its rows; `halo`
  // (>= the plan's) must cover the graph's row bandwidth (checked at upload).
  void setup_shard(int64_t row0, int64_t row1, int halo) {
    const Domain* D = nullptr;
    auto same = [&](const Domain& d) {
      if (!D) D = &d;
      check(d == *D, Err::kBindError, "strip sharding needs every field on one grid domain");
    };
    for (const Field& f : P_.unknowns) same(f.dom);
    for (const Field& f : P_.arrays) same(f.dom);
    for (const Field& f : P_.computed) same(f.dom);
    for (const GridSet& g : P_.grid_sets) same(g.dom);
    for (const GatherSet& g : P_.gather_sets) same(g.dom);
    for (const ExcludeKernel& e : P_.exclude_kernels) same(e.dom);
    check(D && !D->dims.empty(), Err::kBindError, "strip sharding needs a grid domain");
    sh_.dom = *D;
    sh_.d0 = P_.shape_of(*D)[0];
    sh_.S = P_.extent_of(*D) / std::max<int64_t>(sh_.d0, 1);
    if (row1 < 0) row1 = sh_.d0;
    check(row0 >= 0 && row0 < row1 && row1 <= sh_.d0, Err::kBindError, "strip rows out of range");
    sh_.R = std::max(halo_rows(P_), halo);
    check(comm_->world == 1 || row1 - row0 >= sh_.R, Err::kBindError, "strip thinner than the halo");
    sh_.row0 = row0;
    sh_.row1 = row1;
    sh_.lo = std::max<int64_t>(0, row0 - sh_.R);
    sh_.hi = std::min<int64_t>(sh_.d0, row1 + sh_.R);
    sh_.on = true;
    int64_t col = 0;  // local column layout: each field's [lo, hi) rows, field-major
    for (size_t f = 0; f < P_.unknowns.size(); ++f) {
      P_.ubase[f] = col;
      col += lext(P_.unknowns[f].dom) * P_.unknowns[f].channels;
    }
    P_.num_cols = col;
  }
  // Local (stored) element count of a domain.
  int64_t lext(const Domain& d) const {
    return sh_.on && d == sh_.dom ? (sh_.hi - sh_.lo) * sh_.S : P_.extent_of(d);
  }
  HaloSeg seg(void* base, size_t row_bytes) const {
    HaloSeg s;
    s.base = static_cast<char*>(base);
    s.row_bytes = row_bytes;
    s.top = int(sh_.row0 - sh_.lo);
    s.owned = int(sh_.row1 - sh_.row0);
    s.bottom = int(sh_.hi - sh_.row1);
    s.send_up = int(std::min<int64_t>(sh_.d0, sh_.row0 + sh_.R) - sh_.row0);
    s.send_down = int(std::min<int64_t>(sh_.R, sh_.row1));
    if (comm_->rank == 0) s.send_up = 0;
    if (comm_->rank == comm_->world - 1) s.send_down = 0;
    return s;
  }
  // Halo rows of a column-layout vector (p, x, x_trial, delta).
  void exchange_cols(Real* v, cudaStream_t s = nullptr) {
    if (!sh_.on) return;
    std::vector<HaloSeg> segs;
    for (size_t f = 0; f < P_.unknowns.size(); ++f)
      segs.push_back(seg(v + P_.ubase[f], size_t(sh_.S) * size_t(P_.unknowns[f].channels) * sizeof(Real)));
    comm_->halo(segs, s ? s : st_);
  }
  void exchange_computed() {
    if (!sh_.on || comp_.empty()) return;
    std::vector<HaloSeg> segs;
    for (size_t c = 0; c < comp_.size(); ++c)
      segs.push_back(seg(comp_[c], size_t(sh_.S) * size_t(P_.computed[c].channels) * sizeof(Real)));
    comm_->halo(segs, st_);
  }
  // After the kernels of one reduction: every rank's partial is gathered in
  // rank order and finalised identically everywhere (deterministic).
  void reduce_done(int op, int arg) {
    if (!sh_.on) return;
    if (peer_on_ && peer_ready_) {
      kl(k_peer_fin<Real>, dim3(1), dim3(64), state_, peer_, rankbuf_, op, arg, 0);
      ++launches_;
      return;
    }
    comm_->allgather(&state_->sums[4], rankbuf_, 2, st_);
    kl(k_global_fin<Real>, dim3(1), dim3(32), state_, rankbuf_, comm_->world, op, arg);
    ++launches_;
  }
  void reduce_flags() {
    if (!sh_.on) return;
    if (peer_on_ && peer_ready_) {
      kl(k_peer_fin<Real>, dim3(1), dim3(64), state_, peer_, rankbuf_, 0, 0, 1);
      ++launches_;
      return;
    }
    kl(k_flags_out, dim3(1), dim3(1), state_);
    comm_->allgather(&state_->sums[4], rankbuf_, 2, st_);
    kl(k_flags_in, dim3(1), dim3(1), state_, rankbuf_, comm_->world);
    launches_ += 2;
  }
  void mark_halo_cols() {
    for (size_t f = 0; f < P_.unknowns.size(); ++f) {
      const long long rowc = sh_.S * P_.unknowns[f].channels;
      const long long top = (sh_.row0 - sh_.lo) * rowc, own = (sh_.row1 - sh_.row0) * rowc;
      const long long bot = (sh_.hi - sh_.row1) * rowc;
      unsigned char* base = colmask_ + P_.ubase[f];
      if (top) kl(k_or_bits, dim3(vgrid(top, nsm_)), dim3(MO_THREADS), base, top, 2);
      if (bot) kl(k_or_bits, dim3(vgrid(bot, nsm_)), dim3(MO_THREADS), base + top + own, bot, 2);
      launches_ += (top ? 1 : 0) + (bot ? 1 : 0);
    }
  }

 public:
  void local_layout(int64_t* lo, int64_t* hi, int64_t* row0, int64_t* row1) const override {
    *lo = sh_.on ? sh_.lo : 0;
    *hi = sh_.on ? sh_.hi : 0;
    *row0 = sh_.on ? sh_.row0 : 0;
    *row1 = sh_.on ? sh_.row1 : 0;
  }

 private:
  int64_t array_size(int i) const {
    return lext(P_.arrays[size_t(i)].dom) * P_.arrays[size_t(i)].channels;
  }

  void ensure_refreshed() {
    if (!refreshed_) refresh();
  }

  // validate(): solver.hpp:529-546
  void validate() {
    check(x_bound_, Err::kBindError, "unknown vector size does not match the plan layout");
    check(params_bound_ || P_.params.empty(), Err::kBindError, "parameter count does not match the declaration");
    for (size_t i = 0; i < P_.arrays.size(); ++i)
      check(arr_n_[i] == array_size(int(i)), Err::kBindError,
            "array '" + P_.arrays[i].name + "' has the wrong size");
    for (size_t i = 0; i < P_.graphs.size(); ++i) {
      check(graphs_[i].bound, Err::kBindError, "graph count does not match the declaration");
      check(graphs_[i].arity == P_.graphs[i].second, Err::kBindError,
            "graph '" + P_.graphs[i].first + "' arity does not match the declaration");
    }
  }

  void setup_graph_set(int gi) {
    const GraphSet& g = P_.graph_sets[size_t(gi)];
    GSet& gs = gsets_[size_t(gi)];
    gs.rowbase = dalloc<long long>(std::max<size_t>(g.templates.size(), 1));
    const int ar = P_.graphs[size_t(g.graph)].second;
    // Vertex bounds per slot: fields read through the slot and scatter
    // targets (exec.hpp:238-259).
    gs.slot_bound.assign(size_t(std::max(ar, 1)), INT64_MAX);
    for (const Program* pg : {&g.cost, &g.evalf, &g.bm, &g.jtj})
      for (const Instr& in : pg->instrs) {
        if (in.op != kLoadU && in.op != kLoadA && in.op != kLoadC && in.op != kLoadP) continue;
        if (!in.graph) continue;
        check(in.slot >= 0 && in.slot < ar, Err::kShapeMismatch, "kernel reads a slot beyond the edge arity");
        const Field* f = in.op == kLoadA ? &P_.arrays[size_t(in.field)]
                        : in.op == kLoadC ? &P_.computed[size_t(in.field)]
                                          : &P_.unknowns[size_t(in.field)];
        gs.slot_bound[size_t(in.slot)] = std::min(gs.slot_bound[size_t(in.slot)], P_.extent_of(f->dom));
      }
    for (const Scat& s : g.scats) {
      check(s.slot >= 0 && s.slot < ar, Err::kShapeMismatch, "graph output scatters through a slot beyond the edge arity");
      gs.slot_bound[size_t(s.slot)] =
          std::min(gs.slot_bound[size_t(s.slot)], P_.extent_of(P_.unknowns[size_t(s.field)].dom));
    }
    // One gather launch per target domain.
    for (const Scat& s : g.scats) {
      const Domain& d = P_.unknowns[size_t(s.field)].dom;
      GatherDom* gd = nullptr;
      for (auto& x : gs.doms)
        if (x.dom == d) gd = &x;
      if (!gd) {
        gs.doms.push_back({});
        gd = &gs.doms.back();
        gd->dom = d;
        gd->nverts = lext(d);  // (a strip: its stored rows, local vertex ids)
      }
      if (std::find(gd->slots.begin(), gd->slots.end(), s.slot) == gd->slots.end()) gd->slots.push_back(s.slot);
    }
    const size_t K = g.scats.size();
    for (auto& gd : gs.doms) {
      std::vector<mo_gather_out> obm(2 * K), ojtj(K);
      for (size_t k = 0; k < K; ++k) {
        const Scat& s = g.scats[k];
        const UnknownLike u = unknown(s.field);
        mo_gather_out o{};
        o.slot = s.slot;
        o.C = u.channels;
        o.active = P_.unknowns[size_t(s.field)].dom == gd.dom;
        o.cbase = P_.ubase[size_t(s.field)] + s.channel;
        o.sel = 0;
        ojtj[k] = o;
        obm[2 * k] = o;
        o.sel = 1;
        obm[2 * k + 1] = o;
      }
      gd.outs_bm = dalloc<mo_gather_out>(2 * K);
      gd.outs_jtj = dalloc<mo_gather_out>(K);
      gd.vptr = dalloc<int>(size_t(gd.nverts) + 1);
      if (K) {
        CK(cudaMemcpyAsync(gd.outs_bm, obm.data(), obm.size() * sizeof(mo_gather_out), cudaMemcpyHostToDevice, st_));
        CK(cudaMemcpyAsync(gd.outs_jtj, ojtj.data(), ojtj.size() * sizeof(mo_gather_out), cudaMemcpyHostToDevice, st_));
      }
      CK(cudaStreamSynchronize(st_));
    }
  }
  struct UnknownLike {
    int channels;
  };
  UnknownLike unknown(int f) const { return {P_.unknowns[size_t(f)].channels}; }

  // Upload changed graphs: int32 vertex table, contribution buffers and the
  // per-domain incidence CSR (edges ascending) of the deterministic gather.
  void upload_graphs() {
    for (size_t gi = 0; gi < graphs_.size(); ++gi) {
      GraphData& g = graphs_[gi];
      if (!g.dirty) continue;
      g.E = g.arity > 0 ? int64_t(g.verts.size()) / g.arity : 0;
      const size_t ne = g.verts.size();
      if (ne > g.cap) {
        cudaFree(g.d_verts);
        g.d_verts = dalloc<int>(ne);
        g.cap = ne;
        invalidate_graphs();
      }
      // Vertex validation before any write (exec.hpp:255-259).
      for (size_t si = 0; si < P_.graph_sets.size(); ++si) {
        if (P_.graph_sets[si].graph != int(gi)) continue;
        const GSet& gs = gsets_[si];
        for (int64_t e = 0; e < g.E; ++e)
          for (int s = 0; s < g.arity; ++s)
            check(g.verts[size_t(e * g.arity + s)] < uint64_t(gs.slot_bound[size_t(s)]), Err::kIndexOutOfRange,
                  "edge references a vertex beyond the bound extent");
      }
      std::vector<int> v32(ne);
      for (size_t k = 0; k < ne; ++k) {
        check(g.verts[k] < (uint64_t(1) << 31), Err::kIndexOutOfRange, "vertex index exceeds int32");
        v32[k] = int(g.verts[k]);
      }
      g.E_own = g.E;
      std::vector<int> ord;  // local edges in global edge order (the gathers' accumulation order)
      if (sh_.on) {  // strip: edges touching the owned rows, local vertex ids, owned edges first
        const int64_t a = sh_.row0 * sh_.S, b = sh_.row1 * sh_.S, la = sh_.lo * sh_.S, lb = sh_.hi * sh_.S;
        std::vector<int> own, other;
        for (int64_t e = 0; e < g.E; ++e) {
          bool touch = false;
          for (int k = 0; k < g.arity; ++k) {
            const int64_t v = v32[size_t(e * g.arity + k)];
            touch = touch || (v >= a && v < b);
          }
          if (!touch) continue;
          for (int k = 0; k < g.arity; ++k) {
            const int64_t v = v32[size_t(e * g.arity + k)];
            check(v >= la && v < lb, Err::kBindError, "graph edge spans more rows than the strip halo");
          }
          const int64_t v0 = v32[size_t(e * g.arity)];
          (v0 >= a && v0 < b ? own : other).push_back(int(e));
        }
        std::vector<int> loc;
        loc.reserve((own.size() + other.size()) * size_t(g.arity));
        for (const std::vector<int>* lst : {&own, &other})
          for (int e : *lst)
            for (int k = 0; k < g.arity; ++k) loc.push_back(int(v32[size_t(e * g.arity + k)] - la));
        v32.swap(loc);
        g.E = int64_t(own.size() + other.size());
        g.E_own = int64_t(own.size());
        size_t i = 0, j = 0;
        while (i < own.size() || j < other.size()) {
          if (j == other.size() || (i < own.size() && own[i] < other[j])) ord.push_back(int(i++));
          else ord.push_back(int(own.size() + j++));
        }
      } else {
        ord.resize(size_t(g.E));
        for (int64_t e = 0; e < g.E; ++e) ord[size_t(e)] = int(e);
      }
      const size_t nl = v32.size();
      if (nl) CK(cudaMemcpyAsync(g.d_verts, v32.data(), nl * sizeof(int), cudaMemcpyHostToDevice, st_));
      for (size_t si = 0; si < P_.graph_sets.size(); ++si) {
        const GraphSet& gset = P_.graph_sets[si];
        if (gset.graph != int(gi)) continue;
        GSet& gs = gsets_[si];
        const size_t no = std::max<size_t>(gset.bm.outputs.size(), 1);
        if (size_t(g.E) * no > gs.cap) {
          cudaFree(gs.contrib);
          gs.contrib = dalloc<Real>(size_t(g.E) * no);
          gs.cap = size_t(g.E) * no;
          invalidate_graphs();
        }
        for (auto& gd : gs.doms) {
          std::vector<int> cnt(size_t(gd.nverts) + 1, 0), last(size_t(gd.nverts), -1);
          for (int e : ord)
            for (int s : gd.slots) {
              int v = v32[size_t(e * g.arity + s)];
              if (last[size_t(v)] != int(e)) {
                last[size_t(v)] = int(e);
                cnt[size_t(v) + 1]++;
              }
            }
          for (size_t v = 0; v < size_t(gd.nverts); ++v) cnt[v + 1] += cnt[v];
          std::vector<int> vedge(static_cast<size_t>(cnt[static_cast<size_t>(gd.nverts)]));
          std::vector<int> pos(cnt.begin(), cnt.end() - 1);
          std::fill(last.begin(), last.end(), -1);
          for (int e : ord)
            for (int s : gd.slots) {
              int v = v32[size_t(e * g.arity + s)];
              if (last[size_t(v)] != int(e)) {
                last[size_t(v)] = int(e);
                vedge[size_t(pos[size_t(v)]++)] = int(e);
              }
            }
          if (vedge.size() > gd.vedge_cap) {
            cudaFree(gd.vedge);
            gd.vedge = dalloc<int>(vedge.size());
            gd.vedge_cap = vedge.size();
            invalidate_graphs();
          }
          CK(cudaMemcpyAsync(gd.vptr, cnt.data(), cnt.size() * sizeof(int), cudaMemcpyHostToDevice, st_));
          if (!vedge.empty())
            CK(cudaMemcpyAsync(gd.vedge, vedge.data(), vedge.size() * sizeof(int), cudaMemcpyHostToDevice, st_));
        }
      }
      CK(cudaStreamSynchronize(st_));
      invalidate_graphs();  // edge counts are baked into the captured PCG graph
      g.dirty = false;
      mt_dirty_ = true;
    }
  }

  void invalidate_graphs() {
    for (auto& kv : stage_exec_) cudaGraphExecDestroy(kv.second);
    stage_exec_.clear();
  }

  void* arena_ = nullptr;
  size_t arena_bytes_ = 0;

  // materialized J (linearize / Materialize::kJ)
  int mat_ = 0;
  bool jvalid_ = false, mt_dirty_ = true, mt_ok_ = false, csr_ok_ = false;
  Module mod_evj_;
  std::vector<Real*> jl_grid_, jl_graph_;
  std::vector<long long*> jl_rb_grid_, jl_rb_graph_;
  std::vector<size_t> jl_graph_cap_;
  std::vector<int*> mat_vptr_, mat_vedge_;
  std::vector<long long> mat_nverts_;
  std::vector<int64_t> mt_rowbase_;
  std::vector<void*> mt_bufs_;
  mo_mat_tables mt_{};
  Real* jtmp_ = nullptr;
  size_t jtmp_cap_ = 0;
  size_t mt_smem_ = 0;         // staged table bytes (mo_mat_stage)
  long long max_trows_ = 1, max_fel_ = 1;
  int* ecol_ = nullptr;  // kJtJ: merged graph rows (k_mat_erows)
  Real* eval_ = nullptr;
  unsigned char* ecnt_ = nullptr;
  size_t erow_cap_ = 0, ecnt_cap_ = 0;
  bool has_graph_rows_ = false;
  int* hcol_ = nullptr;  // kJtJ: H = 2 J^T J, slot-major ELL (int32 columns)
  Real* hval_ = nullptr;
  int* hcnt_ = nullptr;
  int hK_ = 0;
  size_t hn_ = 0;
  std::vector<int64_t> csr_offs_, csr_col_;
  std::vector<Real> csr_val_;

  // ------------------------------------------------------------ launches
  // Every kernel of the solver goes through kl()/klc() with the
  // programmatic-stream-serialization attribute: each kernel starts with
  // griddepcontrol.wait (MO_PDL_ENTRY) and triggers its successor only
  // implicitly at exit, so the successor's launch overlaps the drain of the
  // predecessor (measured -0.5..-1.5% per iteration on B200; an early
  // explicit trigger was 3-8% slower).  MO_B200_NO_PDL=1 launches plainly.
  static bool pdl_on() {
    static const bool on = std::getenv("MO_B200_NO_PDL") == nullptr;
    return on;
  }
  cudaLaunchConfig_t launch_cfg(dim3 grid, dim3 block, size_t smem, cudaLaunchAttribute* at) const {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = st_;
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl_on() ? 1 : 0;
    return lc;
  }
  template <class... K, class... A>
  void kl(void (*k)(K...), dim3 grid, dim3 block, A&&... a) {
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t lc = launch_cfg(grid, block, 0, at);
    CK(cudaLaunchKernelEx(&lc, k, std::forward<A>(a)...));
  }
  template <class... K, class... A>
  void kls(void (*k)(K...), dim3 grid, dim3 block, size_t smem, A&&... a) {
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t lc = launch_cfg(grid, block, smem, at);
    CK(cudaLaunchKernelEx(&lc, k, std::forward<A>(a)...));
  }
  void klc(const void* f, dim3 grid, dim3 block, void** args, size_t smem) {
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t lc = launch_cfg(grid, block, smem, at);
    CK(cudaLaunchKernelExC(&lc, f, args));
  }
  mo_kparams kp_base(const Real* xv, const Real* pv) {
    mo_kparams k;
    std::memset(&k, 0, sizeof k);
    const int U = int(P_.unknowns.size()), A = int(P_.arrays.size());
    auto view = [&](const void* ptr, const Field& f) {
      mo_view v{};
      v.p = ptr;
      v.ch = f.channels;
      v.nd = int(f.dom.dims.size());
      auto s = P_.shape_of(f.dom);
      v.s0 = int(s[0]);
      v.s1 = int(s[1]);
      v.s2 = int(s[2]);
      v.row_lo = sh_.on ? int(sh_.lo) : 0;
      return v;
    };
    for (int f = 0; f < U; ++f) {
      k.v[f] = view(xv + P_.ubase[size_t(f)], P_.unknowns[size_t(f)]);
      k.v[U + f] = view(pv ? pv + P_.ubase[size_t(f)] : nullptr, P_.unknowns[size_t(f)]);
      k.ubase[f] = P_.ubase[size_t(f)];
    }
    for (int a = 0; a < A; ++a) k.v[2 * U + a] = view(arr_[size_t(a)], P_.arrays[size_t(a)]);
    for (size_t c = 0; c < P_.computed.size(); ++c) k.v[2 * U + A + int(c)] = view(comp_[c], P_.computed[c]);
    k.params = params_d_;
    for (size_t i = 0; i < params_h_.size() && i < MO_MAX_PARAMS; ++i) k.pv[i] = params_h_[i];
    k.colmask = colmask_;
    k.state = state_;
    return k;
  }
  mo_kparams kp_grid(const Domain& d, const Real* xv, const Real* pv) {
    mo_kparams k = kp_base(xv, pv);
    auto s = P_.shape_of(d);
    k.dnd = std::max<int>(1, int(d.dims.size()));
    k.d0 = int(s[0]);
    k.d1 = int(s[1]);
    k.d2 = int(s[2]);
    k.row0 = sh_.on ? int(sh_.row0) : 0;
    k.row1 = sh_.on ? int(sh_.row1) : int(s[0]);
    k.row_lo = sh_.on ? int(sh_.lo) : 0;
    for (size_t i = 0; i < P_.exclude_kernels.size(); ++i)
      if (P_.exclude_kernels[i].dom == d) k.mask = masks_[i];
    return k;
  }
  mo_kparams kp_graph(int gi, const Real* xv, const Real* pv) {
    mo_kparams k = kp_base(xv, pv);
    const GraphData& g = graphs_[size_t(P_.graph_sets[size_t(gi)].graph)];
    k.dnd = 1;  // graph env: default DomainInfo (shape {1,1,1}, nd 1)
    k.d0 = k.d1 = k.d2 = 1;
    k.verts = g.d_verts;
    k.arity = g.arity;
    k.nedges = g.E_own;  // edge kernels (cost, residuals): the edges this strip owns
    return k;
  }

  int tiles_of(const Domain& d) const {
    auto s = P_.shape_of(d);
    const int nd = std::max<int>(1, int(d.dims.size()));
    long long rows = ov0_ >= 0 ? ov1_ - ov0_ : s[0];
    if (rows <= 0) return 0;
    if (nd == 1) return int((rows + MO_THREADS - 1) / MO_THREADS);
    if (nd == 2) return int(((s[1] + MO_TILE_X - 1) / MO_TILE_X) * ((rows + MO_TILE_Y - 1) / MO_TILE_Y));
    return int(((s[2] + MO_TILE_X - 1) / MO_TILE_X) * rows * ((s[1] + MO_TILE_Y - 1) / MO_TILE_Y));
  }
  int occupancy(const void* f, size_t smem = 0, int threads = MO_THREADS) {
    auto it = occ_.find(f);
    if (it != occ_.end()) return it->second;
    if (smem > 48 * 1024)
      CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, threads, smem) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 1;
    }
    occ_[f] = n;
    return n;
  }
  // Rows per work item of the row-wise streaming kernels (variants 4, 7 and
  // mo_gather_bm8): items are dealt to a fixed grid of resident blocks, so a
  // launch takes ceil(items / grid) rounds of (chunk + 2H) phase-1 rows plus a
  // small per-item cost; the larger chunk on ties.
  static int stream_chunk(long long rows, long long nb, long long grid, int halo) {
    static const int force = std::getenv("MO_B200_CHUNK") ? std::atoi(std::getenv("MO_B200_CHUNK")) : 0;
    if (force > 0) return force;
    int best = 0;
    double best_cost = 1e300;
    for (int ch = 1; ch <= 256; ++ch) {
      const long long items = nb * ((rows + ch - 1) / ch);
      const double cost = double((items + grid - 1) / grid) * (ch + 2 * halo + 4);
      if (cost <= best_cost) {
        best_cost = cost;
        best = ch;
      }
    }
    return std::max(best, 1);
  }
  int grid_blocks(const std::string& name, const Domain& d, size_t smem = 0) {
    const void* f = mod_.kernel(name);
    long long g = std::min<long long>(tiles_of(d), (long long)nsm_ * occupancy(f, smem));
    return int(std::max<long long>(g, 1));
  }
  int edge_blocks(const std::string& name, long long E) {
    const void* f = mod_.kernel(name);
    long long g = std::min<long long>((E + MO_THREADS - 1) / MO_THREADS, (long long)nsm_ * occupancy(f));
    return int(std::max<long long>(g, 1));
  }
  void launch_grid(const std::string& name, const Domain& d, const mo_kparams& kp, int grid = 0, size_t smem = 0) {
    const void* f = mod_.kernel(name);
    if (grid <= 0) grid = grid_blocks(name, d, smem);
    dim3 block = d.dims.size() <= 1 ? dim3(MO_THREADS, 1, 1) : dim3(MO_TILE_X, MO_TILE_Y, 1);
    void* args[] = {const_cast<mo_kparams*>(&kp)};
    klc(f, dim3(grid), block, args, smem);
    ++launches_;
  }
  // Apply kernel variants of gather set i: 0 = the reference's gather program
  // (exact mode always uses it), 1 = two-phase 32x8 tiles, 2 = row-streaming
  // two-phase bands, 3 = TMA-staged row-streaming bands (block-wide 8-row
  // steps), 4 = TMA-staged warp-streaming bands, 5 = TMA-staged gather
  // program (2-D domains).
  static constexpr int kVariants = 10;
  // variants 8 and 9 apply from the lane cache (direct loads / TMA-staged)
  static bool lc_variant(int v) { return v == 8 || v == 9; }
  bool uses_lcache(size_t i) const { return lc_variant(variant(i)); }
  static constexpr int kBm4 = 100;  // tma_info id of the TMA build_normal kernel
  static constexpr int kBm8 = 101;  // tma_info id of the warp-specialised build_normal kernel
  static constexpr int kBm8c = 102;  // ... that also writes the lane cache of variant 8
  const ModuleInfo::Tma* tma_info(size_t i, int v) const {
    if (v == kBm4 && i < minfo_.bm4.size()) return &minfo_.bm4[i];
    if (v == kBm8 && i < minfo_.bm8.size()) return &minfo_.bm8[i];
    if (v == kBm8c && i < minfo_.bm8c.size()) return &minfo_.bm8c[i];
    if (v == 7 && i < minfo_.jtj8.size()) return &minfo_.jtj8[i];
    if (v == 8 && i < minfo_.jtj9.size()) return &minfo_.jtj9[i];
    if (v == 9 && i < minfo_.jtj9t.size()) return &minfo_.jtj9t[i];
    if (v == 3 && i < minfo_.jtj4.size()) return &minfo_.jtj4[i];
    if (v == 6 && i < minfo_.jtj7.size()) return &minfo_.jtj7[i];
    if (v == 4 && i < minfo_.jtj5.size()) return &minfo_.jtj5[i];
    if (v == 5 && i < minfo_.jtj6.size()) return &minfo_.jtj6[i];
    return nullptr;
  }
  bool variant_ok(size_t i, int v) const {
    if (v == 0) return true;
    if (P_.exact) return false;
    if (v == 1) return i < minfo_.jtj2.size() && minfo_.jtj2[i].ok;
    if (v == 2) return i < minfo_.jtj3.size() && minfo_.jtj3[i].ok;
    const ModuleInfo::Tma* t = tma_info(i, v);
    if (lc_variant(v) && (sh_.on || !t || t->cache_planes == 0)) return false;  // lane cache: unsharded grids
    return t && t->ok && tma_capable(i, *t);
  }
  int variant(size_t i) const {
    if (i < jtj_choice_.size() && variant_ok(i, jtj_choice_[i])) return jtj_choice_[i];
    for (int v : {9, 8, 7, 3, 6, 5, 4, 2, 1}) if (variant_ok(i, v)) return v;
    return 0;
  }
  static const char* variant_prefix(int v) {
    static const char* n[] = {"mo_gather_jtj_",  "mo_gather_jtj2_", "mo_gather_jtj3_",
                              "mo_gather_jtj4_", "mo_gather_jtj5_", "mo_gather_jtj6_", "mo_gather_jtj7_",
                              "mo_gather_jtj8_", "mo_gather_jtj9_", "mo_gather_jtj9t_"};
    return n[v];
  }

  // ---- TMA tensor maps for the staged applies (variants 3, 4)
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encoder() {
    static EncodeFn fn = [] {
      void* f = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        f = nullptr;
      cudaGetLastError();
      return reinterpret_cast<EncodeFn>(f);
    }();
    return fn;
  }
  // Rows stored per buffer of a grid field (strip shards keep their halo rows).
  long long stored_rows(const Domain& d) const {
    return sh_.on && d == sh_.dom ? (long long)(sh_.hi - sh_.lo) : (long long)P_.shape_of(d)[0];
  }
  // Every staged field must be addressable by TMA: 16-byte aligned base
  // (column-layout fields start at ubase[f]) and 16-byte multiple row pitch.
  bool tma_capable(size_t i, const ModuleInfo::Tma& t) const {
    if (!encoder() || std::getenv("MO_B200_NO_TMA")) return false;
    if (P_.num_cols >= (1LL << 31)) return false;  // 32-bit column indices in the epilogue
    const auto sh = P_.shape_of(P_.gather_sets[i].dom);
    const int U = int(P_.unknowns.size());
    for (auto [sl, C] : t.slots) {
      if ((sh[1] * C * (long long)sizeof(Real)) % 16) return false;
      if (sl < 2 * U && (P_.ubase[size_t(sl % U)] * (long long)sizeof(Real)) % 16) return false;
    }
    return true;
  }
  const mo_tmaps& tmaps_for(size_t i, int v, const mo_kparams& kp) {
    const ModuleInfo::Tma& ti = *tma_info(i, v);
    std::string key = std::to_string(i) + "/" + std::to_string(v);
    for (auto [sl, C] : ti.slots) key += "/" + std::to_string(reinterpret_cast<uintptr_t>(kp.v[sl].p));
    auto it = tmaps_.find(key);
    if (it != tmaps_.end()) return it->second;
    mo_tmaps T;
    std::memset(&T, 0, sizeof T);
    const auto sh = P_.shape_of(P_.gather_sets[i].dom);
    const long long rows = stored_rows(P_.gather_sets[i].dom);
    for (size_t k = 0; k < ti.slots.size(); ++k) {
      const int C = ti.slots[k].second;
      const void* ptr = kp.v[ti.slots[k].first].p;
      check(ptr != nullptr, Err::kInternal, "TMA apply: staged field is not bound");
      // lane-cache planes: the extended-domain plane geometry
      const bool cp = ti.cache_planes && ti.slots[k].first >= ti.cache_slot0;
      const cuuint64_t dims[2] = {cuuint64_t(cp ? ti.cache_pw : sh[1] * C), cuuint64_t(cp ? ti.cache_rows : rows)};
      const cuuint64_t strides[1] = {cuuint64_t((cp ? ti.cache_pw : sh[1] * C) * (long long)sizeof(Real))};
      const cuuint32_t box[2] = {cuuint32_t(ti.win * C), cuuint32_t(ti.rows)};
      const cuuint32_t estr[2] = {1u, 1u};
      CUresult r = encoder()(reinterpret_cast<CUtensorMap*>(&T.m[k]),
                             sizeof(Real) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                             const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      check(r == CUDA_SUCCESS, Err::kCuda, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    }
    return tmaps_.emplace(key, T).first->second;
  }
  // Best of 3 replays of `body` captured as one CUDA graph, in ms.
  template <class F>
  float time_graph(F&& body) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed));
    body();
    CK(cudaStreamEndCapture(st_, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    CK(cudaGraphLaunch(ge, st_));  // warm-up
    for (int round = 0; round < 3; ++round) {
      CK(cudaEventRecord(a, st_));
      CK(cudaGraphLaunch(ge, st_));
      CK(cudaEventRecord(b, st_));
      CK(cudaEventSynchronize(b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaGraphExecDestroy(ge);
    return best;
  }
  // First use: time every available variant on the bound data and keep the
  // fastest per gather set (cheap programs such as Poisson's can win without
  // shared memory, barriers or halo recompute).  MO_B200_JTJ=gather|twophase|
  // stream forces a choice.
  void tune_apply() {
    if (tuned_) return;
    tuned_ = true;
    tune_apply_once();
  }
  void tune_apply_once() {
    if (mat_) return;  // one apply: the materialized J
    // One decision per (module, shape) per process, so every session of a plan
    // runs the same kernel (bitwise run-to-run reproducibility).
    static std::mutex mu;
    static std::map<std::string, std::vector<int>> cache, bm_cache;
    const char* force = std::getenv("MO_B200_JTJ");
    std::string key = module_key_ + (force ? std::string("/force:") + force : "");
    if (const char* bf = std::getenv("MO_B200_BM")) key += std::string("/bm:") + bf;
    for (auto& d : P_.dims) key += "/" + std::to_string(d.second);
    // A strip that owns the whole domain shares the unsharded decision.
    if (sh_.on && sh_.row1 - sh_.row0 != sh_.d0) key += "/s" + std::to_string(sh_.row1 - sh_.row0);
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = cache.find(key);
      if (it != cache.end()) {
        jtj_choice_ = it->second;
        bm_choice_ = bm_cache[key];
        return;
      }
    }
    jtj_choice_.assign(P_.gather_sets.size(), 0);
    for (size_t i = 0; i < P_.gather_sets.size(); ++i) {
      jtj_choice_[i] = -1;
      const std::string fs = force ? force : "";
      const int want = !force ? -1
                       : fs == "gather" ? 0
                       : fs == "twophase" ? 1
                       : fs == "stream" ? 2
                       : fs == "tma" ? 3
                       : fs == "warp" ? 4
                       : fs == "gprog" ? 5
                       : fs == "tma4" ? 6
                       : fs == "ws" ? 7
                       : fs == "lct" ? 9
                                       : 8;
      if (want >= 0) {
        jtj_choice_[i] = variant_ok(i, want) ? want : -1;
        if (jtj_choice_[i] >= 0) continue;
      }
      // Time every variant (best of 3 rounds of 4 launches), then take the
      // first variant in a fixed preference order that is within 5% of the
      // fastest: near-ties resolve the same way in every process, so the
      // kernel choice (and with it the rounding) is stable across runs.
      float t[kVariants];
      float best = 1e30f;
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      for (int v = 0; v < kVariants; ++v) {
        t[v] = 1e30f;
        if (!variant_ok(i, v)) continue;
        jtj_choice_[i] = v;
        if (lc_variant(v)) lanecache_fill(i);
        mo_kparams kp = kp_apply(i, x_, otmp_, MO_F_EXSKIP);  // (stores as inside the PCG)
        const int grid = jtj_grid(i);
        launch_apply(i, kp, grid);  // warm-up (module load, tensor maps)
        // Timed as a captured graph of 8 launches (as the solver runs them):
        // back-to-back host launches of a small kernel measure the launch
        // rate, not the kernel.
        t[v] = time_graph([&] {
          for (int rep = 0; rep < 8; ++rep) launch_apply(i, kp, grid);
        });
        launches_ -= 9;
        best = std::min(best, t[v]);
      }
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      if (std::getenv("MO_B200_TUNE_LOG")) {
        for (int v = 0; v < kVariants; ++v)
          if (t[v] < 1e29f) fprintf(stderr, "[mo tune] gather set %zu variant %d: %.1f us\n", i, v, t[v] * 1e3f / 8);
      }
      int bestv = 0;
      for (int v : {9, 8, 7, 3, 6, 5, 4, 2, 1, 0})
        if (t[v] <= 1.05f * best) {
          bestv = v;
          break;
        }
      jtj_choice_[i] = bestv;
    }
    // build_normal: TMA two-phase kernel vs the reference's bm program.
    bm_choice_.assign(P_.gather_sets.size(), 0);
    const int stage = cur_stage_;
    cur_stage_ = -1;  // no profiling events while tuning
    const int64_t launched = launches_;
    for (size_t i = 0; i < P_.gather_sets.size(); ++i) {
      if (sh_.on || (!bm4_avail(i) && !bm8_avail(i))) continue;  // (strips: normal_device has collectives)
      float tb[3] = {1e30f, 1e30f, 1e30f};
      for (int v = 0; v < 3; ++v) {
        if ((v == 1 && !bm4_avail(i)) || (v == 2 && !bm8_avail(i))) continue;
        bm_choice_[i] = v;
        normal_device();  // warm-up
        tb[v] = time_graph([&] {
          for (int rep = 0; rep < 4; ++rep) normal_device();
        });
      }
      // fp32: the evalj-based kernels form each residual once per element and
      // sum d_l r_t per merged lane, which tracks the fp64 trajectory far
      // more closely than the bm gather program's fp32 root sums (ARAP
      // 1024², 10 x 20: 1192.985 vs 1193.153, fp64 reference 1192.980), so
      // one of them is kept unless it costs more than 30%.  fp64: the
      // fastest.  Between the two evalj kernels: the faster, bm8 on a 5% tie.
      // MO_B200_BM=prog|bm4|bm8 forces one.
      const char* bmf = std::getenv("MO_B200_BM");
      const float slack = sizeof(Real) == 4 ? 1.30f : 0.95f;
      const int ev = tb[2] <= 1.05f * tb[1] ? 2 : 1;
      bm_choice_[i] = tb[ev] < slack * tb[0] ? ev : 0;
      if (std::getenv("MO_B200_TUNE_LOG"))
        fprintf(stderr, "[mo tune] gather set %zu build_normal: program %.1f us, bm4 %.1f us, bm8 %.1f us\n", i,
                tb[0] * 1e3f / 4, tb[1] * 1e3f / 4, tb[2] * 1e3f / 4);
      if (bmf) {
        const std::string b = bmf;
        bm_choice_[i] = b == "bm4" && bm4_avail(i) ? 1 : b == "bm8" && bm8_avail(i) ? 2 : 0;
      }
    }
    launches_ = launched;
    cur_stage_ = stage;
    // Strips: every rank runs rank 0's kernels (one rounding behaviour across
    // the whole grid, run to run).  Collective: all ranks tune in their first
    // solve; later sessions of the same key take the per-process cache.
    if (sh_.on && comm_ && comm_->world > 1) {
      const size_t G = P_.gather_sets.size();
      check(G <= 32, Err::kInternal, "too many gather sets for the kernel-choice broadcast");
      std::vector<double> mine(64, 0.0), all(size_t(comm_->world) * 64);
      for (size_t i = 0; i < G; ++i) {
        mine[i] = jtj_choice_[i];
        mine[32 + i] = bm_choice_.size() > i ? bm_choice_[i] : 0;
      }
      // (chob_ is allocated with the session: a cudaFree here would wait for
      // the whole device, i.e. for another LocalComm rank's peer reduction
      // spinning on this rank's flag)
      CK(cudaMemcpyAsync(chob_, mine.data(), 64 * sizeof(double), cudaMemcpyHostToDevice, st_));
      comm_->allgather(chob_, rankbuf_, 64, st_);
      CK(cudaMemcpyAsync(all.data(), rankbuf_, all.size() * sizeof(double), cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
      for (size_t i = 0; i < G; ++i) {  // rank 0's entries come first
        jtj_choice_[i] = int(all[i]);
        if (bm_choice_.size() > i) bm_choice_[i] = int(all[32 + i]);
      }
    }
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = jtj_choice_;
    bm_cache[key] = bm_choice_;
  }
  std::string jtj_kernel(size_t i) const { return variant_prefix(variant(i)) + std::to_string(i); }
  size_t jtj_smem(size_t i) const {
    const int v = variant(i);
    if (const ModuleInfo::Tma* t = tma_info(i, v)) return t->smem;
    return v == 1 ? minfo_.jtj2[i].smem : v == 2 ? minfo_.jtj3[i].smem : 0;
  }
  int jtj_threads(size_t i) const {
    const ModuleInfo::Tma* t = tma_info(i, variant(i));
    return t ? t->threads : MO_THREADS;
  }
  int jtj_halo(size_t i) const {
    const ModuleInfo::Tma* t = tma_info(i, variant(i));
    return t ? t->halo : minfo_.jtj3[i].halo;
  }
  int jtj_band(size_t i) const {
    const ModuleInfo::Tma* t = tma_info(i, variant(i));
    return t ? t->band : minfo_.jtj3[i].band;
  }
  int jtj_occupancy(size_t i) {
    const void* f = mod_.kernel(jtj_kernel(i));
    const size_t smem = jtj_smem(i);
    const int threads = jtj_threads(i);
    auto it = occ_.find(f);
    if (it != occ_.end()) return it->second;
    if (smem > 48 * 1024) CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, threads, smem) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 1;
    }
    occ_[f] = n;
    return n;
  }
  // Launch the apply kernel of gather set i (variants 3, 4 also take the tensor maps).
  void launch_apply(size_t i, const mo_kparams& kp, int grid) {
    const int v = variant(i);
    if (v < 3) {
      launch_grid(jtj_kernel(i), P_.gather_sets[i].dom, kp, grid, jtj_smem(i));
      return;
    }
    const void* f = mod_.kernel(jtj_kernel(i));
    const size_t smem = jtj_smem(i);
    jtj_occupancy(i);  // sets the dynamic smem attribute once
    const mo_tmaps& T = tmaps_for(i, v, kp);
    void* args[] = {const_cast<mo_kparams*>(&kp), const_cast<mo_tmaps*>(&T)};
    const dim3 block = v == 4 || v >= 7 ? dim3(unsigned(jtj_threads(i)), 1, 1) : dim3(32, unsigned(jtj_threads(i) / 32), 1);
    klc(f, dim3(grid), block, args, smem);
    ++launches_;
  }
  // Rows per work item of the streaming variants.  Work items are dealt to a
  // fixed grid of resident blocks, so an apply takes ceil(items / grid)
  // rounds of (chunk + 2H) phase-1 rows (variants 2-3 step 8 rows at a time,
  // chunk + 2H a multiple of 8): pick the chunk minimising that plus a
  // per-item pipeline fill, the larger one on ties.
  int jtj3_chunk(size_t i) {
    static const int force = std::getenv("MO_B200_CHUNK") ? std::atoi(std::getenv("MO_B200_CHUNK")) : 0;
    if (force > 0) return force;
    const auto sh = P_.shape_of(P_.gather_sets[i].dom);
    const long long rows = apply_rows(sh[0]);
    const int halo = jtj_halo(i), band = jtj_band(i);
    const long long nb = (sh[1] + band - 1) / band;
    const long long grid = (long long)nsm_ * jtj_occupancy(i);
    const bool rowwise = variant(i) == 4 || variant(i) >= 7;
    if (rowwise) return stream_chunk(rows, nb, grid, halo);
    const ModuleInfo::Tma* ti = tma_info(i, variant(i));
    const int step = ti && !rowwise ? ti->rows : 8;  // rows per step of the block-stepped variants
    int best = 0;
    double best_cost = 1e300;
    for (int m = 1; m <= (rowwise ? 256 : 128 / step); ++m) {
      const int ch = rowwise ? m : step * m - 2 * halo;
      if (ch <= 0) continue;
      const long long items = nb * ((rows + ch - 1) / ch);
      const long long rounds = (items + grid - 1) / grid;
      const double cost = rowwise ? double(rounds) * (ch + 2 * halo + 4) : double(rounds) * (m + 0.5);
      if (cost <= best_cost) {
        best_cost = cost;
        best = ch;
      }
    }
    return std::max(best, 1);
  }
  // Output rows of one apply launch: the strip's, the whole domain's, or the
  // sub-range of an overlapped strip apply (ov0_/ov1_).
  long long apply_rows(long long d0) const {
    if (ov0_ >= 0) return ov1_ - ov0_;
    return sh_.on ? sh_.row1 - sh_.row0 : d0;
  }
  int jtj_grid(size_t i) {
    if (variant(i) == 0 && ov0_ < 0 && cm_any_ && i < tl_count_.size() && tl_count_[i] >= 0)
      return std::max(1, std::min(tl_count_[i], grid_blocks(jtj_kernel(i), P_.gather_sets[i].dom, jtj_smem(i))));
    if (variant(i) < 2) return grid_blocks(jtj_kernel(i), P_.gather_sets[i].dom, jtj_smem(i));
    const auto sh = P_.shape_of(P_.gather_sets[i].dom);
    const long long rows = apply_rows(sh[0]);
    const int band = jtj_band(i);
    const long long nb = (sh[1] + band - 1) / band;
    const int ch = jtj3_chunk(i);
    const long long items = nb * ((rows + ch - 1) / ch);
    const long long cap = (long long)nsm_ * jtj_occupancy(i);
    return int(std::max<long long>(1, std::min(items, cap)));
  }
  mo_kparams kp_apply(size_t i, const Real* pv, Real* out, int flags) {
    mo_kparams kp = kp_grid(P_.gather_sets[i].dom, x_, pv);
    kp.out0 = out;
    kp.in0 = pv;
    kp.in1 = damp_;
    kp.flags = flags;
    if (ov0_ >= 0) {
      kp.row0 = int(ov0_);
      kp.row1 = int(ov1_);
    } else if (cm_any_ && variant(i) == 0 && i < tiles_.size() && tiles_[i]) {
      kp.in3 = tiles_[i];  // active-tile list (read under MO_F_EXSKIP)
    }
    if (variant(i) >= 2) kp.chunk = jtj3_chunk(i);
    if (uses_lcache(i)) {  // lane-cache planes (read directly, or as TMA-staged views)
      ensure_lanecache(i);
      kp.in2 = lcache_[i];
      const ModuleInfo::Tma& ti = *tma_info(i, variant(i));
      if (ti.cache_tma) {
        const size_t ps = size_t(ti.cache_pw) * size_t(ti.cache_rows);
        for (int j = 0; j < ti.cache_planes; ++j) kp.v[ti.cache_slot0 + j].p = lcache_[i] + size_t(j) * ps;
      }
    }
    return kp;
  }
  // ---- lane cache (variant 8): planes of the x-dependent evalj lanes and
  // guard outcomes, rewritten once per linearisation (normal_device) and
  // before every standalone apply.
  void ensure_lanecache(size_t i) {
    if (lcache_.size() < P_.gather_sets.size()) lcache_.resize(P_.gather_sets.size(), nullptr);
    if (lcache_[i]) return;
    const ModuleInfo::Tma& ti = minfo_.jtj9[i];  // (the same planes for jtj9t)
    const size_t bytes = size_t(ti.cache_planes) * size_t(ti.cache_pw) * size_t(ti.cache_rows) * sizeof(Real);
    CK(cudaMalloc(&lcache_[i], bytes));
    CK(cudaMemsetAsync(lcache_[i], 0, bytes, st_));
  }
  void lanecache_fill(size_t i) {
    ensure_lanecache(i);
    const std::string kn = "mo_lanecache_" + std::to_string(i);
    mo_kparams kp = kp_grid(P_.gather_sets[i].dom, x_, nullptr);
    kp.out0 = lcache_[i];
    const void* f = mod_.kernel(kn);
    const int grid = nsm_ * occupancy(f);
    void* args[] = {&kp};
    klc(f, dim3(grid), dim3(MO_TILE_X, MO_TILE_Y, 1), args, 0);
    ++launches_;
  }
  void lanecache_fill() {
    if (mat_) return;
    tune_apply();
    for (size_t i = 0; i < P_.gather_sets.size(); ++i)
      if (uses_lcache(i)) lanecache_fill(i);
  }
  void launch_edges(const std::string& name, int gi, const mo_kparams& kp, int grid = 0) {
    const void* f = mod_.kernel(name);
    (void)gi;
    if (grid <= 0) grid = edge_blocks(name, kp.nedges);
    void* args[] = {const_cast<mo_kparams*>(&kp)};
    klc(f, dim3(grid), dim3(MO_THREADS), args, 0);
    ++launches_;
  }
  mo_red red(int base, int total, int op, int arg) {
    check(total <= kPartCap, Err::kInternal, "reduction exceeds the partial buffer");
    mo_red R;
    R.partials = partials_;
    R.counter = &state_->counters[0];
    R.state = state_;
    R.part_base = base;
    R.part_total = total;
    // Shard mode: kernels only produce this rank's partial (sums[4..5]);
    // reduce_done() gathers and finalises.
    R.fin_op = sh_.on ? MO_FIN_STORE2 : op;
    R.fin_arg = sh_.on ? 4 : arg;
    return R;
  }

  // One-pass graph apply (mo_graph_vjtjf_0): grid gather program, incident
  // edges in order and the apply epilogue per vertex, one launch.
  bool vertex_apply_one_pass() const {
    static const bool off = std::getenv("MO_B200_NO_VFUSE") != nullptr;
    return !off && minfo_.fused_vertex_apply && !sh_.on && vertex_path(0);
  }
  void apply_vertex_fused(const Real* pv, Real* out, int flags) {
    GSet& gs = gsets_[0];
    const GatherDom& gd = gs.doms[0];
    mo_kparams kp = kp_grid(P_.gather_sets[0].dom, x_, pv);  // grid env (InBounds, mask) of the vertex domain
    const GraphData& g = graphs_[size_t(P_.graph_sets[0].graph)];
    kp.verts = g.d_verts;
    kp.arity = g.arity;
    kp.nedges = g.E;
    kp.vptr = gd.vptr;
    kp.vedge = gd.vedge;
    kp.nverts = gd.nverts;
    kp.out0 = out;
    kp.in0 = pv;
    kp.in1 = damp_;
    kp.flags = flags;
    const void* f = mod_.kernel("mo_graph_vjtjf_0");
    const int grid = int(std::max<long long>(
        1, std::min<long long>((gd.nverts + MO_THREADS - 1) / MO_THREADS, (long long)nsm_ * occupancy(f))));
    kp.red = red(0, grid, consumer_ ? MO_FIN_PARTIALS : MO_FIN_PCG_ALPHA, 0);
    apply_parts_ = grid;
    void* args[] = {&kp};
    klc(f, dim3(grid), dim3(MO_THREADS), args, 0);
    ++launches_;
    if ((flags & MO_F_REDUCE) && !consumer_) reduce_done(MO_FIN_PCG_ALPHA, 0);
  }

  // Vertex-centric recompute kernels (generated per scatter-target domain).
  bool vertex_path(size_t gi) const {
    static const bool off = std::getenv("MO_B200_EDGE_SCATTER") != nullptr;
    return !off && gi < minfo_.vertex_kernels.size() && minfo_.vertex_kernels[gi];
  }
  void launch_vertex(const char* prefix, int gi, mo_kparams kp, Real* dst0, Real* dst1) {
    GSet& gs = gsets_[size_t(gi)];
    for (size_t di = 0; di < gs.doms.size(); ++di) {
      const GatherDom& gd = gs.doms[di];
      kp.out0 = dst0;
      kp.out1 = dst1;
      kp.vptr = gd.vptr;
      kp.vedge = gd.vedge;
      kp.nverts = gd.nverts;
      const std::string name = prefix + std::to_string(gi) + "_" + std::to_string(di);
      const void* f = mod_.kernel(name);
      long long g = std::min<long long>((gd.nverts + MO_THREADS - 1) / MO_THREADS, (long long)nsm_ * occupancy(f));
      void* args[] = {&kp};
      klc(f, dim3(unsigned(std::max<long long>(g, 1))), dim3(MO_THREADS), args, 0);
      ++launches_;
    }
  }

  void gather_graph(int gi, bool bm, Real* dst0, Real* dst1) {
    const GraphSet& g = P_.graph_sets[size_t(gi)];
    GSet& gs = gsets_[size_t(gi)];
    const GraphData& gd0 = graphs_[size_t(g.graph)];
    const int NO = int(bm ? g.bm.outputs.size() : g.jtj.outputs.size());
    if (NO == 0) return;
    for (auto& gd : gs.doms) {
      kl(k_graph_gather<Real>, dim3(vgrid(gd.nverts, nsm_)), dim3(MO_THREADS), 
          gd.nverts, gd.vptr, gd.vedge, gd0.d_verts, gd0.arity, gs.contrib, NO, bm ? gd.outs_bm : gd.outs_jtj,
          dst0, dst1);
      ++launches_;
    }
  }

  // cost_at (solver.hpp:176-193) into state->sums[slot].
  void cost_at(const Real* xv, int slot) {
    int total = 0;
    std::vector<int> grids;
    for (size_t i = 0; i < P_.grid_sets.size(); ++i) {
      grids.push_back(grid_blocks("mo_grid_cost_" + std::to_string(i), P_.grid_sets[i].dom));
      total += grids.back();
    }
    for (size_t i = 0; i < P_.graph_sets.size(); ++i) {
      grids.push_back(edge_blocks("mo_graph_cost_" + std::to_string(i),
                                  graphs_[size_t(P_.graph_sets[i].graph)].E_own));
      total += grids.back();
    }
    if (total == 0) {
      CK(cudaMemsetAsync(&state_->sums[sh_.on ? 4 : slot], 0, sizeof(double) * (sh_.on ? 2 : 1), st_));
      reduce_done(MO_FIN_STORE, slot);
      return;
    }
    int base = 0, gi = 0;
    for (size_t i = 0; i < P_.grid_sets.size(); ++i, ++gi) {
      mo_kparams kp = kp_grid(P_.grid_sets[i].dom, xv, nullptr);
      kp.red = red(base, total, MO_FIN_STORE, slot);
      launch_grid("mo_grid_cost_" + std::to_string(i), P_.grid_sets[i].dom, kp, grids[size_t(gi)]);
      base += grids[size_t(gi)];
    }
    for (size_t i = 0; i < P_.graph_sets.size(); ++i, ++gi) {
      mo_kparams kp = kp_graph(int(i), xv, nullptr);
      kp.red = red(base, total, MO_FIN_STORE, slot);
      launch_edges("mo_graph_cost_" + std::to_string(i), int(i), kp, grids[size_t(gi)]);
      base += grids[size_t(gi)];
    }
    reduce_done(MO_FIN_STORE, slot);
  }

  // build_normal (solver.hpp:220-251) on the device.
  // GN: the bm gather kernels can also start the PCG (k_pcg_init's work on
  // the patched b, m), when they write every column (no graph scatters, every
  // unknown channel an output of exactly one gather set).  On a strip the
  // kernels cover the owned rows only; halo p arrives by the exchange.
  // TMA two-phase build_normal (mo_gather_bm4_<i>), fast mode only;
  // MO_B200_NO_BM4=1 keeps the reference's bm gather program.
  bool bm4_avail(size_t i) const {
    if (std::getenv("MO_B200_NO_BM4") || P_.exact || i >= minfo_.bm4.size() || !minfo_.bm4[i].ok) return false;
    return tma_capable(i, minfo_.bm4[i]);
  }
  // chosen by tune_apply (timed against the bm gather program; kept only
  // when >5% faster: it wins on large grids, loses on small ones)
  bool bm4_ok(size_t i) const { return i < bm_choice_.size() && bm_choice_[i] == 1 && bm4_avail(i); }
  // Warp-specialised streaming build_normal (mo_gather_bm8_<i>), fast mode only.
  bool bm8_avail(size_t i) const {
    if (std::getenv("MO_B200_NO_BM4") || P_.exact || i >= minfo_.bm8.size() || !minfo_.bm8[i].ok) return false;
    return tma_capable(i, minfo_.bm8[i]);
  }
  bool bm8_ok(size_t i) const { return i < bm_choice_.size() && bm_choice_[i] == 2 && bm8_avail(i); }
  // build_normal writes variant 8's lane cache itself (mo_gather_bm8c): no
  // separate mo_lanecache pass per linearisation.
  bool bm8c_fuses(size_t i) const {
    return bm8_ok(i) && uses_lcache(i) && i < minfo_.bm8c.size() && minfo_.bm8c[i].ok &&
           tma_capable(i, minfo_.bm8c[i]) && !std::getenv("MO_B200_NO_BM8C");
  }
  // Grid and rows per work item of mo_gather_bm8 / bm8c (the apply's row model).
  int bm8_grid(size_t i, int* chunk) {
    const bool fz = bm8c_fuses(i);
    const ModuleInfo::Tma& ti = fz ? minfo_.bm8c[i] : minfo_.bm8[i];
    const void* f = mod_.kernel((fz ? "mo_gather_bm8c_" : "mo_gather_bm8_") + std::to_string(i));
    const int occ = occupancy(f, ti.smem, ti.threads);
    const auto sh = P_.shape_of(P_.gather_sets[i].dom);
    const long long rows = sh_.on ? sh_.row1 - sh_.row0 : sh[0];
    const long long nb = (sh[1] + ti.band - 1) / ti.band, grid = (long long)nsm_ * occ;
    *chunk = stream_chunk(rows, nb, grid, ti.halo);
    const long long items = nb * ((rows + *chunk - 1) / *chunk);
    return int(std::max<long long>(1, std::min(items, grid)));
  }
  int bm4_grid(size_t i, int* chunk) {
    const ModuleInfo::Tma& ti = minfo_.bm4[i];
    const void* f = mod_.kernel("mo_gather_bm4_" + std::to_string(i));
    const int occ = occupancy(f, ti.smem);
    const auto sh = P_.shape_of(P_.gather_sets[i].dom);
    const long long rows = sh_.on ? sh_.row1 - sh_.row0 : sh[0];
    const long long nb = (sh[1] + ti.band - 1) / ti.band, grid = (long long)nsm_ * occ;
    int best = 0;
    double best_cost = 1e300;
    for (int m = 1; m <= 16; ++m) {  // same round model as the apply (jtj3_chunk)
      const int ch = 8 * m - 2 * ti.halo;
      if (ch <= 0) continue;
      const long long items = nb * ((rows + ch - 1) / ch);
      const double cost = double((items + grid - 1) / grid) * (m + 0.5);
      if (cost <= best_cost) {
        best_cost = cost;
        best = ch;
      }
    }
    *chunk = std::max(best, 1);
    const long long items = nb * ((rows + *chunk - 1) / *chunk);
    return int(std::max<long long>(1, std::min(items, grid)));
  }
  bool bm_init_ok() const {
    static const bool off = std::getenv("MO_B200_NO_BMINIT") != nullptr;
    if (off || !P_.graph_sets.empty() || P_.gather_sets.empty()) return false;
    size_t outs = 0, chans = 0;
    for (const GatherSet& g : P_.gather_sets) outs += g.chans.size();
    for (const Field& f : P_.unknowns) chans += size_t(f.channels);
    return outs == chans;
  }
  void normal_device(bool pcg_init = false) {
    if (tuned_ && !mat_)  // the linearisation point moved: refresh the lane cache
      for (size_t i = 0; i < P_.gather_sets.size(); ++i)
        if (uses_lcache(i) && !bm8c_fuses(i)) lanecache_fill(i);
    prof_begin(2);
    const bool fused = P_.graph_sets.empty();
    const long long n = P_.num_cols;
    std::vector<int> grids, chunks;
    int total = 0;
    for (size_t i = 0; i < P_.gather_sets.size(); ++i) {
      if (bm8_ok(i)) {
        int ch = 0;
        grids.push_back(bm8_grid(i, &ch));
        chunks.push_back(ch);
      } else if (bm4_ok(i)) {
        int ch = 0;
        grids.push_back(bm4_grid(i, &ch));
        chunks.push_back(ch);
      } else {
        grids.push_back(grid_blocks("mo_gather_bm_" + std::to_string(i), P_.gather_sets[i].dom));
        chunks.push_back(0);
      }
      total += grids.back();
    }
    if (!fused) total = vgrid(n, nsm_);
    int base = 0;
    for (size_t i = 0; i < P_.gather_sets.size(); ++i) {
      mo_kparams kp = kp_grid(P_.gather_sets[i].dom, x_, nullptr);
      kp.chunk = chunks[i];
      kp.out0 = b_;
      kp.out1 = m_;
      kp.flags = fused ? (MO_F_PATCH | MO_F_REDUCE) : 0;
      kp.red = red(base, total, MO_FIN_UNCONSTRAINED, 0);
      if (pcg_init) {
        kp.flags |= MO_F_PCGINIT;
        kp.red = red(base, total, MO_FIN_BM_INIT, 0);
        kp.out2 = p_;
        kp.out3 = delta_;
        kp.out4 = r_;
      }
      if (chunks[i] && bm8_ok(i)) {  // warp-specialised streaming build_normal
        const bool fz = tuned_ && bm8c_fuses(i);  // (+ the lane cache of the apply)
        const ModuleInfo::Tma& ti = fz ? minfo_.bm8c[i] : minfo_.bm8[i];
        if (fz) {
          ensure_lanecache(i);
          kp.in2 = lcache_[i];
          kp.flags |= MO_F_LCACHE;
        }
        const void* f = mod_.kernel((fz ? "mo_gather_bm8c_" : "mo_gather_bm8_") + std::to_string(i));
        const mo_tmaps& T = tmaps_for(i, fz ? kBm8c : kBm8, kp);
        void* args[] = {&kp, const_cast<mo_tmaps*>(&T)};
        klc(f, dim3(grids[i]), dim3(unsigned(ti.threads), 1, 1), args, ti.smem);
        ++launches_;
      } else if (chunks[i]) {  // TMA two-phase build_normal
        const void* f = mod_.kernel("mo_gather_bm4_" + std::to_string(i));
        const mo_tmaps& T = tmaps_for(i, kBm4, kp);
        void* args[] = {&kp, const_cast<mo_tmaps*>(&T)};
        klc(f, dim3(grids[i]), dim3(MO_TILE_X, MO_TILE_Y, 1), args, minfo_.bm4[i].smem);
        ++launches_;
      } else {
        launch_grid("mo_gather_bm_" + std::to_string(i), P_.gather_sets[i].dom, kp, grids[i]);
      }
      base += grids[i];
    }
    if (!fused) {
      for (size_t i = 0; i < P_.graph_sets.size(); ++i) {
        mo_kparams kp = kp_graph(int(i), x_, nullptr);
        if (vertex_path(i)) {
          launch_vertex("mo_graph_vbm_", int(i), kp, b_, m_);
          continue;
        }
        kp.out0 = gsets_[i].contrib;
        // contributions of EVERY stored edge: the incidence CSR the gather
        // walks also holds the strip's non-owned edges touching owned vertices
        kp.nedges = graphs_[size_t(P_.graph_sets[i].graph)].E;
        launch_edges("mo_graph_bm_" + std::to_string(i), int(i), kp);
        gather_graph(int(i), true, b_, m_);
      }
      kl(k_bm_patch<Real>, dim3(vgrid(n, nsm_)), dim3(MO_THREADS), red(0, vgrid(n, nsm_), MO_FIN_UNCONSTRAINED, 0), n,
                                                                colmask_, b_, m_);
      ++launches_;
      reduce_done(MO_FIN_UNCONSTRAINED, 0);  // (strips only)
    } else if (P_.gather_sets.empty()) {
      CK(cudaMemsetAsync(&state_->unconstrained, 0, sizeof(long long), st_));
    } else {
      reduce_done(pcg_init ? MO_FIN_BM_INIT : MO_FIN_UNCONSTRAINED, 0);
    }
    prof_end(2);
  }

  // out = 2 J^T J pv (+ damp pv), optionally zeroing excluded columns and
  // reducing p'Ap into alpha (flags: MO_F_DAMP | MO_F_REDUCE | MO_F_ZEROEXCL).
  void apply(const Real* pv, Real* out, int flags) {
    if (pending_p_) {
      const bool split = !mat_ && P_.graph_sets.empty() && pending_p_ == pv && comm_ && comm_->world > 1 &&
                         !std::getenv("MO_B200_NO_OVERLAP") && sh_.row1 - sh_.row0 > 2 * int64_t(sh_.R);
      if (split) {
        apply_overlapped(pv, out, flags);
        return;
      }
      exchange_cols(const_cast<Real*>(pending_p_));
      pending_p_ = nullptr;
    }
    if (mat_) {
      mat_apply(pv, out, flags);
      return;
    }
    if (vertex_apply_one_pass()) {
      apply_vertex_fused(pv, out, flags);
      return;
    }
    const bool fused = P_.graph_sets.empty();
    const long long n = P_.num_cols;
    std::vector<int> grids;
    int total = 0;
    for (size_t i = 0; i < P_.gather_sets.size(); ++i) {
      grids.push_back(jtj_grid(i));
      total += grids.back();
    }
    if (!fused) total = vgrid(n, nsm_);
    apply_parts_ = total;
    int base = 0;
    for (size_t i = 0; i < P_.gather_sets.size(); ++i) {
      mo_kparams kp = kp_apply(i, pv, out, fused ? flags : (flags & MO_F_SKIPDONE));
      kp.red = red(base, total, consumer_ && fused ? MO_FIN_PARTIALS : MO_FIN_PCG_ALPHA, 0);
      launch_apply(i, kp, grids[i]);
      base += grids[i];
    }
    if (fused && (flags & MO_F_REDUCE) && !consumer_) reduce_done(MO_FIN_PCG_ALPHA, 0);
    if (!fused) {
      for (size_t i = 0; i < P_.graph_sets.size(); ++i) {
        mo_kparams kp = kp_graph(int(i), x_, pv);
        kp.flags = flags & MO_F_SKIPDONE;
        if (vertex_path(i)) {
          launch_vertex("mo_graph_vjtj_", int(i), kp, out, nullptr);
          continue;
        }
        kp.out0 = gsets_[i].contrib;
        kp.nedges = graphs_[size_t(P_.graph_sets[i].graph)].E;  // (all stored edges, as for b/m)
        launch_edges("mo_graph_jtj_" + std::to_string(i), int(i), kp);
        gather_graph(int(i), false, out, nullptr);
      }
      if (flags & (MO_F_DAMP | MO_F_REDUCE | MO_F_ZEROEXCL)) {
        kl(k_apply_finish<Real>, dim3(vgrid(n, nsm_)), dim3(MO_THREADS), red(0, vgrid(n, nsm_), MO_FIN_PCG_ALPHA, 0), n,
                                                                     colmask_, pv, damp_, out, flags);
        ++launches_;
        if (flags & MO_F_REDUCE) reduce_done(MO_FIN_PCG_ALPHA, 0);  // (strips only)
      }
    }
  }

  // Strip apply with the p halo exchange overlapped (pcg_body defers the
  // exchange of p to here): the interior rows [row0+R, row1-R), whose
  // stencils read owned p rows only, are launched first on st_; the exchange
  // runs on sd_ meanwhile (forked after the p update); st_ joins it and
  // applies the R border rows on each side.  One reduction spans the three
  // launches (disjoint partial slots, the last block of the last launch
  // finalises), so alpha is the same deterministic fixed-order sum on every
  // run.  LocalComm's host barriers sit between the interior launch and the
  // border launches, so the overlap is real for both transports.
  void apply_overlapped(const Real* pv, Real* out, int flags) {
    pending_p_ = nullptr;
    const int64_t a = sh_.row0, b = sh_.row1, M = sh_.R;
    const int64_t parts[3][2] = {{a + M, b - M}, {a, a + M}, {b - M, b}};
    const size_t ng = P_.gather_sets.size();
    std::vector<int> grids;
    int total = 0;
    for (const auto& pr : parts) {
      ov0_ = pr[0];
      ov1_ = pr[1];
      for (size_t i = 0; i < ng; ++i) {
        grids.push_back(jtj_grid(i));
        total += grids.back();
      }
    }
    CK(cudaEventRecord(ev_p_, st_));
    int base = 0;
    size_t gi = 0;
    for (int part = 0; part < 3; ++part) {
      if (part == 1) {
        CK(cudaStreamWaitEvent(sd_, ev_p_, 0));
        exchange_cols(p_, sd_);
        CK(cudaEventRecord(ev_h_, sd_));
        CK(cudaStreamWaitEvent(st_, ev_h_, 0));
      }
      ov0_ = parts[part][0];
      ov1_ = parts[part][1];
      for (size_t i = 0; i < ng; ++i, ++gi) {
        mo_kparams kp = kp_apply(i, pv, out, flags);
        kp.red = red(base, total, MO_FIN_PCG_ALPHA, 0);
        launch_apply(i, kp, grids[gi]);
        base += grids[gi];
      }
    }
    ov0_ = ov1_ = -1;
    apply_parts_ = total;
    if (flags & MO_F_REDUCE) reduce_done(MO_FIN_PCG_ALPHA, 0);
  }

  // ------------------------------------------------------------ materialized J
  // linearize (solver.hpp:291-376) keeps J as the reference does before its
  // CSR assembly: the evalj lanes, [lane][element] per template set.  In
  // Materialize::kJ plans the apply is 2 J^T (J v) from those lanes
  // (k_mat_rows / k_mat_cols, sparse.hpp spmv / spmv_t order); jacobian()
  // assembles the reference's CSR on the host for callers that want it.
  bool plan_has_evalj() const {
    for (const GridSet& g : P_.grid_sets)
      if (!g.templates.empty() && !g.has_evalj) return false;
    for (const GraphSet& g : P_.graph_sets)
      if (!g.templates.empty() && !g.has_evalj) return false;
    return true;
  }
  const void* evj_kernel(const std::string& name) {
    if (mat_) return mod_.kernel(name);
    if (!mod_evj_.loaded())  // matrix-free plan with lanes: compile the linearize kernels on demand
      mod_evj_.load(compile_cubin(generate_module(P_, sizeof(Real) == 8, device_prelude(), nullptr, true),
                                  "mo_evalj.cu", P_.exact));
    return mod_evj_.kernel(name);
  }
  // linear_index(coord + off) - linear_index(coord) (problem.hpp:131-136)
  static long long lane_lin(const Lane& l, const std::array<int64_t, 3>& sh) {
    return ((long long)l.off[0] * sh[1] + l.off[1]) * sh[2] + l.off[2];
  }
  void check_mat_bad() {
    if (state_h_->mat_bad & 1) fail(Err::kIndexOutOfRange, "CSR column out of range");
    if (state_h_->mat_bad & 2) fail(Err::kInternal, "CSR row entries must arrive in increasing column order");
    if (state_h_->mat_bad & 4) fail(Err::kInternal, "normal matrix row exceeds its assembled width");
  }
  // max over vertices of |union of the columns of the edge rows incident to it|
  size_t graph_row_union(const std::vector<uint64_t>& verts, int64_t E, int arity, long long nv,
                         const std::vector<const JTemplate*>& jts) const {
    std::vector<int> deg(size_t(nv) + 1, 0), edge_of;
    for (int64_t e = 0; e < E; ++e)
      for (int k = 0; k < arity; ++k) deg[size_t(verts[size_t(e * arity + k)]) + 1] += 1;
    for (size_t i = 0; i < size_t(nv); ++i) deg[i + 1] += deg[i];
    edge_of.resize(size_t(deg[size_t(nv)]));
    std::vector<int> pos(deg.begin(), deg.end() - 1);
    for (int64_t e = 0; e < E; ++e)
      for (int k = 0; k < arity; ++k) edge_of[size_t(pos[size_t(verts[size_t(e * arity + k)])]++)] = int(e);
    size_t best = 0;
    std::set<long long> cols;
    for (size_t vtx = 0; vtx < size_t(nv); ++vtx) {
      cols.clear();
      for (int k = deg[vtx]; k < deg[vtx + 1]; ++k) {
        const int64_t e = edge_of[size_t(k)];
        for (const JTemplate* jt : jts)
          for (const Lane& l : jt->lanes)
            cols.insert(P_.ubase[size_t(l.field)] +
                        (long long)verts[size_t(e * arity + l.slot)] * P_.unknowns[size_t(l.field)].channels + l.channel);
      }
      best = std::max(best, cols.size());
    }
    return best;
  }
  static std::vector<long long> lane_rowbase(size_t nout, long long n) {
    std::vector<long long> rb(std::max<size_t>(nout, 1));
    for (size_t k = 0; k < rb.size(); ++k) rb[k] = (long long)k * n;
    return rb;
  }
  // Lane buffers, row tables and per-graph incidence; rebuilt when the
  // residual rows or the graphs change (never inside a captured stage).
  void mat_prepare() {
    if (!mt_dirty_ && mt_rowbase_ == rowbase_ && mt_ok_) return;
    bool realloc = false;
    for (size_t i = 0; i < P_.grid_sets.size(); ++i) {
      const GridSet& g = P_.grid_sets[i];
      if (g.jtemplates.empty() || jl_grid_[i]) continue;
      const long long ext = P_.extent_of(g.dom);
      const size_t no = g.evalj.outputs.size();
      jl_grid_[i] = dalloc<Real>(std::max<size_t>(no * size_t(ext), 1));
      const auto rb = lane_rowbase(no, ext);
      jl_rb_grid_[i] = dalloc<long long>(rb.size());
      CK(cudaMemcpyAsync(jl_rb_grid_[i], rb.data(), rb.size() * sizeof(long long), cudaMemcpyHostToDevice, st_));
      realloc = true;
    }
    for (size_t i = 0; i < P_.graph_sets.size(); ++i) {
      const GraphSet& g = P_.graph_sets[i];
      if (g.jtemplates.empty()) continue;
      const long long E = graphs_[size_t(g.graph)].E;
      const size_t no = g.evalj.outputs.size(), need = std::max<size_t>(no * size_t(E), 1);
      if (need > jl_graph_cap_[i]) {
        cudaFree(jl_graph_[i]);
        jl_graph_[i] = dalloc<Real>(need);
        jl_graph_cap_[i] = need;
      }
      const auto rb = lane_rowbase(no, E);
      if (!jl_rb_graph_[i]) jl_rb_graph_[i] = dalloc<long long>(rb.size());
      CK(cudaMemcpyAsync(jl_rb_graph_[i], rb.data(), rb.size() * sizeof(long long), cudaMemcpyHostToDevice, st_));
      realloc = true;
    }
    if (size_t(rows_) > jtmp_cap_) {
      cudaFree(jtmp_);
      jtmp_ = dalloc<Real>(size_t(rows_));
      jtmp_cap_ = size_t(rows_);
    }
    // Per-graph vertex -> incident edges (each edge once, ascending): the
    // row order of spmv_t for a vertex column.
    for (size_t gi = 0; gi < graphs_.size(); ++gi) {
      const GraphData& g = graphs_[gi];
      long long nv = 0;
      for (uint64_t v : g.verts) nv = std::max<long long>(nv, (long long)v + 1);
      std::vector<int> cnt(size_t(nv) + 1, 0), last(size_t(nv), -1), vedge;
      for (int64_t e = 0; e < g.E; ++e)
        for (int k = 0; k < g.arity; ++k) {
          const size_t v = size_t(g.verts[size_t(e * g.arity + k)]);
          if (last[v] != int(e)) {
            last[v] = int(e);
            cnt[v + 1]++;
          }
        }
      for (size_t v = 0; v < size_t(nv); ++v) cnt[v + 1] += cnt[v];
      vedge.resize(size_t(cnt[size_t(nv)]));
      std::vector<int> pos(cnt.begin(), cnt.end() - 1);
      std::fill(last.begin(), last.end(), -1);
      for (int64_t e = 0; e < g.E; ++e)
        for (int k = 0; k < g.arity; ++k) {
          const size_t v = size_t(g.verts[size_t(e * g.arity + k)]);
          if (last[v] != int(e)) {
            last[v] = int(e);
            vedge[size_t(pos[v]++)] = int(e);
          }
        }
      cudaFree(mat_vptr_[gi]);
      cudaFree(mat_vedge_[gi]);
      mat_vptr_[gi] = dalloc<int>(cnt.size());
      mat_vedge_[gi] = dalloc<int>(std::max<size_t>(vedge.size(), 1));
      CK(cudaMemcpyAsync(mat_vptr_[gi], cnt.data(), cnt.size() * sizeof(int), cudaMemcpyHostToDevice, st_));
      if (!vedge.empty())
        CK(cudaMemcpyAsync(mat_vedge_[gi], vedge.data(), vedge.size() * sizeof(int), cudaMemcpyHostToDevice, st_));
      mat_nverts_[gi] = nv;
      CK(cudaStreamSynchronize(st_));
    }
    // Row tables, one per residual template, in template (= row) order.
    const size_t NT = P_.residuals.size();
    std::vector<mo_mat_tmpl> tm(NT);
    std::vector<bool> seen(NT, false);
    std::vector<mo_mat_lane> lanes;
    long long erow_n = 0, ecnt_n = 0;
    for (size_t i = 0; i < P_.grid_sets.size(); ++i) {
      const GridSet& g = P_.grid_sets[i];
      const auto sh = P_.shape_of(g.dom);
      for (const JTemplate& jt : g.jtemplates) {
        mo_mat_tmpl& M = tm[size_t(jt.tmpl)];
        M = mo_mat_tmpl{};
        M.rowbase = rowbase_[size_t(jt.tmpl)];
        M.nrows = P_.extent_of(g.dom);
        M.buf = jl_grid_[i];
        M.kind = 0;
        M.guard = jt.guard_out;
        M.lane0 = int(lanes.size());
        M.nlanes = int(jt.lanes.size());
        for (const Lane& l : jt.lanes) {
          check(P_.unknowns[size_t(l.field)].dom == g.dom, Err::kBindError,
                "materialized J: an unknown read on a different domain than its residual's");
          lanes.push_back({l.out, l.field, l.channel, -1, lane_lin(l, sh)});
        }
        seen[size_t(jt.tmpl)] = true;
      }
    }
    for (size_t i = 0; i < P_.graph_sets.size(); ++i) {
      const GraphSet& g = P_.graph_sets[i];
      const GraphData& gd = graphs_[size_t(g.graph)];
      for (const JTemplate& jt : g.jtemplates) {
        check(jt.lanes.size() <= MO_MAT_MAXL, Err::kInternal, "materialized J: too many lanes per edge row");
        mo_mat_tmpl& M = tm[size_t(jt.tmpl)];
        M = mo_mat_tmpl{};
        M.rowbase = rowbase_[size_t(jt.tmpl)];
        M.nrows = gd.E;
        M.buf = jl_graph_[i];
        M.kind = 1;
        M.guard = -1;
        M.lane0 = int(lanes.size());
        M.nlanes = int(jt.lanes.size());
        M.verts = gd.d_verts;
        M.arity = gd.arity;
        M.vptr = mat_vptr_[size_t(g.graph)];
        M.vedge = mat_vedge_[size_t(g.graph)];
        M.nverts = mat_nverts_[size_t(g.graph)];
        M.eoff = erow_n;  // kJtJ: merged edge rows (k_mat_erows)
        M.ecoff = ecnt_n;
        erow_n += (long long)jt.lanes.size() * gd.E;
        ecnt_n += gd.E;
        for (const Lane& l : jt.lanes) lanes.push_back({l.out, l.field, l.channel, l.slot, 0});
        seen[size_t(jt.tmpl)] = true;
      }
    }
    for (size_t t = 0; t < NT; ++t) check(seen[t], Err::kBindError, "plan was compiled without Jacobian kernels");
    // Column entry lists per (field, channel): templates ascending; within a
    // grid template the rows holding the column ascend as the offset descends.
    std::vector<int> cbase(P_.unknowns.size() + 1, 0);
    for (size_t f = 0; f < P_.unknowns.size(); ++f) cbase[f + 1] = cbase[f] + P_.unknowns[f].channels;
    std::vector<std::vector<mo_mat_centry>> per(size_t(cbase.back()));
    for (size_t t = 0; t < NT; ++t) {
      const mo_mat_tmpl& M = tm[t];
      std::vector<int> idx;
      for (int k = 0; k < M.nlanes; ++k) idx.push_back(M.lane0 + k);
      if (M.kind == 0) {
        std::stable_sort(idx.begin(), idx.end(),
                         [&](int a, int b) { return lanes[size_t(a)].lin > lanes[size_t(b)].lin; });
        for (int k : idx) per[size_t(cbase[size_t(lanes[size_t(k)].field)] + lanes[size_t(k)].ch)].push_back({int(t), k});
      } else {
        for (int k : idx) {  // one entry per (template, column pair): ~mask of its lanes
          auto& v = per[size_t(cbase[size_t(lanes[size_t(k)].field)] + lanes[size_t(k)].ch)];
          if (v.empty() || v.back().t != int(t)) v.push_back({int(t), ~0});
          v.back().lane = ~(~v.back().lane | int(1u << unsigned(k - M.lane0)));
        }
      }
    }
    std::vector<mo_mat_centry> ce;
    std::vector<int> ceptr{0};
    for (auto& v : per) {
      ce.insert(ce.end(), v.begin(), v.end());
      ceptr.push_back(int(ce.size()));
    }
    for (void* p : mt_bufs_) cudaFree(p);
    mt_bufs_.clear();
    auto up = [&](const void* src, size_t bytes) {
      void* d = dalloc<unsigned char>(std::max<size_t>(bytes, 1));
      if (bytes) CK(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st_));
      mt_bufs_.push_back(d);
      return d;
    };
    mt_ = mo_mat_tables{};
    mt_.tm = static_cast<const mo_mat_tmpl*>(up(tm.data(), tm.size() * sizeof(mo_mat_tmpl)));
    mt_.ntm = int(NT);
    mt_.lanes = static_cast<const mo_mat_lane*>(up(lanes.data(), lanes.size() * sizeof(mo_mat_lane)));
    mt_.ce = static_cast<const mo_mat_centry*>(up(ce.data(), ce.size() * sizeof(mo_mat_centry)));
    mt_.ceptr = static_cast<const int*>(up(ceptr.data(), ceptr.size() * sizeof(int)));
    for (size_t f = 0; f < P_.unknowns.size(); ++f) {
      mt_.ubase[f] = P_.ubase[f];
      mt_.chans[f] = P_.unknowns[f].channels;
      mt_.cbase[f] = cbase[f];
    }
    mt_.nfields = int(P_.unknowns.size());
    mt_.nrows = rows_;
    mt_.ncols = P_.num_cols;
    max_trows_ = 1;
    for (const mo_mat_tmpl& M : tm) max_trows_ = std::max<long long>(max_trows_, M.nrows);
    max_fel_ = 1;
    for (size_t f = 0; f < P_.unknowns.size(); ++f) max_fel_ = std::max<long long>(max_fel_, P_.extent_of(P_.unknowns[f].dom));
    for (const mo_mat_tmpl& M : tm) check(M.nlanes <= MO_MAT_MAXL, Err::kInternal, "materialized J: too many lanes per row");
    for (size_t k = 0; k + 1 < ceptr.size(); ++k)
      check(ceptr[k + 1] - ceptr[k] <= MO_MAT_MAXCE, Err::kInternal, "materialized J: too many rows per column");
    mt_.ntl = int(lanes.size());
    mt_.nce = int(ce.size());
    mt_.nk = int(per.size());
    auto r16 = [](size_t b) { return (b + 15) & ~size_t(15); };
    mt_smem_ = r16(sizeof(mo_mat_tmpl) * NT) + r16(sizeof(mo_mat_lane) * lanes.size()) +
               r16(sizeof(mo_mat_centry) * ce.size()) + r16(sizeof(int) * ceptr.size());
    check(mt_smem_ <= 200 * 1024, Err::kBindError, "materialized J: lane tables exceed shared memory");
    if (mt_smem_ > 48 * 1024)  // (k_mat_hbuild stages the tables)
      CK(cudaFuncSetAttribute((const void*)k_mat_hbuild<Real>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              int(mt_smem_)));
    if (mat_ == 2 && (size_t(erow_n) > erow_cap_ || size_t(ecnt_n) > ecnt_cap_)) {
      cudaFree(ecol_);
      cudaFree(eval_);
      cudaFree(ecnt_);
      ecol_ = dalloc<int>(size_t(std::max<long long>(erow_n, 1)));
      eval_ = dalloc<Real>(size_t(std::max<long long>(erow_n, 1)));
      ecnt_ = dalloc<unsigned char>(size_t(std::max<long long>(ecnt_n, 1)));
      erow_cap_ = size_t(erow_n);
      ecnt_cap_ = size_t(ecnt_n);
      realloc = true;
    }
    has_graph_rows_ = ecnt_n > 0;
    if (mat_ == 2) {  // ELL width of H = 2 J^T J: an upper bound on the row widths
      std::vector<std::set<std::tuple<int, int, long long>>> S(size_t(cbase.back()));
      for (size_t t = 0; t < NT; ++t) {
        const mo_mat_tmpl& M = tm[t];
        if (M.kind != 0) continue;
        for (int a = 0; a < M.nlanes; ++a) {
          const mo_mat_lane& A = lanes[size_t(M.lane0 + a)];
          for (int b = 0; b < M.nlanes; ++b) {
            const mo_mat_lane& B = lanes[size_t(M.lane0 + b)];
            S[size_t(cbase[size_t(A.field)] + A.ch)].insert({B.field, B.ch, B.lin - A.lin});
          }
        }
      }
      size_t K = 0;
      for (auto& x : S) K = std::max(K, x.size());
      for (size_t gi = 0; gi < graphs_.size(); ++gi) {  // per vertex: columns of the incident rows
        const GraphData& g = graphs_[gi];
        std::vector<const JTemplate*> jts;
        for (const GraphSet& gs : P_.graph_sets)
          if (gs.graph == int(gi))
            for (const JTemplate& jt : gs.jtemplates) jts.push_back(&jt);
        if (jts.empty()) continue;
        K += graph_row_union(g.verts, g.E, g.arity, mat_nverts_[gi], jts);
      }
      K = std::max<size_t>(K, 1);
      check(K <= MO_MAT_MAXK, Err::kBindError, "normal matrix rows too wide for the device's assembled H (kJtJ)");
      const size_t n = size_t(P_.num_cols);
      if (int(K) != hK_ || n != hn_) {
        cudaFree(hcol_);
        cudaFree(hval_);
        cudaFree(hcnt_);
        check(P_.num_cols < (int64_t(1) << 31), Err::kBindError, "kJtJ: more than 2^31 columns");
        hcol_ = dalloc<int>(K * n + 1);
        hval_ = dalloc<Real>(K * n + 1);
        hcnt_ = dalloc<int>(n + 1);
        // (ELL slots past a row's count are never written; normal_matrix()
        // downloads whole slot planes, so they hold defined zeros)
        CK(cudaMemsetAsync(hcol_, 0, (K * n + 1) * sizeof(int), st_));
        CK(cudaMemsetAsync(hval_, 0, (K * n + 1) * sizeof(Real), st_));
        hK_ = int(K);
        hn_ = n;
        realloc = true;
      }
    }
    CK(cudaStreamSynchronize(st_));
    if (realloc || mt_ok_) invalidate_graphs();  // captured stages hold the old pointers
    mt_rowbase_ = rowbase_;
    mt_dirty_ = false;
    mt_ok_ = true;
    jvalid_ = false;
  }
  // (x blocks per row of the y extent: ~8 resident blocks per SM in total)
  dim3 mat_grid(long long n, int ny) const {
    const long long want = std::max<long long>(1, (8LL * nsm_ + ny - 1) / std::max(ny, 1));
    return dim3(unsigned(std::max<long long>(1, std::min<long long>((n + MO_THREADS - 1) / MO_THREADS, want))),
                unsigned(std::max(ny, 1)));
  }
  void linearize_device() {
    CK(cudaMemsetAsync(&state_->mat_bad, 0, sizeof(int), st_));
    bool grid_rows = false;
    for (size_t i = 0; i < P_.grid_sets.size(); ++i) {
      const GridSet& g = P_.grid_sets[i];
      if (g.jtemplates.empty()) continue;
      mo_kparams kp = kp_grid(g.dom, x_, nullptr);
      kp.out0 = jl_grid_[i];
      kp.rowbase = jl_rb_grid_[i];
      const void* f = evj_kernel("mo_grid_evalj_" + std::to_string(i));
      const long long nb = std::min<long long>(tiles_of(g.dom), (long long)nsm_ * occupancy(f));
      dim3 block = g.dom.dims.size() <= 1 ? dim3(MO_THREADS, 1, 1) : dim3(MO_TILE_X, MO_TILE_Y, 1);
      void* args[] = {&kp};
      klc(f, dim3(unsigned(std::max<long long>(nb, 1))), block, args, 0);
      ++launches_;
      grid_rows = true;
    }
    if (grid_rows && mt_ok_ && rows_ > 0) {
      kl(k_mat_check<Real>, mat_grid(max_trows_, mt_.ntm), dim3(MO_THREADS), mt_, state_);
      ++launches_;
    }
    bool pending_h = mat_ == 2;
    for (size_t i = 0; i < P_.graph_sets.size(); ++i) {
      const GraphSet& g = P_.graph_sets[i];
      if (g.jtemplates.empty() || graphs_[size_t(g.graph)].E == 0) continue;
      mo_kparams kp = kp_graph(int(i), x_, nullptr);
      kp.out0 = jl_graph_[i];
      kp.rowbase = jl_rb_graph_[i];
      const void* f = evj_kernel("mo_graph_evalj_" + std::to_string(i));
      const long long nb =
          std::min<long long>((graphs_[size_t(g.graph)].E + MO_THREADS - 1) / MO_THREADS, (long long)nsm_ * occupancy(f));
      void* args[] = {&kp};
      klc(f, dim3(unsigned(std::max<long long>(nb, 1))), dim3(MO_THREADS), args, 0);
      ++launches_;
    }
    if (pending_h && mt_ok_) {  // assemble H = 2 J^T J (solver.hpp:370-374)
      const long long n = P_.num_cols;
      if (has_graph_rows_) {
        kl(k_mat_erows<Real>, mat_grid(max_trows_, mt_.ntm), dim3(MO_THREADS), mt_, ecol_, eval_, ecnt_);
        ++launches_;
      }
      kls(k_mat_hbuild<Real>, dim3(unsigned(std::max<long long>(1, std::min<long long>((n + 127) / 128, 8LL * nsm_)))),
          dim3(128), mt_smem_, mt_, state_, hK_, hcol_, hval_, hcnt_, static_cast<const int*>(ecol_),
          static_cast<const Real*>(eval_), static_cast<const unsigned char*>(ecnt_));
      ++launches_;
    }
    jvalid_ = true;
  }
  // apply_jtj, materialized branch (solver.hpp:278-283) + apply_damped's
  // damping, exclusion and p'Ap (pcg.hpp:100-102) in k_apply_finish.
  void mat_apply(const Real* pv, Real* out, int flags) {
    check(jvalid_, Err::kInternal, "normal-matrix apply before linearize()");
    const long long n = P_.num_cols;
    const int skip = (flags & MO_F_SKIPDONE) ? 1 : 0;
    if (mat_ == 2) {  // spmv(H, v) (solver.hpp:284)
      kl(k_mat_happly<Real>, dim3(vgrid(n, nsm_, 8)), dim3(MO_THREADS), n, hK_, static_cast<const int*>(hcol_),
         static_cast<const Real*>(hval_), static_cast<const int*>(hcnt_), static_cast<const mo_state*>(state_), skip, pv,
         out);
      ++launches_;
    } else {
      if (rows_ > 0) {
        kl(k_mat_rows<Real>, mat_grid(max_trows_, mt_.ntm), dim3(MO_THREADS), mt_, static_cast<const mo_state*>(state_),
           skip, pv, jtmp_);
        ++launches_;
      }
      kl(k_mat_cols<Real>, mat_grid(max_fel_, mt_.nk), dim3(MO_THREADS), mt_, static_cast<const mo_state*>(state_),
         skip, static_cast<const Real*>(jtmp_), out);
      ++launches_;
    }
    apply_parts_ = vgrid(n, nsm_);
    if (flags & (MO_F_DAMP | MO_F_REDUCE | MO_F_ZEROEXCL)) {
      kl(k_apply_finish<Real>, dim3(vgrid(n, nsm_)), dim3(MO_THREADS), red(0, vgrid(n, nsm_), MO_FIN_PCG_ALPHA, 0), n,
         colmask_, pv, damp_, out, flags);
      ++launches_;
    }
  }

 public:
  void linearize() override {
    Range nv("minopt::linearize");
    ensure_refreshed();
    check(plan_has_evalj(), Err::kBindError, "plan was compiled without Jacobian kernels");
    cur_stage_ = -1;
    mat_prepare();
    linearize_device();
    sync_state();
    csr_ok_ = false;
    if (state_h_->mat_bad) jvalid_ = false;
    check_mat_bad();
  }
  void jacobian(int64_t* rows, int64_t* cols, std::vector<int64_t>* offs, std::vector<int64_t>* col,
                std::vector<double>* val) override {
    check(jvalid_, Err::kBindError, "no Jacobian has been materialized");
    if (!csr_ok_) assemble_csr();
    *rows = rows_;
    *cols = P_.num_cols;
    if (offs) *offs = csr_offs_;
    if (col) *col = csr_col_;
    if (val) val->assign(csr_val_.begin(), csr_val_.end());
  }

  void normal_matrix(std::vector<int64_t>* offs, std::vector<int64_t>* col, std::vector<double>* val) override {
    check(jvalid_ && mat_ == 2, Err::kBindError, "no normal matrix has been assembled");
    const size_t n = size_t(P_.num_cols), K = size_t(hK_);
    std::vector<int> cnt(n);
    std::vector<int> hc(K * n);
    std::vector<Real> hv(K * n);
    if (n) {
      CK(cudaMemcpyAsync(cnt.data(), hcnt_, n * sizeof(int), cudaMemcpyDeviceToHost, st_));
      CK(cudaMemcpyAsync(hc.data(), hcol_, K * n * sizeof(int), cudaMemcpyDeviceToHost, st_));
      CK(cudaMemcpyAsync(hv.data(), hval_, K * n * sizeof(Real), cudaMemcpyDeviceToHost, st_));
    }
    CK(cudaStreamSynchronize(st_));
    offs->assign(1, 0);
    col->clear();
    val->clear();
    for (size_t q = 0; q < n; ++q) {
      for (int k = 0; k < cnt[q]; ++k) {
        col->push_back(hc[size_t(k) * n + q]);
        val->push_back(double(hv[size_t(k) * n + q]));
      }
      offs->push_back(int64_t(col->size()));
    }
  }

 private:
  // The reference's CSR assembly (solver.hpp:323-369) over the device lanes.
  void assemble_csr() {
    std::vector<std::vector<Real>> hg(P_.grid_sets.size()), hr(P_.graph_sets.size());
    for (size_t i = 0; i < P_.grid_sets.size(); ++i) {
      const GridSet& g = P_.grid_sets[i];
      if (g.jtemplates.empty()) continue;
      hg[i].resize(g.evalj.outputs.size() * size_t(P_.extent_of(g.dom)));
      if (!hg[i].empty())
        CK(cudaMemcpyAsync(hg[i].data(), jl_grid_[i], hg[i].size() * sizeof(Real), cudaMemcpyDeviceToHost, st_));
    }
    for (size_t i = 0; i < P_.graph_sets.size(); ++i) {
      const GraphSet& g = P_.graph_sets[i];
      if (g.jtemplates.empty()) continue;
      hr[i].resize(g.evalj.outputs.size() * size_t(graphs_[size_t(g.graph)].E));
      if (!hr[i].empty())
        CK(cudaMemcpyAsync(hr[i].data(), jl_graph_[i], hr[i].size() * sizeof(Real), cudaMemcpyDeviceToHost, st_));
    }
    CK(cudaStreamSynchronize(st_));
    csr_offs_.assign(1, 0);
    csr_col_.clear();
    csr_val_.clear();
    auto begin_row = [&] { csr_offs_.push_back(int64_t(csr_col_.size())); };
    auto push = [&](int64_t c, Real v) {
      csr_col_.push_back(c);
      csr_val_.push_back(v);
      csr_offs_.back() = int64_t(csr_col_.size());
    };
    for (size_t t = 0; t < P_.residuals.size(); ++t) {
      bool done = false;
      for (size_t i = 0; i < P_.grid_sets.size() && !done; ++i) {
        const GridSet& g = P_.grid_sets[i];
        for (const JTemplate& jt : g.jtemplates) {
          if (size_t(jt.tmpl) != t) continue;
          const auto sh = P_.shape_of(g.dom);
          const int64_t ext = P_.extent_of(g.dom);
          const std::vector<Real>& buf = hg[i];
          for (int64_t e = 0; e < ext; ++e) {
            begin_row();
            if (buf[size_t(jt.guard_out) * size_t(ext) + size_t(e)] == Real(0)) continue;
            for (const Lane& l : jt.lanes)
              push(P_.ubase[size_t(l.field)] + (e + lane_lin(l, sh)) * P_.unknowns[size_t(l.field)].channels +
                       l.channel,
                   buf[size_t(l.out) * size_t(ext) + size_t(e)]);
          }
          done = true;
          break;
        }
      }
      for (size_t i = 0; i < P_.graph_sets.size() && !done; ++i) {
        const GraphSet& g = P_.graph_sets[i];
        for (const JTemplate& jt : g.jtemplates) {
          if (size_t(jt.tmpl) != t) continue;
          const GraphData& gd = graphs_[size_t(g.graph)];
          const std::vector<Real>& buf = hr[i];
          std::vector<std::pair<int64_t, Real>> row;
          for (int64_t e = 0; e < gd.E; ++e) {
            begin_row();
            row.clear();
            for (const Lane& l : jt.lanes)
              row.emplace_back(P_.ubase[size_t(l.field)] +
                                   int64_t(gd.verts[size_t(e * gd.arity + l.slot)]) *
                                       P_.unknowns[size_t(l.field)].channels +
                                   l.channel,
                               buf[size_t(l.out) * size_t(gd.E) + size_t(e)]);
            std::stable_sort(row.begin(), row.end(),
                             [](const auto& x, const auto& y) { return x.first < y.first; });
            for (size_t k = 0; k < row.size();) {
              const int64_t c = row[k].first;
              Real v = row[k].second;
              for (++k; k < row.size() && row[k].first == c; ++k) v += row[k].second;
              push(c, v);
            }
          }
          done = true;
          break;
        }
      }
    }
    csr_ok_ = true;
  }

  // Jacobi PCG (pcg.hpp:63-130) as a captured CUDA graph.  (Fusing the
  // direction update into the apply's p staging was measured slower: the
  // apply is issue-bound, the p update streams at HBM speed on its own.)
  void pcg_body(bool lm, bool init_done = false) {
    const long long n = P_.num_cols;
    const int vg = vgrid(n, nsm_);
    // Update / direction kernels: one wave of 4 blocks per SM while a thread
    // has few float4 groups (small grids are latency-bound), 16 blocks per SM
    // (several waves) for large ones; both measured on B200 (1024^2 vs 8192^2
    // ARAP).  MO_B200_VEC_PER_SM overrides.
    static const int vper_env = std::getenv("MO_B200_VEC_PER_SM") ? std::atoi(std::getenv("MO_B200_VEC_PER_SM")) : 0;
    const int vper = vper_env > 0 ? vper_env : (n / 4 > 8LL * nsm_ * 4 * MO_THREADS ? 16 : 4);
    // (over the active groups when the kernels walk the list)
    const int vgu = gl() && gl_count_ >= 0 ? vgrid(std::max<long long>(gl_count_, 1), nsm_, vper)  // (a thread per group)
                                          : vgrid(n, nsm_, vper);
    const Real* mdv = lm ? md_ : m_;
    const int pre = cfg_.use_preconditioner ? 1 : 0;
    if (!init_done) {
      kl(k_pcg_init<Real>, dim3(vg), dim3(MO_THREADS), red(0, vg, MO_FIN_PCG_INIT, 0), n, colmask_, b_, mdv, delta_, r_,
         p_, pre);
      ++launches_;
      reduce_done(MO_FIN_PCG_INIT, 0);
    }
    pending_p_ = sh_.on ? p_ : nullptr;  // strips: neighbours' p rows, exchanged by apply()
    const int flags = MO_F_REDUCE | MO_F_ZEROEXCL | MO_F_SKIPDONE | MO_F_EXSKIP | (lm ? MO_F_DAMP : 0);
    // Consumer-side reductions (unsharded grid plans): the apply and the
    // update only store block partials; the next kernel sums them in every
    // block (same fixed order, bitwise the same total) and derives alpha /
    // beta itself, removing the atomic + last-block tail from the producers.
    static const bool nocons = std::getenv("MO_B200_NO_CONSUMER") != nullptr;
    const bool cons = !nocons && !sh_.on && !mat_ && (P_.graph_sets.empty() || vertex_apply_one_pass());
    // Deferred delta (k_pcg_update_r / k_pcg_dp) moves 42 instead of 46 bytes
    // per column and wins where the pair streams from HBM (8192^2: 1.40 vs
    // 1.46 ms per iteration); on L2-sized grids the extra stream in the
    // direction kernel costs more than it saves (ARAP 1024^2: 40 vs 34 us),
    // so it is used on the large-grid configuration of the vector kernels.
    // MO_B200_NO_DEFER=1 / MO_B200_DEFER=1 force either.
    const bool nodefer = std::getenv("MO_B200_NO_DEFER") != nullptr;
    const bool fdefer = std::getenv("MO_B200_DEFER") != nullptr;
    const bool defer = cons && !nodefer && (fdefer || vper == 16);
    for (int k = 0; k < cfg_.linear_iters; ++k) {
      prof_begin(0);
      consumer_ = cons;
      apply(p_, ap_, flags);
      consumer_ = false;
      prof_end(0);
      prof_begin(1);
      if (defer) {  // deferred-delta pair (k_pcg_update_r / k_pcg_dp, mo_kernels.cuh)
        mo_red ru = red(0, vgu, MO_FIN_PARTIALS, 0);
        ru.partials = partials2_;
        kl(gl() ? k_pcg_update_r<Real, true> : k_pcg_update_r<Real, false>, dim3(vgu), dim3(MO_THREADS), ru, n, cmv(), mdv, r_, ap_, pre,
           (const double*)partials_, apply_parts_, k, gl());
        const int last = k + 1 < cfg_.linear_iters ? 0 : 1;  // the last direction is never applied
        kl(gl() ? k_pcg_dp<Real, true> : k_pcg_dp<Real, false>, dim3(vgu), dim3(MO_THREADS), state_, n, cmv(), mdv, r_, delta_, p_, pre,
           (const double*)partials2_, vgu, k, last, gl());
        launches_ += 2;
        prof_end(1);
        continue;
      }
      // (A cooperative single-kernel update + direction with a grid barrier
      // was measured slower on B200 than this pair at every config size.)
      mo_red ru = red(0, vgu, cons ? MO_FIN_PARTIALS : MO_FIN_PCG_BETA, 0);
      if (cons) ru.partials = partials2_;
      const double* pap_part = cons ? partials_ : nullptr;
      kl(gl() ? k_pcg_update<Real, true> : k_pcg_update<Real, false>, dim3(vgu), dim3(MO_THREADS), ru, n, cmv(), mdv, delta_, r_, p_, ap_, pre, pap_part,
         apply_parts_, k, gl());
      ++launches_;
      if (!cons) reduce_done(MO_FIN_PCG_BETA, 0);
      const double* rz_part = cons ? partials2_ : nullptr;
      if (k + 1 < cfg_.linear_iters) {  // the last direction is never applied
        kl(gl() ? k_pcg_p<Real, true> : k_pcg_p<Real, false>, dim3(vgu), dim3(MO_THREADS), state_, n, cmv(), mdv, r_, p_, pre, rz_part, vgu, k, gl());
        ++launches_;
        pending_p_ = sh_.on ? p_ : nullptr;
      } else if (cons) {  // bookkeeping of the last r'z
        kl(k_pcg_fin<Real>, dim3(1), dim3(MO_THREADS), state_, rz_part, vgu, k);
        ++launches_;
      }
      prof_end(1);
    }
    pending_p_ = nullptr;
  }

  // Replay `body` as a CUDA graph captured on first use (per stage key);
  // MO_B200_NOGRAPH=1 launches it directly.  Kernels count individually.
  template <class F>
  void run_stage(int key, F&& body) {
    static const bool nograph = std::getenv("MO_B200_NOGRAPH") != nullptr;
    cur_stage_ = key;
    // Strips over NCCL capture like the unsharded stages (halo send/recv and
    // the all-gathers are stream operations); the single-process transport
    // (LocalComm) orders its peer copies with host barriers and runs eagerly.
    if (nograph || (sh_.on && !(comm_ && comm_->capturable()))) {
      stage_pos_[key] = 0;
      body();
      return;
    }
    auto it = stage_exec_.find(key);
    if (it == stage_exec_.end()) {
      stage_pos_[key] = 0;
      const int64_t before = launches_;
      cudaGraph_t graph;
      CK(cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed));
      try {
        body();
      } catch (...) {
        cudaGraph_t g2;
        cudaStreamEndCapture(st_, &g2);
        if (g2) cudaGraphDestroy(g2);
        throw;
      }
      CK(cudaStreamEndCapture(st_, &graph));
      cudaGraphExec_t exec;
      CK(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      stage_nodes_[key] = launches_ - before;
      launches_ = before;
      it = stage_exec_.emplace(key, exec).first;
    }
    CK(cudaGraphLaunch(it->second, st_));
    launches_ += stage_nodes_[key];
  }

  // ------------------------------------------------------------ profiling
  // Inside stream capture an event record must be an external event node to
  // be timed; outside capture it is a plain record.
  unsigned capture_flags() {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st_, &cs));
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
  }
  void prof_begin(int kind) {
    if (!profiling_ || cur_stage_ < 0) return;
    auto& v = stage_ev_[cur_stage_];
    size_t& pos = stage_pos_[cur_stage_];
    if (pos == v.size()) {
      ProfEv e;
      CK(cudaEventCreate(&e.a));
      CK(cudaEventCreate(&e.b));
      v.push_back(e);
    }
    v[pos].kind = kind;
    CK(cudaEventRecordWithFlags(v[pos].a, st_, capture_flags()));
    open_.push_back(pos++);
  }
  void prof_end(int) {
    if (!profiling_ || cur_stage_ < 0 || open_.empty()) return;
    auto& v = stage_ev_[cur_stage_];
    CK(cudaEventRecordWithFlags(v[open_.back()].b, st_, capture_flags()));
    open_.pop_back();
  }
  void collect_profile(int stage) {
    if (!profiling_) return;
    auto& v = stage_ev_[stage];
    for (size_t i = 0; i < stage_pos_[stage] && i < v.size(); ++i) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, v[i].a, v[i].b) == cudaSuccess) {
        prof_[size_t(v[i].kind)].total_ms += ms;
        prof_[size_t(v[i].kind)].count++;
      } else {
        cudaGetLastError();
      }
    }
  }

  void sync_state() {
    CK(cudaMemcpyAsync(state_h_, state_, sizeof(mo_state), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    if (state_h_->peer_timeout) fail(Err::kInternal, "peer reduction timed out: the strip ranks are out of step");
  }
  void download(const Real* src, void* out, int64_t n) {
    check(n == P_.num_cols, Err::kShapeMismatch, "vector size mismatch");
    if (n) CK(cudaMemcpyAsync(out, src, size_t(n) * sizeof(Real), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
  }

  Plan P_;
  Config cfg_;
  int dev_ = 0, nsm_ = 148;
  cudaStream_t st_ = nullptr;
  cudaStream_t sd_ = nullptr;                      // strips: p halo exchange beside the interior apply
  cudaEvent_t ev_p_ = nullptr, ev_h_ = nullptr;    // (fork after the p update / join after the exchange)
  const Real* pending_p_ = nullptr;                // p whose halo the next apply exchanges
  int64_t ov0_ = -1, ov1_ = -1;                    // apply row range override (overlapped strips)
  Module mod_;
  Real *x_ = nullptr, *xt_ = nullptr, *b_ = nullptr, *m_ = nullptr, *md_ = nullptr, *damp_ = nullptr;
  Real *delta_ = nullptr, *r_ = nullptr, *p_ = nullptr, *ap_ = nullptr, *vtmp_ = nullptr, *otmp_ = nullptr;
  Real* resid_ = nullptr;
  size_t resid_cap_ = 0;
  double* bd_ = nullptr;
  std::vector<Real*> arr_, comp_;
  std::vector<int64_t> arr_n_;
  std::vector<unsigned char*> masks_;
  unsigned char* colmask_ = nullptr;
  bool cm_any_ = true;     // some column mask bit set (see refresh())
  int* anyflag_ = nullptr;  // (device flag of that test)
  double* params_d_ = nullptr;
  std::vector<double> params_h_;
  mo_state* state_ = nullptr;
  mo_state* state_h_ = nullptr;
  double* partials_ = nullptr;
  double* partials2_ = nullptr;   // r'z block partials (consumer-side reductions)
  bool consumer_ = false;         // PCG applies store p'Ap block partials only
  int apply_parts_ = 0;           // block partials of the last captured apply
  std::vector<GraphData> graphs_;
  std::vector<GSet> gsets_;
  std::vector<long long*> grid_rowbase_;
  std::vector<int64_t> rowbase_, rowbase_dev_;
  int64_t rows_ = 0;
  int64_t unconstrained_ = 0;
  Comm* comm_ = nullptr;      // strip-shard communicator (not owned)
  Shard sh_;
  double* rankbuf_ = nullptr;  // gathered per-rank partials
  double* chob_ = nullptr;     // this rank's kernel choices (tuning broadcast)
  std::vector<int*> tiles_;              // active-tile lists of masked gather domains
  std::vector<unsigned char*> tflags_;   // (their per-tile flags)
  void* tl_temp_ = nullptr;              // cub::DeviceSelect scratch
  int* glist_ = nullptr;                 // active-group list [count, groups] (build_group_list)
  long long gl_count_ = -1;              // (its count on the host, -1 unknown)
  std::vector<int> tl_count_;            // active-tile counts on the host
  int* gvals_ = nullptr;
  unsigned char* gflags_ = nullptr;
  void* gl_temp_ = nullptr;
  size_t gl_temp_bytes_ = 0;
  size_t tl_temp_bytes_ = 0;
  bool peer_on_ = false;       // reductions through k_peer_fin (peer-mapped blocks)
  bool peer_ready_ = false;    // (after the first tuning)
  mo_peer peer_{};
  bool x_bound_ = false, params_bound_ = false, refreshed_ = false;
  std::map<const void*, int> occ_;
  ModuleInfo minfo_;
  std::map<int, cudaGraphExec_t> stage_exec_;
  bool tuned_ = false;
  std::vector<Real*> lcache_;    // per gather set: lane-cache planes (variant 8)
  std::vector<int> bm_choice_;   // per gather set: 1 = TMA two-phase build_normal
  std::vector<int> jtj_choice_;  // per gather set: 0 gather program, 1 two-phase tiles, 2 streaming, 3 TMA streaming
  std::map<std::string, mo_tmaps> tmaps_;  // per (gather set, staged buffers)
  std::string module_key_;
  std::map<int, int64_t> stage_nodes_;
  std::vector<void*> owned_;
  int64_t launches_ = 0;
  bool profiling_ = false;
  std::vector<Prof> prof_ = std::vector<Prof>(4);
  std::map<int, std::vector<ProfEv>> stage_ev_;
  std::map<int, size_t> stage_pos_;
  std::vector<size_t> open_;
  int cur_stage_ = -1;
  double* mu_h_ = nullptr;  // pinned staging of the LM radius
};

// ---------------------------------------------------------------- standalone PCG
// pcg<Real>(apply_a, b, m, delta, opt, ws, excluded) (pcg.hpp:59-130) over
// a caller-supplied operator: the session's PCG kernels (init, alpha from
// p'Ap with the excluded outputs zeroed, update, direction), one host sync
// per iteration for the stop test.  Not a hot path: the solver's own PCG
// runs inside captured CUDA graphs with the generated J^T J p.
namespace {
template <class Real>
PcgOutcome run_pcg_t(int device, int64_t n, PcgApply apply, void* user, const void* b, const void* m, void* delta,
                     const PcgOpts& o, const uint8_t* excluded) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(Err::kNoDevice, "no CUDA device available (the B200 path has no CPU fallback)");
  check(device >= 0 && device < ndev, Err::kNoDevice, "device index out of range");
  check(n >= 0, Err::kShapeMismatch, "pcg operand sizes do not match");
  CK(cudaSetDevice(device));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const size_t N = size_t(std::max<int64_t>(n, 1));
  std::vector<void*> owned;
  auto alloc = [&](size_t bytes) {
    void* q = nullptr;
    CK(cudaMalloc(&q, std::max<size_t>(bytes, 16)));
    owned.push_back(q);
    return q;
  };
  Real* bd = static_cast<Real*>(alloc(N * sizeof(Real)));
  Real* md = static_cast<Real*>(alloc(N * sizeof(Real)));
  Real* dd = static_cast<Real*>(alloc(N * sizeof(Real)));
  Real* r = static_cast<Real*>(alloc(N * sizeof(Real)));
  Real* p = static_cast<Real*>(alloc(N * sizeof(Real)));
  Real* ap = static_cast<Real*>(alloc(N * sizeof(Real)));
  unsigned char* cm = excluded ? static_cast<unsigned char*>(alloc(N)) : nullptr;
  mo_state* state = static_cast<mo_state*>(alloc(sizeof(mo_state)));
  double* partials = static_cast<double*>(alloc(2 * size_t(kPartCap) * sizeof(double)));
  mo_state h{};
  h.tol_rel = o.tol_rel;
  h.tol_abs = o.tol_abs;
  h.use_precond = o.use_preconditioner;
  PcgOutcome out;
  try {
    if (n) {
      CK(cudaMemcpyAsync(bd, b, size_t(n) * sizeof(Real), cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(md, m, size_t(n) * sizeof(Real), cudaMemcpyHostToDevice, st));
      if (cm) CK(cudaMemcpyAsync(cm, excluded, size_t(n), cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemcpyAsync(state, &h, sizeof(mo_state), cudaMemcpyHostToDevice, st));
    const int vg = vgrid(std::max<int64_t>(n, 1), nsm);
    auto red = [&](int op) {
      mo_red R;
      R.partials = partials;
      R.counter = &state->counters[0];
      R.state = state;
      R.part_base = 0;
      R.part_total = vg;
      R.fin_op = op;
      R.fin_arg = 0;
      return R;
    };
    const int pre = o.use_preconditioner ? 1 : 0;
    k_pcg_init<Real><<<vg, MO_THREADS, 0, st>>>(red(MO_FIN_PCG_INIT), n, cm, bd, md, dd, r, p, pre);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&h, state, sizeof(mo_state), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int k = 0; k < o.max_iters && !h.done; ++k) {
      apply(p, ap, st, user);  // y = A x, complete on return or enqueued on `st`
      k_apply_finish<Real><<<vg, MO_THREADS, 0, st>>>(red(MO_FIN_PCG_ALPHA), n, cm, p, nullptr, ap,
                                                        MO_F_ZEROEXCL | MO_F_REDUCE);
      k_pcg_update<Real, false><<<vg, MO_THREADS, 0, st>>>(red(MO_FIN_PCG_BETA), n, cm, md, dd, r, p, ap, pre, nullptr, 0, k,
                                                    nullptr);
      k_pcg_p<Real, false><<<vg, MO_THREADS, 0, st>>>(state, n, cm, md, r, p, pre, nullptr, 0, k, nullptr);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(&h, state, sizeof(mo_state), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    if (n) CK(cudaMemcpyAsync(delta, dd, size_t(n) * sizeof(Real), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out.iterations = h.iters;
    out.indefinite = h.indefinite != 0;
    out.nonfinite = h.nonfinite != 0;
  } catch (...) {
    for (void* q : owned) cudaFree(q);
    cudaStreamDestroy(st);
    throw;
  }
  for (void* q : owned) cudaFree(q);
  cudaStreamDestroy(st);
  return out;
}
}  // namespace

PcgOutcome run_pcg(int device, int precision, int64_t n, PcgApply apply, void* user, const void* b, const void* m,
                   void* delta, const PcgOpts& opt, const uint8_t* excluded) {
  check(apply != nullptr, Err::kBindError, "pcg needs an operator");
  if (precision == 0) return run_pcg_t<float>(device, n, apply, user, b, m, delta, opt, excluded);
  return run_pcg_t<double>(device, n, apply, user, b, m, delta, opt, excluded);
}

std::unique_ptr<SessionBase> make_session(const Plan& plan, int device) {
  if (plan.cfg.precision == 0) return std::make_unique<Session<float>>(plan, device);
  return std::make_unique<Session<double>>(plan, device);
}

std::unique_ptr<SessionBase> make_shard_session(const Plan& plan, int device, Comm* comm, int64_t row0,
                                                int64_t row1, int halo) {
  check(comm != nullptr, Err::kBindError, "shard session needs a communicator");
  if (plan.cfg.precision == 0) return std::make_unique<Session<float>>(plan, device, comm, row0, row1, halo);
  return std::make_unique<Session<double>>(plan, device, comm, row0, row1, halo);
}

int halo_rows(const Plan& P) {
  int reach = 0, H = 0;
  auto scan = [&](const Program& pg) {
    for (const Instr& in : pg.instrs) {
      const bool load = in.op == kLoadU || in.op == kLoadA || in.op == kLoadC || in.op == kLoadP;
      if ((load && !in.graph) || in.op == kInB) reach = std::max(reach, std::abs(int(in.off[0])));
    }
  };
  for (const GridSet& g : P.grid_sets) {
    scan(g.cost);
    scan(g.evalf);
    if (g.has_evalj) {
      scan(g.evalj);
      for (const JTemplate& jt : g.jtemplates)
        for (const Lane& l : jt.lanes) H = std::max(H, std::abs(l.off[0]));
    }
  }
  for (const GatherSet& g : P.gather_sets) {
    scan(g.bm);
    scan(g.jtj);
  }
  for (const ComputedKernel& c : P.computed_kernels) scan(c.prog);
  for (const ExcludeKernel& e : P.exclude_kernels) scan(e.prog);
  return reach + H;
}

}  // namespace mo
