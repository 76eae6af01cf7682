// mo_device.cuh — device-side definitions shared by the hand-written kernels
// (mo_kernels.cu, compiled by nvcc into libmo_b200.so) and the per-element
// kernels generated at plan time from the reference's KernelPrograms
// (mo_codegen.cpp, compiled by NVRTC for sm_100a).  The file is embedded
// verbatim into every generated module, so it must stay self-contained
// (no standard headers).
#ifndef MO_DEVICE_CUH_
#define MO_DEVICE_CUH_

#define MO_MAX_VIEWS 32
#define MO_MAX_UNK 16
#define MO_THREADS 256
#define MO_TILE_X 32
#define MO_TILE_Y 8

// One bound field: channel-interleaved values over the field's own grid
// domain (reference eval.hpp:15-21).  Shapes are GLOBAL extents; `row_lo` is
// the global axis-0 row stored first in this (possibly strip-sharded) buffer.
struct mo_view {
  const void* p;
  int ch;
  int nd;
  int s0, s1, s2;
  int row_lo;
};

// Device-resident solver scalars.  Real-typed quantities are stored as double
// (exact for float) and always recomputed in Real to follow pcg.hpp:63-130.
struct mo_state {
  double rz, pap, alpha, beta, stop, rz_next;
  double tol_rel, tol_abs;
  int done, iters, indefinite, nonfinite;
  int use_precond, nonfinite_kernel;
  int any_nonzero, mat_bad;  // mat_bad: linearize's CSR checks (k_mat_check)
  long long unconstrained;
  double sums[8];
  unsigned counters[8];
  double mu;  // LM trust-region radius of the current trial
  double rzs[2];  // consumer-side reductions: rz of PCG iteration k in rzs[k & 1]
  // Deferred-delta PCG: where the PCG stopped, 2k (the update of iteration k
  // found p'Ap unusable: no alpha_k) or 2k + 1 (r'z of iteration k ended it
  // after alpha_k); INT_MAX while running.  Unlike `done`, a kernel of
  // iteration k can test it against its own k while its block 0 writes it.
  int stop_code;
  int peer_timeout;  // k_peer_fin gave up waiting for a rank (ranks out of step)
};

// Finalisation ops run by the last block of a reduction.
enum {
  MO_FIN_STORE = 0,      // sums[slot] = total (slot in fin_arg)
  MO_FIN_PCG_INIT = 1,   // rz0, stop test          (pcg.hpp:88-95)
  MO_FIN_PCG_ALPHA = 2,  // p'Ap checks, alpha      (pcg.hpp:100-110)
  MO_FIN_PCG_BETA = 3,   // rz', stop test, beta    (pcg.hpp:116-124)
  MO_FIN_UNCONSTRAINED = 4,
  MO_FIN_STORE2 = 5,     // sums[slot], sums[slot+1] = pair totals
  MO_FIN_BM_INIT = 6,    // unconstrained count + rz0 / stop test (fused bm + pcg init)
  MO_FIN_PARTIALS = 7,   // store the block partials only; the consuming kernel sums them
};

enum {
  MO_F_DAMP = 1,       // jtj: out += damp * p              (solver.hpp:401-405)
  MO_F_REDUCE = 2,     // kernel contributes to a reduction
  MO_F_PATCH = 4,      // bm: identity patch + unconstrained (solver.hpp:241-250)
  MO_F_ZEROEXCL = 8,   // jtj: zero excluded columns        (pcg.hpp:101)
  MO_F_SKIPDONE = 16,  // return at once when the PCG has already stopped
  MO_F_PCGINIT = 64,   // bm: also delta = 0, r = b, p = z = b/m, rz0 (pcg.hpp:75-97)
  MO_F_LCACHE = 128,   // bm8: also write the lane cache of the J^T J p apply (in2)
  MO_F_EXSKIP = 256,   // jtj (PCG): no stores for excluded elements (their Ap is never read)
};

// One deterministic reduction: partial slots [part_base, part_base+gridDim)
// of [0, part_total); the last arriving block finalises with fin_op.
struct mo_red {
  double* partials;
  unsigned* counter;
  mo_state* state;
  int part_base, part_total;
  int fin_op, fin_arg;
};

#define MO_MAX_PARAMS 16
struct mo_kparams {
  mo_view v[MO_MAX_VIEWS];
  const double* params;
  double pv[MO_MAX_PARAMS];  // parameter values (constant bank); params[] beyond MO_MAX_PARAMS
  int dnd, d0, d1, d2;  // iteration domain, global shape
  int row0, row1;       // axis-0 rows this launch iterates (global)
  int row_lo;           // first global row of the per-element storage
  int flags;
  void* out0;
  void* out1;
  const void* in0;  // p for damp / p'Ap
  const void* in1;  // damp
  const void* in2;  // (unused)
  const void* in3;  // (unused)
  void* out2;       // PCGINIT: p
  void* out3;       // PCGINIT: delta
  void* out4;       // PCGINIT: r
  const unsigned char* mask;     // per-element exclusion (uint8) or null
  const unsigned char* colmask;  // per-column exclusion (uint8) or null
  long long ubase[MO_MAX_UNK];   // local column base per unknown field
  const long long* rowbase;      // evalf: residual row base per output
  const int* verts;              // graph: int32 vertex table, edge-major
  int arity;
  int chunk;                     // jtj3: rows per work item (chunk + 2*halo is a multiple of 8)
  long long nedges;
  const int* vptr;               // graph vertex kernels: incident-edge CSR of one domain
  const int* vedge;
  long long nverts;
  mo_red red;
  mo_state* state;
};

// TMA tensor maps of the fields a staged apply kernel streams into shared
// memory (second __grid_constant__ kernel parameter).  Same 128-byte, 64-byte
// aligned layout as the driver's CUtensorMap.
#define MO_MAX_TMAPS 16
struct __align__(64) mo_tmap {
  unsigned long long w[16];
};
struct mo_tmaps {
  mo_tmap m[MO_MAX_TMAPS];
};

// Programmatic dependent launch: every kernel first waits for its stream
// predecessor to complete (memory visible); the successor is triggered
// implicitly when this grid exits.  Harmless without the PDL attribute.
// (MO_PDL_EARLY: trigger at entry instead - measured slower.)
#ifndef MO_PDL_EARLY
#define MO_PDL_ENTRY() asm volatile("griddepcontrol.wait;" ::: "memory")
#else
#define MO_PDL_ENTRY() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")
#endif

// ---------------------------------------------------------------- TMA / mbarrier
__device__ __forceinline__ unsigned mo_smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mo_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mo_smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mo_mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// One arrival that also announces `bytes` of TMA transactions for this phase.
__device__ __forceinline__ void mo_mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mo_smem_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mo_mbar_wait(unsigned long long* b, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(mo_smem_addr(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
// One plain arrival (release): a consumer is done with a ring slot.
__device__ __forceinline__ void mo_mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mo_smem_addr(b)) : "memory");
}
// Generic-proxy reads of a ring slot are ordered before the async-proxy
// (TMA) writes that refill it.
__device__ __forceinline__ void mo_fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// 2-D tiled TMA load: box at (c_inner, c_outer) of tensor map `m` into smem
// `dst`, completing `bytes` on barrier `b`.  Out-of-bounds box elements are
// zero-filled, which is exactly the reference's OOB->0 read (eval.hpp:47-51).
__device__ __forceinline__ void mo_tma_load_2d(void* dst, const mo_tmap* m, int c_inner, int c_outer,
                                               unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(mo_smem_addr(dst)), "l"(reinterpret_cast<unsigned long long>(m)), "r"(c_inner), "r"(c_outer),
      "r"(mo_smem_addr(b))
      : "memory");
}

// The same with an L2 eviction-priority hint (createpolicy): streamed-once
// data (the lane cache) marked evict_first so it does not push the PCG
// vectors out of L2 on grids whose working set nearly fits.
__device__ __forceinline__ unsigned long long mo_l2_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void mo_tma_load_2d_hint(void* dst, const mo_tmap* m, int c_inner, int c_outer,
                                                    unsigned long long* b, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(mo_smem_addr(dst)), "l"(reinterpret_cast<unsigned long long>(m)), "r"(c_inner), "r"(c_outer),
      "r"(mo_smem_addr(b)), "l"(pol)
      : "memory");
}

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ bool mo_finite(double x) { return x == x && fabs(x) <= 1.7976931348623157e308; }

// pow_eval / ipow (reference common.hpp:102-124): one rounding rule everywhere.
template <class Real>
__device__ __forceinline__ Real mo_ipow(Real x, long long n) {
  if (n < 0) return Real(1) / mo_ipow(x, -n);
  Real r = Real(1);
  while (n > 0) {
    if (n & 1) r *= x;
    x *= x;
    n >>= 1;
  }
  return r;
}
__device__ __forceinline__ float mo_pow_(float x, float y) { return powf(x, y); }
__device__ __forceinline__ double mo_pow_(double x, double y) { return pow(x, y); }
__device__ __forceinline__ float mo_sqrt_(float x) { return sqrtf(x); }
__device__ __forceinline__ double mo_sqrt_(double x) { return sqrt(x); }
template <class Real>
__device__ __forceinline__ Real mo_pow_eval(Real x, long long num, long long den) {
  if (den == 1) {
    if (num >= -32 && num <= 32) return mo_ipow(x, num);
    return mo_pow_(x, Real(num));
  }
  if (den == 2) return mo_ipow(mo_sqrt_(x), num);
  return mo_pow_(x, Real(num) / Real(den));
}

// Deterministic block sum (fixed shuffle tree, fixed warp order).
__device__ __forceinline__ double mo_block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int nw = (blockDim.x * blockDim.y + 31) >> 5;
  if ((tid & 31) == 0) sh[tid >> 5] = v;
  __syncthreads();
  double t = 0;
  if (tid < 32) {
    t = tid < nw ? sh[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

// Scalar finalisation: a single thread, after the reduction total is known.
template <class Real>
__device__ void mo_finalize(mo_state* st, int op, int arg, double total, double total2) {
  switch (op) {
    case MO_FIN_STORE: st->sums[arg] = total; break;
    case MO_FIN_STORE2:
      st->sums[arg] = total;
      st->sums[arg + 1] = total2;
      break;
    case MO_FIN_UNCONSTRAINED: st->unconstrained = (long long)total; break;
    case MO_FIN_BM_INIT:
      st->unconstrained = (long long)total;
      total = total2;
      [[fallthrough]];
    case MO_FIN_PCG_INIT: {
      Real rz = Real(total);
      st->rz = double(rz);
      st->rzs[0] = double(rz);
      if (!mo_finite(double(rz))) {
        st->nonfinite = 1;
        st->done = 1;
        st->stop_code = -1;  // before iteration 0
        break;
      }
      Real tr = Real(st->tol_rel);
      Real stop = tr * tr * rz;
      Real ta = Real(st->tol_abs);
      if (ta > stop) stop = ta;
      st->stop = double(stop);
      if (rz <= stop) {
        st->done = 1;
        st->stop_code = -1;
      }
      break;
    }
    case MO_FIN_PCG_ALPHA: {
      Real pap = Real(total);
      st->pap = double(pap);
      if (!mo_finite(double(pap))) {
        st->nonfinite = 1;
        st->done = 1;
      } else if (pap <= Real(0)) {
        st->indefinite = 1;
        st->done = 1;
      } else {
        st->alpha = double(Real(st->rz) / pap);
      }
      break;
    }
    case MO_FIN_PCG_BETA: {
      Real rzn = Real(total);
      st->rz_next = double(rzn);
      if (!mo_finite(double(rzn))) {
        st->nonfinite = 1;
        st->done = 1;
        break;
      }
      st->iters += 1;
      if (rzn <= Real(st->stop)) {
        st->done = 1;
        break;
      }
      st->beta = double(rzn / Real(st->rz));
      st->rz = double(rzn);
      break;
    }
  }
}

// Block epilogue of a (possibly multi-kernel) deterministic reduction: each
// block writes its partial(s); the last block to arrive sums all partials in
// index order (fixed assignment to threads, fixed tree) and finalises.
// Must be called by every thread of the block.
template <class Real>
__device__ void mo_reduce_epilogue(const mo_red& P, double v, double v2, bool two) {
  __shared__ double sh[32];
  __shared__ bool am_last;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int nt = blockDim.x * blockDim.y;
  const int bid = blockIdx.x;
  double s = mo_block_sum(v, sh);
  double s2 = two ? mo_block_sum(v2, sh) : 0.0;
  if (P.fin_op == MO_FIN_PARTIALS) {  // the next kernel sums (mo_sum_partials)
    if (tid == 0) {
      P.partials[P.part_base + bid] = s;
      if (two) P.partials[P.part_total + P.part_base + bid] = s2;
    }
    return;
  }
  if (tid == 0) {
    P.partials[P.part_base + bid] = s;
    if (two) P.partials[P.part_total + P.part_base + bid] = s2;
    __threadfence();
    unsigned t = atomicAdd(P.counter, 1u);
    am_last = (t == unsigned(P.part_total - 1));
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  double a = 0, a2 = 0;
  // Fixed thread->partial assignment; loads batched 4 deep (L2, bypassing L1)
  // so the last block's sum costs ~one L2 round trip, not one per partial.
  int i = tid;
  for (; i + 3 * nt < P.part_total; i += 4 * nt) {
    const double x0 = __ldcg(P.partials + i), x1 = __ldcg(P.partials + i + nt);
    const double x2 = __ldcg(P.partials + i + 2 * nt), x3 = __ldcg(P.partials + i + 3 * nt);
    a += x0;
    a += x1;
    a += x2;
    a += x3;
    if (two) {
      const double y0 = __ldcg(P.partials + P.part_total + i), y1 = __ldcg(P.partials + P.part_total + i + nt);
      const double y2 = __ldcg(P.partials + P.part_total + i + 2 * nt);
      const double y3 = __ldcg(P.partials + P.part_total + i + 3 * nt);
      a2 += y0;
      a2 += y1;
      a2 += y2;
      a2 += y3;
    }
  }
  for (; i < P.part_total; i += nt) {
    a += __ldcg(P.partials + i);
    if (two) a2 += __ldcg(P.partials + P.part_total + i);
  }
  double tot = mo_block_sum(a, sh);
  double tot2 = two ? mo_block_sum(a2, sh) : 0.0;
  if (tid == 0) {
    *P.counter = 0u;
    mo_finalize<Real>(P.state, P.fin_op, P.fin_arg, tot, tot2);
  }
}

// Consumer side of a MO_FIN_PARTIALS reduction: every block sums the n block
// partials of the previous kernel in the same fixed order (the last-block
// scheme's order), so all blocks obtain the bitwise same total without the
// producer's atomic + last-block tail.  All threads call it; total in all.
__device__ __forceinline__ double mo_sum_partials(const double* p, int n) {
  __shared__ double sh[32];
  __shared__ double tot;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int nt = blockDim.x * blockDim.y;
  double a = 0;
  int i = tid;
  for (; i + 3 * nt < n; i += 4 * nt) {
    const double x0 = __ldcg(p + i), x1 = __ldcg(p + i + nt), x2 = __ldcg(p + i + 2 * nt), x3 = __ldcg(p + i + 3 * nt);
    a += x0;
    a += x1;
    a += x2;
    a += x3;
  }
  for (; i < n; i += nt) a += __ldcg(p + i);
  const double t = mo_block_sum(a, sh);
  if (tid == 0) tot = t;
  __syncthreads();
  return tot;
}
// alpha from p'Ap (pcg.hpp:100-110); block 0 (writer) records the state.
// Returns false when the PCG stops here (indefinite / non-finite).
template <class Real>
__device__ __forceinline__ bool mo_alpha_from(mo_state* st, double total, int k, bool writer, Real* alpha) {
  const Real pap = Real(total);
  if (!mo_finite(double(pap))) {
    if (writer) { st->pap = double(pap); st->nonfinite = 1; st->done = 1; st->stop_code = 2 * k; }
    return false;
  }
  if (pap <= Real(0)) {
    if (writer) { st->pap = double(pap); st->indefinite = 1; st->done = 1; st->stop_code = 2 * k; }
    return false;
  }
  *alpha = Real(st->rzs[k & 1]) / pap;
  if (writer) { st->pap = double(pap); st->alpha = double(*alpha); }
  return true;
}
// beta from r'z (pcg.hpp:116-124): rz of iteration k is rzs[k & 1], the new
// one goes to rzs[(k + 1) & 1].  Returns false when the PCG stops here.
template <class Real>
__device__ __forceinline__ bool mo_beta_from(mo_state* st, double total, int k, bool writer, Real* beta) {
  const Real rzn = Real(total);
  if (!mo_finite(double(rzn))) {
    if (writer) { st->rz_next = double(rzn); st->nonfinite = 1; st->done = 1; st->stop_code = 2 * k + 1; }
    return false;
  }
  const bool stop = rzn <= Real(st->stop);
  if (writer) {
    st->rz_next = double(rzn);
    st->iters += 1;
    if (stop) { st->done = 1; st->stop_code = 2 * k + 1; }
  }
  if (stop) return false;
  *beta = rzn / Real(st->rzs[k & 1]);
  if (writer) { st->beta = double(*beta); st->rz = double(rzn); st->rzs[(k + 1) & 1] = double(rzn); }
  return true;
}

// Grid-stride tile iteration for a grid domain (reference exec.hpp:151-214:
// one program run per element; here one thread per element of a 32x8 tile,
// fastest axis on threadIdx.x).  Returns the number of tiles.
__device__ __forceinline__ int mo_num_tiles(const mo_kparams& P) {
  const int rows = P.row1 - P.row0;
  if (rows <= 0) return 0;
  if (P.dnd == 1) return (rows + MO_THREADS - 1) / MO_THREADS;
  const int fx = P.dnd == 2 ? P.d1 : P.d2;
  const int ntx = (fx + MO_TILE_X - 1) / MO_TILE_X;
  const int nty = P.dnd == 2 ? (rows + MO_TILE_Y - 1) / MO_TILE_Y : rows * ((P.d1 + MO_TILE_Y - 1) / MO_TILE_Y);
  return ntx * nty;
}

// Coordinates (global) of this thread's element in tile t; false if outside.
__device__ __forceinline__ bool mo_tile_coord(const mo_kparams& P, int t, int& p0, int& p1, int& p2) {
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  if (P.dnd == 1) {
    p0 = P.row0 + t * MO_THREADS + tid;
    p1 = 0;
    p2 = 0;
    return p0 < P.row1;
  }
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (P.dnd == 2) {
    const int ntx = (P.d1 + MO_TILE_X - 1) / MO_TILE_X;
    const int bx = t % ntx, by = t / ntx;
    p0 = P.row0 + by * MO_TILE_Y + ty;
    p1 = bx * MO_TILE_X + tx;
    p2 = 0;
    return p0 < P.row1 && p1 < P.d1;
  }
  const int ntx = (P.d2 + MO_TILE_X - 1) / MO_TILE_X;
  const int nty = (P.d1 + MO_TILE_Y - 1) / MO_TILE_Y;
  const int bx = t % ntx;
  const int r = t / ntx;
  const int by = r % nty;
  p0 = P.row0 + r / nty;
  p1 = by * MO_TILE_Y + ty;
  p2 = bx * MO_TILE_X + tx;
  return p0 < P.row1 && p1 < P.d1 && p2 < P.d2;
}

// Local (storage) element index of a global coordinate on the iteration domain.
__device__ __forceinline__ int mo_local_elem(const mo_kparams& P, int p0, int p1, int p2) {
  if (P.dnd == 1) return p0 - P.row_lo;
  if (P.dnd == 2) return (p0 - P.row_lo) * P.d1 + p1;
  return ((p0 - P.row_lo) * P.d1 + p1) * P.d2 + p2;
}

// InBounds against the iteration domain (eval.hpp:57-61).
__device__ __forceinline__ bool mo_inb(const mo_kparams& P, int c0, int c1, int c2) {
  if ((unsigned)c0 >= (unsigned)P.d0) return false;
  if (P.dnd >= 2 && (unsigned)c1 >= (unsigned)P.d1) return false;
  if (P.dnd >= 3 && (unsigned)c2 >= (unsigned)P.d2) return false;
  return true;
}

// Tile origin (global coordinates), computed once per tile and pinned in
// registers: the integer divisions must not be rematerialised inside the
// per-element code (measured: >10% of a J^T J p kernel's instructions).
struct mo_tile {
  int o0, o1, o2;
};
__device__ __forceinline__ mo_tile mo_tile_at(const mo_kparams& P, int t) {
  mo_tile T;
  if (P.dnd == 1) {
    T.o0 = P.row0 + t * MO_THREADS;
    T.o1 = 0;
    T.o2 = 0;
  } else if (P.dnd == 2) {
    const int ntx = (P.d1 + MO_TILE_X - 1) / MO_TILE_X;
    const int by = t / ntx;
    T.o0 = P.row0 + by * MO_TILE_Y;
    T.o1 = (t - by * ntx) * MO_TILE_X;
    T.o2 = 0;
  } else {
    const int ntx = (P.d2 + MO_TILE_X - 1) / MO_TILE_X;
    const int nty = (P.d1 + MO_TILE_Y - 1) / MO_TILE_Y;
    const int r = t / ntx;
    const int rr = r / nty;
    T.o0 = P.row0 + rr;
    T.o1 = (r - rr * nty) * MO_TILE_Y;
    T.o2 = (t - r * ntx) * MO_TILE_X;
  }
  asm volatile("" : "+r"(T.o0), "+r"(T.o1), "+r"(T.o2));
  return T;
}
__device__ __forceinline__ bool mo_tile_in(const mo_kparams& P, const mo_tile& T, int R) {
  if (P.dnd == 1) return T.o0 - R >= 0 && T.o0 + MO_THREADS - 1 + R < P.d0;
  if (P.dnd == 2)
    return T.o0 - R >= 0 && T.o0 + MO_TILE_Y - 1 + R < P.d0 && T.o1 - R >= 0 && T.o1 + MO_TILE_X - 1 + R < P.d1;
  return T.o0 - R >= 0 && T.o0 + R < P.d0 && T.o1 - R >= 0 && T.o1 + MO_TILE_Y - 1 + R < P.d1 && T.o2 - R >= 0 &&
         T.o2 + MO_TILE_X - 1 + R < P.d2;
}
__device__ __forceinline__ bool mo_tile_elem(const mo_kparams& P, const mo_tile& T, int& p0, int& p1, int& p2) {
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  if (P.dnd == 1) {
    p0 = T.o0 + tid;
    p1 = 0;
    p2 = 0;
    return p0 < P.row1;
  }
  if (P.dnd == 2) {
    p0 = T.o0 + (int)threadIdx.y;
    p1 = T.o1 + (int)threadIdx.x;
    p2 = 0;
    return p0 < P.row1 && p1 < P.d1;
  }
  p0 = T.o0;
  p1 = T.o1 + (int)threadIdx.y;
  p2 = T.o2 + (int)threadIdx.x;
  return p0 < P.row1 && p1 < P.d1 && p2 < P.d2;
}

// Is tile t at least R elements away from every border of the iteration
// domain?  Then every InBounds(off) with |off| <= R is true and every read of
// a field living on the iteration domain is in shape (uniform per block).
__device__ __forceinline__ bool mo_tile_interior(const mo_kparams& P, int t, int R) {
  if (P.dnd == 1) {
    const int lo = P.row0 + t * MO_THREADS;
    return lo - R >= 0 && lo + MO_THREADS - 1 + R < P.d0;
  }
  if (P.dnd == 2) {
    const int ntx = (P.d1 + MO_TILE_X - 1) / MO_TILE_X;
    const int r0 = P.row0 + (t / ntx) * MO_TILE_Y, c0 = (t % ntx) * MO_TILE_X;
    return r0 - R >= 0 && r0 + MO_TILE_Y - 1 + R < P.d0 && c0 - R >= 0 && c0 + MO_TILE_X - 1 + R < P.d1;
  }
  const int ntx = (P.d2 + MO_TILE_X - 1) / MO_TILE_X;
  const int nty = (P.d1 + MO_TILE_Y - 1) / MO_TILE_Y;
  const int r = t / ntx;
  const int p0 = P.row0 + r / nty, y0 = (r % nty) * MO_TILE_Y, x0 = (t % ntx) * MO_TILE_X;
  return p0 - R >= 0 && p0 + R < P.d0 && y0 - R >= 0 && y0 + MO_TILE_Y - 1 + R < P.d1 && x0 - R >= 0 &&
         x0 + MO_TILE_X - 1 + R < P.d2;
}

// Grid read with the OOB->0 rule against the FIELD's own shape (eval.hpp:41-55).
// UNCHECKED: caller proved the coordinate in shape (interior tile).
template <class Real, int ND, int C, bool UNCHECKED = false>
__device__ __forceinline__ Real mo_ld(const mo_view& v, int c0, int c1, int c2, int ch) {
  if (!UNCHECKED) {
    if ((unsigned)c0 >= (unsigned)v.s0) return Real(0);
    if (ND >= 2 && (unsigned)c1 >= (unsigned)v.s1) return Real(0);
    if (ND >= 3 && (unsigned)c2 >= (unsigned)v.s2) return Real(0);
  }
  int e = c0 - v.row_lo;
  if (ND >= 2) e = e * v.s1 + c1;
  if (ND >= 3) e = e * v.s2 + c2;
  return __ldg(reinterpret_cast<const Real*>(v.p) + (long long)e * C + ch);
}

// Interior read by precomputed local element index (field on the iteration
// domain, coordinate proven in shape).
template <class Real, int C>
__device__ __forceinline__ Real mo_ldi(const mo_view& v, int e, int ch) {
  return __ldg(reinterpret_cast<const Real*>(v.p) + (long long)e * C + ch);
}

// Slot read (eval.hpp:43-45): vertex validated on the host before any launch.
template <class Real, int C>
__device__ __forceinline__ Real mo_ldv(const mo_view& v, int vert, int ch) {
  return __ldg(reinterpret_cast<const Real*>(v.p) + (long long)vert * C + ch);
}

#endif  // MO_DEVICE_CUH_
