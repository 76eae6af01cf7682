// mo_kernels.cuh — hand-written sm_100a kernels of the solver loop: Jacobi PCG
// vector updates with fused deterministic reductions (pcg.hpp:63-130), LM
// bookkeeping (solver.hpp:427-501), the build_normal identity patch
// (solver.hpp:241-250), exclusion column masks (solver.hpp:137-157) and the
// deterministic vertex-centric graph gather that replaces the reference's
// atomic scatter (exec.hpp:265-282).
//
// Vector kernels are grid-stride over columns with a FIXED grid, so the
// assignment of columns to threads (and therefore every reduction) is
// reproducible run to run.  Column i of every vector is excluded iff
// colmask[i] != 0 (the reference's per-column `excluded_`).
#pragma once

#include "mo_device.cuh"

namespace mo {

// colmask bit 0: excluded column (solver.hpp:149-157).  Bit 1: halo column of
// a strip shard — owned by a neighbour, never updated or reduced here.
__device__ __forceinline__ bool ex_at(const unsigned char* cm, long long i) { return cm && (cm[i] & 1); }
__device__ __forceinline__ bool halo_at(const unsigned char* cm, long long i) { return cm && (cm[i] & 2); }

// Strip shards: fixed rank-order sum of the gathered partials, then the same
// finalisation every rank (pcg.hpp scalar logic via mo_finalize).
template <class Real>
__global__ void k_global_fin(mo_state* st, const double* rb, int world, int op, int arg) {
  MO_PDL_ENTRY();
  if (threadIdx.x != 0) return;
  if ((op == MO_FIN_PCG_ALPHA || op == MO_FIN_PCG_BETA) && st->done) return;
  double t = 0, t2 = 0;
  for (int r = 0; r < world; ++r) {
    t += rb[2 * r];
    t2 += rb[2 * r + 1];
  }
  mo_finalize<Real>(st, op, arg, t, t2);
}
// Peer-memory all-gather + finalisation (mo_comm.hpp PeerTable): thread q
// stores this rank's pair into slot `rank` of rank q's block, fences, raises
// the slot's flag (release, system scope), then waits for rank q's flag in
// this rank's block (acquire) and copies its pair; thread 0 sums the pairs
// in rank order exactly as k_global_fin does.  Every rank runs every
// exchange (the `done` skip applies to the finalisation only), so the
// per-block epoch counters stay in step.  A bounded wait (60 s) raises
// peer_timeout instead of hanging the device.  kind 0: finalise (op, arg);
// kind 1: OR of the nonfinite / any-nonzero flags (reduce_flags).
struct mo_peer {
  char* block[64];
  int rank, world;
  unsigned long long timeout_ns;
};
__device__ __forceinline__ void mo_st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long mo_ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long mo_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
template <class Real>
__global__ void k_peer_fin(mo_state* st, mo_peer P, double* rb, int op, int arg, int kind) {
  MO_PDL_ENTRY();
  constexpr int KP = 64;  // = kPeerMax
  __shared__ unsigned long long e_s;
  const int t = threadIdx.x;
  char* const mine = P.block[P.rank];
  unsigned long long* const ep = reinterpret_cast<unsigned long long*>(mine + 3072);
  if (t == 0) {
    e_s = *ep + 1;
    *ep = e_s;
  }
  __syncthreads();
  const unsigned long long e = e_s;
  const int par = int(e & 1);
  const double s0 = kind ? double(st->nonfinite_kernel) : st->sums[4];
  const double s1 = kind ? double(st->any_nonzero) : st->sums[5];
  if (t < P.world) {
    char* const dst = P.block[t];
    double* const v = reinterpret_cast<double*>(dst) + (par * KP + P.rank) * 2;
    v[0] = s0;
    v[1] = s1;
    __threadfence_system();
    mo_st_release_sys(reinterpret_cast<unsigned long long*>(dst + 2048) + par * KP + P.rank, e);
    const unsigned long long* f = reinterpret_cast<const unsigned long long*>(mine + 2048) + par * KP + t;
    const unsigned long long t0 = mo_globaltimer();
    while (mo_ld_acquire_sys(f) < e) {
      if (mo_globaltimer() - t0 > P.timeout_ns) {
        st->peer_timeout = 1;
        break;
      }
      __nanosleep(100);
    }
    const volatile double* w = reinterpret_cast<const volatile double*>(mine) + (par * KP + t) * 2;
    rb[2 * t] = w[0];
    rb[2 * t + 1] = w[1];
  }
  __syncthreads();
  if (t != 0) return;
  if (kind) {
    int nf = 0, nz = 0;
    for (int r = 0; r < P.world; ++r) {
      nf |= rb[2 * r] != 0.0;
      nz |= rb[2 * r + 1] != 0.0;
    }
    st->nonfinite_kernel = nf;
    st->any_nonzero = nz;
    return;
  }
  if ((op == MO_FIN_PCG_ALPHA || op == MO_FIN_PCG_BETA) && st->done) return;
  double a = 0, a2 = 0;
  for (int r = 0; r < P.world; ++r) {
    a += rb[2 * r];
    a2 += rb[2 * r + 1];
  }
  mo_finalize<Real>(st, op, arg, a, a2);
}
__global__ void k_flags_out(mo_state* st) {
  MO_PDL_ENTRY();
  st->sums[4] = double(st->nonfinite_kernel);
  st->sums[5] = double(st->any_nonzero);
}
__global__ void k_flags_in(mo_state* st, const double* rb, int world) {
  MO_PDL_ENTRY();
  int nf = 0, nz = 0;
  for (int r = 0; r < world; ++r) {
    nf |= rb[2 * r] != 0.0;
    nz |= rb[2 * r + 1] != 0.0;
  }
  st->nonfinite_kernel = nf;
  st->any_nonzero = nz;
}
// *flag |= any byte of p[0, n) nonzero.
__global__ void k_any_byte(const unsigned char* p, long long n, int* flag) {
  MO_PDL_ENTRY();
  bool any = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    any |= p[i] != 0;
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(flag, 1);
}
__global__ void k_or_bits(unsigned char* p, long long n, unsigned char bits) {
  MO_PDL_ENTRY();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] |= bits;
}

// Jacobi z = r / m (pcg.hpp:79, 117, 124), bitwise.  r == +-0 with m > 0
// gives r itself (the IEEE quotient): a zero numerator otherwise sends every
// column through the division's slow path (FCHK), and the residual of a
// matrix-free solve is exactly zero on most of the domain while it spreads
// from the data terms (measured: the slow path was ~40% of k_pcg_update).
template <class Real>
__device__ __forceinline__ Real mo_precond_div(Real r, Real m) {
  return (r == Real(0) && m > Real(0)) ? r : r / m;
}

// delta = 0; r = b; z = r/m; p = z; rz = r'z   (pcg.hpp:75-97)
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_pcg_init(mo_red R, long long n, const unsigned char* cm, const Real* __restrict__ b,
           const Real* __restrict__ md, Real* __restrict__ delta, Real* __restrict__ r,
           Real* __restrict__ p, int precond) {
  MO_PDL_ENTRY();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    R.state->done = 0;
    R.state->stop_code = 0x7fffffff;
    R.state->iters = 0;
    R.state->indefinite = 0;
    R.state->nonfinite = 0;
  }
  double acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (halo_at(cm, i)) continue;
    const bool ex = ex_at(cm, i);
    const Real ri = ex ? Real(0) : b[i];
    const Real zi = ex ? Real(0) : (precond ? mo_precond_div(ri, md[i]) : ri);
    delta[i] = Real(0);
    r[i] = ri;
    p[i] = zi;
    acc += double(ri * zi);
  }
  mo_reduce_epilogue<Real>(R, acc, 0.0, false);
}

// 4-wide vector access (16-byte for float, 2 x 16-byte for double).  Column
// vectors come from cudaMalloc (256-byte aligned) and are indexed from 0.
template <class Real>
struct V4 {
  Real a[4];
};
__device__ __forceinline__ V4<float> ld4(const float* p) {
  const float4 t = *reinterpret_cast<const float4*>(p);
  return {{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ V4<double> ld4(const double* p) {
  const double2 t0 = reinterpret_cast<const double2*>(p)[0], t1 = reinterpret_cast<const double2*>(p)[1];
  return {{t0.x, t0.y, t1.x, t1.y}};
}
__device__ __forceinline__ void st4(float* p, const V4<float>& v) {
  *reinterpret_cast<float4*>(p) = make_float4(v.a[0], v.a[1], v.a[2], v.a[3]);
}
__device__ __forceinline__ void st4(double* p, const V4<double>& v) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v.a[0], v.a[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(v.a[2], v.a[3]);
}
__device__ __forceinline__ uchar4 ldm4(const unsigned char* cm, long long i) {
  return cm ? *reinterpret_cast<const uchar4*>(cm + i) : make_uchar4(0, 0, 0, 0);
}

// Four excluded (non-halo) columns: every PCG vector holds +0 there from the
// start (pcg_init / the fused build_normal start write them, pcg.hpp:75-80)
// and every update writes +0 again (zero_excluded, pcg.hpp:50-55), so the
// vector kernels skip such a group without loading or storing anything:
// bitwise the same vectors, and excluded regions (Poisson's frozen 3/4 of
// the image) cost no bandwidth.
__device__ __forceinline__ bool mo_all_excluded(uchar4 e) {
  return (e.x & e.y & e.z & e.w & 1) && !((e.x | e.y | e.z | e.w) & 2);
}

// Active-group list (unsharded grids with excluded columns, mo_session.cu
// build_group_list): gl[0] = count, gl[1..] = the 4-column groups holding a
// non-excluded column, ascending; bit 31 marks a group with an excluded
// column (its mask is loaded).  The vector kernels then walk only the active
// groups: no mask stream, no loop trips over excluded regions (Poisson: 3/4
// of the columns).  Calls body(i, mask) for column i = 4 * group; the next
// entry is loaded one trip ahead.
template <class F>
__device__ __forceinline__ void mo_for_groups(const int* __restrict__ gl, const unsigned char* cm, F&& body) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long cnt = __ldg(gl);
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int an = v < cnt ? __ldg(gl + 1 + v) : 0;
  for (; v < cnt; v += stride) {
    const int a = an;
    if (v + stride < cnt) an = __ldg(gl + 1 + v + stride);
    const long long i = (long long)(a & 0x7fffffff) << 2;
    body(i, a < 0 ? ldm4(cm, i) : make_uchar4(0, 0, 0, 0));
  }
}

// delta += alpha p; r -= alpha Ap; z = r/m; rz' = r'z   (pcg.hpp:111-118)
template <class Real>
__device__ __forceinline__ double pcg_update1(Real alpha, unsigned char m, Real& d, Real& r, Real p, Real ap, Real md,
                                              int precond) {
  if (m & 2) return 0.0;  // halo column: a neighbour's
  if (m & 1) {
    d = Real(0);
    r = Real(0);
    return 0.0;
  }
  d = d + alpha * p;
  r = r - alpha * ap;
  const Real z = precond ? mo_precond_div(r, md) : r;
  return double(r * z);
}

template <class Real, bool GL>
__global__ void __launch_bounds__(MO_THREADS)
k_pcg_update(mo_red R, long long n, const unsigned char* cm, const Real* __restrict__ md,
             Real* __restrict__ delta, Real* __restrict__ r, const Real* __restrict__ p,
             const Real* __restrict__ ap, int precond, const double* pap_part, int pap_n, int k,
             const int* gl) {
  MO_PDL_ENTRY();
  if (R.state->done) return;
  Real alpha;
  if (pap_part) {  // consumer-side p'Ap (the apply only stored block partials)
    const double tot = mo_sum_partials(pap_part, pap_n);
    const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
    if (!mo_alpha_from<Real>(R.state, tot, k, writer, &alpha)) return;
  } else {
    alpha = Real(R.state->alpha);
  }
  double acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long n4 = n >> 2;
  if constexpr (GL) {
    mo_for_groups(gl, cm, [&](long long i, uchar4 e) {
      V4<Real> D = ld4(delta + i), Rr = ld4(r + i);
      const V4<Real> Pp = ld4(p + i), A = ld4(ap + i), M = ld4(md + i);
      const unsigned char ex[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) acc += pcg_update1(alpha, ex[q], D.a[q], Rr.a[q], Pp.a[q], A.a[q], M.a[q], precond);
      st4(delta + i, D);
      st4(r + i, Rr);
    });
  }
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; !GL && v < n4; v += stride) {
    const long long i = v << 2;
    const uchar4 e = ldm4(cm, i);
    if (mo_all_excluded(e)) continue;
    V4<Real> D = ld4(delta + i), Rr = ld4(r + i);
    const V4<Real> Pp = ld4(p + i), A = ld4(ap + i), M = ld4(md + i);
    const unsigned char ex[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += pcg_update1(alpha, ex[k], D.a[k], Rr.a[k], Pp.a[k], A.a[k], M.a[k], precond);
    st4(delta + i, D);
    st4(r + i, Rr);
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    acc += pcg_update1(alpha, cm ? cm[i] : (unsigned char)0, delta[i], r[i], p[i], ap[i], md[i], precond);
  mo_reduce_epilogue<Real>(R, acc, 0.0, false);
}

// p = z + beta p with z = r/m recomputed   (pcg.hpp:124-126)
template <class Real>
__device__ __forceinline__ Real pcg_p1(Real beta, unsigned char m, Real r, Real md, Real p, int precond) {
  if (m & 2) return p;  // halo column: refreshed by the exchange
  if (m & 1) return Real(0);
  const Real z = precond ? mo_precond_div(r, md) : r;
  return z + beta * p;
}

template <class Real, bool GL>
__global__ void __launch_bounds__(MO_THREADS)
k_pcg_p(mo_state* st, long long n, const unsigned char* cm, const Real* __restrict__ md,
        const Real* __restrict__ r, Real* __restrict__ p, int precond, const double* rz_part, int rz_n, int k,
        const int* gl) {
  MO_PDL_ENTRY();
  if (st->done) return;
  Real beta;
  if (rz_part) {  // consumer-side r'z of the update kernel
    const double tot = mo_sum_partials(rz_part, rz_n);
    const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
    if (!mo_beta_from<Real>(st, tot, k, writer, &beta)) return;
  } else {
    beta = Real(st->beta);
  }
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long n4 = n >> 2;
  if constexpr (GL) {
    mo_for_groups(gl, cm, [&](long long i, uchar4 e) {
      const V4<Real> Rr = ld4(r + i), M = ld4(md + i);
      V4<Real> Pp = ld4(p + i);
      const unsigned char ex[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) Pp.a[q] = pcg_p1(beta, ex[q], Rr.a[q], M.a[q], Pp.a[q], precond);
      st4(p + i, Pp);
    });
  }
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; !GL && v < n4; v += stride) {
    const long long i = v << 2;
    const uchar4 e = ldm4(cm, i);
    if (mo_all_excluded(e)) continue;
    const V4<Real> Rr = ld4(r + i), M = ld4(md + i);
    V4<Real> Pp = ld4(p + i);
    const unsigned char ex[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) Pp.a[k] = pcg_p1(beta, ex[k], Rr.a[k], M.a[k], Pp.a[k], precond);
    st4(p + i, Pp);
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    p[i] = pcg_p1(beta, cm ? cm[i] : (unsigned char)0, r[i], md[i], p[i], precond);
}

// Deferred-delta PCG (consumer-side reductions, unsharded grids).  The
// update of iteration k only moves r (r -= alpha_k Ap; z = r/m; r'z
// partials); the direction kernel of the same iteration first folds
// delta += alpha_k p_k with the p it is about to replace, then p = z + beta p.
// delta receives the same alpha_k p_k terms in the same order as
// pcg.hpp:111-112, so every value is bitwise the eager scheme's, and a
// column moves 42 instead of 46 bytes per iteration (the update no longer
// reads p or reads and writes delta).  After the last iteration (or an r'z
// stop) the same kernel runs with last = 1: delta only.  Iteration k's
// kernels proceed while stop_code > 2k (update) / >= 2k + 1 (direction).
template <class Real>
__device__ __forceinline__ double pcg_update_r1(Real alpha, unsigned char m, Real& r, Real ap, Real md, int precond) {
  if (m & 3) {  // excluded (halo columns do not occur on unsharded grids)
    r = Real(0);
    return 0.0;
  }
  r = r - alpha * ap;
  const Real z = precond ? mo_precond_div(r, md) : r;
  return double(r * z);
}

template <class Real, bool GL>
__global__ void __launch_bounds__(MO_THREADS)
k_pcg_update_r(mo_red R, long long n, const unsigned char* cm, const Real* __restrict__ md, Real* __restrict__ r,
               const Real* __restrict__ ap, int precond, const double* pap_part, int pap_n, int k, const int* gl) {
  MO_PDL_ENTRY();
  if (R.state->done) return;
  Real alpha;
  const double tot = mo_sum_partials(pap_part, pap_n);
  const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
  if (!mo_alpha_from<Real>(R.state, tot, k, writer, &alpha)) return;
  double acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long n4 = n >> 2;
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if constexpr (GL) {
    mo_for_groups(gl, cm, [&](long long i, uchar4 e) {
      V4<Real> Rr = ld4(r + i);
      const V4<Real> A = ld4(ap + i), M = ld4(md + i);
      const unsigned char ex[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) acc += pcg_update_r1(alpha, ex[q], Rr.a[q], A.a[q], M.a[q], precond);
      st4(r + i, Rr);
    });
    v = n4;  // (the tail below still runs)
  }
  // two 4-wide groups per step, every load issued before the first use (few
  // streams per column: the loads in flight per thread set the bandwidth)
  // (the masks of a pair are loaded one pair ahead, so the skip test never
  // holds back the vector loads it guards)
  uchar4 n0 = make_uchar4(0, 0, 0, 0), n1 = n0;
  if (v + stride < n4) {
    n0 = ldm4(cm, v << 2);
    n1 = ldm4(cm, (v + stride) << 2);
  }
  for (; v + stride < n4; v += 2 * stride) {
    const long long i = v << 2, j = (v + stride) << 2;
    const uchar4 e0 = n0, e1 = n1;
    if (v + 3 * stride < n4) {
      n0 = ldm4(cm, (v + 2 * stride) << 2);
      n1 = ldm4(cm, (v + 3 * stride) << 2);
    }
    if (mo_all_excluded(e0) && mo_all_excluded(e1)) continue;
    V4<Real> R0 = ld4(r + i), R1 = ld4(r + j);
    const V4<Real> A0 = ld4(ap + i), A1 = ld4(ap + j), M0 = ld4(md + i), M1 = ld4(md + j);
    const unsigned char x0[4] = {e0.x, e0.y, e0.z, e0.w}, x1[4] = {e1.x, e1.y, e1.z, e1.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += pcg_update_r1(alpha, x0[q], R0.a[q], A0.a[q], M0.a[q], precond);
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += pcg_update_r1(alpha, x1[q], R1.a[q], A1.a[q], M1.a[q], precond);
    st4(r + i, R0);
    st4(r + j, R1);
  }
  for (; v < n4; v += stride) {
    const long long i = v << 2;
    const uchar4 e = ldm4(cm, i);
    if (mo_all_excluded(e)) continue;
    V4<Real> Rr = ld4(r + i);
    const V4<Real> A = ld4(ap + i), M = ld4(md + i);
    const unsigned char ex[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += pcg_update_r1(alpha, ex[q], Rr.a[q], A.a[q], M.a[q], precond);
    st4(r + i, Rr);
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    acc += pcg_update_r1(alpha, cm ? cm[i] : (unsigned char)0, r[i], ap[i], md[i], precond);
  mo_reduce_epilogue<Real>(R, acc, 0.0, false);
}

template <class Real, bool GL>
__global__ void __launch_bounds__(MO_THREADS)
k_pcg_dp(mo_state* st, long long n, const unsigned char* cm, const Real* __restrict__ md, const Real* __restrict__ r,
         Real* __restrict__ delta, Real* __restrict__ p, int precond, const double* rz_part, int rz_n, int k, int last,
         const int* gl) {
  MO_PDL_ENTRY();
  if (st->stop_code < 2 * k + 1) return;  // stopped before alpha_k existed
  const double tot = mo_sum_partials(rz_part, rz_n);
  const bool writer = blockIdx.x == 0 && threadIdx.x == 0;
  Real beta = Real(0);
  const bool go = mo_beta_from<Real>(st, tot, k, writer, &beta) && !last;  // (writer: bookkeeping of r'z)
  const Real alpha = Real(st->alpha);  // alpha_k, recorded by the update of iteration k
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long n4 = n >> 2;
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if constexpr (GL) {
    mo_for_groups(gl, cm, [&](long long i, uchar4 e) {
      V4<Real> D = ld4(delta + i), Pp = ld4(p + i);
      const unsigned char ex[4] = {e.x, e.y, e.z, e.w};
      if (go) {
        const V4<Real> Rr = ld4(r + i), M = ld4(md + i);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          D.a[q] = (ex[q] & 1) ? Real(0) : D.a[q] + alpha * Pp.a[q];
          Pp.a[q] = pcg_p1(beta, ex[q], Rr.a[q], M.a[q], Pp.a[q], precond);
        }
        st4(p + i, Pp);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) D.a[q] = (ex[q] & 1) ? Real(0) : D.a[q] + alpha * Pp.a[q];
      }
      st4(delta + i, D);
    });
    v = n4;  // (the tail below still runs)
  }
  if (go && !GL) {  // two 4-wide groups per step, loads first (see k_pcg_update_r)
    uchar4 n0 = make_uchar4(0, 0, 0, 0), n1 = n0;  // (masks one pair ahead)
    if (v + stride < n4) {
      n0 = ldm4(cm, v << 2);
      n1 = ldm4(cm, (v + stride) << 2);
    }
    for (; v + stride < n4; v += 2 * stride) {
      const long long i = v << 2, j = (v + stride) << 2;
      const uchar4 e0 = n0, e1 = n1;
      if (v + 3 * stride < n4) {
        n0 = ldm4(cm, (v + 2 * stride) << 2);
        n1 = ldm4(cm, (v + 3 * stride) << 2);
      }
      if (mo_all_excluded(e0) && mo_all_excluded(e1)) continue;
      V4<Real> D0 = ld4(delta + i), D1 = ld4(delta + j), P0 = ld4(p + i), P1 = ld4(p + j);
      const V4<Real> R0 = ld4(r + i), R1 = ld4(r + j), M0 = ld4(md + i), M1 = ld4(md + j);
      const unsigned char x0[4] = {e0.x, e0.y, e0.z, e0.w}, x1[4] = {e1.x, e1.y, e1.z, e1.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        D0.a[q] = (x0[q] & 1) ? Real(0) : D0.a[q] + alpha * P0.a[q];
        P0.a[q] = pcg_p1(beta, x0[q], R0.a[q], M0.a[q], P0.a[q], precond);
        D1.a[q] = (x1[q] & 1) ? Real(0) : D1.a[q] + alpha * P1.a[q];
        P1.a[q] = pcg_p1(beta, x1[q], R1.a[q], M1.a[q], P1.a[q], precond);
      }
      st4(delta + i, D0);
      st4(delta + j, D1);
      st4(p + i, P0);
      st4(p + j, P1);
    }
  }
  for (; v < n4; v += stride) {
    const long long i = v << 2;
    const uchar4 e = ldm4(cm, i);
    if (mo_all_excluded(e)) continue;
    V4<Real> D = ld4(delta + i), Pp = ld4(p + i);
    const unsigned char ex[4] = {e.x, e.y, e.z, e.w};
    if (go) {
      const V4<Real> Rr = ld4(r + i), M = ld4(md + i);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        D.a[q] = (ex[q] & 1) ? Real(0) : D.a[q] + alpha * Pp.a[q];
        Pp.a[q] = pcg_p1(beta, ex[q], Rr.a[q], M.a[q], Pp.a[q], precond);
      }
      st4(p + i, Pp);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) D.a[q] = (ex[q] & 1) ? Real(0) : D.a[q] + alpha * Pp.a[q];
    }
    st4(delta + i, D);
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned char m = cm ? cm[i] : (unsigned char)0;
    const Real pi = p[i];
    delta[i] = (m & 1) ? Real(0) : delta[i] + alpha * pi;
    if (go) p[i] = pcg_p1(beta, m, r[i], md[i], pi, precond);
  }
}

// Last PCG iteration under consumer-side reductions: no direction update,
// only the r'z bookkeeping (iteration count, stop / non-finite flags).
template <class Real>
__global__ void k_pcg_fin(mo_state* st, const double* rz_part, int rz_n, int k) {
  MO_PDL_ENTRY();
  if (st->done) return;
  const double tot = mo_sum_partials(rz_part, rz_n);
  Real beta;
  if (threadIdx.x == 0) mo_beta_from<Real>(st, tot, k, true, &beta);
}

// Unfused apply epilogue (plans with graph scatters): LM damping, excluded
// zeroing, p'Ap -> alpha.
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_apply_finish(mo_red R, long long n, const unsigned char* cm, const Real* __restrict__ p,
               const Real* __restrict__ damp, Real* __restrict__ ap, int flags) {
  MO_PDL_ENTRY();
  if ((flags & MO_F_REDUCE) && R.state->done) return;
  double acc = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (halo_at(cm, i)) continue;  // a strip's halo column: owned (and reduced) by a neighbour
    Real v = ap[i];
    if (flags & MO_F_DAMP) v = v + damp[i] * p[i];
    if ((flags & MO_F_ZEROEXCL) && ex_at(cm, i)) v = Real(0);
    ap[i] = v;
    acc += double(p[i] * v);
  }
  if (flags & MO_F_REDUCE) mo_reduce_epilogue<Real>(R, acc, 0.0, false);
}

// Identity rows for excluded columns, m==0 -> 1 (solver.hpp:241-250).
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_bm_patch(mo_red R, long long n, const unsigned char* cm, Real* __restrict__ b, Real* __restrict__ m) {
  MO_PDL_ENTRY();
  double cnt = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (halo_at(cm, i)) continue;
    if (ex_at(cm, i)) {
      b[i] = Real(0);
      m[i] = Real(1);
    } else if (m[i] == Real(0)) {
      cnt += 1.0;
      m[i] = Real(1);
    }
  }
  mo_reduce_epilogue<Real>(R, cnt, 0.0, false);
}

// Active tiles of a masked grid domain: flag[t] = some element of tile t is
// not excluded (the PCG apply of the gather program then walks only those
// tiles, mo_session.cu build_tile_lists).
__global__ void __launch_bounds__(MO_THREADS) k_tile_active(const __grid_constant__ mo_kparams P, unsigned char* flag,
                                                           int nt) {
  MO_PDL_ENTRY();
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const mo_tile T = mo_tile_at(P, t);
    int p0, p1, p2;
    const bool in = mo_tile_elem(P, T, p0, p1, p2);
    const bool act = in && !P.mask[mo_local_elem(P, p0, p1, p2)];
    const int any = __syncthreads_or(act);
    if (threadIdx.x == 0 && threadIdx.y == 0) flag[t] = any ? 1 : 0;
  }
}

// Active-group list source (mo_for_groups): per 4-column group, flag = not
// all excluded, val = group | bit 31 if some column is excluded.
__global__ void __launch_bounds__(MO_THREADS) k_group_flags(const unsigned char* __restrict__ cm, long long n4,
                                                           int* __restrict__ val, unsigned char* __restrict__ flag) {
  MO_PDL_ENTRY();
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n4; g += (long long)gridDim.x * blockDim.x) {
    const uchar4 e = ldm4(cm, g << 2);
    flag[g] = mo_all_excluded(e) ? 0 : 1;
    val[g] = int(g) | ((e.x | e.y | e.z | e.w) ? int(0x80000000u) : 0);
  }
}

// Per-column exclusion from a per-element mask (solver.hpp:149-157).
__global__ void __launch_bounds__(MO_THREADS)
k_colmask(long long nelem, int C, const unsigned char* __restrict__ mask, unsigned char* __restrict__ cm) {
  MO_PDL_ENTRY();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nelem;
       e += (long long)gridDim.x * blockDim.x) {
    const unsigned char v = mask[e];
    for (int c = 0; c < C; ++c) cm[e * C + c] = v;
  }
}

// LM: base_diag = clamp(m/2, dmin, dmax) in double (solver.hpp:427-429).
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_lm_base_diag(long long n, const Real* __restrict__ m, double* __restrict__ bd, double dmin, double dmax) {
  MO_PDL_ENTRY();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double v = double(m[i]) / 2.0;
    bd[i] = v < dmin ? dmin : (dmax < v ? dmax : v);
  }
}

// LM: damp = excluded ? 0 : 2/mu * base_diag; md = m + damp (solver.hpp:433-438).
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_lm_damp(const mo_state* st, long long n, const unsigned char* cm, const Real* __restrict__ m,
          const double* __restrict__ bd, Real* __restrict__ damp, Real* __restrict__ md) {
  MO_PDL_ENTRY();
  const double s = 2.0 / st->mu;  // mu staged by the host before each trial
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (halo_at(cm, i)) continue;
    const Real d = ex_at(cm, i) ? Real(0) : Real(s * bd[i]);
    damp[i] = d;
    md[i] = m[i] + d;
  }
}

// x_trial = excluded ? x : x + delta; flags any delta != 0 (solver.hpp:448-449, 486-492).
// in_place (GN, commit unconditional unless cost_old / PCG were non-finite).
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_xtrial(mo_state* st, long long n, const unsigned char* cm, Real* __restrict__ x,
         const Real* __restrict__ delta, Real* __restrict__ xt, int in_place, int cost_slot) {
  MO_PDL_ENTRY();
  if (in_place && (st->nonfinite || !mo_finite(st->sums[cost_slot]))) return;
  bool nz = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long n4 = n >> 2;  // 4-wide body (16-byte accesses), scalar tail
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n4; v += stride) {
    const long long i = v << 2;
    const uchar4 e = ldm4(cm, i);
    if (in_place && mo_all_excluded(e)) continue;  // x stays, delta is 0 there
    const V4<Real> D = ld4(delta + i);
    V4<Real> X = ld4(x + i);
    const unsigned char ex[4] = {e.x, e.y, e.z, e.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (ex[q] & 2) continue;  // halo column: refreshed by the exchange
      if (D.a[q] != Real(0)) nz = true;
      if (!(ex[q] & 1)) X.a[q] = X.a[q] + D.a[q];
    }
    if (in_place) {
      if (cm && (e.x | e.y | e.z | e.w) & 2) {  // (strips) never write a neighbour's halo column
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (!(ex[q] & 2)) x[i + q] = X.a[q];
      } else {
        st4(x + i, X);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (!(ex[q] & 2)) xt[i + q] = X.a[q];
    }
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    if (halo_at(cm, i)) continue;  // refreshed by the halo exchange
    const Real d = delta[i];
    if (d != Real(0)) nz = true;
    const Real xi = x[i];
    const Real v = ex_at(cm, i) ? xi : xi + d;
    if (in_place) x[i] = v;
    else xt[i] = v;
  }
  if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(&st->any_nonzero, 1);
}

// LM predicted decrease pieces in double (solver.hpp:468-473):
// sums[arg] = sum b*delta, sums[arg+1] = sum (0.5*delta)*JtJdelta.
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_lm_predicted(mo_red R, long long n, const unsigned char* cm, const Real* __restrict__ b, const Real* __restrict__ delta,
               const Real* __restrict__ ap) {
  MO_PDL_ENTRY();
  double s1 = 0, s2 = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (halo_at(cm, i)) continue;
    s1 += double(b[i]) * double(delta[i]);
    s2 += 0.5 * double(delta[i]) * double(ap[i]);
  }
  mo_reduce_epilogue<Real>(R, s1, s2, true);
}

// Deterministic graph scatter (replaces exec.hpp:265-282's sequential `+=` /
// parallel atomics).  One thread per target vertex v of one domain; incident
// edges are visited in ascending edge order and, within an edge, outputs in
// program order — exactly the per-column accumulation order of the
// reference's sequential executor, without any floating-point atomics.
struct mo_gather_out {
  int slot;     // edge slot the output scatters through
  int sel;      // 0 -> dst0, 1 -> dst1 (bm: b/m)
  int C;        // channels of the target field
  int active;   // target field lives on this launch's domain
  long long cbase;  // ubase[field] + channel
};

template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_graph_gather(long long nverts, const int* __restrict__ vptr, const int* __restrict__ vedge,
               const int* __restrict__ verts, int arity, const Real* __restrict__ contrib, int NO,
               const mo_gather_out* __restrict__ outs, Real* dst0, Real* dst1) {
  MO_PDL_ENTRY();
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nverts;
       v += (long long)gridDim.x * blockDim.x) {
    const int j0 = vptr[v], j1 = vptr[v + 1];
    for (int j = j0; j < j1; ++j) {
      const long long e = vedge[j];
      for (int k = 0; k < NO; ++k) {
        const mo_gather_out o = outs[k];
        if (!o.active || verts[e * arity + o.slot] != int(v)) continue;
        Real* d = o.sel ? dst1 : dst0;
        const long long col = o.cbase + v * o.C;
        d[col] = d[col] + contrib[e * NO + k];
      }
    }
  }
}

// ------------------------------------------------------------ materialized J
// Materialize::kJ (solver.hpp:278-283, 291-376; sparse.hpp spmv / spmv_t).
// J is kept as the reference keeps it before CSR assembly: one value lane
// buffer per template set, [lane][row element] (jlanes_grid_ / jlanes_graph_),
// plus these tables describing where each lane's column lies.  The apply is
//   jtmp = J v          (k_mat_rows: one thread per row, entries in the CSR's
//                        column order, acc = 0 then acc + val * v[col])
//   out  = 2 J^T jtmp   (k_mat_cols: one thread per column, its entries in the
//                        CSR's row order, i.e. spmv_t's scatter order)
// with round-to-nearest intrinsics (no FMA contraction), so both products
// round exactly like the reference's CPU loops.  A grid lane's column is
// ubase + (e + lin) * C + ch with lin the lane offset linearised over the
// domain shape, exactly linear_index(coord + off) (problem.hpp:131-136).
#define MO_MAT_MAXL 32
struct mo_mat_tmpl {
  long long rowbase, nrows;  // rows [rowbase, rowbase + nrows); lane stride nrows
  const void* buf;           // lane values, [out][nrows]
  int kind;                  // 0 grid, 1 graph
  int guard;                 // grid: boundary-guard lane (0 -> the row is empty)
  int lane0, nlanes;         // into the lane table
  const int* verts;          // graph: int32 edge-major vertex table
  int arity;
  const int* vptr;           // graph: vertex -> incident edges (unique, ascending)
  const int* vedge;
  long long nverts;
  long long eoff, ecoff;     // kJtJ graph: offsets of this template's merged edge rows / counts (k_mat_erows)
};
struct mo_mat_lane {
  int out, field, ch, slot;
  long long lin;  // grid: linearised stencil offset
};
struct mo_mat_centry {  // one source of entries of a (field, channel) column
  int t, lane;          // grid: the lane; graph: ~(bitmask of the template's lanes on this column)
};
struct mo_mat_tables {
  const mo_mat_tmpl* tm;
  int ntm;
  const mo_mat_lane* lanes;
  const mo_mat_centry* ce;
  const int* ceptr;  // per (field, channel) index cbase[f] + ch: [ceptr[k], ceptr[k+1])
  long long ubase[MO_MAX_UNK];
  int chans[MO_MAX_UNK];
  int cbase[MO_MAX_UNK];
  int nfields;
  long long nrows, ncols;
  int ntl, nce, nk;  // table sizes: lanes, column entries, (field, channel) pairs
};

// Stage the (few-KB) tables in shared memory: every row / column walks them,
// and from global memory those walks were the kernels' dominant issue cost.
__device__ __forceinline__ mo_mat_tables mo_mat_stage(const mo_mat_tables& G) {
  extern __shared__ __align__(16) unsigned char mo_mat_sm[];
  mo_mat_tables T = G;
  size_t off = 0;
  auto copy = [&](const void* src, size_t bytes) -> const void* {
    unsigned char* dst = mo_mat_sm + off;
    const int tid = threadIdx.x + threadIdx.y * blockDim.x, nt = blockDim.x * blockDim.y;
    for (size_t i = size_t(tid) * 4; i < bytes; i += size_t(nt) * 4)
      *reinterpret_cast<unsigned*>(dst + i) = *reinterpret_cast<const unsigned*>(static_cast<const unsigned char*>(src) + i);
    off += (bytes + 15) & ~size_t(15);
    return dst;
  };
  T.tm = static_cast<const mo_mat_tmpl*>(copy(G.tm, sizeof(mo_mat_tmpl) * size_t(G.ntm)));
  T.lanes = static_cast<const mo_mat_lane*>(copy(G.lanes, sizeof(mo_mat_lane) * size_t(G.ntl)));
  T.ce = static_cast<const mo_mat_centry*>(copy(G.ce, sizeof(mo_mat_centry) * size_t(G.nce)));
  T.ceptr = static_cast<const int*>(copy(G.ceptr, sizeof(int) * size_t(G.nk + 1)));
  __syncthreads();
  return T;
}

__device__ __forceinline__ float mo_mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mo_mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mo_add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double mo_add_rn(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ int mo_mat_find(const mo_mat_tables& T, long long r) {
  int t = 0;
  while (t + 1 < T.ntm && T.tm[t + 1].rowbase <= r) ++t;
  return t;
}

// The reference's CSR assembly checks (sparse.hpp:30-37) on every non-empty
// grid row: column inside the field (bit 0: kIndexOutOfRange; the reference
// throws for columns outside [0, cols) and would silently read a neighbouring
// field's column otherwise - the device refuses both) and strictly ascending
// (bit 1: kInternal).
template <class Real>
__global__ void __launch_bounds__(MO_THREADS) k_mat_check(const __grid_constant__ mo_mat_tables G, mo_state* st) {
  MO_PDL_ENTRY();
  // gridDim.y = template (as k_mat_rows); graph rows need no check
  const mo_mat_tmpl M = G.tm[blockIdx.y];
  if (M.kind != 0) return;
  __shared__ mo_mat_lane sl[MO_MAT_MAXL];
  const int nl = M.nlanes < MO_MAT_MAXL ? M.nlanes : MO_MAT_MAXL;
  if (threadIdx.x < nl) sl[threadIdx.x] = G.lanes[M.lane0 + threadIdx.x];
  __syncthreads();
  int bad = 0;
  const Real* buf = static_cast<const Real*>(M.buf);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < M.nrows;
       e += (long long)gridDim.x * blockDim.x) {
    if (buf[(long long)M.guard * M.nrows + e] == Real(0)) continue;
    long long prev = -1;
    for (int k = 0; k < nl; ++k) {
      const long long el = e + sl[k].lin;
      if (el < 0 || el >= M.nrows) {
        bad |= 1;
        continue;
      }
      const long long col = G.ubase[sl[k].field] + el * G.chans[sl[k].field] + sl[k].ch;
      if (col <= prev) bad |= 2;
      prev = col;
    }
  }
  if (bad) atomicOr(&st->mat_bad, bad);
}

// gridDim.y = template: the block's template (and its lanes) are uniform,
// read once; threads stride over the template's rows.
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_mat_rows(const __grid_constant__ mo_mat_tables G, const mo_state* st, int skipdone, const Real* __restrict__ v,
           Real* __restrict__ jtmp) {
  MO_PDL_ENTRY();
  if (skipdone && st->done) return;
  const mo_mat_tmpl M = G.tm[blockIdx.y];
  const Real* __restrict__ buf = static_cast<const Real*>(M.buf);
  __shared__ mo_mat_lane sl[MO_MAT_MAXL];
  __shared__ long long sb[MO_MAT_MAXL];  // grid: column base of the lane, ubase + lin * C + ch
  __shared__ int sc[MO_MAT_MAXL];        // channels of the lane's field
  const int nl = M.nlanes < MO_MAT_MAXL ? M.nlanes : MO_MAT_MAXL;
  if (threadIdx.x < nl) {
    const mo_mat_lane L = G.lanes[M.lane0 + threadIdx.x];
    sl[threadIdx.x] = L;
    sc[threadIdx.x] = G.chans[L.field];
    sb[threadIdx.x] = G.ubase[L.field] + L.lin * G.chans[L.field] + L.ch;
  }
  __syncthreads();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < M.nrows;
       e += (long long)gridDim.x * blockDim.x) {
    Real acc = Real(0);
    if (M.kind == 0) {
      // All loads of the row issue together (none depends on the guard).
      const Real g = buf[(long long)M.guard * M.nrows + e];
      for (int k0 = 0; k0 < nl; k0 += 4) {
        Real a[4], b[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u;
          const long long el = e + (k < nl ? sl[k].lin : 0);
          ok[u] = k < nl && el >= 0 && el < M.nrows;  // (out-of-field lanes are refused by k_mat_check)
          a[u] = ok[u] ? buf[(long long)sl[k].out * M.nrows + e] : Real(0);
          b[u] = ok[u] ? v[sb[k] + e * sc[k]] : Real(0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (ok[u]) acc = mo_add_rn(acc, mo_mul_rn(a[u], b[u]));
      }
      if (g == Real(0)) acc = Real(0);  // boundary guard false: the row is empty
    } else {
      // Edge row: entries sorted by column (stable: repeated vertices keep
      // lane order) and merged (solver.hpp:350-366).
      long long cols[MO_MAT_MAXL];
      Real vals[MO_MAT_MAXL];
      int n = 0;
      for (int k = 0; k < nl; ++k) {
        const mo_mat_lane L = sl[k];
        const long long col = G.ubase[L.field] + (long long)M.verts[e * M.arity + L.slot] * sc[k] + L.ch;
        const Real val = buf[(long long)L.out * M.nrows + e];
        int j = n++;
        while (j > 0 && cols[j - 1] > col) {
          cols[j] = cols[j - 1];
          vals[j] = vals[j - 1];
          --j;
        }
        cols[j] = col;
        vals[j] = val;
      }
      for (int k = 0; k < n;) {
        const long long col = cols[k];
        Real mv = vals[k];
        for (++k; k < n && cols[k] == col; ++k) mv = mo_add_rn(mv, vals[k]);
        acc = mo_add_rn(acc, mo_mul_rn(mv, v[col]));
      }
    }
    jtmp[M.rowbase + e] = acc;
  }
}

// gridDim.y = (field, channel) pair: the block's column-entry list is uniform
// and staged in shared memory; threads stride over the field's elements.
#define MO_MAT_MAXCE 128
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_mat_cols(const __grid_constant__ mo_mat_tables G, const mo_state* st, int skipdone, const Real* __restrict__ jtmp,
           Real* __restrict__ out) {
  MO_PDL_ENTRY();
  if (skipdone && st->done) return;
  const int k = blockIdx.y;
  int f = 0;
  while (f + 1 < G.nfields && G.cbase[f + 1] <= k) ++f;
  const int ch = k - G.cbase[f], C = G.chans[f];
  const long long nel = (f + 1 < G.nfields ? G.ubase[f + 1] : G.ncols) - G.ubase[f];
  const long long ne = nel / C;
  const int c0 = G.ceptr[k], nce = min(G.ceptr[k + 1] - c0, MO_MAT_MAXCE);
  // per entry: template rows, lane value row, guard row, rowbase, lin (or graph template index)
  __shared__ const Real* s_val[MO_MAT_MAXCE];
  __shared__ const Real* s_grd[MO_MAT_MAXCE];
  __shared__ long long s_rb[MO_MAT_MAXCE], s_lin[MO_MAT_MAXCE], s_n[MO_MAT_MAXCE];
  __shared__ int s_t[MO_MAT_MAXCE];
  __shared__ unsigned s_mask[MO_MAT_MAXCE];
  for (int c = threadIdx.x; c < nce; c += blockDim.x) {
    const mo_mat_centry E = G.ce[c0 + c];
    const mo_mat_tmpl& M = G.tm[E.t];
    const Real* buf = static_cast<const Real*>(M.buf);
    s_t[c] = E.lane >= 0 ? -1 : E.t;
    s_mask[c] = E.lane >= 0 ? 0u : ~unsigned(E.lane);
    s_rb[c] = M.rowbase;
    s_n[c] = M.nrows;
    if (E.lane >= 0) {
      const mo_mat_lane L = G.lanes[E.lane];
      s_val[c] = buf + (long long)L.out * M.nrows;
      s_grd[c] = buf + (long long)M.guard * M.nrows;
      s_lin[c] = L.lin;
    }
  }
  __syncthreads();
  for (long long el = blockIdx.x * (long long)blockDim.x + threadIdx.x; el < ne;
       el += (long long)gridDim.x * blockDim.x) {
    Real y = Real(0);
    for (int c = 0; c < nce; ++c) {
      if (s_t[c] < 0) {  // grid: the one row of this template holding the column through the lane
        // batch the consecutive grid entries' loads (independent of the guards)
        Real g[4], a[4], b[4];
        bool ok[4];
        int m = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int cc = c + u;
          const bool grid = cc < nce && s_t[cc] < 0 && (u == 0 || m == u);
          const long long e = el - (grid ? s_lin[cc] : 0);
          ok[u] = grid && e >= 0 && e < s_n[cc];
          if (grid) m = u + 1;
          g[u] = ok[u] ? s_grd[cc][e] : Real(0);
          a[u] = ok[u] ? s_val[cc][e] : Real(0);
          b[u] = ok[u] ? jtmp[s_rb[cc] + e] : Real(0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (ok[u] && g[u] != Real(0)) y = mo_add_rn(y, mo_mul_rn(a[u], b[u]));
        c += m - 1;
      } else {  // graph: incident edges in row order, the merged entry of the column
        const mo_mat_tmpl& M = G.tm[s_t[c]];
        const Real* buf = static_cast<const Real*>(M.buf);
        if (el >= M.nverts) continue;
        for (int j = M.vptr[el]; j < M.vptr[el + 1]; ++j) {
          const int e = M.vedge[j];
          bool has = false;
          Real mv = Real(0);
          for (unsigned mk = s_mask[c]; mk; mk &= mk - 1) {  // this column's lanes, in lane order
            const mo_mat_lane L = G.lanes[M.lane0 + __ffs(mk) - 1];
            if (M.verts[(long long)e * M.arity + L.slot] != el) continue;
            const Real val = buf[(long long)L.out * M.nrows + e];
            mv = has ? mo_add_rn(mv, val) : val;
            has = true;
          }
          if (has) y = mo_add_rn(y, mo_mul_rn(mv, jtmp[M.rowbase + e]));
        }
      }
    }
    out[G.ubase[f] + el * C + ch] = mo_mul_rn(y, Real(2));
  }
}

// Materialize::kJtJ (solver.hpp:370-374; sparse.hpp transpose + spgemm +
// scale_inplace): row q of H = 2 J^T J, one thread per column q.  Rows r of
// J holding q are visited in ascending order (transpose's row order), each
// row's entries in column order, H[q][j] accumulating a * b from 0 exactly
// as Gustavson's dense accumulator does; the row is then emitted in column
// order (slot-major ELL: slot k of column q at k * ncols + q) and doubled.
template <class Real>
__device__ __forceinline__ void mo_h_acc(long long* cols, Real* vals, int& n, int K, long long j, Real p, int& bad) {
  for (int k = 0; k < n; ++k)
    if (cols[k] == j) {
      vals[k] = mo_add_rn(vals[k], p);
      return;
    }
  if (n == K) {
    bad |= 4;
    return;
  }
  cols[n] = j;
  vals[n] = mo_add_rn(Real(0), p);
  ++n;
}
// kJtJ: each graph row's sorted, merged entries, once per edge (slot-major:
// entry k of edge e of template t at eoff + k * E + e); k_mat_hbuild reads
// them for every column the row holds instead of re-sorting per column.
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_mat_erows(const __grid_constant__ mo_mat_tables G, int* __restrict__ ecol, Real* __restrict__ eval,
            unsigned char* __restrict__ ecnt) {
  MO_PDL_ENTRY();
  const mo_mat_tmpl M = G.tm[blockIdx.y];
  if (M.kind != 1) return;
  const Real* buf = static_cast<const Real*>(M.buf);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < M.nrows;
       e += (long long)gridDim.x * blockDim.x) {
    long long rc[MO_MAT_MAXL];
    Real rv[MO_MAT_MAXL];
    int rn = 0;
    for (int l = 0; l < M.nlanes; ++l) {
      const mo_mat_lane B = G.lanes[M.lane0 + l];
      const long long col = G.ubase[B.field] + (long long)M.verts[e * M.arity + B.slot] * G.chans[B.field] + B.ch;
      const Real val = buf[(long long)B.out * M.nrows + e];
      int x = rn++;
      while (x > 0 && rc[x - 1] > col) {
        rc[x] = rc[x - 1];
        rv[x] = rv[x - 1];
        --x;
      }
      rc[x] = col;
      rv[x] = val;
    }
    int w = 0;
    for (int k = 0; k < rn;) {
      const long long col = rc[k];
      Real mv = rv[k];
      for (++k; k < rn && rc[k] == col; ++k) mv = mo_add_rn(mv, rv[k]);
      ecol[M.eoff + (long long)w * M.nrows + e] = int(col);
      eval[M.eoff + (long long)w * M.nrows + e] = mv;
      ++w;
    }
    ecnt[M.ecoff + e] = (unsigned char)w;
  }
}

#define MO_MAT_MAXK 64
template <class Real>
__global__ void __launch_bounds__(128)
k_mat_hbuild(const __grid_constant__ mo_mat_tables G, mo_state* st, int K, int* __restrict__ hcol,
             Real* __restrict__ hval, int* __restrict__ hcnt, const int* __restrict__ ecol,
             const Real* __restrict__ eval, const unsigned char* __restrict__ ecnt) {
  MO_PDL_ENTRY();
  const mo_mat_tables T = mo_mat_stage(G);
  int bad = 0;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < T.ncols;
       q += (long long)gridDim.x * blockDim.x) {
    long long cols[MO_MAT_MAXK];
    Real vals[MO_MAT_MAXK];
    int n = 0;
    int f = 0;
    while (f + 1 < T.nfields && T.ubase[f + 1] <= q) ++f;
    const long long rel = q - T.ubase[f];
    const long long el = T.ncols < 2147483647LL ? (long long)(int(rel) / T.chans[f]) : rel / T.chans[f];
    const int ch = int(rel - el * T.chans[f]);
    const int kk = T.cbase[f] + ch;
    for (int c = T.ceptr[kk]; c < T.ceptr[kk + 1]; ++c) {
      const mo_mat_centry E = T.ce[c];
      const mo_mat_tmpl M = T.tm[E.t];
      const Real* buf = static_cast<const Real*>(M.buf);
      if (E.lane >= 0) {
        const mo_mat_lane L = T.lanes[E.lane];
        const long long e = el - L.lin;
        if (e < 0 || e >= M.nrows) continue;
        if (buf[(long long)M.guard * M.nrows + e] == Real(0)) continue;
        const Real a = buf[(long long)L.out * M.nrows + e];
        for (int l = 0; l < M.nlanes; ++l) {
          const mo_mat_lane B = T.lanes[M.lane0 + l];
          const long long e2 = e + B.lin;
          if (e2 < 0 || e2 >= M.nrows) continue;
          mo_h_acc(cols, vals, n, K, T.ubase[B.field] + e2 * T.chans[B.field] + B.ch,
                   mo_mul_rn(a, buf[(long long)B.out * M.nrows + e]), bad);
        }
      } else {
        if (el >= M.nverts) continue;
        (void)buf;
        const long long eo = M.eoff, E = M.nrows;
        const unsigned char* cnt = ecnt + M.ecoff;
        for (int j = M.vptr[el]; j < M.vptr[el + 1]; ++j) {
          const int e = M.vedge[j];
          const int w = cnt[e];  // the row's sorted, merged entries (k_mat_erows)
          Real a = Real(0);
          bool has = false;
          for (int k = 0; k < w; ++k)
            if (ecol[eo + k * E + e] == q) {
              a = eval[eo + k * E + e];
              has = true;
            }
          if (!has) continue;
          for (int k = 0; k < w; ++k)
            mo_h_acc(cols, vals, n, K, (long long)ecol[eo + k * E + e], mo_mul_rn(a, eval[eo + k * E + e]), bad);
        }
      }
    }
    for (int k = 1; k < n; ++k) {  // emit in column order
      const long long cc = cols[k];
      const Real vv = vals[k];
      int x = k;
      while (x > 0 && cols[x - 1] > cc) {
        cols[x] = cols[x - 1];
        vals[x] = vals[x - 1];
        --x;
      }
      cols[x] = cc;
      vals[x] = vv;
    }
    hcnt[q] = n;
    for (int k = 0; k < n; ++k) {  // slot-major ELL: coalesced in the apply
      hcol[k * T.ncols + q] = int(cols[k]);
      hval[k * T.ncols + q] = mo_mul_rn(vals[k], Real(2));
    }
  }
  if (bad) atomicOr(&st->mat_bad, bad);
}

// spmv(H, v) (sparse.hpp spmv): out[q] = sum over row q in column order.
template <class Real>
__global__ void __launch_bounds__(MO_THREADS)
k_mat_happly(long long n, int K, const int* __restrict__ hcol, const Real* __restrict__ hval,
             const int* __restrict__ hcnt, const mo_state* st, int skipdone, const Real* __restrict__ v,
             Real* __restrict__ out) {
  MO_PDL_ENTRY();
  if (skipdone && st->done) return;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    Real acc = Real(0);
    const int c = hcnt[q];
    for (int k = 0; k < c; ++k) acc = mo_add_rn(acc, mo_mul_rn(hval[k * n + q], v[hcol[k * n + q]]));
    out[q] = acc;
  }
}

}  // namespace mo
