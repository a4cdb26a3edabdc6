// sm_100a kernels for the batched MLS-MPM substep and its adjoint.
//
// Layout:
//   particle state  AoSoA fp32, blocks of 32 particles x 24 fields
//                   (x 3, v 3, F 9 row-major, C 9), env-major; plus one packed
//                   u32 attribute per particle (original index | material |
//                   actuation group).  Fluid G2P outputs store F(0,0) only.
//   bins            4x4x4-cell tiles; per env a dense table of tile start /
//                   count into the env's stably sorted particle order, an
//                   env-ordered active-tile list and a largest-first work list
//   grid            per active tile a 6x6x6 node block (fp32 mass, momentum)
//                   accumulated in shared memory and written once; a node's
//                   value is the sum of the (<= 8) blocks that cover it, taken
//                   in ascending tile order, so every transfer is
//                   deterministic and atomic-free
//
// Persistent warps take tiles from the work list through a per-launch atomic
// counter; one warp owns one tile at a time.  Constitutive / per-particle
// math runs with lanes = particles; the stencil scatter runs with lanes = the
// 27 stencil nodes (3 groups x 9 columns), serially over each group's
// segment of the staged chunk, so shared-memory accumulation needs no atomics
// and has a fixed order (bit-reproducible replays: the recompute-on-backward
// contract of tape.hpp:234-241).  Particle and grid loads are software
// pipelined (next chunk in flight during the current one; cp.async for tile
// grids and the P2G-adjoint staging).
#pragma once

#include <cuda.h>  // CUtensorMap (TMA descriptors are encoded by the context)

#include <cstdint>

#include "dm_transfer.cuh"

namespace dm {

constexpr int kTile = 4;
constexpr int kExt = 6;  // tile + quadratic stencil reach
constexpr int kExt3 = kExt * kExt * kExt;
constexpr int kWarps = 4;  // warps per CTA in tile kernels
constexpr int kGridCoopParticlesPerWarp = 64;  // the grid kernels' COOP threshold (dm_create)
constexpr int kCoopParticlesPerWarp = 640;  // below this many particles per resident warp: COOP tiles (r02 A/B: cfg4 x128 envs +24 %, x256 -3 %)
// the scatter kernels (p2g, p2g_adj, g2p_adj) keep COOP up to larger batches
// (r02 A/B at 256 envs, 2-warp groups: g2p_adj -6 % in COOP, g2p +3 %; at
// 512 envs COOP loses everywhere)
constexpr int kCoopP2gParticlesPerWarp = 1280;
constexpr int kPay = 28;   // payload stride (floats; 7 float4, conflict-free STS.128 / 3-way LDS.128)
constexpr int kNacc = 64;  // per-tile cotangent accumulators
constexpr int kAccMu = 0, kAccLam = 4, kAccMuG = 8, kAccCol = 12, kAccAct = 48;

struct ColShape {
  int kind;
  float nrm[3], radius, half[3], length, thickness;
};

struct DevParams {
  int E, N;                // envs, particles per env
  int dims[3], td[3], Tn;  // grid dims, tile dims, tiles per env
  float dx, inv_dx, dt;
  float dx_lo;  // dx - (float)dx (node_rel)
  float grav[3];
  int boundary;
  float alpha_c, mu_b;
  int K, G, nmat;
  int fiso;  // input state's F isotropic (fluid: every g2p output, F = J^(1/3) I)
  int tauv;  // elastoplastic: the input state carries tau (S.tau), P2G skips the stress SVD
  Law<float> law[4];
  double dmu_dE[4], dlam_dE[4];  // Lame derivatives w.r.t. Young's modulus (fp64)
  ColShape shape[4];
};

// Particle-state layout: DM_AOSOA (default) stores blocks of 32 particles
// with their 24 fields contiguous ([i/32][24][32]: a warp's access to one
// field is one 128-byte segment, a particle's state one 3 KB region);
// otherwise plain SoA [24][Ntot].  Allocations round Ntot up to 32.
#ifndef DM_AOSOA
#define DM_AOSOA 1
#endif
#ifndef DM_AOSOA_LOG2
#define DM_AOSOA_LOG2 5  // particles per block = 32
#endif
constexpr size_t kAB = (size_t)1 << DM_AOSOA_LOG2;

// Bounds checks of the debug build (tools/bounds_check.sh: -DDM_DEBUG_BOUNDS,
// the GPU suite against it; compute-sanitizer is not available on the pool):
// a failed check prints the condition and traps, so the test fails loudly.
#ifdef DM_DEBUG_BOUNDS
#define DM_CHECK(cond)                                                          \
  do {                                                                          \
    if (!(cond)) {                                                              \
      printf("DM_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      __trap();                                                                 \
    }                                                                           \
  } while (0)
#else
#define DM_CHECK(cond) \
  do {                 \
  } while (0)
#endif
__host__ __device__ __forceinline__ size_t state_index(int comp, size_t i, size_t stride) {
#if DM_AOSOA
  (void)stride;
  return ((i >> DM_AOSOA_LOG2) * 24 + comp) * kAB + (i & (kAB - 1));
#else
  return comp * stride + i;
#endif
}

// Adjoint buffers share the layout: the state cotangent (24 fields) like the
// state, the particle-side partial cotangents (12 fields) in blocks of 32 x 12.
// kFluidTraceCot: in a fluid context the cotangent of a G2P-produced state's
// F is stored as its trace (field 6 / part field 3): such an F is J^(1/3) I,
// so every consumer of its cotangent (the next G2P projection's VJP,
// tr(F'bar) cof(F_new) / (3 J^(2/3))) reads only the trace.  The initial
// state (general F) keeps all nine.
__host__ __device__ __forceinline__ size_t adj_index(int comp, size_t i, size_t stride) {
  return state_index(comp, i, stride);
}
__host__ __device__ __forceinline__ size_t part_index(int comp, size_t i, size_t stride) {
#if DM_AOSOA
  (void)stride;
  return ((i >> DM_AOSOA_LOG2) * 12 + comp) * kAB + (i & (kAB - 1));
#else
  return comp * stride + i;
#endif
}

// tau (elastoplastic batches, G2P outputs inside a segment): the Kirchhoff
// stress P F^T of the state's F as the G2P projection computed it, 6
// symmetric components, AoSoA [N/32][6][32]; nullptr elsewhere.
struct StateView {
  float* f;
  uint32_t* attr;
  size_t stride;
  float* tau = nullptr;
  __device__ __forceinline__ float& c(int comp, size_t i) const {
    DM_CHECK(i < stride && comp >= 0 && comp < 24);
    return f[state_index(comp, i, stride)];
  }
  __device__ __forceinline__ float& t(int comp, size_t i) const {
    DM_CHECK(tau != nullptr && i < stride && comp >= 0 && comp < 6);
    return tau[((i >> 5) * 6 + comp) * 32 + (i & 31)];
  }
};

struct DevFlags {
  unsigned long long err_key;  // min over (env, substep, stage, particle, axis, code)
  unsigned int vmax_bits;      // max |v| component (CFL warning, mpm.hpp:355-361)
  int max_active;              // largest active-tile count seen (sizes the replay block pool)
};

__device__ __forceinline__ uint32_t attr_index(uint32_t a) { return a & 0xFFFFFu; }
__device__ __forceinline__ int attr_mat(uint32_t a) { return (a >> 20) & 0x3; }
__device__ __forceinline__ int attr_group(uint32_t a) { return (a >> 24) & 0xFF; }

// error key: substep(16) | env(16) | stage(2) | particle(24) | axis(2) | code(4).
// The minimum over a launch sequence is the first error in substep order
// (the reference throws at the first failing substep; within it at the
// lowest env, the P2G check before the G2P one, and the lowest particle
// index), so the flags can be read lazily after several control steps.
// sub = global substep index since the tape start.
__device__ __forceinline__ void report(DevFlags* fl, int env, int sub, int stage, uint32_t particle, int axis,
                                       int code) {
  const unsigned long long k = ((unsigned long long)(sub & 0xFFFF) << 48) |
                               ((unsigned long long)(env & 0xFFFF) << 32) | ((unsigned long long)(stage & 3) << 30) |
                               ((unsigned long long)(particle & 0xFFFFFF) << 6) | ((unsigned long long)(axis & 3) << 4) |
                               (unsigned long long)(code & 0xF);
  atomicMin(&fl->err_key, k);
}

// Dynamic tile scheduling: warps take active-tile indices from a per-launch
// counter (a wq ring slot zeroed by the previous tile kernel), so the load balances to within one
// tile; lane 0 grabs and broadcasts.
__device__ __forceinline__ int grab_tile(int* ctr, int lane, int n = 1) {
  int a = 0;
  if (lane == 0) a = atomicAdd(ctr, n);
  return __shfl_sync(0xffffffffu, a, 0);
}

// ---- launch chaining (programmatic dependent launch) ----
// Every kernel opens with dm_pdl(): it waits until the previous grid in the
// stream has completed and its writes are visible, then lets the next kernel
// be scheduled, so the next launch's setup and CTA rasterisation overlap this
// grid's tail instead of following it (small batches: ~2 us per boundary).
// Launched without the PDL attribute (DIFFMPM_NO_PDL=1) both are no-ops.
__device__ __forceinline__ void dm_pdl() {
#if DM_PDL_EARLY  // A/B: trigger first (the next-but-one kernel may then be scheduled too)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#else
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
}
// Tile-scheduling counters: a ring of kWqRing ints (one per tile-kernel
// launch, the ring aligned to its size).  Each tile kernel zeroes the next
// slot for the next tile kernel, so no memset node sits between launches
// (which would also break the PDL chain).
constexpr int kWqRing = 32;
constexpr int kOrdBuckets = 16;  // k_order_hist / k_order_scatter buckets
__device__ __forceinline__ void wq_clear_next(int* wq) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uintptr_t m = kWqRing * sizeof(int) - 1, u = reinterpret_cast<uintptr_t>(wq);
    *reinterpret_cast<int*>((u & ~m) | ((u + sizeof(int)) & m)) = 0;
  }
}

// Local base inside the tile, in [0, 4).  Always in range for valid particles
// (the bin key comes from the same fp32 base); clamped for particles already
// reported outside the interior so shared-memory indices stay in bounds.
__device__ __forceinline__ int tile_local(int base, int origin) {
  const int l = base - origin;
  return l < 0 ? 0 : (l > kTile - 1 ? kTile - 1 : l);
}

// Constitutive law with its kind fixed at compile time (LAW >= 0): the
// law switch folds away, so a kernel instantiated for the fluid or
// neo-Hookean law carries no SVD code and needs far fewer registers.
// LAW < 0 keeps the runtime dispatch (mixed-law batches).
template <int LAW>
__device__ __forceinline__ Law<float> law_of(const DevParams& P, int mi) {
  Law<float> L = P.law[mi];
  if (LAW >= 0) L.kind = LAW;
  return L;
}
#ifndef DM_G2P_MINB
#define DM_G2P_MINB 4
#endif
// 4 CTAs/SM (r02, with the staging ring: fluid -1.7 % vs 5; round 1 without it: 5 was 4 % faster)
constexpr int kG2pBlocks(int law) { return law == kFluid ? DM_G2P_MINB : 4; }

__device__ __forceinline__ TransferCtx<float> tctx(const DevParams& P) {
  TransferCtx<float> t;
  t.dims[0] = P.dims[0];
  t.dims[1] = P.dims[1];
  t.dims[2] = P.dims[2];
  t.dx = P.dx;
  t.inv_dx = P.inv_dx;
  t.dt = P.dt;
  t.dx64 = P.dx;
  return t;
}

__device__ __forceinline__ NodeCtx<float> nctx(const DevParams& P) {
  NodeCtx<float> g;
  g.dims[0] = P.dims[0];
  g.dims[1] = P.dims[1];
  g.dims[2] = P.dims[2];
  g.dx = P.dx;
  g.dx_lo = P.dx_lo;
  g.dt = P.dt;
  g.gravity = mk3(P.grav[0], P.grav[1], P.grav[2]);
  g.boundary = P.boundary;
  g.alpha_c = P.alpha_c;
  g.mu_b = P.mu_b;
  return g;
}

template <int MAXC>
__device__ __forceinline__ void load_cols(const DevParams& P, const float* cvo_env, Col<float>* cols) {
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    if (c >= P.K) break;
    const ColShape& s = P.shape[c];
    const float* q = cvo_env + 9 * c;
    cols[c].kind = s.kind;
    cols[c].c = mk3(q[0], q[1], q[2]);
    cols[c].vel = mk3(q[3], q[4], q[5]);
    cols[c].om = mk3(q[6], q[7], q[8]);
    cols[c].nrm = mk3(s.nrm[0], s.nrm[1], s.nrm[2]);
    cols[c].radius = s.radius;
    cols[c].length = s.length;
    cols[c].thickness = s.thickness;
    cols[c].half = mk3(s.half[0], s.half[1], s.half[2]);
  }
}

// The stored deviation D = F - I of the state.  The fluid projection
// (mpm.hpp:207) makes every G2P output F exactly J^(1/3) I (off-diagonals
// stored as +0), so for a fluid batch and a state produced by G2P (P.fiso)
// one word is read instead of nine; the reconstructed matrix holds the
// identical values.
template <int LAW>
__device__ __forceinline__ void load_F(const StateView& S, size_t i, m3<float>& F, int fiso) {
  if (LAW == kFluid && fiso) {
    const float sF = S.c(6, i);
    F = mdiag(sF, sF, sF);
  } else {
#pragma unroll
    for (int q = 0; q < 9; ++q) F.a[q] = S.c(6 + q, i);
  }
}

template <int LAW = -1>
__device__ __forceinline__ void load_state(const StateView& S, size_t i, float x[3], v3<float>& v, m3<float>& F,
                                           m3<float>& C, int fiso = 0) {
#pragma unroll
  for (int a = 0; a < 3; ++a) x[a] = S.c(a, i);
  v = mk3(S.c(3, i), S.c(4, i), S.c(5, i));
  load_F<LAW>(S, i, F, fiso);
#pragma unroll
  for (int q = 0; q < 9; ++q) C.a[q] = S.c(15 + q, i);
}

// G2P and its adjoint only read x and F of the start-of-substep state
// (v and C are outputs): 48 B (fluid after the first substep: 16 B).
template <int LAW = -1>
__device__ __forceinline__ void load_xF(const StateView& S, size_t i, float x[3], m3<float>& F, int fiso = 0) {
#pragma unroll
  for (int a = 0; a < 3; ++a) x[a] = S.c(a, i);
  load_F<LAW>(S, i, F, fiso);
}

// The F fields hold the deviation D = F - I (law_stress_fwd).  A fluid G2P
// output stores only D(0,0) (F = J^(1/3) I, D = (J^(1/3) - 1) I); readers of
// such a state reconstruct the rest (load_F, k_soa_to_aos, k_fiso_expand).
template <int LAW = -1>
__device__ __forceinline__ void store_state(const StateView& S, size_t i, v3<float> x, v3<float> v, const m3<float>& F,
                                            const m3<float>& C) {
  S.c(0, i) = x.x;
  S.c(1, i) = x.y;
  S.c(2, i) = x.z;
  S.c(3, i) = v.x;
  S.c(4, i) = v.y;
  S.c(5, i) = v.z;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    if (LAW != kFluid || q == 0) S.c(6 + q, i) = F.a[q];
    S.c(15 + q, i) = C.a[q];
  }
}

// ============================ binning ============================
// One CTA per env (nw warps): keys + interior check (p2g's stencil_base,
// mpm.hpp:149-161), per-warp tile histograms over contiguous particle chunks,
// dense tile table, active-tile list, and a stable counting sort: every warp
// scatters its chunk in index order from its own per-tile cursor, so the
// permutation equals std::stable_sort by key.
// CT: histogram / cursor word (unsigned short when particles per env fit in
// 16 bits: half the shared memory, twice the resident CTAs).
// vref[e]: the substep's reference velocity (node_update_rel): the mean
// velocity of the env's first min(N, 256) particles in physical order, in a
// fixed summation order (a deterministic function of the state: the replay
// reproduces it bitwise).
constexpr int kVrefParticles = 256;
constexpr int kBinU = 4;  // chunks whose loads k_bin / k_cellsort issue together
template <class CT>
__global__ void __launch_bounds__(1024, 2) k_bin(DevParams P, StateView S, int* keys, int* perm, int* tile_start,
                                             int* tile_count, int4* active, int* env_abase, int* env_acount,
                                             DevFlags* flags, int* nact, int substep, int check_vmax,
                                             float4* __restrict__ vref, int* __restrict__ ord) {
  dm_pdl();
  wq_clear_next(nact);  // nact: a zeroed ring slot here (k_order_hist stores the total in the slot's nact)
  // the bucket counters of k_order_hist / k_order_scatter (no memset node)
  if (blockIdx.x == 0 && threadIdx.x < 2 * kOrdBuckets) ord[threadIdx.x] = 0;
  extern __shared__ __align__(16) unsigned char bin_smem[];
  CT* cnt = reinterpret_cast<CT*>(bin_smem);  // [nw][Tn]
  __shared__ int s_part[1024 / 32 + 1][2];
  __shared__ int s_base;
  const int e = blockIdx.x;
  const int nw = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t base = (size_t)e * P.N;
  if (wid == 0) {
    const int nv = P.N < kVrefParticles ? P.N : kVrefParticles;
    float sx = 0.f, sy = 0.f, sz = 0.f;
    for (int p = lane; p < nv; p += 32) {
      sx += S.c(3, base + p);
      sy += S.c(4, base + p);
      sz += S.c(5, base + p);
    }
    for (int o = 16; o > 0; o >>= 1) {
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
      sy += __shfl_xor_sync(0xffffffffu, sy, o);
      sz += __shfl_xor_sync(0xffffffffu, sz, o);
    }
    const float inv = 1.f / (float)nv;
    // a non-finite reference (a blown-up particle) would poison every node: use 0
    const bool ok = isfinite(sx) && isfinite(sy) && isfinite(sz);
    if (lane == 0) vref[e] = ok ? make_float4(sx * inv, sy * inv, sz * inv, 0.f) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int t = threadIdx.x; t < nw * P.Tn; t += blockDim.x) cnt[t] = 0;
  __syncthreads();
  const int chunk = (P.N + nw - 1) / nw;
  const int p0 = wid * chunk, p1 = min(P.N, p0 + chunk);
  CT* my = cnt + wid * P.Tn;
  float vmax = 0.f;
  // kBinU chunks per step: their position loads are all in flight before the
  // first key is computed (latency-bound at small batches)
  for (int c0 = p0; c0 < p1; c0 += 32 * kBinU) {
    float xs[kBinU][3];
#pragma unroll
    for (int u = 0; u < kBinU; ++u) {
      const int p = c0 + 32 * u + lane;
      if (p < p1)
#pragma unroll
        for (int a = 0; a < 3; ++a) xs[u][a] = S.c(a, base + p);
    }
#pragma unroll
    for (int u = 0; u < kBinU; ++u) {
      const int p = c0 + 32 * u + lane;
      if (c0 + 32 * u >= p1) break;
      int key = -1 - lane;
      if (p < p1) {
        const size_t i = base + p;
        int b[3];
        float fx[3];
        const int bad = stencil_base(xs[u], P.inv_dx, (double)P.dx, P.dims, b, fx);
        if (bad >= 0) {
          report(flags, e, substep, 0, attr_index(S.attr[i]), bad, kErrP2GInterior);
#pragma unroll
          for (int a = 0; a < 3; ++a) b[a] = b[a] < 1 ? 1 : (b[a] > P.dims[a] - 4 ? P.dims[a] - 4 : b[a]);
        }
        key = ((b[0] >> 2) * P.td[1] + (b[1] >> 2)) * P.td[2] + (b[2] >> 2);
        keys[i] = key * 64 + ((b[0] & 3) * 4 + (b[1] & 3)) * 4 + (b[2] & 3);  // full key: tile * 64 + cell
        if (check_vmax) vmax = fmaxf(vmax, fmaxf(fabsf(S.c(3, i)), fmaxf(fabsf(S.c(4, i)), fabsf(S.c(5, i)))));
      }
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      if (p < p1 && lane == __ffs(peers) - 1) my[key] = (CT)(my[key] + __popc(peers));
      __syncwarp();
    }
  }
  if (check_vmax) {
    for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    if (lane == 0) atomicMax(&flags->vmax_bits, __float_as_uint(vmax));
  }
  __syncthreads();
  // per bin: total count; exclusive scan over bins of (count, active)
  const int nt = blockDim.x;
  const int per = (P.Tn + nt - 1) / nt;
  const int t0 = threadIdx.x * per, t1 = min(P.Tn, t0 + per);
  int sc = 0, sa = 0;
  for (int t = t0; t < t1; ++t) {
    int h = 0;
    for (int w = 0; w < nw; ++w) h += cnt[w * P.Tn + t];
    sc += h;
    sa += h > 0;
  }
  int ic = sc, ia = sa;
  for (int o = 1; o < 32; o <<= 1) {
    const int yc = __shfl_up_sync(0xffffffffu, ic, o);
    const int ya = __shfl_up_sync(0xffffffffu, ia, o);
    if (lane >= o) {
      ic += yc;
      ia += ya;
    }
  }
  if (lane == 31) {
    s_part[wid][0] = ic;
    s_part[wid][1] = ia;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int rc = 0, ra = 0;
    for (int w = 0; w < nw; ++w) {
      const int c = s_part[w][0], a = s_part[w][1];
      s_part[w][0] = rc;
      s_part[w][1] = ra;
      rc += c;
      ra += a;
    }
    s_base = atomicAdd(nact, ra);
    env_abase[e] = s_base;
    env_acount[e] = ra;
  }
  __syncthreads();
  int oc = s_part[wid][0] + ic - sc, oa = s_part[wid][1] + ia - sa;
  const size_t tb = (size_t)e * P.Tn;
  for (int t = t0; t < t1; ++t) {
    const int st = oc;
    for (int w = 0; w < nw; ++w) {  // per-warp cursors in warp (= index) order
      const int c = cnt[w * P.Tn + t];
      cnt[w * P.Tn + t] = (CT)oc;
      oc += c;
    }
    const int c = oc - st;
    tile_start[tb + t] = st;
    tile_count[tb + t] = c;
    if (c > 0) {
      active[s_base + oa] = make_int4(e, t, st, c);
      ++oa;
    }
  }
  __syncthreads();
  for (int c0 = p0; c0 < p1; c0 += 32 * kBinU) {
    int ks[kBinU];
#pragma unroll
    for (int u = 0; u < kBinU; ++u) {
      const int p = c0 + 32 * u + lane;
      ks[u] = p < p1 ? keys[base + p] >> 6 : -1 - lane;
    }
#pragma unroll
    for (int u = 0; u < kBinU; ++u) {  // in index order: the cursors advance stably
      if (c0 + 32 * u >= p1) break;
      const int p = c0 + 32 * u + lane;
      const int key = ks[u];
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int leader = __ffs(peers) - 1;
      const int rank = __popc(peers & ((1u << lane) - 1u));
      int pos = 0;
      if (lane == leader && p < p1) {
        pos = my[key];
        my[key] = (CT)(pos + __popc(peers));
      }
      pos = __shfl_sync(0xffffffffu, pos, leader);
      if (p < p1) perm[base + pos + rank] = (int)(base + p);
      __syncwarp();
    }
  }
}

// ---- work order: active tiles by descending particle count ----
// The tile kernels take tiles from a work list ordered largest-first (16
// buckets of 64 particles), so the dynamic scheduler ends on small tiles
// (longest-processing-time-first).  Only the schedule depends on the order:
// every tile's result is order-independent, and the replay and the adjoint of
// a substep share their slot's list, so the work index also names the tile's
// stored grid blocks consistently.  ord[0..15]: bucket counts, ord[16..31]:
// bucket cursors (zeroed by k_bin).
__device__ __forceinline__ int ord_bucket(int count) {
  const int b = count >> 6;
  return kOrdBuckets - 1 - (b < kOrdBuckets - 1 ? b : kOrdBuckets - 1);  // 0 = largest
}

__global__ void __launch_bounds__(256) k_order_hist(const int4* __restrict__ active, const int* acc, int* ord,
                                                    int* __restrict__ nact) {
  dm_pdl();
  __shared__ int h[kOrdBuckets];
  if (threadIdx.x < kOrdBuckets) h[threadIdx.x] = 0;
  __syncthreads();
  const int n = *(const volatile int*)acc;  // k_bin's ring-slot total -> the slot's nact
  if (blockIdx.x == 0 && threadIdx.x == 0) *nact = n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&h[ord_bucket(active[i].w)], 1);
  __syncthreads();
  if (threadIdx.x < kOrdBuckets && h[threadIdx.x]) atomicAdd(&ord[threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_order_scatter(const int4* __restrict__ active, const int* nact,
                                                       int* ord, int4* __restrict__ work) {
  dm_pdl();
  __shared__ int h[kOrdBuckets], base[kOrdBuckets];
  if (threadIdx.x < kOrdBuckets) h[threadIdx.x] = 0;
  __syncthreads();
  const int n = *(const volatile int*)nact;
  const int i0 = blockIdx.x * blockDim.x * 8, i1 = min(n, i0 + (int)blockDim.x * 8);
  int4 d[8];
  int b[8], r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = i0 + k * blockDim.x + threadIdx.x;
    b[k] = -1;
    if (i < i1) {
      d[k] = active[i];
      b[k] = ord_bucket(d[k].w);
      r[k] = atomicAdd(&h[b[k]], 1);
    }
  }
  __syncthreads();
  if (threadIdx.x < kOrdBuckets) {
    int start = 0;
    for (int q = 0; q < threadIdx.x; ++q) start += ord[q];
    base[threadIdx.x] = h[threadIdx.x] ? start + atomicAdd(&ord[kOrdBuckets + threadIdx.x], h[threadIdx.x]) : 0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (b[k] >= 0) work[base[b[k]] + r[k]] = d[k];
}

// ============================ sort records ============================
// The forward's binning of substep s (perm, dense tile counts, the active
// and work lists, per-env ranges, vref) copied into the rollout's record s,
// so the backward's segment replay reuses it instead of binning again (the
// replay's state is bit-identical, so is its sort).  Lists longer than the
// record's capacity set ovf (that substep is re-binned in the replay).
struct SortRec {
  int* perm;
  int* tile_count;
  int4* active;
  int4* work;
  int* abase;
  int* acount;
  int* nact;
  float4* vref;
  int* ovf;
};
// The sort record's copy of the capacity-limited binning tables, done by
// the cell-sort kernel's threads (grid-stride) instead of a k_rec_save
// launch; rec.nact == nullptr: no record for this substep.
struct RecSrc {
  const int4* active;
  const int4* work;
  const int* abase;
  const int* acount;
  const int* nact;
  const float4* vref;
  int cap, E;
};
__device__ __forceinline__ void rec_copy(const SortRec& r, const RecSrc& q) {
  if (!r.nact) return;
  const int n = *(const volatile int*)q.nact;
  const bool fits = n <= q.cap;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i0 == 0) {
    *r.nact = n;
    *r.ovf = fits ? 0 : 1;
  }
  if (fits)
    for (size_t i = i0; i < (size_t)n; i += stride) {
      r.active[i] = q.active[i];
      r.work[i] = q.work[i];
    }
  for (size_t i = i0; i < (size_t)q.E; i += stride) {
    r.abase[i] = q.abase[i];
    r.acount[i] = q.acount[i];
    r.vref[i] = q.vref[i];
  }
}

// Small batches (a few thousand active tiles at most): both passes in one
// CTA -- bucket counts, scan, scatter -- one launch instead of two.  Same
// bucket order as k_order_hist + k_order_scatter (the order inside a bucket
// is not fixed by either; every tile's result is independent of it).
// With a sort record (rec.nact != nullptr) it also writes the record's
// copies of the lists and per-env tables (off the cell sort's critical path).
__global__ void __launch_bounds__(1024) k_order_small(const int4* __restrict__ active, const int* acc,
                                                      int* __restrict__ nact, int4* __restrict__ work, SortRec rec,
                                                      RecSrc rs) {
  dm_pdl();
  __shared__ int h[kOrdBuckets], cur[kOrdBuckets];
  if (threadIdx.x < kOrdBuckets) h[threadIdx.x] = 0;
  __syncthreads();
  const int n = *(const volatile int*)acc;  // k_bin's ring-slot total -> the slot's nact
  const bool keep = rec.nact && n <= rs.cap;
  if (threadIdx.x == 0) {
    *nact = n;
    if (rec.nact) {
      *rec.nact = n;
      *rec.ovf = keep ? 0 : 1;
    }
  }
  if (rec.nact)
    for (int i = threadIdx.x; i < rs.E; i += blockDim.x) {
      rec.abase[i] = rs.abase[i];
      rec.acount[i] = rs.acount[i];
      rec.vref[i] = rs.vref[i];
    }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int4 d = active[i];
    atomicAdd(&h[ord_bucket(d.w)], 1);
    if (keep) rec.active[i] = d;
  }
  __syncthreads();
  if (threadIdx.x < kOrdBuckets) {
    int start = 0;
    for (int q = 0; q < (int)threadIdx.x; ++q) start += h[q];
    cur[threadIdx.x] = start;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int4 d = active[i];
    const int pos = atomicAdd(&cur[ord_bucket(d.w)], 1);
    work[pos] = d;
    if (keep) rec.work[pos] = d;
  }
}

// Second sort level: within every active tile, a stable counting sort by the
// cell inside the tile (64 buckets).  Final key = tile * 64 + cell; particles
// of one cell become contiguous so the stencil scatters can accumulate runs in
// registers.  Equals std::stable_sort by the full key (the tile pass is stable).
__global__ void __launch_bounds__(kWarps * 32) k_cellsort(DevParams P, StateView S, const int* __restrict__ ptile,
                                                          int* __restrict__ perm, int* __restrict__ keys,
                                                          const int* __restrict__ tile_start,
                                                          const int* __restrict__ tile_count,
                                                          const int4* __restrict__ active, const int* nact,
                                                          DevFlags* flags, int* __restrict__ wq, SortRec rec, RecSrc rsrc) {
  dm_pdl();
  wq_clear_next(wq);
  rec_copy(rec, rsrc);
  __shared__ int c64[kWarps][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* cnt = c64[warp];
  const int n_active = *(const volatile int*)nact;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(&flags->max_active, n_active);
  for (int a = grab_tile(wq, lane), an = a < n_active ? grab_tile(wq, lane) : n_active; a < n_active;
       a = an, an = a < n_active ? grab_tile(wq, lane) : n_active) {
    const int4 et = active[a];
    const int e = et.x;
    const int start = et.z, n = et.w;
    const size_t base = (size_t)e * P.N + start;
    cnt[lane] = 0;
    cnt[lane + 32] = 0;
    __syncwarp();
    auto cell_of = [&](int src) { return keys[src] & 63; };  // k_bin stored the full key
    // kBinU chunks per step, their dependent (perm -> key) loads in flight together
    auto load_cells = [&](int c0, int (&src)[kBinU], int (&cell)[kBinU]) __attribute__((always_inline)) {
#pragma unroll
      for (int u = 0; u < kBinU; ++u) src[u] = c0 + 32 * u + lane < n ? ptile[base + c0 + 32 * u + lane] : -1;
#pragma unroll
      for (int u = 0; u < kBinU; ++u) cell[u] = src[u] >= 0 ? cell_of(src[u]) : 64 + lane;
    };
    for (int c0 = 0; c0 < n; c0 += 32 * kBinU) {
      int src[kBinU], cl[kBinU];
      load_cells(c0, src, cl);
#pragma unroll
      for (int u = 0; u < kBinU; ++u) {
        if (c0 + 32 * u >= n) break;
        const bool ok = src[u] >= 0;
        const unsigned peers = __match_any_sync(0xffffffffu, cl[u]);
        if (ok && lane == __ffs(peers) - 1) cnt[cl[u]] += __popc(peers);
        __syncwarp();
      }
    }
    // exclusive scan over the 64 buckets (2 per lane)
    const int a0 = cnt[2 * lane], a1 = cnt[2 * lane + 1];
    int incl = a0 + a1;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int ex = incl - a0 - a1;
    __syncwarp();
    cnt[2 * lane] = ex;
    cnt[2 * lane + 1] = ex + a0;
    __syncwarp();
    for (int c0 = 0; c0 < n; c0 += 32 * kBinU) {
      int src[kBinU], cl[kBinU];
      load_cells(c0, src, cl);
#pragma unroll
      for (int u = 0; u < kBinU; ++u) {  // in index order: stable
        if (c0 + 32 * u >= n) break;
        const bool ok = src[u] >= 0;
        const unsigned peers = __match_any_sync(0xffffffffu, cl[u]);
        const int leader = __ffs(peers) - 1;
        const int rank = __popc(peers & ((1u << lane) - 1u));
        int pos = 0;
        if (ok && lane == leader) {
          pos = cnt[cl[u]];
          cnt[cl[u]] = pos + __popc(peers);
        }
        pos = __shfl_sync(0xffffffffu, pos, leader);
        if (ok) perm[base + pos + rank] = src[u];
        __syncwarp();
      }
    }
  }
}

// ---- run-accumulated deterministic scatter ----
// Phase 1 (lanes = particles) stages a payload per particle: the local base
// node (linear in the 6^3 block), the 3x3 separable weights, and the affine
// contribution (m, q, Ad) with node value w_o (m, q + Ad o).  Phase 2 (lanes =
// the 27 stencil nodes) walks the chunk's particles in order; particles are
// cell-sorted, so a lane accumulates the run of particles sharing a base cell
// in registers and touches shared memory once per run.  Fixed order: no
// atomics, bit-reproducible.
struct RunAcc {
  int cur;
  float4 acc[3];
};

// Payload (7 float4 per particle, stride 28 floats):
//   0: (lbl, m, wz0, wz1)  1: (wz2, w00, w01, w02)  2: (w10, w11, w12, w20)
//   3: (w21, w22, -, -)    4..6: row r of (q | Ad) = (q_r, Ad_r0, Ad_r1, Ad_r2)
// with w_ij = wx_i * wy_j precomputed (float index 5 + 3 i + j).
__device__ __forceinline__ void stage_payload(float* __restrict__ pp, int lbl, const Stencil<float>& sc, float m,
                                              v3<float> q, const m3<float>& Ad) {
  float4* p4 = reinterpret_cast<float4*>(pp);
  float w[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) w[3 * i + j] = sc.w[0][i] * sc.w[1][j];
  p4[0] = make_float4(__int_as_float(lbl), sc.w[2][0], sc.w[2][1], sc.w[2][2]);
  p4[1] = make_float4(m, w[0], w[1], w[2]);
  p4[2] = make_float4(w[3], w[4], w[5], w[6]);
  p4[3] = make_float4(w[7], w[8], 0.f, 0.f);
  p4[4] = make_float4(q.x, Ad.a[0], Ad.a[1], Ad.a[2]);
  p4[5] = make_float4(q.y, Ad.a[3], Ad.a[4], Ad.a[5]);
  p4[6] = make_float4(q.z, Ad.a[6], Ad.a[7], Ad.a[8]);
}

// cur starts at node 0 of the block: the first flush then adds zeros there
// (x + 0 == x), so the flush needs no branch.
__device__ __forceinline__ void run_reset(RunAcc& ra) {
  ra.cur = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) ra.acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Adds the lane's three run sums (nodes (i, j, 0..2) of the run's base) into
// its group's block copy.
__device__ __forceinline__ void run_flush(float4* __restrict__ blk, RunAcc& ra, int off) {
  DM_CHECK(ra.cur >= 0 && ra.cur + off + 2 < kExt3);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float4 b = blk[ra.cur + off + k];
    b.x += ra.acc[k].x;
    b.y += ra.acc[k].y;
    b.z += ra.acc[k].z;
    b.w += ra.acc[k].w;
    blk[ra.cur + off + k] = b;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) ra.acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Lanes 0..26 = 3 groups x 9 stencil columns (i, j).  A staged chunk of 32
// cell-sorted particles is cut into three contiguous segments (kSeg each) and
// group g walks segment g in order, so a run is a cell's particles within the
// segment and a lane flushes about once per cell; each lane accumulates the 3
// nodes (i, j, 0..2) of its column.  Each group flushes into its own block
// copy (no write races); the copies are summed in fixed order by
// scatter_store.  The next particle's payload is loaded while the current one
// accumulates (shared-memory latency off the critical path).
constexpr int kSeg = 11;

struct PayLane {
  int lb;
  float m, wij, wz[3];
  float4 r[3];
};

// Payload: (label, wz0, wz1, wz2), (m, w_00 .. w_22), (q_a, Ad row a) x 3:
// the mass-free adjoint scatter reads 5 shared-memory words-groups per
// particle, P2G 6 (g2p_adj -2.8 %; a register mass for one-material batches
// made P2G slower, +3.7 %).
template <bool HASM>
__device__ __forceinline__ void load_pay(const float* __restrict__ pk, int wi, PayLane& p) {
  const float4* p4 = reinterpret_cast<const float4*>(pk);
  const float4 h = p4[0];
  p.lb = __float_as_int(h.x);
  p.wz[0] = h.y;
  p.wz[1] = h.z;
  p.wz[2] = h.w;
  p.m = HASM ? pk[4] : 0.f;
  p.wij = pk[wi];
  p.r[0] = p4[4];
  p.r[1] = p4[5];
  p.r[2] = p4[6];
}

// One particle's contribution to the lane's column run.
#ifndef DM_RUN_SHIFT
#define DM_RUN_SHIFT 1
#endif
template <bool HASM>
__device__ __forceinline__ void run_add(float4* __restrict__ blk, RunAcc& ra, int off, float fi, float fj,
                                        const PayLane& p) {
  if (p.lb != ra.cur) {
    if (DM_RUN_SHIFT && HASM && p.lb == ra.cur + 1) {
      // next cell in z (the sort's innermost order): the run's nodes k = 1, 2
      // are the new run's k = 0, 1 -- flush only node k = 0 and shift
      // (P2G only: measured slower in the G2P adjoint)
      float4 b = blk[ra.cur + off];
      b.x += ra.acc[0].x;
      b.y += ra.acc[0].y;
      b.z += ra.acc[0].z;
      b.w += ra.acc[0].w;
      blk[ra.cur + off] = b;
      ra.acc[0] = ra.acc[1];
      ra.acc[1] = ra.acc[2];
      ra.acc[2] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      run_flush(blk, ra, off);
    }
    ra.cur = p.lb;
  }
  // node (i, j, kk) value: b + kk a  (b = q + Ad_0 i + Ad_1 j, a = Ad_2)
  const float bx = fmaf(p.r[0].z, fj, fmaf(p.r[0].y, fi, p.r[0].x));
  const float by = fmaf(p.r[1].z, fj, fmaf(p.r[1].y, fi, p.r[1].x));
  const float bz = fmaf(p.r[2].z, fj, fmaf(p.r[2].y, fi, p.r[2].x));
  const float ax = p.r[0].w, ay = p.r[1].w, az = p.r[2].w;
  const float cx[3] = {bx, bx + ax, fmaf(ax, 2.f, bx)};
  const float cy[3] = {by, by + ay, fmaf(ay, 2.f, by)};
  const float cz[3] = {bz, bz + az, fmaf(az, 2.f, bz)};
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    const float w = p.wij * p.wz[kk];
    if (HASM) ra.acc[kk].x += w * p.m;
    ra.acc[kk].y += w * cx[kk];
    ra.acc[kk].z += w * cy[kk];
    ra.acc[kk].w += w * cz[kk];
  }
}

// Two payload register sets alternate (no register moves between particles).
template <bool HASM>
__device__ __forceinline__ void scatter_runs(float4* __restrict__ blk3, const float* __restrict__ pay, int nv, int lane,
                                             RunAcc& ra) {
  if (lane < 27) {
    const int g = lane / 9, i = (lane % 9) / 3, j = lane % 3;
    float4* blk = blk3 + g * kExt3;
    const int off = (i * kExt + j) * kExt;
    const int wi = 5 + 3 * i + j;
    const float fi = (float)i, fj = (float)j;
    const int k0 = g * kSeg, k1 = min(nv, k0 + kSeg);
    if (k0 < k1) {
      PayLane pa, pb;
      load_pay<HASM>(pay + k0 * kPay, wi, pa);
      int k = k0;
      for (; k + 1 < k1; k += 2) {
        load_pay<HASM>(pay + (k + 1) * kPay, wi, pb);
        run_add<HASM>(blk, ra, off, fi, fj, pa);
        if (k + 2 < k1) load_pay<HASM>(pay + (k + 2) * kPay, wi, pa);
        run_add<HASM>(blk, ra, off, fi, fj, pb);
      }
      if (k < k1) run_add<HASM>(blk, ra, off, fi, fj, pa);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void scatter_zero(float4* __restrict__ blk3, int lane) {
  for (int i = lane; i < 3 * kExt3; i += 32) blk3[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Final flush, then block = copy0 + copy1 + copy2 (fixed order) -> dst.
__device__ __forceinline__ void scatter_store(float4* __restrict__ blk3, int lane, RunAcc& ra, float4* __restrict__ dst) {
  if (lane < 27) run_flush(blk3 + (lane / 9) * kExt3, ra, (((lane % 9) / 3) * kExt + lane % 3) * kExt);
  __syncwarp();
  for (int i = lane; i < kExt3; i += 32) {
    const float4 a = blk3[i], b = blk3[kExt3 + i], c = blk3[2 * kExt3 + i];
    dst[i] = make_float4((a.x + b.x) + c.x, (a.y + b.y) + c.y, (a.z + b.z) + c.z, (a.w + b.w) + c.w);
  }
  __syncwarp();
}

// dynamic shared memory of the scatter kernels (bytes per CTA)
constexpr size_t kP2gSmem = (size_t)kWarps * (3 * kExt3 * sizeof(float4) + 32 * kPay * sizeof(float));
constexpr size_t kG2pAdjSmem = (size_t)kWarps * (4 * kExt3 * sizeof(float4) + 32 * kPay * sizeof(float));

// Persistent tile loop: the next two tiles' descriptors (env, tile, start,
// count) are loaded ahead (`nxt` is known when the current tile starts, so
// its grid block can be prefetched) and the index after them is grabbed
// ahead, so neither the atomic nor the descriptor load is on the critical path.
struct TileIter {
  int a, a1, a2, a3, n, lane;
  int* ctr;
  int4 cur, nxt, nxt2;
  __device__ __forceinline__ TileIter(const int4* __restrict__ active, int* ctr_, int n_, int lane_) {
    n = n_;
    lane = lane_;
    ctr = ctr_;
    a = grab_tile(ctr, lane, 2);
    a1 = a + 1;
    a2 = grab_tile(ctr, lane);
    a3 = n;
    cur = a < n ? active[a] : make_int4(0, 0, 0, 0);
    nxt = a1 < n ? active[a1] : make_int4(0, 0, 0, 0);
    nxt2 = make_int4(0, 0, 0, 0);
  }
  __device__ __forceinline__ bool valid() const { return a < n; }
  __device__ __forceinline__ bool has_next() const { return a1 < n; }
  __device__ __forceinline__ void prefetch(const int4* __restrict__ active) {
    if (a2 < n) nxt2 = active[a2];
    a3 = a2 < n ? grab_tile(ctr, lane) : n;
  }
  __device__ __forceinline__ void advance() {
    a = a1;
    a1 = a2;
    a2 = a3;
    cur = nxt;
    nxt = nxt2;
  }
};

// cp.async (LDGSTS) 16-byte copies; src_size 0 zero-fills (out-of-grid nodes)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- TMA / bulk async copies (sm_90+ async proxy; mbarrier completion) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
// the issuing thread's arrival, expecting `bytes` of async-proxy writes
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// generic-proxy accesses of a buffer are ordered before a following async-proxy write into it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// 1-D bulk copy global -> shared (UBLKCP), completing on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  mbar_expect_tx(bar, bytes);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 1-D bulk copy shared -> global (bulk async group of the issuing thread)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// the issuing thread's bulk stores have finished reading shared memory
__device__ __forceinline__ void bulk_s2g_read_wait() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_s2g_wait() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// cp.async (LDGSTS) load of tile d's 6^3 block of a dense grid, zero-filling
// nodes past the grid's far faces (src-size 0).
__device__ __forceinline__ void prefetch_tile_grid(const DevParams& P, const float4* __restrict__ grid, int4 d,
                                                   float4* dst, int lane) {
  const int t = d.y;
  const int o[3] = {(t / (P.td[2] * P.td[1])) * kTile, ((t / P.td[2]) % P.td[1]) * kTile, (t % P.td[2]) * kTile};
  const size_t eb = (size_t)d.x * P.dims[0] * P.dims[1] * P.dims[2];
  for (int i = lane; i < kExt3; i += 32) {
    const int g0 = o[0] + i / 36, g1 = o[1] + (i / 6) % 6, g2 = o[2] + i % 6;
    const bool in = g0 < P.dims[0] && g1 < P.dims[1] && g2 < P.dims[2];
    cp_async16(dst + i, in ? grid + eb + ((size_t)g0 * P.dims[1] + g1) * P.dims[2] + g2 : grid, in);
  }
}

// TMA tensor load (UTMALDG) of tile d's 6^3 node block of a dense per-env grid
// [E][d0][d1][d2] float4, described by the 4-D map tm (4 d2 floats, d1, d0,
// E; box 24 x 6 x 6 x 1, dm_context.cu make_grid_tmap).  Nodes past the
// grid's far faces are zero-filled by the TMA unit (the cp.async path's
// src-size-0 copies).  One thread issues it; completion lands on bar.
__device__ __forceinline__ void tma_tile_grid(const DevParams& P, const CUtensorMap* tm, int4 d, float4* dst,
                                              uint64_t* bar) {
  const int t = d.y;
  const int o0 = (t / (P.td[2] * P.td[1])) * kTile, o1 = ((t / P.td[2]) % P.td[1]) * kTile, o2 = (t % P.td[2]) * kTile;
  mbar_expect_tx(bar, kExt3 * (uint32_t)sizeof(float4));
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(4 * o2), "r"(o1), "r"(o0), "r"(d.x), "r"(smem_u32(bar))
      : "memory");
}

// Particle state of one chunk slot held in registers (software pipeline:
// the next chunk's loads are issued before the current chunk's scatter).
struct PState {
  float x[3];
  v3<float> v;
  m3<float> F, C;
  uint32_t at;
};

// tauv (elastoplastic, a G2P output inside a segment): the cached stress's 6
// components go into F.a[0..5] instead of F (P2G needs F only for the stress).
template <int LAW>
__device__ __forceinline__ void load_pstate(const StateView& S, int src, PState& p, int fiso, int tauv = 0) {
  if (LAW == kElastoplastic && tauv) {
#pragma unroll
    for (int a = 0; a < 3; ++a) p.x[a] = S.c(a, src);
    p.v = mk3(S.c(3, src), S.c(4, src), S.c(5, src));
#pragma unroll
    for (int q = 0; q < 6; ++q) p.F.a[q] = S.t(q, src);
#pragma unroll
    for (int q = 0; q < 9; ++q) p.C.a[q] = S.c(15 + q, src);
  } else {
    load_state<LAW>(S, src, p.x, p.v, p.F, p.C, fiso);
  }
  p.at = S.attr[src];
}

// ---- cooperative tiles (small batches) ----
// With few tiles per resident warp (a small env batch: cfg 1, cfg 2, a
// strong-scaling shard) one warp per tile leaves most of the GPU idle and a
// launch lasts as long as its largest tile's chunk chain.  COOP kernels let
// the 4 warps of a CTA share a tile: warp w takes the tile's 32-particle
// chunks w, w + 4, w + 8, ...  Each warp runs the usual per-chunk code on a
// virtual particle range: its virtual index v maps to the tile's index
// coop_idx(v, w); the last (partial) chunk belongs to one warp.  Scatter
// kernels sum the 4 warps' block copies in a fixed order (deterministic;
// the replay uses the same mode), gathers need no reduction.
// CG (warps per tile group) divides kWarps: CG < kWarps lets a CTA work on
// kWarps / CG tiles at once (groups synchronise on named barriers).
template <bool COOP, int CG = kWarps>
__device__ __forceinline__ int coop_idx(int v, int w) {
  return COOP ? (((v >> 5) * CG + w) << 5) + (v & 31) : v;
}
template <bool COOP, int CG = kWarps>
__device__ __forceinline__ int coop_count(int cnt, int w) {
  if (!COOP) return cnt;
  const int nc = (cnt + 31) >> 5;
  if (w >= nc) return 0;
  const int k = (nc - 1 - w) / CG + 1;  // chunks w, w + CG, ... below nc
  return 32 * k - ((((nc - 1) % CG) == w) ? 32 * nc - cnt : 0);
}
template <int CG>
__device__ __forceinline__ void group_sync(int g) {
  if (CG == kWarps)
    __syncthreads();
  else
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + g), "n"(CG * 32) : "memory");
}

// Group-level item loop of the COOP kernels: the group's first thread takes
// the next item, the group (the CTA when CG = kWarps) processes it, a
// barrier closes it.
template <int CG = kWarps, class Body>
__device__ __forceinline__ void coop_loop(const int4* __restrict__ work, int* ctr, int n, Body& body) {
  __shared__ int s_item[kWarps / CG];
  const int g = (threadIdx.x >> 5) / CG;
  const int tig = threadIdx.x - g * CG * 32;
  for (;;) {
    if (tig == 0) s_item[g] = atomicAdd(ctr, 1);
    group_sync<CG>(g);
    const int a = s_item[g];
    if (a >= n) break;
    body(work[a], a);
    group_sync<CG>(g);
  }
}

// Fixed-order sum of the group's CG x 3 scatter copies (warp w's copies at
// base + w * wstride, kExt3 apart) into dst, after every warp flushed.
template <int CG = kWarps>
__device__ __forceinline__ void coop_store_blocks(const float4* __restrict__ base, int wstride,
                                                  float4* __restrict__ dst) {
  const int g = (threadIdx.x >> 5) / CG;
  group_sync<CG>(g);
  for (int i = threadIdx.x - g * CG * 32; i < kExt3; i += CG * 32) {
    float4 acc = base[i];
#pragma unroll
    for (int c = 1; c < 3 * CG; ++c) {
      const float4 b = base[(c / 3) * wstride + (c % 3) * kExt3 + i];
      acc.x += b.x;
      acc.y += b.y;
      acc.z += b.z;
      acc.w += b.w;
    }
    dst[i] = acc;
  }
}

// Fixed-order group sum of a per-warp value (after the warp's butterfly; lane 0 holds it).
template <int CG = kWarps, class V>
__device__ __forceinline__ V coop_sum(V v) {
  __shared__ V s_part[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = warp / CG;
  group_sync<CG>(g);
  if (lane == 0) s_part[warp] = v;
  group_sync<CG>(g);
  V acc = s_part[g * CG];
#pragma unroll
  for (int w = 1; w < CG; ++w) acc += s_part[g * CG + w];
  return acc;
}
// COOP group size CG (warps per tile; the tile kernels' last template
// parameter, chosen per context): 2 for small batches -- each CTA works on
// two tiles, half the block copies to combine, shorter barrier waits (r02
// A/B: cfg2 +12 %, cfg4 at 128 envs +11 %) -- and 4 for tiny ones, where a
// tile's chunk chain is the critical path (cfg1: CG = 2 was 25 % slower).

// k_cellsort with CTA-shared tiles (small batches: a tile's chunk chain is
// the launch's critical path).  Warp w takes the w-th contiguous quarter of
// the tile (whole chunks), counts it, the CTA scans the 64 buckets in
// (bucket, warp) order, and each warp scatters its quarter in index order
// from its cursors: the same stable permutation as k_cellsort.
__global__ void __launch_bounds__(kWarps * 32) k_cellsort_coop(DevParams P, const int* __restrict__ ptile,
                                                               int* __restrict__ perm, const int* __restrict__ keys,
                                                               const int4* __restrict__ active, const int* nact,
                                                               DevFlags* flags, int* __restrict__ wq, SortRec rec, RecSrc rsrc) {
  dm_pdl();
  wq_clear_next(wq);
  rec_copy(rec, rsrc);
  __shared__ int c64[kWarps][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_active = *(const volatile int*)nact;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicMax(&flags->max_active, n_active);
  auto item = [&](const int4 et, int) __attribute__((always_inline)) {
    const int n = et.w;
    const size_t base = (size_t)et.x * P.N + et.z;
    const int nch = (n + 31) >> 5, per = (nch + kWarps - 1) / kWarps;
    const int q0 = min(n, warp * per * 32), q1 = min(n, (warp + 1) * per * 32);  // this warp's quarter
    int* cnt = c64[warp];
    cnt[lane] = 0;
    cnt[lane + 32] = 0;
    __syncwarp();
    auto load_cells = [&](int c0, int (&src)[kBinU], int (&cell)[kBinU]) __attribute__((always_inline)) {
#pragma unroll
      for (int u = 0; u < kBinU; ++u) src[u] = c0 + 32 * u + lane < q1 ? ptile[base + c0 + 32 * u + lane] : -1;
#pragma unroll
      for (int u = 0; u < kBinU; ++u) cell[u] = src[u] >= 0 ? (keys[src[u]] & 63) : 64 + lane;
    };
    for (int c0 = q0; c0 < q1; c0 += 32 * kBinU) {
      int src[kBinU], cl[kBinU];
      load_cells(c0, src, cl);
#pragma unroll
      for (int u = 0; u < kBinU; ++u) {
        if (c0 + 32 * u >= q1) break;
        const unsigned peers = __match_any_sync(0xffffffffu, cl[u]);
        if (src[u] >= 0 && lane == __ffs(peers) - 1) cnt[cl[u]] += __popc(peers);
        __syncwarp();
      }
    }
    __syncthreads();
    if (warp == 0) {  // bucket-major exclusive scan of (bucket, warp) counts -> cursors
      int t0 = 0, t1 = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        t0 += c64[w][2 * lane];
        t1 += c64[w][2 * lane + 1];
      }
      int incl = t0 + t1;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int e0 = incl - t0 - t1, e1 = incl - t1;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const int a0 = c64[w][2 * lane], a1 = c64[w][2 * lane + 1];
        c64[w][2 * lane] = e0;
        c64[w][2 * lane + 1] = e1;
        e0 += a0;
        e1 += a1;
      }
    }
    __syncthreads();
    for (int c0 = q0; c0 < q1; c0 += 32 * kBinU) {
      int src[kBinU], cl[kBinU];
      load_cells(c0, src, cl);
#pragma unroll
      for (int u = 0; u < kBinU; ++u) {  // in index order: stable
        if (c0 + 32 * u >= q1) break;
        const bool ok = src[u] >= 0;
        const unsigned peers = __match_any_sync(0xffffffffu, cl[u]);
        const int leader = __ffs(peers) - 1;
        const int rank = __popc(peers & ((1u << lane) - 1u));
        int pos = 0;
        if (ok && lane == leader) {
          pos = cnt[cl[u]];
          cnt[cl[u]] = pos + __popc(peers);
        }
        pos = __shfl_sync(0xffffffffu, pos, leader);
        if (ok) perm[base + pos + rank] = src[u];
        __syncwarp();
      }
    }
  };
  coop_loop(active, wq, n_active, item);
}

// ============================ P2G ============================
// Per active tile: stage particle payloads (lanes = particles), scatter runs
// into the warp's 6^3 shared block (lanes = stencil nodes), write the block.
// The next chunk's state loads are in flight during the current scatter.

// Drives a per-chunk body (32 particles; chunk k + 1's perm index sits in
// parity slot (k + 1) & 1; the body loads that chunk and returns chunk
// k + 3's index for the slot).  Two call sites per iteration suit the short
// bodies (fluid; neo-Hookean in k_p2g: -8 %, but +2 % in k_g2p_adj); the
// SVD laws take one call site with the slot selected by parity (their bodies
// are 3-4x larger and ran 14-70 % faster as a single copy; as a plain lambda
// called twice they were outlined onto an 880-byte stack).
template <bool TWO, class Body>
__device__ __forceinline__ void chunk_loop(Body& body, int cnt, int& s0, int& s1) {
  if constexpr (TWO) {
    for (int c0 = 0; c0 < cnt; c0 += 64) {
      s1 = body(c0, s1);
      if (c0 + 32 >= cnt) break;
      s0 = body(c0 + 32, s0);
    }
  } else {
    for (int c0 = 0, k = 0; c0 < cnt; c0 += 32, ++k) {
      const int sn = body(c0, (k & 1) ? s0 : s1);
      s0 = (k & 1) ? sn : s0;
      s1 = (k & 1) ? s1 : sn;
    }
  }
}

#ifndef DM_P2G_MINB
#define DM_P2G_MINB 4
#endif

template <int LAW, bool COOP, int CG>
__global__ void __launch_bounds__(kWarps * 32, DM_P2G_MINB) k_p2g(DevParams P, StateView S, const int* __restrict__ perm,
                                                     const int* __restrict__ tile_start,
                                                     const int* __restrict__ tile_count, const int4* __restrict__ active,
                                                     const float* __restrict__ act, float4* __restrict__ blocks,
                                                     DevFlags* flags, const int* nact, int substep, int* __restrict__ wq,
                                                     const float4* __restrict__ vref) {
  dm_pdl();
  wq_clear_next(wq);
  extern __shared__ float4 dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_active = *(const volatile int*)nact;
  const TransferCtx<float> T = tctx(P);
  float4* bw = dsm + warp * 3 * kExt3;  // 3 group copies of the 6^3 block
  float* pw = reinterpret_cast<float*>(dsm + kWarps * 3 * kExt3) + warp * 32 * kPay;
  auto tile = [&](const int4 cur) __attribute__((always_inline)) {
    const int e = cur.x, t = cur.y, start = cur.z;
    const int cnt = coop_count<COOP, CG>(cur.w, warp % CG);  // this warp's (virtual) particle count
    const int tz = t % P.td[2], ty = (t / P.td[2]) % P.td[1], tx = t / (P.td[2] * P.td[1]);
    const int o[3] = {tx * kTile, ty * kTile, tz * kTile};
    const size_t tix = (size_t)e * P.Tn + t;
    const int* prow = perm + (size_t)e * P.N + start;
    auto pidx = [&](int v) {
      DM_CHECK((coop_idx<COOP, CG>(v, warp % CG) < cur.w));
      const int r = prow[coop_idx<COOP, CG>(v, warp % CG)];
      DM_CHECK(r >= 0 && (size_t)r < (size_t)P.E * P.N);
      return r;
    };
    const float4 vr4 = vref[e];
    const v3<float> vr = mk3(vr4.x, vr4.y, vr4.z);  // momentum relative to the env's reference velocity
    // perm indices two chunks ahead in two parity slots (no register moves
    // between chunks, so a refill never waits on the load it replaces)
    PState ps;
    if (lane < cnt) load_pstate<LAW>(S, pidx(lane), ps, P.fiso, P.tauv);
    int s1 = 32 + lane < cnt ? pidx(32 + lane) : 0;
    int s0 = 64 + lane < cnt ? pidx(64 + lane) : 0;
    scatter_zero(bw, lane);
    RunAcc ra;
    run_reset(ra);
    auto chunk = [&](int c0, int s_next) __attribute__((always_inline)) -> int {
      if (c0 + lane < cnt) {
        Stencil<float> sc;
        make_stencil(ps.x, P.inv_dx, (double)P.dx, P.dims, sc);
        const Law<float> L = law_of<LAW>(P, attr_mat(ps.at));
        const float av = act ? act[e * P.G + min(attr_group(ps.at), P.G - 1)] : 0.f;
        bool bad = false;
        // fluid with an isotropic F (fiso): a literal-zero diagonal F lets the
        // compiler drop the off-diagonal work (same values: the products with
        // the zeros vanish exactly)
        const m3<float> A = (LAW == kFluid && P.fiso)
                                ? p2g_affine(L, T, mdiag(ps.F.a[0], ps.F.a[0], ps.F.a[0]), ps.C, av, &bad)
                            : (LAW == kElastoplastic && P.tauv) ? p2g_affine_tau(L, T, sym6(ps.F.a), ps.C)
                                                                : p2g_affine(L, T, ps.F, ps.C, av, &bad);
        if (bad) report(flags, e, substep, 0, attr_index(ps.at), attr_mat(ps.at), kErrDetF);
        v3<float> q;
        m3<float> Ad;
        p2g_payload(A, L.mass, ps.v - vr, sc, P.dx, q, Ad);
        const int lbl = (tile_local(sc.base[0], o[0]) * kExt + tile_local(sc.base[1], o[1])) * kExt +
                        tile_local(sc.base[2], o[2]);
        stage_payload(pw + lane * kPay, lbl, sc, L.mass, q, Ad);
      }
      __syncwarp();
      // software pipeline: issue the next chunk's loads before this chunk's scatter
      if (c0 + 32 + lane < cnt) load_pstate<LAW>(S, s_next, ps, P.fiso, P.tauv);
      const int s_new = c0 + 96 + lane < cnt ? pidx(c0 + 96 + lane) : 0;
      scatter_runs<true>(bw, pw, min(32, cnt - c0), lane, ra);
      return s_new;
    };
    chunk_loop<LAW == kFluid || LAW == kNeoHookean>(chunk, cnt, s0, s1);
    if constexpr (COOP) {  // flush, then the CTA sums the 4 warps' copies
      if (lane < 27) run_flush(bw + (lane / 9) * kExt3, ra, (((lane % 9) / 3) * kExt + lane % 3) * kExt);
      coop_store_blocks<CG>(dsm + (warp / CG) * CG * 3 * kExt3, 3 * kExt3, blocks + tix * kExt3);
    } else {
      scatter_store(bw, lane, ra, blocks + tix * kExt3);
    }
  };
  if constexpr (COOP) {
    auto item = [&](const int4 cur, int) __attribute__((always_inline)) { tile(cur); };
    coop_loop<CG>(active, wq, n_active, item);
  } else {
    for (TileIter ti(active, wq, n_active, lane); ti.valid(); ti.advance()) {
      ti.prefetch(active);
      tile(ti.cur);
    }
  }
}

// ---- node ownership ----
// A node is covered by the extended blocks of up to 2 tiles per axis; its
// value is the sum of the covering active tiles' blocks in ascending tile
// order and it is computed (owned) by the first active covering tile.
// nbr: 27-bit activity mask of the 3x3x3 tile neighbourhood (bit = (rx+1)*9 +
// (ry+1)*3 + (rz+1)).
// nbt[bit]: the neighbour's block index e * Tn + tile when active, else -1.
__device__ __forceinline__ unsigned neighbour_mask(const DevParams& P, const int* __restrict__ tile_count, int e,
                                                   const int tc[3], int lane, int* nbt) {
  bool act = false;
  __syncwarp();  // the previous tile's readers are done with nbt
  if (lane < 27) {
    const int sx = tc[0] + lane / 9 - 1, sy = tc[1] + (lane / 3) % 3 - 1, sz = tc[2] + lane % 3 - 1;
    int slot = -1;
    if (sx >= 0 && sx < P.td[0] && sy >= 0 && sy < P.td[1] && sz >= 0 && sz < P.td[2]) {
      const int st = e * P.Tn + (sx * P.td[1] + sy) * P.td[2] + sz;
      act = tile_count[st] > 0;
      slot = act ? st : -1;
    }
    nbt[lane] = slot;
  }
  const unsigned m = __ballot_sync(0xffffffffu, act);
  __syncwarp();
  return m;
}

// candidate range per axis for local coordinate a in [0, 6): rel in [lo, hi]
__device__ __forceinline__ void cand_range(int a, int& lo, int& hi) {
  lo = a < 2 ? -1 : 0;
  hi = a >= 4 ? 1 : 0;
}

// Per local node i of the 6^3 block: `cand` = neighbourhood bits of the tiles
// whose extended block covers it (<= 8, self included), `prior` = the subset
// ordered before self.  Ascending bit order = ascending tile order, so
// iterating the set bits of nbr & cand sums the covering blocks in the fixed
// order, and a tile owns node i iff nbr & prior == 0.  Built once per CTA.
// cl[i][0..nc[i]): the covering tiles of node i in ascending order, packed
// (neighbourhood bit << 8) | (node i's index in that tile's block).
struct NodeMasks {
  unsigned cand[kExt3], prior[kExt3];
  unsigned short cl[kExt3][8];
  unsigned char nc[kExt3];
};

__device__ __forceinline__ void build_node_masks(NodeMasks& m) {
  for (int i = threadIdx.x; i < kExt3; i += blockDim.x) {
    const int l[3] = {i / 36, (i / 6) % 6, i % 6};
    int lo[3], hi[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) cand_range(l[d], lo[d], hi[d]);
    unsigned c = 0u, pr = 0u;
    bool before = true;
    int k = 0;
    for (int rx = lo[0]; rx <= hi[0]; ++rx)
      for (int ry = lo[1]; ry <= hi[1]; ++ry)
        for (int rz = lo[2]; rz <= hi[2]; ++rz) {
          const int code = (rx + 1) * 9 + (ry + 1) * 3 + (rz + 1);
          const unsigned bit = 1u << code;
          if (rx == 0 && ry == 0 && rz == 0) before = false;
          c |= bit;
          if (before) pr |= bit;
          m.cl[i][k++] = (unsigned short)((code << 8) | (((l[0] - 4 * rx) * kExt + (l[1] - 4 * ry)) * kExt + (l[2] - 4 * rz)));
        }
    m.nc[i] = (unsigned char)k;
    m.cand[i] = c;
    m.prior[i] = pr & ~(1u << 13);
  }
  __syncthreads();
}

// Compacted list (ascending) of the tile's owned, in-grid nodes; returns count.
__device__ __forceinline__ int owned_nodes(const DevParams& P, const NodeMasks& nm, unsigned nbr, const int tc[3],
                                           short* list, int lane) {
  __syncwarp();  // previous tile's readers are done with the list
  int n = 0;
  for (int i0 = 0; i0 < kExt3; i0 += 32) {
    const int i = i0 + lane;
    bool ok = false;
    if (i < kExt3) {
      const int g[3] = {tc[0] * kTile + i / 36, tc[1] * kTile + (i / 6) % 6, tc[2] * kTile + i % 6};
      ok = g[0] < P.dims[0] && g[1] < P.dims[1] && g[2] < P.dims[2] && (nbr & nm.prior[i]) == 0u;
    }
    const unsigned b = __ballot_sync(0xffffffffu, ok);
    if (ok) list[n + __popc(b & ((1u << lane) - 1u))] = (short)i;
    n += __popc(b);
  }
  __syncwarp();
  return n;
}

__device__ __forceinline__ float4 sum_blocks(const NodeMasks& nm, const float4* __restrict__ blocks,
                                             const int* __restrict__ nbt, int i) {
  // all (<= 8) covering blocks' loads are issued before the fixed-order sum
  // (ascending tile order = lexicographic (rx, ry, rz), as the cover mask bits)
  const int k = nm.nc[i];
  float4 v[8];
  bool ok[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    ok[c] = false;
    if (c < k) {
      const unsigned cc = nm.cl[i][c];
      const int b = nbt[cc >> 8];
      ok[c] = b >= 0;
      if (ok[c]) v[c] = blocks[(size_t)b * kExt3 + (cc & 255u)];
    }
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (ok[c]) {
      acc.x += v[c].x;
      acc.y += v[c].y;
      acc.z += v[c].z;
      acc.w += v[c].w;
    }
  return acc;
}

__device__ __forceinline__ size_t node_lin(const DevParams& P, int e, const int g[3]) {
  DM_CHECK(e >= 0 && e < P.E && g[0] >= 0 && g[0] < P.dims[0] && g[1] >= 0 && g[1] < P.dims[1] && g[2] >= 0 &&
           g[2] < P.dims[2]);
  return (size_t)e * P.dims[0] * P.dims[1] * P.dims[2] + ((size_t)g[0] * P.dims[1] + g[1]) * P.dims[2] + g[2];
}

// ============================ grid update ============================
// Owned nodes of every active tile: sum the covering blocks, update
// (mpm.hpp:256-305 + extensions), write (mass, momentum) and velocity to the
// dense per-env grid.
template <int MAXC, int CK, bool COOP>
#ifndef DM_GRID_MINB
#define DM_GRID_MINB 5
#endif
__global__ void __launch_bounds__(kWarps * 32, DM_GRID_MINB) k_grid(DevParams P, const int* __restrict__ tile_count,
                                                      const int4* __restrict__ active, const float* __restrict__ cvo,
                                                      const float4* __restrict__ blocks, float4* __restrict__ gmp,
                                                      float4* __restrict__ gv, const int* nact, int* __restrict__ wq,
                                                      const float4* __restrict__ vref) {
  dm_pdl();
  wq_clear_next(wq);
  __shared__ short own[kWarps][kExt3];
  __shared__ NodeMasks nm;
  __shared__ int nbt[kWarps][27];  // the tile's neighbour block indices (neighbour_mask)
  __shared__ Col<float> scol[kWarps][MAXC];
  build_node_masks(nm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_active = *(const volatile int*)nact;
  const NodeCtx<float> G = nctx(P);
  // COOP (small batches): the CTA's 4 warps share a tile's owned nodes (each
  // warp builds the tile's masks itself; node q goes to warp (q / 32) % 4)
  auto tile = [&](const int4 et) __attribute__((always_inline)) {
    const int e = et.x, t = et.y;
    const int tc[3] = {t / (P.td[2] * P.td[1]), (t / P.td[2]) % P.td[1], t % P.td[2]};
    const unsigned nbr = neighbour_mask(P, tile_count, e, tc, lane, nbt[warp]);
    Col<float>* cols = scol[warp];  // the env's colliders, in shared memory (frees registers)
    __syncwarp();
    if (lane == 0) load_cols<MAXC>(P, cvo + (size_t)e * P.K * 9, cols);
    __syncwarp();
    const int n_own = owned_nodes(P, nm, nbr, tc, own[warp], lane);
    const float4 vr4 = vref[e];
    const v3<float> vr = mk3(vr4.x, vr4.y, vr4.z);
    for (int q = COOP ? 32 * warp + lane : lane; q < n_own; q += COOP ? 32 * kWarps : 32) {
      const int i = own[warp][q];
      const int l[3] = {i / 36, (i / 6) % 6, i % 6};
      const int g[3] = {tc[0] * kTile + l[0], tc[1] * kTile + l[1], tc[2] * kTile + l[2]};
      const float4 mm = sum_blocks(nm, blocks, nbt[warp], i);  // (mass, momentum relative to vref)
      const v3<float> v = node_update_rel<float, MAXC, CK>(G, cols, P.K, g, mm.x, mk3(mm.y, mm.z, mm.w), vr);
      const size_t n = node_lin(P, e, g);
      if (gmp) gmp[n] = mm;  // (mass, momentum) only when the replay dumps them
      gv[n] = make_float4(v.x, v.y, v.z, 0.f);
    }
  };
  if constexpr (COOP) {
    auto item = [&](const int4 cur, int) __attribute__((always_inline)) { tile(cur); };
    coop_loop(active, wq, n_active, item);
  } else {
    for (int a = grab_tile(wq, lane), an = a < n_active ? grab_tile(wq, lane) : n_active; a < n_active;
         a = an, an = a < n_active ? grab_tile(wq, lane) : n_active)
      tile(active[a]);
  }
}

// Loads the tile's 6^3 block of a dense grid into shared memory.
__device__ __forceinline__ void load_tile_grid(const DevParams& P, const float4* __restrict__ grid, int e,
                                               const int o[3], float4* dst, int lane) {
  for (int i = lane; i < kExt3; i += 32) {
    const int g[3] = {o[0] + i / 36, o[1] + (i / 6) % 6, o[2] + i % 6};
    dst[i] = (g[0] < P.dims[0] && g[1] < P.dims[1] && g[2] < P.dims[2]) ? grid[node_lin(P, e, g)]
                                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// ============================ G2P ============================
// Tile grids are double-buffered in shared memory with cp.async (the next
// tile's 6^3 velocity block streams in while the current tile computes) and
// the next chunk's particle loads are issued before the current chunk's math.
#ifndef DM_G2P_RING
#define DM_G2P_RING 3
#endif
constexpr int kG2pRing = DM_G2P_RING;  // 3: k_g2p -7 % vs registers one chunk ahead; 4: same at 1,024 envs, +3 % at 128
template <int LAW, bool COOP, int CG>
__global__ void __launch_bounds__(kWarps * 32, kG2pBlocks(LAW)) k_g2p(DevParams P, StateView S, StateView Sout,
                                                     const int* __restrict__ perm, const int* __restrict__ tile_start,
                                                     const int* __restrict__ tile_count, const int4* __restrict__ active,
                                                     const __grid_constant__ CUtensorMap tm_gv, DevFlags* flags, const int* nact,
                                                     int substep, const float4* __restrict__ gmp,
                                                     float4* __restrict__ out_gv, float4* __restrict__ out_gmp, int* __restrict__ wq,
                                                     int dump_cap, const float4* __restrict__ vref) {
  dm_pdl();
  wq_clear_next(wq);
  __shared__ __align__(128) float4 vg[kWarps][2][kExt3];
  __shared__ uint64_t vbar[kWarps][2];  // TMA completion of vg[w][b]
  // fluid, isotropic F: a ring of kG2pRing chunk slots per warp (x, F word,
  // attr: 5 x 32 words each) filled by cp.async kG2pRing - 1 chunks ahead
  __shared__ float gst[LAW == kFluid ? kWarps : 1][kG2pRing][5 * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    mbar_init(&vbar[warp][0]);
    mbar_init(&vbar[warp][1]);
    mbar_init_fence();
  }
  __syncwarp();
  const int n_active = *(const volatile int*)nact;
  const TransferCtx<float> T = tctx(P);
  // one tile (item a) with its grid block landed in vw
  auto tile = [&](const int4 cur, const int a, const float4* vw) __attribute__((always_inline)) {
    const int e = cur.x, t = cur.y, start = cur.z;
    const int cnt = coop_count<COOP, CG>(cur.w, warp % CG);  // this warp's (virtual) particle count
    const int tc[3] = {t / (P.td[2] * P.td[1]), (t / P.td[2]) % P.td[1], t % P.td[2]};
    const int o[3] = {tc[0] * kTile, tc[1] * kTile, tc[2] * kTile};
    const size_t row = (size_t)e * P.N + start;
    auto pidx = [&](int v) {
      DM_CHECK((coop_idx<COOP, CG>(v, warp % CG) < cur.w));
      const int r = perm[row + coop_idx<COOP, CG>(v, warp % CG)];
      DM_CHECK(r >= 0 && (size_t)r < (size_t)P.E * P.N);
      return r;
    };
    const float4 vr4 = vref[e];
    const v3<float> vr = mk3(vr4.x, vr4.y, vr4.z);
    auto dump = [&]() __attribute__((always_inline)) {
      if (out_gv && a < dump_cap && (!COOP || warp % CG == 0)) {  // segment replay: keep the tile's grid for the adjoint
        if (lane == 0) bulk_s2g(out_gv + (size_t)a * kExt3, vw, kExt3 * (uint32_t)sizeof(float4));
        load_tile_grid(P, gmp, e, o, out_gmp + (size_t)a * kExt3, lane);
      }
    };
    auto body = [&](int c0, const float x[3], m3<float> F, uint32_t at) {
      if (c0 + lane >= cnt) return;
      const size_t dst = row + coop_idx<COOP, CG>(c0 + lane, warp % CG);
      Stencil<float> sc;
      make_stencil(x, P.inv_dx, (double)P.dx, P.dims, sc);
      const int lb[3] = {tile_local(sc.base[0], o[0]), tile_local(sc.base[1], o[1]), tile_local(sc.base[2], o[2])};
      auto getv = [&](int i, int j, int k) {
        const float4 q = vw[((lb[0] + i) * kExt + (lb[1] + j)) * kExt + lb[2] + k];
        return mk3(q.x, q.y, q.z);
      };
      v3<float> xn = mk3(x[0], x[1], x[2]), v;
      m3<float> C;
      bool bad_adv = false, bad_det = false;
      m3<float> tau;
      g2p_particle_sep(law_of<LAW>(P, attr_mat(at)), T, sc, getv, xn, v, C, F, &bad_adv, &bad_det, vr,
                       LAW == kElastoplastic && Sout.tau ? &tau : nullptr);
      if (bad_adv) report(flags, e, substep, 1, attr_index(at), 0, kErrG2PInterior);
      if (bad_det) report(flags, e, substep, 1, attr_index(at), attr_mat(at), kErrDetF);
      store_state<LAW>(Sout, dst, xn, v, F, C);
      if (LAW == kElastoplastic && Sout.tau) {  // the next P2G's stress (SURVEY 8 "stress source")
        Sout.t(0, dst) = tau.a[0];
        Sout.t(1, dst) = tau.a[1];
        Sout.t(2, dst) = tau.a[2];
        Sout.t(3, dst) = tau.a[4];
        Sout.t(4, dst) = tau.a[5];
        Sout.t(5, dst) = tau.a[8];
      }
      Sout.attr[dst] = at;
    };
    if (LAW == kFluid && P.fiso) {
      // staged: chunk k + kG2pRing - 1's loads are issued (perm index one
      // chunk earlier) before chunk k computes -- no state registers held
      float* ring = &gst[LAW == kFluid ? warp : 0][0][0];
      auto issue = [&](int c0, int src, int slot) __attribute__((always_inline)) {
        if (c0 + lane < cnt) {
          float* d = ring + slot * 160 + lane;
          cp_async4(d, &S.c(0, src));
          cp_async4(d + 32, &S.c(1, src));
          cp_async4(d + 64, &S.c(2, src));
          cp_async4(d + 96, &S.c(6, src));
          cp_async4(d + 128, S.attr + src);
        }
        cp_async_commit();
      };
#pragma unroll
      for (int r = 0; r < kG2pRing - 1; ++r) issue(32 * r, 32 * r + lane < cnt ? pidx(32 * r + lane) : 0, r);
      int pn = 32 * (kG2pRing - 1) + lane < cnt ? pidx(32 * (kG2pRing - 1) + lane) : 0;
      dump();
      for (int c0 = 0, slot = 0, nslot = kG2pRing - 1; c0 < cnt; c0 += 32) {
        issue(c0 + 32 * (kG2pRing - 1), pn, nslot);
        pn = c0 + 32 * kG2pRing + lane < cnt ? pidx(c0 + 32 * kG2pRing + lane) : 0;
        cp_async_wait<kG2pRing - 1>();  // chunk c0 has landed
        __syncwarp();
        const float* sl = ring + slot * 160 + lane;
        const float x[3] = {sl[0], sl[32], sl[64]};
        const float f0 = sl[96];
        body(c0, x, mdiag(f0, f0, f0), __float_as_uint(sl[128]));
        __syncwarp();  // slot is refilled kG2pRing - 1 chunks later
        slot = slot == kG2pRing - 1 ? 0 : slot + 1;
        nslot = nslot == kG2pRing - 1 ? 0 : nslot + 1;
      }
      cp_async_wait<0>();
      __syncwarp();  // every lane is done with vw before it is refilled
      return;
    }
    // two particle-state buffers (chunks alternate) and perm indices two
    // chunks ahead in parity slots: no register moves between chunks
    float xa[3], xb[3];
    m3<float> Fa, Fb;
    uint32_t ata = 0, atb = 0;
    if (lane < cnt) {
      const int src = pidx(lane);
      load_xF<LAW>(S, src, xa, Fa, P.fiso);
      ata = S.attr[src];
    }
    int s1 = lane + 32 < cnt ? pidx(lane + 32) : 0;
    int s0 = lane + 64 < cnt ? pidx(lane + 64) : 0;
    dump();
    for (int c0 = 0; c0 < cnt; c0 += 64) {
      if (c0 + 32 + lane < cnt) {  // chunk c0 + 32 -> buffer b
        load_xF<LAW>(S, s1, xb, Fb, P.fiso);
        atb = S.attr[s1];
      }
      s1 = c0 + 96 + lane < cnt ? pidx(c0 + 96 + lane) : 0;
      body(c0, xa, Fa, ata);
      if (c0 + 32 >= cnt) break;
      if (c0 + 64 + lane < cnt) {  // chunk c0 + 64 -> buffer a
        load_xF<LAW>(S, s0, xa, Fa, P.fiso);
        ata = S.attr[s0];
      }
      s0 = c0 + 128 + lane < cnt ? pidx(c0 + 128 + lane) : 0;
      body(c0 + 32, xb, Fb, atb);
    }
    __syncwarp();  // every lane is done with vw before it is refilled
  };
  // tile grids arrive by TMA; lane 0 (thread 0 in COOP) issues, after its
  // bulk dump stores of the buffer's previous tile have read it
  uint32_t ph = 0;
  if constexpr (COOP) {
    const int gw = warp - warp % CG;  // the group's first warp: its buffer holds the group's tile grid
    auto item = [&](const int4 cur, int a) __attribute__((always_inline)) {
      if (warp == gw && lane == 0) {  // one copy of the tile's grid for the group
        bulk_s2g_read_wait();
        fence_proxy_async();
        tma_tile_grid(P, &tm_gv, cur, vg[gw][0], &vbar[gw][0]);
      }
      mbar_wait(&vbar[gw][0], ph);
      ph ^= 1;
      tile(cur, a, vg[gw][0]);
    };
    coop_loop<CG>(active, wq, n_active, item);
  } else {
    TileIter ti(active, wq, n_active, lane);
    if (ti.valid() && lane == 0) tma_tile_grid(P, &tm_gv, ti.cur, vg[warp][0], &vbar[warp][0]);
    for (int buf = 0; ti.valid(); ti.advance(), buf ^= 1) {
      if (ti.has_next() && lane == 0) {  // the next tile's grid streams in during this tile
        bulk_s2g_read_wait();
        fence_proxy_async();
        tma_tile_grid(P, &tm_gv, ti.nxt, vg[warp][buf ^ 1], &vbar[warp][buf ^ 1]);
      }
      ti.prefetch(active);
      mbar_wait(&vbar[warp][buf], (ph >> buf) & 1);
      ph ^= 1u << buf;
      tile(ti.cur, ti.a, vg[warp][buf]);
    }
  }
  if (lane == 0) bulk_s2g_read_wait();  // shared memory outlives the dump stores' reads
}

// ============================ G2P adjoint ============================
// Reads the start-of-substep state (via perm) and the cotangent of the
// end-of-substep state (sorted position); writes particle-side partial
// cotangents (sorted position) and a 6^3 block of node-velocity cotangents.
// The next chunk's gathered (x, F) loads are in flight during the current
// chunk's scatter.
#ifndef DM_G2PADJ_MINB
#define DM_G2PADJ_MINB 3
#endif
template <int LAW, int NM, bool COOP, int CG>
__global__ void __launch_bounds__(kWarps * 32, DM_G2PADJ_MINB) k_g2p_adj(DevParams P, StateView S, StateView Sn, const float* __restrict__ adj_in,
                                                         size_t astride, const int* __restrict__ perm,
                                                         const int* __restrict__ tile_start,
                                                         const int* __restrict__ tile_count,
                                                         const int4* __restrict__ active, const float4* __restrict__ gvb,
                                                         float4* __restrict__ ablocks, float* __restrict__ part,
                                                         float* __restrict__ tile_acc, const int* nact, int* __restrict__ wq,
                                                         const float4* __restrict__ vref) {
  dm_pdl();
  wq_clear_next(wq);
  extern __shared__ __align__(128) float4 dsm[];
  __shared__ uint64_t vbar[kWarps];  // COOP: bulk-copy completion of the warp's vw
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (COOP && lane == 0) {
    mbar_init(&vbar[warp]);
    mbar_init_fence();
  }
  __syncwarp();
  uint32_t ph = 0;
  const TransferCtx<float> T = tctx(P);
  float4* vw = dsm + warp * 4 * kExt3;  // the tile's node velocities
  float4* aw = vw + kExt3;              // 3 group copies of the cotangent block
  float* pw = reinterpret_cast<float*>(dsm + kWarps * 4 * kExt3) + warp * 32 * kPay;
  const int n_active = *(const volatile int*)nact;
  auto tile = [&](const int4 cur, const int a) __attribute__((always_inline)) {
    const int e = cur.x, t = cur.y, start = cur.z;
    const int cnt = coop_count<COOP, CG>(cur.w, warp % CG);  // this warp's (virtual) particle count
    const int tc[3] = {t / (P.td[2] * P.td[1]), (t / P.td[2]) % P.td[1], t % P.td[2]};
    const int o[3] = {tc[0] * kTile, tc[1] * kTile, tc[2] * kTile};
    // the replayed substep's grid, by slot (asynchronous; overlaps the first loads)
    // the replayed substep's grid, by slot (asynchronous; overlaps the first
    // loads): one bulk copy (UBLKCP) in COOP mode, per-lane LDGSTS otherwise
    // (r02 A/B: the bulk copy is 7 % faster with CTA-shared tiles, 2.5 %
    // slower with one tile per warp)
    if constexpr (COOP) {
      if (lane == 0) {  // the previous tile's readers passed its closing __syncwarp
        fence_proxy_async();
        bulk_g2s(vw, gvb + (size_t)a * kExt3, kExt3 * (uint32_t)sizeof(float4), &vbar[warp]);
      }
    } else {
      for (int i = lane; i < kExt3; i += 32) cp_async16(vw + i, gvb + (size_t)a * kExt3 + i, true);
      cp_async_commit();
    }
    const size_t tix = (size_t)e * P.Tn + t;
    const size_t row = (size_t)e * P.N + start;
    auto pidx = [&](int v) {
      DM_CHECK((coop_idx<COOP, CG>(v, warp % CG) < cur.w));
      const int r = perm[row + coop_idx<COOP, CG>(v, warp % CG)];
      DM_CHECK(r >= 0 && (size_t)r < (size_t)P.E * P.N);
      return r;
    };
    const float4 vr4 = vref[e];
    float x[3];
    m3<float> F;
    uint32_t at = 0;
    if (lane < cnt) {
      const int src = pidx(lane);
      load_xF<LAW>(S, src, x, F, P.fiso);
      at = S.attr[src];
    }
    int s1 = 32 + lane < cnt ? pidx(32 + lane) : 0;  // perm two chunks ahead, parity slots
    int s0 = 64 + lane < cnt ? pidx(64 + lane) : 0;
    scatter_zero(aw, lane);
    double mub[NM];  // fp64: cancelling per-particle sums (NM = materials)
#pragma unroll
    for (int m = 0; m < NM; ++m) mub[m] = 0.0;
    RunAcc ra;
    run_reset(ra);
    if constexpr (COOP) {
      mbar_wait(&vbar[warp], ph);
      ph ^= 1;
    } else {
      cp_async_wait<0>();
      __syncwarp();
    }
    auto chunk = [&](int c0, int s_next) __attribute__((always_inline)) -> int {
      if (c0 + lane < cnt) {
        const size_t dst = row + coop_idx<COOP, CG>(c0 + lane, warp % CG);
        Stencil<float> sc;
        make_stencil(x, P.inv_dx, (double)P.dx, P.dims, sc);
        const int lb[3] = {tile_local(sc.base[0], o[0]), tile_local(sc.base[1], o[1]), tile_local(sc.base[2], o[2])};
        auto getv = [&](int i, int j, int k) {  // node velocity relative to vref (g2p_vjp_given adds vref's part)
          const float4 q = vw[((lb[0] + i) * kExt + (lb[1] + j)) * kExt + lb[2] + k];
          return mk3(q.x, q.y, q.z);
        };
        v3<float> xb = mk3(adj_in[adj_index(0, dst, astride)], adj_in[adj_index(1, dst, astride)], adj_in[adj_index(2, dst, astride)]);
        v3<float> vb = mk3(adj_in[adj_index(3, dst, astride)], adj_in[adj_index(4, dst, astride)], adj_in[adj_index(5, dst, astride)]);
        m3<float> Fb, Cb;
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          // fluid: the cotangent of the (isotropic) next state's F is kept as its trace (kFluidTraceCot)
          Fb.a[q] = LAW == kFluid ? (q == 0 ? adj_in[adj_index(6, dst, astride)] : 0.f)
                                  : adj_in[adj_index(6 + q, dst, astride)];
          Cb.a[q] = adj_in[adj_index(15 + q, dst, astride)];
        }
        v3<float> xp, gq;
        m3<float> Fp, Bd;
        const int mi = attr_mat(at);
        float mu_l = 0.f;
        // the replay's G2P outputs for this particle: the next state at the same sorted slot
        const v3<float> vn = mk3(Sn.c(3, dst), Sn.c(4, dst), Sn.c(5, dst));
        m3<float> Cn;
#pragma unroll
        for (int q = 0; q < 9; ++q) Cn.a[q] = Sn.c(15 + q, dst);
        if (LAW == kFluid && P.fiso)  // literal-zero diagonal F (see k_p2g)
          g2p_vjp_given(law_of<LAW>(P, mi), T, sc, getv, mdiag(1.f + F.a[0], 1.f + F.a[0], 1.f + F.a[0]), vn, Cn, xb,
                        vb, Cb, Fb, xp, Fp, gq, Bd, mu_l, mk3(vr4.x, vr4.y, vr4.z));
        else  // the adjoint linearises at F = I + D (fp32)
          g2p_vjp_given(law_of<LAW>(P, mi), T, sc, getv, eye_plus(F), vn, Cn, xb, vb, Cb, Fb, xp, Fp, gq, Bd, mu_l,
                        mk3(vr4.x, vr4.y, vr4.z));
#pragma unroll
        for (int m = 0; m < NM; ++m)
          if (m == mi) mub[m] += mu_l;
        part[part_index(0, dst, astride)] = xp.x;
        part[part_index(1, dst, astride)] = xp.y;
        part[part_index(2, dst, astride)] = xp.z;
        if (LAW == kFluid && P.fiso)  // isotropic input F: its cotangent matters only through the trace
          part[part_index(3, dst, astride)] = Fp.a[0] + Fp.a[4] + Fp.a[8];
        else
#pragma unroll
          for (int q = 0; q < 9; ++q) part[part_index(3 + q, dst, astride)] = Fp.a[q];
        stage_payload(pw + lane * kPay, (lb[0] * kExt + lb[1]) * kExt + lb[2], sc, 0.f, gq, Bd);
      }
      __syncwarp();
      if (c0 + 32 + lane < cnt) {
        load_xF<LAW>(S, s_next, x, F, P.fiso);
        at = S.attr[s_next];
      }
      const int s_new = c0 + 96 + lane < cnt ? pidx(c0 + 96 + lane) : 0;
      scatter_runs<false>(aw, pw, min(32, cnt - c0), lane, ra);
      return s_new;
    };
    chunk_loop<LAW == kFluid>(chunk, cnt, s0, s1);
    if constexpr (COOP) {
      if (lane < 27) run_flush(aw + (lane / 9) * kExt3, ra, (((lane % 9) / 3) * kExt + lane % 3) * kExt);
      coop_store_blocks<CG>(dsm + kExt3 + (warp - warp % CG) * 4 * kExt3, 4 * kExt3, ablocks + tix * kExt3);
    } else {
      scatter_store(aw, lane, ra, ablocks + tix * kExt3);
    }
#pragma unroll
    for (int m = 0; m < NM; ++m)
      for (int off = 16; off > 0; off >>= 1) mub[m] += __shfl_xor_sync(0xffffffffu, mub[m], off);
    if constexpr (COOP) {
#pragma unroll
      for (int m = 0; m < NM; ++m) mub[m] = coop_sum<CG>(mub[m]);
      if (warp % CG == 0 && lane == 0)
#pragma unroll
        for (int m = 0; m < NM; ++m) tile_acc[tix * kNacc + kAccMuG + m] = (float)mub[m];
    } else {
      if (lane == 0)
#pragma unroll
        for (int m = 0; m < NM; ++m) tile_acc[tix * kNacc + kAccMuG + m] = (float)mub[m];
    }
    __syncwarp();
  };
  if constexpr (COOP) {
    coop_loop<CG>(active, wq, n_active, tile);
  } else {
    for (TileIter ti(active, wq, n_active, lane); ti.valid(); ti.advance()) {
      ti.prefetch(active);
      tile(ti.cur, ti.a);
    }
  }
}

// ============================ grid adjoint ============================
// Owned nodes: node-velocity cotangent (sum of the covering adjoint blocks)
// -> (mass, momentum) cotangents in the dense grid; collider cotangents
// reduced per tile (each node counted once, by its owner).
template <int MAXC, int CK, bool COOP>
#ifndef DM_GRIDADJ_MINB
#define DM_GRIDADJ_MINB 5  // r02: 96 B of spills but -8 % on cfg4 (the hollow-box query record), -1 % cfg3, +6 % cfg2
#endif
__global__ void __launch_bounds__(kWarps * 32, DM_GRIDADJ_MINB) k_grid_adj(DevParams P, const int* __restrict__ tile_count,
                                                          const int4* __restrict__ active, const float* __restrict__ cvo,
                                                          const float4* __restrict__ ablocks,
                                                          const float4* __restrict__ gmpb, float4* __restrict__ gmb,
                                                          float* __restrict__ tile_acc, const int* nact, int* __restrict__ wq,
                                                          const float4* __restrict__ vref) {
  dm_pdl();
  wq_clear_next(wq);
  __shared__ short own[kWarps][kExt3];
  __shared__ NodeMasks nm;
  __shared__ int nbt[kWarps][27];  // the tile's neighbour block indices (neighbour_mask)
  __shared__ Col<float> scol[kWarps][MAXC];
  build_node_masks(nm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_active = *(const volatile int*)nact;
  const NodeCtx<float> G = nctx(P);
  __shared__ float cred[kWarps][MAXC * 9];  // COOP: the warps' collider cotangents, summed in warp order
  auto tile = [&](const int4 et, const int a) __attribute__((always_inline)) {
    const int e = et.x, t = et.y;
    const int tc[3] = {t / (P.td[2] * P.td[1]), (t / P.td[2]) % P.td[1], t % P.td[2]};
    const unsigned nbr = neighbour_mask(P, tile_count, e, tc, lane, nbt[warp]);
    Col<float>* cols = scol[warp];  // the env's colliders, in shared memory (frees registers)
    __syncwarp();
    if (lane == 0) load_cols<MAXC>(P, cvo + (size_t)e * P.K * 9, cols);
    __syncwarp();
    float cg[MAXC * 9];
#pragma unroll
    for (int q = 0; q < MAXC * 9; ++q) cg[q] = 0.f;
    const int n_own = owned_nodes(P, nm, nbr, tc, own[warp], lane);
    for (int q = COOP ? 32 * warp + lane : lane; q < n_own; q += COOP ? 32 * kWarps : 32) {
      const int i = own[warp][q];
      const int l[3] = {i / 36, (i / 6) % 6, i % 6};
      const int g[3] = {tc[0] * kTile + l[0], tc[1] * kTile + l[1], tc[2] * kTile + l[2]};
      const float4 vb = sum_blocks(nm, ablocks, nbt[warp], i);
      const size_t n = node_lin(P, e, g);
      float4 mm = gmpb[(size_t)a * kExt3 + i];  // this tile's stored (mass, momentum relative to vref) block
      {  // the adjoint linearises in the lab frame: momentum + mass vref
        const float4 vr4 = vref[e];
        mm.y += mm.x * vr4.x;
        mm.z += mm.x * vr4.y;
        mm.w += mm.x * vr4.z;
      }
      float mbar;
      v3<float> pbar;
      // adjoint blocks carry (unused, vbar.x, vbar.y, vbar.z) -- emit_contrib layout
      node_update_vjp<float, MAXC, CK>(G, cols, P.K, g, mm.x, mk3(mm.y, mm.z, mm.w), mk3(vb.y, vb.z, vb.w), mbar, pbar,
                                   cg);
      gmb[n] = make_float4(mbar, pbar.x, pbar.y, pbar.z);
    }
#pragma unroll
    for (int q = 0; q < MAXC * 9; ++q)
      for (int off = 16; off > 0; off >>= 1) cg[q] += __shfl_xor_sync(0xffffffffu, cg[q], off);
    float* ta = tile_acc + ((size_t)e * P.Tn + t) * kNacc;
    if constexpr (COOP) {
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < MAXC * 9; ++q) cred[warp][q] = cg[q];
      __syncthreads();
      if (threadIdx.x < MAXC * 9) {
        float acc = cred[0][threadIdx.x];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) acc += cred[w][threadIdx.x];
        ta[kAccCol + threadIdx.x] = acc;
      }
    } else {
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < MAXC * 9; ++q) ta[kAccCol + q] = cg[q];
    }
    __syncwarp();
  };
  if constexpr (COOP) {
    coop_loop(active, wq, n_active, tile);
  } else {
    for (int a = grab_tile(wq, lane), an = a < n_active ? grab_tile(wq, lane) : n_active; a < n_active;
         a = an, an = a < n_active ? grab_tile(wq, lane) : n_active)
      tile(active[a], a);
  }
}

// ============================ P2G adjoint ============================
// Per tile: the (mass, momentum) cotangent block and chunk 0 stream in with
// cp.async; each chunk's particle data is staged in shared memory by cp.async
// while the previous chunk computes (no registers held for the prefetch).
constexpr int kP2gAdjStage = 38;  // staged words per particle: state 24, attr, part 12, perm index
#ifndef DM_P2GADJ_MINB
#define DM_P2GADJ_MINB 3
#endif
template <int LAW, int NG, int NM, bool COOP, int CG>
__global__ void __launch_bounds__(kWarps * 32, DM_P2GADJ_MINB) k_p2g_adj(DevParams P, StateView S, const int* __restrict__ perm,
                                                         const int* __restrict__ tile_start,
                                                         const int* __restrict__ tile_count,
                                                         const int4* __restrict__ active, const float* __restrict__ act,
                                                         const float4* __restrict__ gmb, const __grid_constant__ CUtensorMap tm_gmb,
                                                         const float* __restrict__ part,
                                                         float* __restrict__ adj_out, size_t astride,
                                                         float* __restrict__ tile_acc, const int* nact, int* __restrict__ wq) {
  dm_pdl();
  wq_clear_next(wq);
  __shared__ __align__(128) float4 mb[kWarps][kExt3];
  __shared__ uint64_t mbar[kWarps];  // COOP: TMA completion of mb[w]
  __shared__ float stg[kWarps][kP2gAdjStage * 32];  // next chunk: [field][lane]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TransferCtx<float> T = tctx(P);
  const int n_active = *(const volatile int*)nact;
  if (COOP && lane == 0) {
    mbar_init(&mbar[warp]);
    mbar_init_fence();
  }
  __syncwarp();
  uint32_t ph = 0;
  float* sg = stg[warp];
  // The tile's (mass, momentum) cotangent block: a TMA box load in COOP mode
  // (r02 A/B: -6 % with CTA-shared tiles), per-lane LDGSTS in the staging
  // group otherwise (a TMA load, single or double-buffered, was 1.5-3 % slower
  // with one tile per warp).
  float4* bw = mb[warp];
  auto tile = [&](const int4 cur) __attribute__((always_inline)) {
    const int e = cur.x, t = cur.y, start = cur.z;
    const int cnt = coop_count<COOP, CG>(cur.w, warp % CG);  // this warp's (virtual) particle count
    const int tc[3] = {t / (P.td[2] * P.td[1]), (t / P.td[2]) % P.td[1], t % P.td[2]};
    const int o[3] = {tc[0] * kTile, tc[1] * kTile, tc[2] * kTile};
    const size_t tix = (size_t)e * P.Tn + t;
    const size_t row = (size_t)e * P.N + start;
    auto pidx = [&](int v) {
      DM_CHECK((coop_idx<COOP, CG>(v, warp % CG) < cur.w));
      const int r = perm[row + coop_idx<COOP, CG>(v, warp % CG)];
      DM_CHECK(r >= 0 && (size_t)r < (size_t)P.E * P.N);
      return r;
    };
    double mub[NM], lab[NM];  // fp64: cancelling sums (NM = materials)
#pragma unroll
    for (int m = 0; m < NM; ++m) mub[m] = lab[m] = 0.0;
    float actb[NG];
#pragma unroll
    for (int q = 0; q < NG; ++q) actb[q] = 0.f;
    // cp.async staging of one chunk's particle data (state + attr via perm,
    // particle-side cotangents at the sorted slot, and the perm index itself)
    auto stage = [&](int c0, int src) {
#pragma unroll
      for (int f = 0; f < 24; ++f)
        if (!(LAW == kFluid && P.fiso && f > 6 && f < 15)) cp_async4(sg + f * 32 + lane, &S.c(f, src));
      cp_async4(sg + 24 * 32 + lane, S.attr + src);
#pragma unroll
      for (int f = 0; f < 12; ++f)
        if (!(LAW == kFluid && P.fiso && f > 3)) cp_async4(sg + (25 + f) * 32 + lane, part + part_index(f, row + coop_idx<COOP, CG>(c0 + lane, warp % CG), astride));
      sg[37 * 32 + lane] = __int_as_float(src);
    };
    int s1 = 32 + lane < cnt ? pidx(32 + lane) : 0;  // perm two chunks ahead, parity slots
    int s0 = lane < cnt ? pidx(lane) : 0;
    __syncwarp();  // previous tile's readers are done with bw and sg
    if constexpr (COOP) {
      if (lane == 0) {
        fence_proxy_async();
        tma_tile_grid(P, &tm_gmb, cur, bw, &mbar[warp]);
      }
    } else {
      prefetch_tile_grid(P, gmb, cur, bw, lane);
    }
    if (lane < cnt) stage(0, s0);
    cp_async_commit();
    s0 = 64 + lane < cnt ? pidx(64 + lane) : 0;
    if constexpr (COOP) {  // the cotangent block has landed
      mbar_wait(&mbar[warp], ph);
      ph ^= 1;
    }
    for (int c0 = 0, k = 0; c0 < cnt; c0 += 32, ++k) {
      cp_async_wait<0>();
      __syncwarp();
      const bool ok = c0 + lane < cnt;
      float x[3];
      v3<float> v, xb;
      m3<float> F, C, Fb;
      uint32_t at = 0;
      int src = 0;
      if (ok) {
#pragma unroll
        for (int a = 0; a < 3; ++a) x[a] = sg[a * 32 + lane];
        v = mk3(sg[3 * 32 + lane], sg[4 * 32 + lane], sg[5 * 32 + lane]);
#pragma unroll
        for (int q = 0; q < 9; ++q) {
          F.a[q] = sg[(6 + q) * 32 + lane];
          C.a[q] = sg[(15 + q) * 32 + lane];
          Fb.a[q] = (LAW == kFluid && P.fiso) ? (q == 0 ? sg[28 * 32 + lane] : 0.f) : sg[(28 + q) * 32 + lane];
        }
        // the stored deviation D -> F = I + D (fp32; the adjoint's linearisation point)
        F = (LAW == kFluid && P.fiso) ? mdiag(1.f + F.a[0], 1.f + F.a[0], 1.f + F.a[0]) : eye_plus(F);
        at = __float_as_uint(sg[24 * 32 + lane]);
        xb = mk3(sg[25 * 32 + lane], sg[26 * 32 + lane], sg[27 * 32 + lane]);
        src = __float_as_int(sg[37 * 32 + lane]);
      }
      __syncwarp();  // every lane has its chunk in registers: refill the staging buffer
      // chunk k + 1's index sits in parity slot (k + 1) & 1; refill it with chunk k + 3's
      const bool odd = k & 1;
      if (c0 + 32 + lane < cnt) stage(c0 + 32, odd ? s0 : s1);
      cp_async_commit();
      const int s_new = c0 + 96 + lane < cnt ? pidx(c0 + 96 + lane) : 0;
      s0 = odd ? s_new : s0;
      s1 = odd ? s1 : s_new;
      if (!ok) continue;
      Stencil<float> sc;
      make_stencil(x, P.inv_dx, (double)P.dx, P.dims, sc);
      const int lb[3] = {tile_local(sc.base[0], o[0]), tile_local(sc.base[1], o[1]), tile_local(sc.base[2], o[2])};
      auto getmb = [&](int i, int jj, int k, float& m_, v3<float>& p_) {
        const float4 q = bw[((lb[0] + i) * kExt + (lb[1] + jj)) * kExt + lb[2] + k];
        m_ = q.x;
        p_ = mk3(q.y, q.z, q.w);
      };
      m3<float> Cb = mzero<float>();
      v3<float> vb = zero3<float>();
      const int mi = attr_mat(at), gi = min(attr_group(at), P.G > 0 ? P.G - 1 : 0);
      const float av = act ? act[e * P.G + gi] : 0.f;
      float mu_l = 0.f, la_l = 0.f, ac_l = 0.f;
      if (LAW == kFluid && P.fiso)  // literal-zero diagonal F (see k_p2g)
        p2g_vjp_sep(law_of<LAW>(P, mi), T, sc, getmb, v, mdiag(F.a[0], F.a[0], F.a[0]), C, av, xb, vb, Fb, Cb, mu_l,
                    la_l, ac_l);
      else
        p2g_vjp_sep(law_of<LAW>(P, mi), T, sc, getmb, v, F, C, av, xb, vb, Fb, Cb, mu_l, la_l, ac_l);
#pragma unroll
      for (int m = 0; m < NM; ++m)
        if (m == mi) {
          mub[m] += mu_l;
          lab[m] += la_l;
        }
#pragma unroll
      for (int q = 0; q < NG; ++q)
        if (q == gi) actb[q] += ac_l;
      adj_out[adj_index(0, src, astride)] = xb.x;
      adj_out[adj_index(1, src, astride)] = xb.y;
      adj_out[adj_index(2, src, astride)] = xb.z;
      adj_out[adj_index(3, src, astride)] = vb.x;
      adj_out[adj_index(4, src, astride)] = vb.y;
      adj_out[adj_index(5, src, astride)] = vb.z;
      if (LAW == kFluid && P.fiso)  // the trace of an isotropic state's F cotangent (kFluidTraceCot)
        adj_out[adj_index(6, src, astride)] = Fb.a[0] + Fb.a[4] + Fb.a[8];
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        if (!(LAW == kFluid && P.fiso)) adj_out[adj_index(6 + q, src, astride)] = Fb.a[q];
        adj_out[adj_index(15 + q, src, astride)] = Cb.a[q];
      }
    }
#pragma unroll
    for (int m = 0; m < NM; ++m)
      for (int off = 16; off > 0; off >>= 1) {
        mub[m] += __shfl_xor_sync(0xffffffffu, mub[m], off);
        lab[m] += __shfl_xor_sync(0xffffffffu, lab[m], off);
      }
#pragma unroll
    for (int q = 0; q < NG; ++q)
      for (int off = 16; off > 0; off >>= 1) actb[q] += __shfl_xor_sync(0xffffffffu, actb[q], off);
    if constexpr (COOP) {  // fixed-order sum of the 4 warps' partials
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        mub[m] = coop_sum<CG>(mub[m]);
        lab[m] = coop_sum<CG>(lab[m]);
      }
#pragma unroll
      for (int q = 0; q < NG; ++q) actb[q] = coop_sum<CG>(actb[q]);
    }
    if (COOP ? (warp % CG == 0 && lane == 0) : lane == 0) {
      float* ta = tile_acc + tix * kNacc;
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        ta[kAccMu + m] = (float)mub[m];
        ta[kAccLam + m] = (float)lab[m];
      }
#pragma unroll
      for (int q = 0; q < NG; ++q) ta[kAccAct + q] = actb[q];
    }
  };
  if constexpr (COOP) {
    auto item = [&](const int4 cur, int) __attribute__((always_inline)) {
      tile(cur);
      cp_async_wait<0>();  // no staging copy outlives the item
    };
    coop_loop<CG>(active, wq, n_active, item);
  } else {
    for (TileIter ti(active, wq, n_active, lane); ti.valid(); ti.advance()) {
      ti.prefetch(active);
      tile(ti.cur);
    }
  }
  cp_async_wait<0>();
}

// Per env: sum the env's tile accumulators into the step's (double)
// parameter cotangents.  kRedSlices contiguous slices of the env's tile list
// are summed in tile order (4 loads in flight per thread), then the slices in
// slice order: a fixed order, independent of the schedule.
constexpr int kRedSlices = 4;
__global__ void __launch_bounds__(kNacc * kRedSlices) k_env_reduce(DevParams P, const int4* __restrict__ active, const int* __restrict__ env_abase,
                             const int* __restrict__ env_acount, const float* __restrict__ tile_acc,
                             double* __restrict__ gcvo_t, double* __restrict__ gact_t, double* __restrict__ gmu,
                             double* __restrict__ glam) {
  dm_pdl();
  __shared__ double part[kRedSlices][kNacc];
  __shared__ double sacc[kNacc];
  const int e = blockIdx.x, f = threadIdx.x % kNacc, g = threadIdx.x / kNacc;
  const int b = env_abase[e], n = env_acount[e];
  const int i0 = b + (int)((long long)n * g / kRedSlices), i1 = b + (int)((long long)n * (g + 1) / kRedSlices);
  auto acc_of = [&](int i) {
    const int4 et = active[i];
    return tile_acc[((size_t)et.x * P.Tn + et.y) * kNacc + f];
  };
  double s = 0.0;
  int i = i0;
  for (; i + 4 <= i1; i += 4) {
    const float a0 = acc_of(i), a1 = acc_of(i + 1), a2 = acc_of(i + 2), a3 = acc_of(i + 3);
    s += a0;
    s += a1;
    s += a2;
    s += a3;
  }
  for (; i < i1; ++i) s += acc_of(i);
  part[g][f] = s;
  __syncthreads();
  if (g != 0) return;
  s = part[0][f];
#pragma unroll
  for (int q = 1; q < kRedSlices; ++q) s += part[q][f];
  sacc[f] = s;
  asm volatile("bar.sync 1, %0;\n" ::"n"(kNacc) : "memory");  // slice 0's threads (2 whole warps) only
  // dL/dmu has two sources (P2G-adjoint stress term f, G2P-adjoint yield
  // term f + 8): one thread adds both, in that fixed order
  if (f < 4) {
    if (f < P.nmat) gmu[e * 4 + f] += s + sacc[f + 8];
  } else if (f < 8) {
    if (f - 4 < P.nmat) glam[e * 4 + f - 4] += s;
  } else if (f < 12) {
    // added by thread f - 8
  } else if (f < 48) {
    const int q = f - 12;
    if (q < P.K * 9) gcvo_t[(size_t)e * P.K * 9 + q] += s;
  } else {
    const int q = f - 48;
    if (q < P.G) gact_t[(size_t)e * P.G + q] += s;
  }
}

// ============================ observables ============================
__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) r += sh[w];
  return r;
}

// Per env observables after a control step: com(3), var(3), spill(1)
// (tasks.hpp:286-304, 604-615) followed, when ngr > 0, by pooled statistics of
// each actuation group g (config 5's 64-d observation): mean x (3), mean v (3),
// var z (1), mean |v| (1).  fp64 sums in a fixed order (deterministic).
// spc: optional per-env spill centers [E][2] (a task's post-step container
// position, tasks.hpp:599-611); nullptr: collider 0's center from cvo.
__global__ void __launch_bounds__(256) k_obs(DevParams P, StateView S, const float* __restrict__ cvo, float spill_half,
                                             float spill_temp, int ngr, float* __restrict__ obs, int od,
                                             const float* __restrict__ spc = nullptr) {
  dm_pdl();
  __shared__ double sh[8];
  const int e = blockIdx.x;
  const size_t base = (size_t)e * P.N;
  double s[3] = {0.0, 0.0, 0.0};
  for (int p = threadIdx.x; p < P.N; p += blockDim.x)
#pragma unroll
    for (int a = 0; a < 3; ++a) s[a] += (double)S.c(a, base + p);
  double m[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) m[a] = block_sum(s[a], sh) / P.N;
  double q[3] = {0.0, 0.0, 0.0}, sp = 0.0;
  const bool spill = P.K > 0 && spill_temp > 0.f;
  const float* sc = spc ? spc + (size_t)e * 2 : cvo + (size_t)e * P.K * 9;
  const double cx = spill ? sc[0] : 0.0, cy = spill ? sc[1] : 0.0;
  for (int p = threadIdx.x; p < P.N; p += blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double d = (double)S.c(a, base + p) - m[a];
      q[a] += d * d;
    }
    if (spill) {
      const double sd = fmax(fabs((double)S.c(0, base + p) - cx), fabs((double)S.c(1, base + p) - cy)) - spill_half;
      sp += 1.0 / (1.0 + exp(-sd / spill_temp));
    }
  }
  double v[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) v[a] = block_sum(q[a], sh) / P.N;
  const double spt = block_sum(sp, sh) / P.N;
  float* o = obs + (size_t)e * od;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      o[a] = (float)m[a];
      o[3 + a] = (float)v[a];
    }
    o[6] = (float)spt;
  }
  for (int g = 0; g < ngr; ++g) {
    double c = 0.0, sx[3] = {0.0, 0.0, 0.0}, sv[3] = {0.0, 0.0, 0.0}, sa = 0.0;
    for (int p = threadIdx.x; p < P.N; p += blockDim.x) {
      const size_t i = base + p;
      if (attr_group(S.attr[i]) != g) continue;
      c += 1.0;
      double v2 = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        sx[a] += (double)S.c(a, i);
        const double va = (double)S.c(3 + a, i);
        sv[a] += va;
        v2 += va * va;
      }
      sa += sqrt(v2);
    }
    const double n = fmax(block_sum(c, sh), 1.0);
    double mx[3], mv[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      mx[a] = block_sum(sx[a], sh) / n;
      mv[a] = block_sum(sv[a], sh) / n;
    }
    const double ma = block_sum(sa, sh) / n;
    double sz = 0.0;
    for (int p = threadIdx.x; p < P.N; p += blockDim.x) {
      const size_t i = base + p;
      if (attr_group(S.attr[i]) != g) continue;
      const double d = (double)S.c(2, i) - mx[2];
      sz += d * d;
    }
    const double vz = block_sum(sz, sh) / n;
    if (threadIdx.x == 0) {
      float* og = o + 7 + 8 * g;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        og[a] = (float)mx[a];
        og[3 + a] = (float)mv[a];
      }
      og[6] = (float)vz;
      og[7] = (float)ma;
    }
  }
}

// Adds the observable cotangent into the state cotangent (physical order of
// that state) and the spill's collider-center cotangent into gcvo_t.
// spc / gspc_t: per-env spill centers and their cotangents (task mode, see
// k_obs); nullptr: collider 0's center, cotangent into gcvo_t.
__global__ void __launch_bounds__(256) k_obs_adj(DevParams P, StateView S, const float* __restrict__ cvo,
                                                 float spill_half, float spill_temp, int ngr,
                                                 const float* __restrict__ dobs, int od, float* __restrict__ adj,
                                                 size_t astride, double* __restrict__ gcvo_t,
                                                 const float* __restrict__ spc = nullptr, double* __restrict__ gspc_t = nullptr) {
  dm_pdl();
  __shared__ double sh[8];
  const int e = blockIdx.x;
  const size_t base = (size_t)e * P.N;
  const float* ob = dobs + (size_t)e * od;
  double s[3] = {0.0, 0.0, 0.0};
  for (int p = threadIdx.x; p < P.N; p += blockDim.x)
#pragma unroll
    for (int a = 0; a < 3; ++a) s[a] += (double)S.c(a, base + p);
  double m[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) m[a] = block_sum(s[a], sh) / P.N;
  const bool spill = P.K > 0 && spill_temp > 0.f && ob[6] != 0.f;
  const float* sc = spc ? spc + (size_t)e * 2 : cvo + (size_t)e * P.K * 9;
  const double cx = spill ? sc[0] : 0.0, cy = spill ? sc[1] : 0.0;
  double gcx = 0.0, gcy = 0.0;
  const double invn = 1.0 / P.N;
  for (int p = threadIdx.x; p < P.N; p += blockDim.x) {
    double g[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = ob[a] * invn + ob[3 + a] * 2.0 * ((double)S.c(a, base + p) - m[a]) * invn;
    if (spill) {
      const double dxp = (double)S.c(0, base + p) - cx, dyp = (double)S.c(1, base + p) - cy;
      const double ax = fabs(dxp), ay = fabs(dyp);
      const double sd = fmax(ax, ay) - spill_half;
      const double sg = 1.0 / (1.0 + exp(-sd / spill_temp));
      const double gg = ob[6] * invn * sg * (1.0 - sg) / spill_temp;
      if (ax > ay) {
        const double sgn = dxp > 0 ? 1.0 : (dxp < 0 ? -1.0 : 0.0);
        g[0] += gg * sgn;
        gcx -= gg * sgn;
      } else if (ay > ax) {
        const double sgn = dyp > 0 ? 1.0 : (dyp < 0 ? -1.0 : 0.0);
        g[1] += gg * sgn;
        gcy -= gg * sgn;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) adj[adj_index(a, base + p, astride)] += (float)g[a];
  }
  if (spill) {
    gcx = block_sum(gcx, sh);
    gcy = block_sum(gcy, sh);
    if (threadIdx.x == 0) {
      double* g = spc ? gspc_t + (size_t)e * 2 : gcvo_t + (size_t)e * P.K * 9;
      g[0] += gcx;
      g[1] += gcy;
    }
  }
  // pooled group statistics
  for (int gi = 0; gi < ngr; ++gi) {
    const float* og = ob + 7 + 8 * gi;
    bool any = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) any = any || og[k] != 0.f;
    if (!any) continue;
    double c = 0.0, sz = 0.0;
    for (int p = threadIdx.x; p < P.N; p += blockDim.x) {
      const size_t i = base + p;
      if (attr_group(S.attr[i]) != gi) continue;
      c += 1.0;
      sz += (double)S.c(2, i);
    }
    const double n = fmax(block_sum(c, sh), 1.0);
    const double mz = block_sum(sz, sh) / n;
    for (int p = threadIdx.x; p < P.N; p += blockDim.x) {
      const size_t i = base + p;
      if (attr_group(S.attr[i]) != gi) continue;
      double vv[3], v2 = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        vv[a] = (double)S.c(3 + a, i);
        v2 += vv[a] * vv[a];
      }
      const double vn = sqrt(v2);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double gx = og[a] / n;
        if (a == 2) gx += og[6] * 2.0 * ((double)S.c(2, i) - mz) / n;
        adj[adj_index(a, i, astride)] += (float)gx;
        double gv = og[3 + a] / n;
        if (vn > 0.0) gv += og[7] * vv[a] / (vn * n);
        adj[adj_index(3 + a, i, astride)] += (float)gv;
      }
    }
  }
}

// Fills D = D(0,0) I for every particle of a fluid G2P-produced state (makes
// it a general state again: used when it becomes a new initial state).
__global__ void k_fiso_expand(size_t Ntot, StateView S) {
  dm_pdl();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < Ntot; i += (size_t)gridDim.x * blockDim.x) {
    const float sF = S.c(6, i);
#pragma unroll
    for (int q = 1; q < 9; ++q) S.c(6 + q, i) = (q % 4 == 0) ? sF : 0.f;
  }
}

// ============================ device-side reset ============================
// RngStream (rng.hpp:11-55): key = mix(seed ^ phi (stream + 1)); the k-th
// draw is mix(key ^ mix(k)), so every particle addresses its own draws.
__device__ __forceinline__ unsigned long long sm64_mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double rng_double(unsigned long long key, unsigned long long k) {
  return (double)(sm64_mix(key ^ sm64_mix(k)) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double rng_uniform(unsigned long long key, unsigned long long k, double lo, double hi) {
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), rng_double(key, k)));
}
__device__ __forceinline__ double box_muller(double u1, double u2) {
  return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586476925286766559, u2)));
}

struct ResetSpec {
  double org[3], sp[3], size[3];
  int cnt[3], odraws;
  double olo, ohi, jlo, jhi, sigma;
  int material, group;
};

// One thread per particle of a masked env.  A stream whose Box-Muller u1
// draw is 0 (probability 2^-53 per draw) is flagged for the exact sequential
// redraw of k_reset_normals_seq.
__global__ void k_reset_lattice(ResetSpec R, int E, int N, unsigned long long seed, int env_offset,
                                const unsigned char* __restrict__ mask, const int* __restrict__ pgroup,
                                double* __restrict__ odelta, int* __restrict__ seq_flag, StateView S) {
  dm_pdl();
  const size_t tot = (size_t)E * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    const int e = (int)(i / N), p = (int)(i % N);
    if (mask && !mask[e]) continue;
    const unsigned long long key =
        sm64_mix(seed ^ (0x9e3779b97f4a7c15ULL * ((unsigned long long)(env_offset + e) + 1ULL)));
    double d[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (a < R.odraws) d[a] = rng_uniform(key, (unsigned long long)a + 1, R.olo, R.ohi);
    if (odelta && p == 0)
#pragma unroll
      for (int a = 0; a < 3; ++a) odelta[(size_t)e * 3 + a] = d[a];
    const int ijk[3] = {p / (R.cnt[1] * R.cnt[2]), (p / R.cnt[2]) % R.cnt[1], p % R.cnt[2]};
    const bool jit = R.jhi > R.jlo;
    unsigned long long ctr = (unsigned long long)R.odraws;
    double x[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      x[a] = __dadd_rn(__dadd_rn(R.org[a], d[a]),
                       R.size[a] > 0.0  // sample_box (mpm.hpp:386-388): size * (i + 0.5) / n
                           ? __ddiv_rn(__dmul_rn(R.size[a], __dadd_rn((double)ijk[a], 0.5)), (double)R.cnt[a])
                           : __dmul_rn(__dadd_rn((double)ijk[a], 0.5), R.sp[a]));
      if (jit) x[a] = __dadd_rn(x[a], rng_uniform(key, ctr + 3ULL * p + a + 1, R.jlo, R.jhi));
    }
    if (jit) ctr += 3ULL * N;
    double v[3] = {0.0, 0.0, 0.0};
    if (R.sigma != 0.0) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const unsigned long long m = 3ULL * p + a;
        const double u1 = rng_double(key, ctr + 2 * m + 1), u2 = rng_double(key, ctr + 2 * m + 2);
        if (u1 <= 0.0) seq_flag[e] = 1;
        v[a] = __dmul_rn(R.sigma, box_muller(u1, u2));
      }
    }
    const size_t o = i;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      S.c(a, o) = __double2float_rn(x[a]);
      S.c(3 + a, o) = __double2float_rn(v[a]);
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      S.c(6 + q, o) = 0.f;  // D = F - I = 0
      S.c(15 + q, o) = 0.f;
    }
    const uint32_t g = pgroup ? (uint32_t)pgroup[p] : (uint32_t)R.group;
    S.attr[o] = (uint32_t)p | (((uint32_t)R.material & 0xF) << 20) | ((g & 0xFF) << 24);
  }
}

// Exact sequential Box-Muller redraw (rng.hpp:35-43: u1 is redrawn while
// u1 <= 0, shifting the stream) for the flagged envs; one thread per env.
__global__ void k_reset_normals_seq(ResetSpec R, int E, int N, unsigned long long seed, int env_offset,
                                    const int* __restrict__ seq_flag, StateView S) {
  dm_pdl();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E || !seq_flag[e]) return;
  const unsigned long long key =
      sm64_mix(seed ^ (0x9e3779b97f4a7c15ULL * ((unsigned long long)(env_offset + e) + 1ULL)));
  unsigned long long ctr = (unsigned long long)R.odraws + (R.jhi > R.jlo ? 3ULL * N : 0ULL);
  for (int m = 0; m < 3 * N; ++m) {
    double u1 = rng_double(key, ++ctr);
    const double u2 = rng_double(key, ++ctr);
    while (u1 <= 0.0) u1 = rng_double(key, ++ctr);
    S.c(3 + m % 3, (size_t)e * N + m / 3) = __double2float_rn(__dmul_rn(R.sigma, box_muller(u1, u2)));
  }
}

// ============================ layout conversion ============================
// host visit order (AoS per env) <-> SoA physical order
__global__ void k_aos_to_soa(int Ntot, const float* __restrict__ x, const float* __restrict__ v,
                             const float* __restrict__ F, const float* __restrict__ C, const int* __restrict__ mat,
                             const int* __restrict__ grp, int N, StateView S) {
  dm_pdl();
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= (size_t)Ntot) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    S.c(a, i) = x[3 * i + a];
    S.c(3 + a, i) = v[3 * i + a];
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    S.c(6 + q, i) = (q % 4 == 0) ? F[9 * i + q] - 1.f : F[9 * i + q];  // stored as D = F - I
    S.c(15 + q, i) = C[9 * i + q];
  }
  const uint32_t idx = (uint32_t)(i % N);
  const uint32_t m = mat ? (uint32_t)mat[i] : 0u, g = grp ? (uint32_t)grp[i] : 0u;
  S.attr[i] = idx | ((m & 0xF) << 20) | ((g & 0xFF) << 24);
}

// physical SoA -> canonical AoS (original order within each env).  eye: the
// F fields hold the stored deviation D (a state: F = I + D) rather than a
// cotangent (dL/dF = dL/dD, no shift).
__global__ void k_soa_to_aos(int Ntot, int N, const float* __restrict__ f, const uint32_t* __restrict__ attr,
                             size_t stride, int state_layout, int fiso, float* __restrict__ x, float* __restrict__ v, float* __restrict__ F,
                             float* __restrict__ C, int eye = 0) {
  dm_pdl();
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= (size_t)Ntot) return;
  const size_t e = i / N;
  const size_t o = e * N + (attr[i] & 0xFFFFFu);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (x) x[3 * o + a] = f[state_layout ? state_index(a, i, stride) : a * stride + i];
    if (v) v[3 * o + a] = f[state_layout ? state_index(3 + a, i, stride) : (3 + a) * stride + i];
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    const float e = (eye && q % 4 == 0) ? 1.f : 0.f;
    if (F) F[9 * o + q] = e + (fiso ? (q % 4 == 0 ? f[state_index(6, i, stride)] : 0.f)
                                    : f[state_layout ? state_index(6 + q, i, stride) : (6 + q) * stride + i]);
    if (C) C[9 * o + q] = f[state_layout ? state_index(15 + q, i, stride) : (15 + q) * stride + i];
  }
}

// canonical AoS cotangent -> physical SoA order of the state with attributes
// attr.  ftrace: a fluid context keeps the cotangent of an isotropic
// (G2P-produced) state's F as its trace in field 6 (kFluidTraceCot).
__global__ void k_aos_to_soa_perm(int Ntot, int N, const float* __restrict__ x, const float* __restrict__ v,
                                  const float* __restrict__ F, const float* __restrict__ C,
                                  const uint32_t* __restrict__ attr, float* __restrict__ f, size_t stride,
                                  int ftrace = 0) {
  dm_pdl();
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= (size_t)Ntot) return;
  const size_t e = i / N;
  const size_t o = e * N + (attr[i] & 0xFFFFFu);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    f[adj_index(a, i, stride)] = x ? x[3 * o + a] : 0.f;
    f[adj_index(3 + a, i, stride)] = v ? v[3 * o + a] : 0.f;
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    f[adj_index(6 + q, i, stride)] = F ? (ftrace ? (q == 0 ? F[9 * o] + F[9 * o + 4] + F[9 * o + 8] : 0.f) : F[9 * o + q])
                                       : 0.f;
    f[adj_index(15 + q, i, stride)] = C ? C[9 * o + q] : 0.f;
  }
}

// ============================ small device epilogues ============================
// fp64 -> fp32 cotangent conversion (stays on the device; the host entry
// points copy the fp32 result out asynchronously).
__global__ void k_f64_to_f32(size_t n, const double* __restrict__ src, float* __restrict__ dst) {
  dm_pdl();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

// dL/dE_m = dL/dmu_m dmu/dE + dL/dlam_m dlam/dE per env (MpmMaterial's Lame
// map, mpm.hpp:33-35; the reference tape cannot produce it).
__global__ void k_dE(int E, int nmat, const double* __restrict__ gmu, const double* __restrict__ glam, DevParams P,
                     double* __restrict__ out) {
  dm_pdl();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E * nmat) return;
  const int e = i / nmat, m = i % nmat;
  out[i] = gmu[e * 4 + m] * P.dmu_dE[m] + glam[e * 4 + m] * P.dlam_dE[m];
}

// Replay verification (Tape::backward_segment, tape.hpp:234-241): the
// segment replay's exit state must equal the stored checkpoint bitwise.  Both
// are written by the same deterministic G2P in the same sorted order, so
// physical slots correspond; a mismatch records min over (env << 40 | k)
// with k the exit value's index in the env's visit order (x 3N, v 3N, F 9N,
// C 9N; tasks.hpp:203-219).  Fluid G2P outputs store F(0,0) only.  Envs
// whose state was replaced by an in-tape reset (cut != 0) are skipped.
__global__ void k_replay_check(DevParams P, StateView R, StateView St, int fluid_iso,
                               const unsigned char* __restrict__ cut, unsigned long long* __restrict__ bad) {
  dm_pdl();
  const size_t tot = (size_t)P.E * P.N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    const int e = (int)(i / P.N);
    if (cut && cut[e]) continue;
    const uint32_t ar = R.attr[i], as = St.attr[i];
    const unsigned long long pn = attr_index(as), N = (unsigned long long)P.N;
    unsigned long long k = ~0ull;
    if (ar != as) k = 3 * pn;
    for (int f = 23; f >= 0; --f) {
      if (fluid_iso && f > 6 && f < 15) continue;
      if (__float_as_uint(R.c(f, i)) != __float_as_uint(St.c(f, i))) {
        const unsigned long long kk = f < 3    ? 3 * pn + f
                                      : f < 6  ? 3 * N + 3 * pn + (f - 3)
                                      : f < 15 ? 6 * N + 9 * pn + (f - 6)
                                               : 15 * N + 9 * pn + (f - 15);
        k = kk < k ? kk : k;
      }
    }
    if (k != ~0ull) atomicMin(bad, ((unsigned long long)e << 40) | k);
  }
}

// Test hook (dm_debug_inject): flips the lowest mantissa bit of x of the
// particle with original index p in env e of state S.
__global__ void k_debug_flip(DevParams P, StateView S, int e, int p) {
  dm_pdl();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.N; i += gridDim.x * blockDim.x) {
    const size_t j = (size_t)e * P.N + i;
    if ((int)attr_index(S.attr[j]) == p) S.c(0, j) = __uint_as_float(__float_as_uint(S.c(0, j)) ^ 1u);
  }
}

// ============================ task support ============================
// Point-cloud observation (tasks.hpp:296-301, 566-569): x of the particles
// with original index p = 0, stride, 2 stride, ... (p / stride < ncloud),
// written to out[e * ostride + ooff + 3 (p / stride) + a].
__global__ void k_cloud(DevParams P, StateView S, int stride, int ncloud, float* __restrict__ out, int ostride,
                        int ooff) {
  dm_pdl();
  const size_t tot = (size_t)P.E * P.N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    const int p = (int)attr_index(S.attr[i]);
    if (p % stride || p / stride >= ncloud) continue;
    float* o = out + (i / P.N) * ostride + ooff + 3 * (p / stride);
    o[0] = S.c(0, i);
    o[1] = S.c(1, i);
    o[2] = S.c(2, i);
  }
}

// Adjoint of k_cloud: dcloud [E][ncloud][3] added into the x cotangent of
// the state with attributes attr (envs with cut[e] != 0 skipped).
__global__ void k_cloud_adj(DevParams P, const uint32_t* __restrict__ attr, int stride, int ncloud,
                            const float* __restrict__ dcloud, const unsigned char* __restrict__ cut,
                            float* __restrict__ adj, size_t astride) {
  dm_pdl();
  const size_t tot = (size_t)P.E * P.N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    const int e = (int)(i / P.N);
    if (cut && cut[e]) continue;
    const int p = (int)attr_index(attr[i]);
    if (p % stride || p / stride >= ncloud) continue;
    const float* d = dcloud + ((size_t)e * ncloud + p / stride) * 3;
#pragma unroll
    for (int a = 0; a < 3; ++a) adj[adj_index(a, i, astride)] += d[a];
  }
}

// EnvBatch::reset_env (env.hpp:93-96) on the device: masked envs of state S
// take the task's particle template (x per particle in visit order; v = 0,
// F = I, C = 0 -- Task::reset copies the sample_box template).
__global__ void k_task_reset(DevParams P, StateView S, const float* __restrict__ tmpl_x,
                             const unsigned char* __restrict__ mask, int material) {
  dm_pdl();
  const size_t tot = (size_t)P.E * P.N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    const int e = (int)(i / P.N), p = (int)(i % P.N);
    if (!mask[e]) continue;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      S.c(a, i) = tmpl_x[3 * p + a];
      S.c(3 + a, i) = 0.f;
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      S.c(6 + q, i) = 0.f;  // D = F - I = 0
      S.c(15 + q, i) = 0.f;
    }
    S.attr[i] = (uint32_t)p | (((uint32_t)material & 0xF) << 20);
  }
}

// Zeroes the state cotangent of envs whose state was replaced by a reset
// (the gradient does not flow across it, algo.hpp:171-178).
__global__ void k_cut_adj(DevParams P, const unsigned char* __restrict__ cut, float* __restrict__ adj, size_t astride) {
  dm_pdl();
  const size_t tot = (size_t)P.E * P.N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    if (!cut[i / P.N]) continue;
#pragma unroll
    for (int f = 0; f < 24; ++f) adj[adj_index(f, i, astride)] = 0.f;
  }
}

__global__ void k_rec_save(size_t Ntot, size_t TT, int E, int cap, const int* __restrict__ perm,
                           const int* __restrict__ tile_count, const int4* __restrict__ active,
                           const int4* __restrict__ work, const int* __restrict__ abase, const int* __restrict__ acount,
                           const int* __restrict__ nact, const float4* __restrict__ vref, SortRec r) {
  dm_pdl();
  const int n = *nact;
  const bool fits = n <= cap;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i0 == 0) {
    *r.nact = n;
    *r.ovf = fits ? 0 : 1;
  }
  if (perm)  // nullptr: the sort wrote the record's permutation itself
    for (size_t i = i0; i < Ntot; i += stride) r.perm[i] = perm[i];
  if (tile_count)
    for (size_t i = i0; i < TT; i += stride) r.tile_count[i] = tile_count[i];
  if (fits)
    for (size_t i = i0; i < (size_t)n; i += stride) {
      r.active[i] = active[i];
      r.work[i] = work[i];
    }
  for (size_t i = i0; i < (size_t)E; i += stride) {
    r.abase[i] = abase[i];
    r.acount[i] = acount[i];
    r.vref[i] = vref[i];
  }
}

}  // namespace dm
