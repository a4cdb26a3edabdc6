// C-ABI implementation: context, device memory plan, substep schedule,
// checkpointed tape (forward stores a state every `checkpoint_every`
// substeps; backward replays each segment and runs the adjoint kernels in
// reverse) -- the B200 replacement for Tape::checkpoint / backward_segment
// (tape.hpp:181-255) driven per control step as step_checkpointed does
// (algo.hpp:79-104).
#include <cuda_runtime.h>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled (driver entry point, no -lcuda)
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges for nsys / ncu --nvtx

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/diffmpm.h"
#include "dm_kernels.cuh"

using namespace dm;

// kernel classes for dm_profile: bin, p2g, g2p, g2p_adj, p2g_adj, env_reduce,
// obs, obs_adj, layout, grid, grid_adj
constexpr int kProfClasses = 11;

struct DmContext {
  DmConfig cfg{};
  int nmat = 0;
  DevParams P{};
  double dmu_dE[4] = {0, 0, 0, 0}, dlam_dE[4] = {0, 0, 0, 0};
  int law_kind[4] = {0, 0, 0, 0};
  cudaStream_t stream = nullptr;
  std::string err;
  bool poisoned = false;
  size_t Ntot = 0;
  int ck = 1;  // substeps per checkpoint segment
  int steps = 0;
  int n_store = 0;
  unsigned long long launches = 0, bytes = 0;
  int grid_tiles = 148 * 4;
  bool coop = false;      // CTA-cooperative tiles in g2p and the cell sort (small batches; see coop_idx)
  bool coop_p2g = false;  // ... in p2g / p2g_adj / g2p_adj (pays up to larger batches)
  int coop_cg = 4;        // COOP group size: warps per tile (4 for tiny batches, else 2)
  bool grid_coop = false;  // CTA-shared tiles in the grid kernels (tiny batches)
  CUtensorMap tm_gv, tm_gmb;  // TMA descriptors of the dense node-velocity / (mass, momentum)-cotangent grids

  float* store = nullptr;  // [n_store][24][Ntot]
  uint32_t* store_attr = nullptr;
  float* seg = nullptr;  // [ck-1][24][Ntot]
  uint32_t* seg_attr = nullptr;
  float* scratch[2] = {nullptr, nullptr};
  // elastoplastic batches: the cached stress of every state buffer
  // (StateView::tau, 6 floats per particle; written by G2P), when memory allows
  bool tau_on = false;
  float* tau_store = nullptr;
  float* tau_scratch[2] = {nullptr, nullptr};
  float* tau_seg = nullptr;
  uint32_t* scratch_attr[2] = {nullptr, nullptr};
  float* adj[2] = {nullptr, nullptr};  // [24][Ntot]
  float* part = nullptr;               // [12][Ntot]
  int *keys = nullptr, *ptile = nullptr;  // sort scratch
  // sort artifacts per substep slot of a recompute segment ([ck][...]); the
  // forward pass uses slot 0, a segment replay fills slot q for substep s0+q
  int *perm_all = nullptr, *tstart_all = nullptr, *tcount_all = nullptr;
  int *abase_all = nullptr, *acount_all = nullptr, *nact_all = nullptr;
  int4* active_all = nullptr;
  int4* work_all = nullptr;
  int* ord_all = nullptr;
  float4* vref_all = nullptr;  // per slot and env: the substep's reference velocity (k_bin)
  // sort records: every forward substep's binning kept for the replay (k_rec_save)
  SortRec rec{};
  int rec_cap = 0;                  // active / work entries per record
  std::vector<int> rec_ovf_h;       // per substep, read at backward_begin: 1 = re-bin in the replay
  void* rec_mem[9] = {};
  // per active tile (by slot) 6^3 grid blocks of the replayed substeps:
  // velocity and (mass, momentum), read by the adjoint substep instead of
  // re-running bin / p2g / grid
  float4 *gvb_pool = nullptr, *gmpb_pool = nullptr;
  size_t blk_cap = 0;
  int max_active_seen = 0;
  int dev_sms = 148;
  // the step that filled the tape kept its segment (states + artifacts) from
  // the forward pass, so the backward skips that segment's replay
  int kept_t = -1;
  bool kept_ok = false;
  float* tail = nullptr;  // replay output of a segment's last substep
  uint32_t* tail_attr = nullptr;
  float4 *blocks = nullptr, *ablocks = nullptr;
  float4 *gmp = nullptr, *gv = nullptr, *gmb = nullptr;  // dense per-env grids
  int bin_warps = 16;
  bool bin_u16 = true;
  int law = -1;  // the batch's single law kind (compile-time specialised kernels), -1: mixed
  int od = DM_OBS_DIM;  // observable dimension per env
  float* dobs_buf = nullptr;  // [E][od] staging for one step's observable cotangent
  int bwd_t = -1;   // next control step the incremental backward processes (-1: not running)
  int bwd_cur = 0;  // which adj buffer holds the running state cotangent
  float* tile_acc = nullptr;
  DevFlags* flags = nullptr;
  bool pdl = false;        // programmatic dependent launch (dm_launch)
  int* wq = nullptr;       // this launch's tile-scheduling counter (a slot of wq_ring)
  int* wq_ring = nullptr;  // kWqRing counters, each zeroed by the previous tile kernel
  unsigned wq_i = 0;
  DevFlags* h_flags = nullptr;
  float *cvo_tape = nullptr, *act_tape = nullptr, *obs_tape = nullptr;
  double *gcvo = nullptr, *gact = nullptr, *gmu = nullptr, *glam = nullptr;
  float *obs_cvo = nullptr, *obs_out = nullptr;  // dm_observe's pose and output (never the tape's slots)
  float* f32_stage = nullptr;                    // fp32 cotangent staging (device)
  double* dE_dev = nullptr;                      // [E][nmat]
  unsigned* vmax_hist = nullptr;                 // per recorded step: max |v| component at its start (CFL)
  int cfl_checked = 0;                           // steps whose CFL word the host has read
  unsigned long long* replay_bad = nullptr;      // replay-verification word (k_replay_check)
  int inj_step = -1, inj_env = 0, inj_particle = 0;  // dm_debug_inject
  // task layer (dm_task_*): per-step spill centers and their cotangents, and
  // the envs reset at the end of each recorded step (the gradient is cut there)
  float* spc_tape = nullptr;     // [max_steps][E][2]
  double* gspc = nullptr;        // [max_steps][E][2]
  unsigned char* cut_tape = nullptr;  // [max_steps][E]
  std::vector<char> cut_any;     // per step: any env reset
  float* dcloud_buf = nullptr;   // [E][cloud] x cotangent staging
  int cloud_n = 0, cloud_stride = 1;
  // optional per-kernel-class CUDA-event timing (bench roofline)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<int> ev_class;
  std::vector<double> prof_ms = std::vector<double>(kProfClasses, 0.0);
  std::vector<long long> prof_n = std::vector<long long>(kProfClasses, 0);
};

namespace {

// Kernel launch, with programmatic dependent launch when `pdl` (every kernel
// opens with dm_pdl(), so it may be scheduled while the previous grid
// drains).  The context enables it for small batches (COOP mode), where the
// ~2 us launch gap per kernel boundary is a visible share of a substep; on
// cfg4's 1,024 envs it measured 2 % slower and stays off.
// DIFFMPM_PDL=0/1 forces it.
template <class... KA, class... A>
void dm_launch(dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, void (*k)(KA...), A&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {grid, block, smem, s, at, pdl ? 1u : 0u};
  cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

// Scoped NVTX range (ncu --nvtx --nvtx-include / nsys timelines).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

#define DM_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      ctx->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call;    \
      ctx->poisoned = true;                                                               \
      return DM_ERR_CUDA;                                                                 \
    }                                                                                     \
  } while (0)

template <class T>
bool dalloc(DmContext* ctx, T** p, size_t n) {
  if (n == 0) n = 1;
  if (cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();  // a failed allocation must not poison later error checks
    *p = nullptr;
    return false;
  }
  ctx->bytes += n * sizeof(T);
  return true;
}

// TMA descriptor of a dense per-env node grid [E][d0][d1][d2] float4 as a 4-D
// fp32 tensor (4 d2, d1, d0, E) with a 24 x 6 x 6 x 1 box: one tile's node
// block (tma_tile_grid), 96-byte rows (a separate 16-byte node dimension
// measured slower).  The encoder comes from the driver entry point table (no
// libcuda link).
bool make_grid_tmap(CUtensorMap* tm, const float4* base, const DevParams& P) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return false;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t d2 = P.dims[2], d1 = P.dims[1], d0 = P.dims[0];
  const cuuint64_t dims[4] = {4 * d2, d1, d0, (cuuint64_t)P.E};
  const cuuint64_t strides[3] = {16 * d2, 16 * d2 * d1, 16 * d2 * d1 * d0};  // bytes, dims 1..3
  const cuuint32_t box[4] = {4 * kExt, kExt, kExt, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float4*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// state buffers hold 24 floats per particle, Ntot rounded up to the AoSoA block
size_t state_floats(const DmContext* c) { return 24 * ((c->Ntot + kAB - 1) / kAB * kAB); }

StateView view(float* f, uint32_t* a, size_t stride) {
  StateView s;
  s.f = f;
  s.attr = a;
  s.stride = stride;
  return s;
}

size_t tau_floats(const DmContext* c) { return 6 * ((c->Ntot + kAB - 1) / kAB * kAB); }

StateView store_view(DmContext* c, int k) {
  StateView v = view(c->store + (size_t)k * state_floats(c), c->store_attr + (size_t)k * c->Ntot, c->Ntot);
  if (c->tau_on) v.tau = c->tau_store + (size_t)k * tau_floats(c);
  return v;
}

// State of global substep index s while running forward.
StateView fwd_state(DmContext* c, int s) {
  if (s % c->ck == 0) return store_view(c, s / c->ck);
  StateView v = view(c->scratch[s & 1], c->scratch_attr[s & 1], c->Ntot);
  if (c->tau_on) v.tau = c->tau_scratch[s & 1];
  return v;
}

// P2G of global substep s reads the cached stress unless s starts a control
// step (set_state, resets and the in-tape cut write fresh particles there).
// The rule does not depend on the checkpoint interval: checkpointed and
// store-every-substep runs stay bit-identical.
void set_tauv(DmContext* c, int s) { c->P.tauv = c->tau_on && s % c->cfg.substeps != 0; }

// State of substep s inside the segment starting at s0 during backward.
StateView seg_state(DmContext* c, int s0, int s) {
  if (s == s0) return store_view(c, s0 / c->ck);
  const int k = s - s0 - 1;
  StateView v = view(c->seg + (size_t)k * state_floats(c), c->seg_attr + (size_t)k * c->Ntot, c->Ntot);
  if (c->tau_on) v.tau = c->tau_seg + (size_t)k * tau_floats(c);
  return v;
}

int maxc_of(int K) { return K <= 1 ? 1 : 4; }

cudaEvent_t next_event(DmContext* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}
void prof_mark(DmContext* c, int cls) {
  if (!c->prof) return;
  cudaEventRecord(next_event(c), c->stream);
  c->ev_class.push_back(cls);
}
// Sum (end - start) per class; events are recorded in begin/end pairs.
void prof_flush(DmContext* c) {
  if (!c->prof || c->ev_used == 0) return;
  cudaStreamSynchronize(c->stream);
  for (size_t i = 0; i + 1 < c->ev_used; i += 2) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev_pool[i], c->ev_pool[i + 1]);
    c->prof_ms[c->ev_class[i]] += ms;
    c->prof_n[c->ev_class[i]] += 1;
  }
  c->ev_used = 0;
  c->ev_class.clear();
}
#define PROF_BEGIN(c, cls) prof_mark(c, cls)
#define PROF_END(c, cls) prof_mark(c, cls)

// Runs `launch` with the kernel template specialised for the batch's law.
#define DM_LAW_DISPATCH(c, LAUNCH)      \
  switch ((c)->law) {                   \
    case kFixedCorotated: LAUNCH(0); break; \
    case kNeoHookean: LAUNCH(1); break;     \
    case kElastoplastic: LAUNCH(2); break;  \
    case kFluid: LAUNCH(3); break;          \
    default: LAUNCH(-1); break;             \
  }

struct Slot {
  int* perm;
  int* tile_start;
  int* tile_count;
  int4* active;  // env-ordered (k_bin)
  int4* work;    // largest-first (k_order_*): the tile kernels' schedule
  int* ord;      // bucket counters of k_order_*
  int* env_abase;
  int* env_acount;
  int* nact;
  float4* gvb;   // per-slot grid blocks (replay only)
  float4* gmpb;
  float4* vref;  // [E] reference velocity of the substep (node_update_rel)
};

// zeroes the dynamic tile-scheduling counter before a tile kernel
// Next tile kernel's counter: the ring slot the previous tile kernel zeroed
// (wq_clear_next); every wq_reset is followed by exactly one tile kernel.
void wq_reset(DmContext* c) { c->wq = c->wq_ring + (c->wq_i++ % kWqRing); }

Slot slot(DmContext* c, int q) {
  const size_t TT = (size_t)c->P.E * c->P.Tn;
  Slot s;
  s.perm = c->perm_all + (size_t)q * c->Ntot;
  s.tile_start = c->tstart_all + (size_t)q * TT;
  s.tile_count = c->tcount_all + (size_t)q * TT;
  s.active = c->active_all + (size_t)q * TT;
  s.work = c->work_all + (size_t)q * TT;
  s.ord = c->ord_all + (size_t)q * 2 * kOrdBuckets;
  s.env_abase = c->abase_all + (size_t)q * c->P.E;
  s.env_acount = c->acount_all + (size_t)q * c->P.E;
  s.nact = c->nact_all + q;
  s.gvb = c->gvb_pool ? c->gvb_pool + (size_t)q * c->blk_cap * kExt3 : nullptr;
  s.gmpb = c->gmpb_pool ? c->gmpb_pool + (size_t)q * c->blk_cap * kExt3 : nullptr;
  s.vref = c->vref_all + (size_t)q * c->P.E;
  return s;
}

#ifndef DM_CS_GRID
#define DM_CS_GRID 2  // k_cellsort is light (32 registers): twice the tile kernels' resident warps
#endif
// CTAs of a tile kernel: every resident slot (grid_tiles), unless the batch
// has few active tiles (max_active_seen, known after the first sync): then a
// CTA per tile in COOP mode (a warp per tile otherwise) with 2x headroom, at
// least one per SM.  Only the schedule changes (every tile's result is
// independent of which CTA runs it); idle CTAs cost a prologue and a
// contended atomic each (cfg1: ~25 of 1,184 CTAs had work).
int tile_ctas(const DmContext* c, bool coop) {
  if (c->max_active_seen <= 0) return c->grid_tiles;
  const long want = coop ? 2L * c->max_active_seen : (2L * c->max_active_seen + kWarps - 1) / kWarps;
  return (int)std::min<long>(c->grid_tiles, std::max<long>(c->dev_sms, want));
}

// active-tile count (as last seen) up to which one CTA orders the work list
constexpr int kOrderSmallMax = 4096;

void launch_bin(DmContext* c, const StateView& S, const Slot& q, int sub, int check_vmax,
                const SortRec* rec = nullptr) {
  wq_reset(c);  // k_bin totals the active tiles in a zeroed ring slot (no memset node)
  PROF_BEGIN(c, 0);
  if (c->bin_u16)
    dm_launch(c->P.E, 32 * c->bin_warps, (size_t)c->bin_warps * c->P.Tn * 2, c->stream, c->pdl, k_bin<unsigned short>, 
        c->P, S, c->keys, c->ptile, q.tile_start, q.tile_count, q.active, q.env_abase, q.env_acount, c->flags, c->wq,
        sub, check_vmax, q.vref, q.ord);
  else
    dm_launch(c->P.E, 32 * c->bin_warps, (size_t)c->bin_warps * c->P.Tn * 4, c->stream, c->pdl, k_bin<int>, 
        c->P, S, c->keys, c->ptile, q.tile_start, q.tile_count, q.active, q.env_abase, q.env_acount, c->flags, c->wq,
        sub, check_vmax, q.vref, q.ord);
  // the sort record's copy of the binning tables: by the one-CTA order kernel
  // or the cell sort (rec_copy)
  const RecSrc rs{q.active, q.work, q.env_abase, q.env_acount, q.nact, q.vref, c->rec_cap, c->P.E};
  const bool small = c->max_active_seen > 0 && c->max_active_seen <= kOrderSmallMax;
  const SortRec no_rec{}, rec_cs = rec && !small ? *rec : no_rec;
  if (small) {  // one CTA orders the list
    dm_launch(1, 1024, 0, c->stream, c->pdl, k_order_small, q.active, c->wq, q.nact, q.work, rec ? *rec : no_rec, rs);
    c->launches += 1;
  } else {
    dm_launch(64, 256, 0, c->stream, c->pdl, k_order_hist, q.active, c->wq, q.ord, q.nact);
    dm_launch((unsigned)((c->P.E * c->P.Tn + 2047) / 2048), 256, 0, c->stream, c->pdl, k_order_scatter, q.active, q.nact,
              q.ord, q.work);
    c->launches += 2;
  }
  wq_reset(c);
  if (c->coop)  // CTA-shared tiles, like the tile kernels of small batches
    dm_launch(tile_ctas(c, true), kWarps * 32, 0, c->stream, c->pdl, k_cellsort_coop, c->P, c->ptile, q.perm, c->keys, q.work, q.nact,
                                                                  c->flags, c->wq, rec_cs, rs);
  else
    dm_launch(tile_ctas(c, false) * DM_CS_GRID, kWarps * 32, 0, c->stream, c->pdl, k_cellsort, c->P, S, c->ptile, q.perm, c->keys,
                                                                         q.tile_start, q.tile_count, q.work, q.nact,
                                                                         c->flags, c->wq, rec_cs, rs);
  ++c->launches;
  PROF_END(c, 0);
  ++c->launches;
}

const float* step_cvo(DmContext* c, int t) { return c->cvo_tape + (size_t)t * c->P.E * (c->P.K > 0 ? c->P.K : 1) * 9; }
const float* step_act(DmContext* c, int t) {
  return c->P.G > 0 ? c->act_tape + (size_t)t * c->P.E * c->P.G : nullptr;
}

template <int LW, bool COOP, int CG>
void launch_p2g_k(DmContext* c, const StateView& S, const Slot& q, int t, int sub) {
  dm_launch(tile_ctas(c, COOP), kWarps * 32, kP2gSmem, c->stream, c->pdl, k_p2g<LW, COOP, CG>, 
      c->P, S, q.perm, q.tile_start, q.tile_count, q.work, step_act(c, t), c->blocks, c->flags, q.nact, sub, c->wq,
      q.vref);
}

void launch_p2g(DmContext* c, const StateView& S, const Slot& q, int t, int sub) {
  wq_reset(c);
  PROF_BEGIN(c, 1);
#define L_P2G(LW)                                   \
  if (!c->coop_p2g)                                 \
    launch_p2g_k<LW, false, 4>(c, S, q, t, sub);    \
  else if (c->coop_cg == 2)                         \
    launch_p2g_k<LW, true, 2>(c, S, q, t, sub);     \
  else                                              \
    launch_p2g_k<LW, true, 4>(c, S, q, t, sub)
  DM_LAW_DISPATCH(c, L_P2G);
#undef L_P2G
  PROF_END(c, 1);
  ++c->launches;
}

// Grid kernels: one collider -> its kind fixed at compile time (CK), else the
// runtime switch over up to 4 colliders.
#define DM_GRID_DISPATCH(c, LAUNCH)                       \
  if (maxc_of((c)->P.K) == 1) {                           \
    switch ((c)->P.K == 1 ? (c)->P.shape[0].kind : -1) {  \
      case kPlane: LAUNCH(1, kPlane); break;              \
      case kSphere: LAUNCH(1, kSphere); break;            \
      case kBox: LAUNCH(1, kBox); break;                  \
      case kCylinder: LAUNCH(1, kCylinder); break;        \
      case kHollowBox: LAUNCH(1, kHollowBox); break;      \
      default: LAUNCH(1, -1); break;                      \
    }                                                     \
  } else {                                                \
    LAUNCH(4, -1);                                        \
  }

void launch_grid(DmContext* c, const Slot& q, int t, bool dump) {
  wq_reset(c);
  PROF_BEGIN(c, 9);
#define L_GRID(MC, CK)                                                                                        \
  if (c->grid_coop)                                                                                     \
    dm_launch(tile_ctas(c, true), kWarps * 32, 0, c->stream, c->pdl, k_grid<MC, CK, true>, c->P, q.tile_count, q.work, step_cvo(c, t), \
                                                               c->blocks, dump ? c->gmp : nullptr, c->gv, q.nact, c->wq, \
                                                               q.vref);                                 \
  else                                                                                                  \
    dm_launch(tile_ctas(c, false), kWarps * 32, 0, c->stream, c->pdl, k_grid<MC, CK, false>, c->P, q.tile_count, q.work, step_cvo(c, t), \
                                                               c->blocks, dump ? c->gmp : nullptr, c->gv, q.nact, c->wq, \
                                                               q.vref)
  DM_GRID_DISPATCH(c, L_GRID);
#undef L_GRID
  PROF_END(c, 9);
  ++c->launches;
}

template <int LW, bool COOP, int CG>
void launch_g2p_k(DmContext* c, const StateView& S, const StateView& So, const Slot& q, int sub, bool dump) {
  dm_launch(tile_ctas(c, COOP), kWarps * 32, 0, c->stream, c->pdl, k_g2p<LW, COOP, CG>, 
      c->P, S, So, q.perm, q.tile_start, q.tile_count, q.work, c->tm_gv, c->flags, q.nact, sub, c->gmp,
      dump ? q.gvb : nullptr, dump ? q.gmpb : nullptr, c->wq, (int)c->blk_cap, q.vref);
}

void launch_g2p(DmContext* c, const StateView& S, const StateView& So, const Slot& q, int t, int sub, bool dump) {
  (void)t;
  wq_reset(c);
  PROF_BEGIN(c, 2);
#define L_G2P(LW)                                        \
  if (!c->coop)                                          \
    launch_g2p_k<LW, false, 4>(c, S, So, q, sub, dump);  \
  else if (c->coop_cg == 2)                              \
    launch_g2p_k<LW, true, 2>(c, S, So, q, sub, dump);   \
  else                                                   \
    launch_g2p_k<LW, true, 4>(c, S, So, q, sub, dump)
  DM_LAW_DISPATCH(c, L_G2P);
#undef L_G2P
  PROF_END(c, 2);
  ++c->launches;
}

// Record s of the sort records.
SortRec rec_at(const DmContext* c, int s) {
  const size_t TT = (size_t)c->P.E * c->P.Tn;
  SortRec r;
  r.perm = c->rec.perm + (size_t)s * c->Ntot;
  r.tile_count = c->rec.tile_count + (size_t)s * TT;
  r.active = c->rec.active + (size_t)s * c->rec_cap;
  r.work = c->rec.work + (size_t)s * c->rec_cap;
  r.abase = c->rec.abase + (size_t)s * c->P.E;
  r.acount = c->rec.acount + (size_t)s * c->P.E;
  r.nact = c->rec.nact + s;
  r.vref = c->rec.vref + (size_t)s * c->P.E;
  r.ovf = c->rec.ovf + s;
  return r;
}

// Slot qi with the sort artifacts of record s (the grid-block dumps stay the slot's).
Slot rec_slot(DmContext* c, int qi, int s) {
  Slot q = slot(c, qi);
  const SortRec r = rec_at(c, s);
  q.perm = r.perm;
  q.tile_count = r.tile_count;
  q.active = r.active;
  q.work = r.work;
  q.env_abase = r.abase;
  q.env_acount = r.acount;
  q.nact = r.nact;
  q.vref = r.vref;
  return q;
}

// whether the replay / adjoint of global substep s can use its sort record
bool rec_usable(const DmContext* c, int s) {
  return c->rec.perm && s < (int)c->rec_ovf_h.size() && c->rec_ovf_h[s] == 0;
}

// One forward substep on slot qi.  rec_s >= 0: the replay of substep rec_s
// with a usable sort record (no binning); record != 0: the forward pass,
// which saves its binning into the record of substep sub.
void forward_substep(DmContext* c, const StateView& S, const StateView& So, int t, int sub, int check_vmax, int qi,
                     bool dump, int rec_s = -1, bool record = false) {
  Slot q = rec_s >= 0 ? rec_slot(c, qi, rec_s) : slot(c, qi);
  // the forward pass sorts straight into the record's permutation and tile
  // counts (always complete: N and E x Tn entries); the cell sort copies the
  // capacity-limited rest of the binning (rec_copy; k_rec_save otherwise)
  if (record && c->rec.perm) {
    const SortRec r = rec_at(c, sub);
    q.perm = r.perm;
    q.tile_count = r.tile_count;
  }
  const bool rec_fused = rec_s < 0 && record && c->rec.perm;
  if (rec_s < 0) {
    const SortRec r = rec_fused ? rec_at(c, sub) : SortRec{};
    launch_bin(c, S, q, sub, check_vmax, rec_fused ? &r : nullptr);
  }
  if (record && c->rec.perm && !rec_fused) {
    const size_t TT = (size_t)c->P.E * c->P.Tn;
    dm_launch(c->grid_tiles, 256, 0, c->stream, c->pdl, k_rec_save, c->Ntot, TT, c->P.E, c->rec_cap, nullptr, nullptr, q.active,
                                                     q.work, q.env_abase, q.env_acount, q.nact, q.vref, rec_at(c, sub));
    ++c->launches;
  }
  launch_p2g(c, S, q, t, sub);
  launch_grid(c, q, t, dump);
  launch_g2p(c, S, So, q, t, sub, dump);
}

template <int LAW, int NG, int NM, bool COOP, int CG>
void launch_p2g_adj_k(DmContext* c, const StateView& S, const Slot& q, int t, float* adj_out) {
  dm_launch(tile_ctas(c, COOP), kWarps * 32, 0, c->stream, c->pdl, k_p2g_adj<LAW, NG, NM, COOP, CG>, 
      c->P, S, q.perm, q.tile_start, q.tile_count, q.work, step_act(c, t), c->gmb, c->tm_gmb, c->part, adj_out, c->Ntot,
      c->tile_acc, q.nact, c->wq);
}

template <int LAW, int NG>
void launch_p2g_adj(DmContext* c, const StateView& S, const Slot& q, int t, float* adj_out) {
  wq_reset(c);
  if (c->P.nmat == 1) {
    if (!c->coop_p2g) launch_p2g_adj_k<LAW, NG, 1, false, 4>(c, S, q, t, adj_out);
    else if (c->coop_cg == 2) launch_p2g_adj_k<LAW, NG, 1, true, 2>(c, S, q, t, adj_out);
    else launch_p2g_adj_k<LAW, NG, 1, true, 4>(c, S, q, t, adj_out);
  } else {
    if (!c->coop_p2g) launch_p2g_adj_k<LAW, NG, 4, false, 4>(c, S, q, t, adj_out);
    else if (c->coop_cg == 2) launch_p2g_adj_k<LAW, NG, 4, true, 2>(c, S, q, t, adj_out);
    else launch_p2g_adj_k<LAW, NG, 4, true, 4>(c, S, q, t, adj_out);
  }
}

template <int LAW, int NM, bool COOP, int CG>
void launch_g2p_adj_k(DmContext* c, const StateView& S, const StateView& Sn, const Slot& q, const float* adj_in) {
  dm_launch(tile_ctas(c, COOP), kWarps * 32, kG2pAdjSmem, c->stream, c->pdl, k_g2p_adj<LAW, NM, COOP, CG>, 
      c->P, S, Sn, adj_in, c->Ntot, q.perm, q.tile_start, q.tile_count, q.work, q.gvb, c->ablocks, c->part,
      c->tile_acc, q.nact, c->wq, q.vref);
}

// Adjoint of one substep from the replay's stored artifacts (slot qi).
void backward_substep(DmContext* c, const StateView& S, const StateView& Sn, int t, int qi, const float* adj_in,
                      float* adj_out, int rec_s = -1, int perm_s = -1) {
  Slot q = rec_s >= 0 ? rec_slot(c, qi, rec_s) : slot(c, qi);
  if (perm_s >= 0) {  // a kept segment: the forward sorted into the record
    q.perm = rec_at(c, perm_s).perm;
    q.tile_count = rec_at(c, perm_s).tile_count;
  }
  wq_reset(c);
  PROF_BEGIN(c, 3);
#define L_G2PA(LW)                                                                                     \
  if (c->P.nmat == 1) {                                                                                 \
    if (!c->coop_p2g) launch_g2p_adj_k<LW, 1, false, 4>(c, S, Sn, q, adj_in);                           \
    else if (c->coop_cg == 2) launch_g2p_adj_k<LW, 1, true, 2>(c, S, Sn, q, adj_in);                    \
    else launch_g2p_adj_k<LW, 1, true, 4>(c, S, Sn, q, adj_in);                                         \
  } else {                                                                                              \
    if (!c->coop_p2g) launch_g2p_adj_k<LW, 4, false, 4>(c, S, Sn, q, adj_in);                           \
    else if (c->coop_cg == 2) launch_g2p_adj_k<LW, 4, true, 2>(c, S, Sn, q, adj_in);                    \
    else launch_g2p_adj_k<LW, 4, true, 4>(c, S, Sn, q, adj_in);                                         \
  }
  DM_LAW_DISPATCH(c, L_G2PA);
#undef L_G2PA
  PROF_END(c, 3);
  ++c->launches;
  wq_reset(c);
  PROF_BEGIN(c, 10);
#define L_GRIDA(MC, CK)                                                                                   \
  if (c->grid_coop)                                                                                 \
    dm_launch(tile_ctas(c, true), kWarps * 32, 0, c->stream, c->pdl, k_grid_adj<MC, CK, true>, c->P, q.tile_count, q.work,  \
                                                                   step_cvo(c, t), c->ablocks, q.gmpb,   \
                                                                   c->gmb, c->tile_acc, q.nact, c->wq, q.vref); \
  else                                                                                              \
    dm_launch(tile_ctas(c, false), kWarps * 32, 0, c->stream, c->pdl, k_grid_adj<MC, CK, false>, c->P, q.tile_count, q.work, \
                                                                   step_cvo(c, t), c->ablocks, q.gmpb,   \
                                                                   c->gmb, c->tile_acc, q.nact, c->wq, q.vref)
  DM_GRID_DISPATCH(c, L_GRIDA);
#undef L_GRIDA
  PROF_END(c, 10);
  ++c->launches;
  const int G = c->P.G;
  PROF_BEGIN(c, 4);
#define L_P2GA(LW)                              \
  if (G <= 1)                                   \
    launch_p2g_adj<LW, 1>(c, S, q, t, adj_out); \
  else if (G <= 8)                              \
    launch_p2g_adj<LW, 8>(c, S, q, t, adj_out); \
  else                                          \
    launch_p2g_adj<LW, 16>(c, S, q, t, adj_out)
  DM_LAW_DISPATCH(c, L_P2GA);
#undef L_P2GA
  PROF_END(c, 4);
  ++c->launches;
  const int Kc = c->P.K > 0 ? c->P.K : 1;
  PROF_BEGIN(c, 5);
  dm_launch(c->P.E, kNacc * kRedSlices, 0, c->stream, c->pdl, k_env_reduce, c->P, q.active, q.env_abase, q.env_acount, c->tile_acc,
                                                c->gcvo + (size_t)t * c->P.E * Kc * 9,
                                                c->gact + (size_t)t * c->P.E * (G > 0 ? G : 1), c->gmu, c->glam);
  PROF_END(c, 5);
  ++c->launches;
}

std::string fmt_error(DmContext* c, unsigned long long key) {
  const int code = (int)(key & 0xF);
  const int axis = (int)((key >> 4) & 3);
  const unsigned particle = (unsigned)((key >> 6) & 0xFFFFFF);
  const int env = (int)((key >> 32) & 0xFFFF);
  const int sub = (int)((key >> 48) & 0xFFFF);
  char buf[256];
  if (code == kErrP2GInterior) {
    std::snprintf(buf, sizeof(buf), "mpm: particle %u outside grid interior (axis %d) [env %d, substep %d]", particle,
                  axis, env, sub);
  } else if (code == kErrG2PInterior) {
    std::snprintf(buf, sizeof(buf), "g2p: particle %u advected outside grid interior [env %d, substep %d]", particle,
                  env, sub);
  } else {
    static const char* names[4] = {"stress_fixed_corotated", "stress_neo_hookean", "stress_elastoplastic",
                                   "stress_fluid"};
    const int kind = c->law_kind[axis];
    std::snprintf(buf, sizeof(buf), "%s: det(F) <= 0 [env %d, particle %u, substep %d]", names[kind & 3], env,
                  particle, sub);
  }
  return buf;
}

// Synchronises the stream and reads the device flags: errors recorded by
// any launch since the last read (the first one in substep order) and the
// CFL word of every control step recorded since (mpm.hpp:355-361: checked
// once per mpm_step on the velocities at its entry; one warning per
// violating step).  Host entry points call it after every control step;
// the *_device entry points only at the points that synchronise anyway.
int check_flags(DmContext* ctx) {
  prof_flush(ctx);
  const int n_cfl = ctx->steps - ctx->cfl_checked;
  std::vector<unsigned> vh(n_cfl > 0 ? n_cfl : 0);
  DM_CUDA(cudaMemcpyAsync(ctx->h_flags, ctx->flags, sizeof(DevFlags), cudaMemcpyDeviceToHost, ctx->stream));
  if (n_cfl > 0)
    DM_CUDA(cudaMemcpyAsync(vh.data(), ctx->vmax_hist + ctx->cfl_checked, n_cfl * sizeof(unsigned),
                            cudaMemcpyDeviceToHost, ctx->stream));
  DM_CUDA(cudaStreamSynchronize(ctx->stream));
  DM_CUDA(cudaGetLastError());
  if (ctx->h_flags->max_active > ctx->max_active_seen) ctx->max_active_seen = ctx->h_flags->max_active;
  if (ctx->h_flags->err_key != ~0ull) {
    ctx->err = fmt_error(ctx, ctx->h_flags->err_key);
    ctx->poisoned = true;
    return DM_ERR_RUNTIME;
  }
  for (int i = 0; i < n_cfl; ++i) {
    float vmax;
    std::memcpy(&vmax, &vh[i], sizeof(float));
    if ((double)vmax * ctx->cfg.dt >= ctx->cfg.dx)
      std::fprintf(stderr, "mpm_step: CFL violated (max|v| dt = %g >= dx = %g)\n", (double)vmax * ctx->cfg.dt,
                   ctx->cfg.dx);
  }
  if (n_cfl > 0) ctx->cfl_checked = ctx->steps;
  return DM_OK;
}

int reset_flags(DmContext* ctx) {
  DevFlags f;
  f.err_key = ~0ull;
  f.vmax_bits = 0;
  f.max_active = 0;
  DM_CUDA(cudaMemcpyAsync(ctx->flags, &f, sizeof(DevFlags), cudaMemcpyHostToDevice, ctx->stream));
  DM_CUDA(cudaStreamSynchronize(ctx->stream));
  return DM_OK;
}

int set_state_impl(DmContext* ctx, const float* x, const float* v, const float* F, const float* C, const int* mat,
                   const int* grp, cudaMemcpyKind kind) {
  if (ctx->poisoned && ctx->h_flags->err_key == ~0ull) ctx->poisoned = false;
  const size_t N = ctx->Ntot;
  float* st = ctx->adj[0];
  int* ints = reinterpret_cast<int*>(ctx->part);
  DM_CUDA(cudaMemcpyAsync(st, x, 3 * N * sizeof(float), kind, ctx->stream));
  DM_CUDA(cudaMemcpyAsync(st + 3 * N, v, 3 * N * sizeof(float), kind, ctx->stream));
  DM_CUDA(cudaMemcpyAsync(st + 6 * N, F, 9 * N * sizeof(float), kind, ctx->stream));
  DM_CUDA(cudaMemcpyAsync(st + 15 * N, C, 9 * N * sizeof(float), kind, ctx->stream));
  if (mat) DM_CUDA(cudaMemcpyAsync(ints, mat, N * sizeof(int), kind, ctx->stream));
  if (grp) DM_CUDA(cudaMemcpyAsync(ints + N, grp, N * sizeof(int), kind, ctx->stream));
  const StateView S0 = store_view(ctx, 0);
  dm_launch((unsigned)((N + 255) / 256), 256, 0, ctx->stream, ctx->pdl, k_aos_to_soa, (int)N, st, st + 3 * N, st + 6 * N, st + 15 * N,
                                                                     mat ? ints : nullptr, grp ? ints + N : nullptr,
                                                                     ctx->P.N, S0);
  ++ctx->launches;
  ctx->steps = 0;
  ctx->cfl_checked = 0;
  ctx->bwd_t = -1;
  ctx->kept_t = -1;
  ctx->kept_ok = false;
  ctx->poisoned = false;
  const int rc = reset_flags(ctx);
  if (rc != DM_OK) return rc;
  DM_CUDA(cudaGetLastError());
  return DM_OK;
}

int get_state_impl(DmContext* ctx, float* x, float* v, float* F, float* C, cudaMemcpyKind kind) {
  const size_t N = ctx->Ntot;
  const int s = ctx->steps * ctx->cfg.substeps;
  const StateView S = fwd_state(ctx, s);
  float* out = ctx->adj[1];
  const int fiso = ctx->law == kFluid && s > 0;  // a fluid G2P output stores F(0,0) only
  dm_launch((unsigned)((N + 255) / 256), 256, 0, ctx->stream, ctx->pdl, k_soa_to_aos, (int)N, ctx->P.N, S.f, S.attr, N, 1, fiso, out,
                                                                     out + 3 * N, out + 6 * N, out + 15 * N, 1);
  ++ctx->launches;
  if (x) DM_CUDA(cudaMemcpyAsync(x, out, 3 * N * sizeof(float), kind, ctx->stream));
  if (v) DM_CUDA(cudaMemcpyAsync(v, out + 3 * N, 3 * N * sizeof(float), kind, ctx->stream));
  if (F) DM_CUDA(cudaMemcpyAsync(F, out + 6 * N, 9 * N * sizeof(float), kind, ctx->stream));
  if (C) DM_CUDA(cudaMemcpyAsync(C, out + 15 * N, 9 * N * sizeof(float), kind, ctx->stream));
  DM_CUDA(cudaStreamSynchronize(ctx->stream));
  return DM_OK;
}

// Allocates the per-slot grid-block pools for `need` active tiles.
int ensure_blk_pool(DmContext* ctx, size_t need) {
  if (ctx->blk_cap >= need) return DM_OK;
  if (ctx->gvb_pool) cudaFree(ctx->gvb_pool);
  if (ctx->gmpb_pool) cudaFree(ctx->gmpb_pool);
  ctx->bytes -= 2 * ctx->blk_cap * ctx->ck * kExt3 * sizeof(float4);
  ctx->gvb_pool = ctx->gmpb_pool = nullptr;
  ctx->blk_cap = 0;
  if (!dalloc(ctx, &ctx->gvb_pool, need * ctx->ck * kExt3) || !dalloc(ctx, &ctx->gmpb_pool, need * ctx->ck * kExt3)) {
    ctx->err = "out of device memory for the replay grid blocks";
    ctx->kept_ok = false;
    return DM_ERR_CUDA;
  }
  ctx->blk_cap = need;
  return DM_OK;
}

int step_impl(DmContext* ctx, const float* cvo, const float* act, float* obs, cudaMemcpyKind kin,
              cudaMemcpyKind kout, const float* spc = nullptr) {
  if (ctx->poisoned) {
    if (ctx->err.empty()) ctx->err = "context poisoned by an earlier error";
    return DM_ERR_RUNTIME;
  }
  if (ctx->steps >= ctx->cfg.max_steps) {
    ctx->err = "tape capacity exceeded (max_steps)";
    return DM_ERR_CAPACITY;
  }
  NvtxRange nv("dm_step");
  const int t = ctx->steps;
  const int E = ctx->P.E, K = ctx->P.K, G = ctx->P.G;
  if (K > 0) {
    if (!cvo) {
      ctx->err = "dm_step: colliders configured but cvo is NULL";
      return DM_ERR_ARG;
    }
    DM_CUDA(cudaMemcpyAsync(const_cast<float*>(step_cvo(ctx, t)), cvo, (size_t)E * K * 9 * sizeof(float), kin,
                            ctx->stream));
  }
  if (G > 0) {
    if (act)
      DM_CUDA(cudaMemcpyAsync(const_cast<float*>(step_act(ctx, t)), act, (size_t)E * G * sizeof(float), kin,
                              ctx->stream));
    else
      DM_CUDA(cudaMemsetAsync(const_cast<float*>(step_act(ctx, t)), 0, (size_t)E * G * sizeof(float), ctx->stream));
  }
  const int S = ctx->cfg.substeps;
  // The step that fills the tape keeps its segment (one segment per control
  // step): intermediate states into the segment buffer, sort and grid blocks
  // into the per-substep slots, exactly as the replay would produce them.
  // (sized from the earlier steps' largest active-tile count plus a margin;
  // tiles beyond it are not dumped and the step is then replayed as usual)
  bool keep = ctx->ck == S && S > 1 && t == ctx->cfg.max_steps - 1;
  if (keep && kout == cudaMemcpyDeviceToDevice) {  // the device path reads the flags lazily: refresh them
    const int rc = check_flags(ctx);
    if (rc != DM_OK) return rc;
  }
  keep = keep && ctx->max_active_seen > 0;
  if (keep) {
    size_t want = (size_t)ctx->max_active_seen + ctx->max_active_seen / 4 + 64;
    if (std::getenv("DIFFMPM_DEBUG_FAIL_KEEP_POOL")) want = (size_t)1 << 40;  // test hook: the pool cannot be allocated
    if (ensure_blk_pool(ctx, want) != DM_OK) {
      keep = false;  // not enough memory to keep it: replay in the backward
      ctx->err.clear();
    }
  }
  ctx->kept_t = -1;
  ctx->kept_ok = false;
  DM_CUDA(cudaMemsetAsync(&ctx->flags->vmax_bits, 0, sizeof(unsigned), ctx->stream));  // this step's CFL word
  for (int q = 0; q < S; ++q) {
    const int s = t * S + q;
    ctx->P.fiso = s > 0;  // every state but the initial one is a G2P output
    set_tauv(ctx, s);
    if (keep)
      forward_substep(ctx, seg_state(ctx, t * S, s), q + 1 < S ? seg_state(ctx, t * S, s + 1) : fwd_state(ctx, s + 1),
                      t, s, q == 0, q, true, -1, true);
    else
      forward_substep(ctx, fwd_state(ctx, s), fwd_state(ctx, s + 1), t, s, q == 0, 0, false, -1, true);
  }
  DM_CUDA(cudaMemcpyAsync(ctx->vmax_hist + t, &ctx->flags->vmax_bits, sizeof(unsigned), cudaMemcpyDeviceToDevice,
                          ctx->stream));
  float* o = ctx->obs_tape + (size_t)t * E * ctx->od;
  float* spc_t = nullptr;
  if (spc) {  // task mode: the spill is measured about the post-step container position
    spc_t = ctx->spc_tape + (size_t)t * E * 2;
    DM_CUDA(cudaMemcpyAsync(spc_t, spc, (size_t)E * 2 * sizeof(float), kin, ctx->stream));
  }
  if (ctx->cut_tape) {
    DM_CUDA(cudaMemsetAsync(ctx->cut_tape + (size_t)t * E, 0, E, ctx->stream));
    ctx->cut_any[t] = 0;
  }
  PROF_BEGIN(ctx, 6);
  dm_launch(E, 256, 0, ctx->stream, ctx->pdl, k_obs, ctx->P, fwd_state(ctx, (t + 1) * S), step_cvo(ctx, t), (float)ctx->cfg.spill_half,
                                    (float)ctx->cfg.spill_temp, ctx->cfg.obs_groups, o, ctx->od, spc_t);
  PROF_END(ctx, 6);
  ++ctx->launches;
  if (obs) DM_CUDA(cudaMemcpyAsync(obs, o, (size_t)E * ctx->od * sizeof(float), kout, ctx->stream));
  ctx->steps = t + 1;
  if (kout != cudaMemcpyDeviceToDevice) {  // host path: errors and the CFL warning of this step now
    const int rc = check_flags(ctx);
    if (rc != DM_OK) {
      ctx->steps = t;
      return rc;
    }
  }
  if (keep && (size_t)ctx->max_active_seen <= ctx->blk_cap) {  // every tile's blocks fit the pool
    ctx->kept_t = t;
    ctx->kept_ok = true;
  }
  return DM_OK;
}

int backward_begin(DmContext* ctx, const float* dfx, const float* dfv, const float* dfF, const float* dfC,
                   cudaMemcpyKind kin) {
  if (ctx->poisoned) return DM_ERR_RUNTIME;
  const int T = ctx->steps, E = ctx->P.E;
  const int Kc = ctx->P.K > 0 ? ctx->P.K : 1, Gc = ctx->P.G > 0 ? ctx->P.G : 1;
  const size_t N = ctx->Ntot;
  if (T == 0) {
    ctx->err = "backward: no recorded steps";
    return DM_ERR_ARG;
  }
  {  // forward errors (lazily read on the device path) surface before the backward
    const int rc = check_flags(ctx);
    if (rc != DM_OK) return rc;
  }
  DM_CUDA(cudaMemsetAsync(ctx->replay_bad, 0xFF, sizeof(unsigned long long), ctx->stream));
  if (ctx->rec.perm) {  // which substeps' sort records the replay can use
    ctx->rec_ovf_h.assign((size_t)T * ctx->cfg.substeps, 1);
    DM_CUDA(cudaMemcpy(ctx->rec_ovf_h.data(), ctx->rec.ovf, ctx->rec_ovf_h.size() * sizeof(int), cudaMemcpyDeviceToHost));
  }
  {
    // grid-block pool for one replayed segment: at least the forward pass's
    // largest active-tile count (the replay is bit-identical to it)
    const size_t need = (size_t)(ctx->max_active_seen > 0 ? ctx->max_active_seen : 1);
    if (ctx->blk_cap < need) {
      ctx->kept_ok = false;  // a reallocated pool loses the kept segment's blocks
      if (ensure_blk_pool(ctx, need) != DM_OK) return DM_ERR_CUDA;
    }
  }
  DM_CUDA(cudaMemsetAsync(ctx->gcvo, 0, (size_t)T * E * Kc * 9 * sizeof(double), ctx->stream));
  DM_CUDA(cudaMemsetAsync(ctx->gact, 0, (size_t)T * E * Gc * sizeof(double), ctx->stream));
  DM_CUDA(cudaMemsetAsync(ctx->gmu, 0, (size_t)E * 4 * sizeof(double), ctx->stream));
  DM_CUDA(cudaMemsetAsync(ctx->glam, 0, (size_t)E * 4 * sizeof(double), ctx->stream));
  // final-state cotangent in the physical order of the final state
  ctx->bwd_cur = 0;
  float* A = ctx->adj[0];
  const StateView Sf = fwd_state(ctx, T * ctx->cfg.substeps);
  if (dfx || dfv || dfF || dfC) {
    float* stg = ctx->adj[1];
    if (dfx) DM_CUDA(cudaMemcpyAsync(stg, dfx, 3 * N * sizeof(float), kin, ctx->stream));
    if (dfv) DM_CUDA(cudaMemcpyAsync(stg + 3 * N, dfv, 3 * N * sizeof(float), kin, ctx->stream));
    if (dfF) DM_CUDA(cudaMemcpyAsync(stg + 6 * N, dfF, 9 * N * sizeof(float), kin, ctx->stream));
    if (dfC) DM_CUDA(cudaMemcpyAsync(stg + 15 * N, dfC, 9 * N * sizeof(float), kin, ctx->stream));
    dm_launch((unsigned)((N + 255) / 256), 256, 0, ctx->stream, ctx->pdl, k_aos_to_soa_perm, 
        (int)N, ctx->P.N, dfx ? stg : nullptr, dfv ? stg + 3 * N : nullptr, dfF ? stg + 6 * N : nullptr,
        dfC ? stg + 15 * N : nullptr, Sf.attr, A, N, ctx->law == kFluid);
    ++ctx->launches;
  } else {
    DM_CUDA(cudaMemsetAsync(A, 0, state_floats(ctx) * sizeof(float), ctx->stream));
  }
  ctx->bwd_t = T - 1;
  return DM_OK;
}

// Converts an fp64 device array to fp32 on the device, into dst (device:
// directly; host: through the device staging buffer and an async copy).
int copy_out_f32(DmContext* ctx, float* dst, const double* src, size_t n, cudaMemcpyKind kout) {
  float* d = kout == cudaMemcpyDeviceToDevice ? dst : ctx->f32_stage;
  dm_launch((unsigned)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024), 256, 0, ctx->stream, ctx->pdl, k_f64_to_f32, n, src, d);
  ++ctx->launches;
  if (d != dst) DM_CUDA(cudaMemcpyAsync(dst, d, n * sizeof(float), kout, ctx->stream));
  DM_CUDA(cudaGetLastError());
  return DM_OK;
}

// dcloud_t (task layer, host): cotangent of the step's point-cloud
// observation [E][cloud_n][3]; gspc_t (host): receives the spill-center
// cotangents [E][2] of a task-mode step.
int backward_step(DmContext* ctx, const float* dobs_t, float* dcvo_t, float* dact_t, cudaMemcpyKind kin,
                  cudaMemcpyKind kout, const float* dcloud_t = nullptr, double* gspc_t = nullptr) {
  if (ctx->poisoned) return DM_ERR_RUNTIME;
  if (ctx->bwd_t < 0) {
    ctx->err = "backward_step: no backward in progress (call dm_backward_begin)";
    return DM_ERR_ARG;
  }
  NvtxRange nv("dm_backward_step");
  const int t = ctx->bwd_t, S = ctx->cfg.substeps, E = ctx->P.E, ck = ctx->ck;
  const int Kc = ctx->P.K > 0 ? ctx->P.K : 1, Gc = ctx->P.G > 0 ? ctx->P.G : 1;
  const size_t N = ctx->Ntot;
  int cur = ctx->bwd_cur;
  const int s_end = (t + 1) * S;
  const bool cut = ctx->cut_tape && ctx->cut_any[t];
  const unsigned char* cut_t = cut ? ctx->cut_tape + (size_t)t * E : nullptr;
  if (cut) {  // envs reset after this step: no cotangent flows back across the reset (algo.hpp:171-178)
    dm_launch(ctx->grid_tiles, 256, 0, ctx->stream, ctx->pdl, k_cut_adj, ctx->P, cut_t, ctx->adj[cur], N);
    ++ctx->launches;
  }
  if (dobs_t) DM_CUDA(cudaMemcpyAsync(ctx->dobs_buf, dobs_t, (size_t)E * ctx->od * sizeof(float), kin, ctx->stream));
  if (dcloud_t)
    DM_CUDA(cudaMemcpyAsync(ctx->dcloud_buf, dcloud_t, (size_t)E * ctx->cloud_n * 3 * sizeof(float),
                            cudaMemcpyHostToDevice, ctx->stream));
  const bool kept = t == ctx->kept_t && ctx->kept_ok;  // the forward kept this step's segment
  const float* spc_t = ctx->spc_tape && gspc_t ? ctx->spc_tape + (size_t)t * E * 2 : nullptr;
  if (spc_t) DM_CUDA(cudaMemsetAsync(ctx->gspc + (size_t)t * E * 2, 0, (size_t)E * 2 * sizeof(double), ctx->stream));
  bool first = true;
  for (int s0 = s_end - ck; s0 >= t * S; s0 -= ck) {
    // replay the segment's forward (tape.hpp:229-233), keeping every
    // substep's sort and grid blocks for its adjoint
    if (!kept) nvtxRangePushA("replay");
    for (int q = 0; q < ck && !kept; ++q) {
      const int s = s0 + q;
      const StateView So = q + 1 < ck ? seg_state(ctx, s0, s + 1) : view(ctx->tail, ctx->tail_attr, ctx->Ntot);
      ctx->P.fiso = s > 0;
      set_tauv(ctx, s);
      forward_substep(ctx, seg_state(ctx, s0, s), So, t, s, 0, q, true, rec_usable(ctx, s) ? s : -1);
    }
    if (!kept) {
      // the replayed exit must equal the stored checkpoint bitwise (tape.hpp:234-241)
      const StateView tl = view(ctx->tail, ctx->tail_attr, ctx->Ntot);
      if (ctx->inj_step == t)  // dm_debug_inject: a non-deterministic forward
        dm_launch((ctx->P.N + 255) / 256, 256, 0, ctx->stream, ctx->pdl, k_debug_flip, ctx->P, tl, ctx->inj_env, ctx->inj_particle);
      dm_launch(ctx->grid_tiles, 256, 0, ctx->stream, ctx->pdl, k_replay_check, ctx->P, tl, store_view(ctx, (s0 + ck) / ck),
                                                                ctx->law == kFluid, s0 + ck == s_end ? cut_t : nullptr,
                                                                ctx->replay_bad);
      ctx->launches += 1 + (ctx->inj_step == t);
      nvtxRangePop();
    }
    if (first) {
      // the step's observables are of its end state before any reset: the
      // replay's exit (== the stored state for envs not reset), or the
      // stored state of a kept segment (never reset)
      first = false;
      const StateView Se = kept ? store_view(ctx, s_end / ck) : view(ctx->tail, ctx->tail_attr, ctx->Ntot);
      if (dobs_t) {
        PROF_BEGIN(ctx, 7);
        dm_launch(E, 256, 0, ctx->stream, ctx->pdl, k_obs_adj, ctx->P, Se, step_cvo(ctx, t), (float)ctx->cfg.spill_half,
                                              (float)ctx->cfg.spill_temp, ctx->cfg.obs_groups, ctx->dobs_buf, ctx->od,
                                              ctx->adj[cur], N, ctx->gcvo + (size_t)t * E * Kc * 9, spc_t,
                                              spc_t ? ctx->gspc + (size_t)t * E * 2 : nullptr);
        PROF_END(ctx, 7);
        ++ctx->launches;
      }
      if (dcloud_t) {
        dm_launch(ctx->grid_tiles, 256, 0, ctx->stream, ctx->pdl, k_cloud_adj, ctx->P, Se.attr, ctx->cloud_stride, ctx->cloud_n,
                                                               ctx->dcloud_buf, nullptr, ctx->adj[cur], N);
        ++ctx->launches;
      }
    }
    for (int q = ck - 1; q >= 0; --q) {
      const int s = s0 + q;
      const StateView Sn = q + 1 < ck ? seg_state(ctx, s0, s + 1)
                       : kept ? store_view(ctx, (s + 1) / ck)
                              : view(ctx->tail, ctx->tail_attr, ctx->Ntot);
      ctx->P.fiso = s > 0;
      backward_substep(ctx, seg_state(ctx, s0, s), Sn, t, q, ctx->adj[cur], ctx->adj[cur ^ 1],
                       !kept && rec_usable(ctx, s) ? s : -1, kept && ctx->rec.perm ? s : -1);
      cur ^= 1;
    }
  }
  ctx->bwd_cur = cur;
  ctx->bwd_t = t - 1;
  if (!kept) ctx->kept_ok = false;  // a replay overwrote the segment buffer and slots
  int rc = DM_OK;
  if (dcvo_t && ctx->P.K > 0)
    rc = copy_out_f32(ctx, dcvo_t, ctx->gcvo + (size_t)t * E * Kc * 9, (size_t)E * Kc * 9, kout);
  if (rc == DM_OK && dact_t && ctx->P.G > 0)
    rc = copy_out_f32(ctx, dact_t, ctx->gact + (size_t)t * E * Gc, (size_t)E * Gc, kout);
  if (rc == DM_OK && spc_t)
    DM_CUDA(cudaMemcpyAsync(gspc_t, ctx->gspc + (size_t)t * E * 2, (size_t)E * 2 * sizeof(double),
                            cudaMemcpyDeviceToHost, ctx->stream));
  if (rc == DM_OK && kout != cudaMemcpyDeviceToDevice && (dcvo_t || dact_t || gspc_t))
    DM_CUDA(cudaStreamSynchronize(ctx->stream));  // host outputs are complete on return
  return rc;
}

int backward_end(DmContext* ctx, float* dx0, float* dv0, float* dF0, float* dC0, double* dE, cudaMemcpyKind kout) {
  if (ctx->poisoned) return DM_ERR_RUNTIME;
  if (ctx->bwd_t != -1) {
    ctx->err = "backward_end: steps remain (call dm_backward_step for every recorded step)";
    return DM_ERR_ARG;
  }
  const int E = ctx->P.E, cur = ctx->bwd_cur;
  const size_t N = ctx->Ntot;
  float* out = ctx->adj[cur ^ 1];
  const StateView S0 = store_view(ctx, 0);
  dm_launch((unsigned)((N + 255) / 256), 256, 0, ctx->stream, ctx->pdl, k_soa_to_aos, (int)N, ctx->P.N, ctx->adj[cur], S0.attr, N, 1, 0, out,
                                                                     out + 3 * N, out + 6 * N, out + 15 * N, 0);
  ++ctx->launches;
  if (dx0) DM_CUDA(cudaMemcpyAsync(dx0, out, 3 * N * sizeof(float), kout, ctx->stream));
  if (dv0) DM_CUDA(cudaMemcpyAsync(dv0, out + 3 * N, 3 * N * sizeof(float), kout, ctx->stream));
  if (dF0) DM_CUDA(cudaMemcpyAsync(dF0, out + 6 * N, 9 * N * sizeof(float), kout, ctx->stream));
  if (dC0) DM_CUDA(cudaMemcpyAsync(dC0, out + 15 * N, 9 * N * sizeof(float), kout, ctx->stream));
  if (dE) {
    double* d = kout == cudaMemcpyDeviceToDevice ? dE : ctx->dE_dev;
    dm_launch((E * ctx->nmat + 127) / 128, 128, 0, ctx->stream, ctx->pdl, k_dE, E, ctx->nmat, ctx->gmu, ctx->glam, ctx->P, d);
    ++ctx->launches;
    if (d != dE) DM_CUDA(cudaMemcpyAsync(dE, d, (size_t)E * ctx->nmat * sizeof(double), kout, ctx->stream));
  }
  unsigned long long bad = ~0ull;
  DM_CUDA(cudaMemcpyAsync(&bad, ctx->replay_bad, sizeof(bad), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->bwd_t = -1;
  const int rc = check_flags(ctx);  // synchronises
  if (rc != DM_OK) return rc;
  if (bad != ~0ull) {
    // Tape::backward_segment's text (tape.hpp:238-240); k indexes the env's
    // segment exit values in visit order
    ctx->err = "checkpoint replay: non-deterministic forward (exit value " + std::to_string(bad & 0xFFFFFFFFFFull) +
               " changed) [env " + std::to_string(bad >> 40) + "]";
    ctx->poisoned = true;
    return DM_ERR_RUNTIME;
  }
  return DM_OK;
}

int backward_impl(DmContext* ctx, const float* dobs, const float* dfx, const float* dfv, const float* dfF,
                  const float* dfC, float* dx0, float* dv0, float* dF0, float* dC0, float* dcvo, float* dact,
                  double* dE, cudaMemcpyKind kin, cudaMemcpyKind kout) {
  int rc = backward_begin(ctx, dfx, dfv, dfF, dfC, kin);
  if (rc != DM_OK) return rc;
  const int T = ctx->steps, E = ctx->P.E;
  const int Kc = ctx->P.K > 0 ? ctx->P.K : 1, Gc = ctx->P.G > 0 ? ctx->P.G : 1;
  for (int t = T - 1; t >= 0; --t) {
    rc = backward_step(ctx, dobs ? dobs + (size_t)t * E * ctx->od : nullptr,
                       dcvo ? dcvo + (size_t)t * E * Kc * 9 : nullptr, dact ? dact + (size_t)t * E * Gc : nullptr,
                       kin, kout);
    if (rc != DM_OK) return rc;
  }
  return backward_end(ctx, dx0, dv0, dF0, dC0, dE, kout);
}

}  // namespace

extern "C" {

DmContext* dm_create(const DmConfig* cfg, const DmMaterial* mats, int num_materials, const DmColliderShape* shapes) {
  DmContext* ctx = new DmContext();
  ctx->cfg = *cfg;
  auto fail = [&](const char* m) {
    ctx->err = m;
    ctx->poisoned = true;
    return ctx;
  };
  if (cfg->substeps < 1) return fail("mpm_step: substeps < 1");
  if (num_materials < 1 || num_materials > DM_MAX_MATERIALS) return fail("dm_create: 1..4 materials supported");
  if (cfg->num_colliders < 0 || cfg->num_colliders > DM_MAX_COLLIDERS) return fail("dm_create: <= 4 colliders");
  if (cfg->num_groups < 0 || cfg->num_groups > DM_MAX_GROUPS) return fail("dm_create: <= 16 actuation groups");
  if (cfg->particles_per_env < 1 || cfg->particles_per_env > (1 << 20)) return fail("dm_create: 1..2^20 particles per env");
  if (cfg->num_envs < 1 || cfg->num_envs > 65535) return fail("dm_create: 1..65535 envs");
  const int ck = cfg->checkpoint_every > 0 ? cfg->checkpoint_every : cfg->substeps;
  if (cfg->substeps % ck != 0) return fail("dm_create: checkpoint_every must divide substeps");
  if (cudaSetDevice(cfg->device) != cudaSuccess) return fail("dm_create: cudaSetDevice failed");
  ctx->ck = ck;
  ctx->nmat = num_materials;
  if (cfg->obs_groups < 0 || cfg->obs_groups > DM_MAX_GROUPS) return fail("dm_create: obs_groups must be 0..16");
  ctx->od = DM_OBS_DIM + 8 * cfg->obs_groups;
  DevParams& P = ctx->P;
  P.E = cfg->num_envs;
  P.N = cfg->particles_per_env;
  for (int a = 0; a < 3; ++a) {
    P.dims[a] = cfg->dims[a];
    P.td[a] = (cfg->dims[a] + kTile - 1) / kTile;
    P.grav[a] = (float)cfg->gravity[a];
  }
  P.Tn = P.td[0] * P.td[1] * P.td[2];
  {
    // 16-bit histogram words when a warp's count and an env's cursor fit
    ctx->bin_u16 = P.N <= 65535;
    const size_t wb = ctx->bin_u16 ? 2 : 4;
    // One CTA per env, nw warps each: pick nw minimising waves x (work per
    // warp) = ceil(E / (SMs x CTAs per SM)) / nw, CTAs per SM bounded by the
    // per-warp histograms (shared memory) and 64 resident warps.
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device);
    const int max_smem = (int)((160 * 1024) / ((size_t)P.Tn * wb));  // warps per CTA by histogram size
    int nw = 0;
    double best = 1e30;
    for (int w = 1; w <= 32 && w <= max_smem; ++w) {
      const size_t shm = (size_t)w * P.Tn * wb + 1024;
      int per_sm = (int)((227 * 1024) / shm);
      per_sm = per_sm < 64 / w ? per_sm : 64 / w;
      if (per_sm < 1) continue;
      const double waves = std::ceil((double)P.E / ((double)sms * per_sm));
      const double cost = waves / w;
      if (cost < best - 1e-12) {
        best = cost;
        nw = w;
      }
    }
    if (nw < 1) return fail("dm_create: grid too large for the bin kernel");
    ctx->bin_warps = nw;
    cudaFuncSetAttribute(k_bin<unsigned short>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(nw * P.Tn * 2));
    cudaFuncSetAttribute(k_bin<int>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(nw * P.Tn * 4));
  }
  P.dx = (float)cfg->dx;
  P.dx_lo = (float)(cfg->dx - (double)P.dx);
  P.inv_dx = (float)(1.0 / cfg->dx);
  P.dt = (float)cfg->dt;
  P.boundary = cfg->boundary;
  P.alpha_c = (float)cfg->alpha_c;
  P.mu_b = (float)cfg->mu_b;
  P.K = cfg->num_colliders;
  P.G = cfg->num_groups;
  P.nmat = num_materials;
  for (int m = 0; m < num_materials; ++m) {
    const DmMaterial& M = mats[m];
    const double nu = M.poisson;
    const double mu = M.youngs / (2.0 * (1.0 + nu));
    double lam = M.youngs * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    ctx->dmu_dE[m] = 1.0 / (2.0 * (1.0 + nu));
    ctx->dlam_dE[m] = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    if (M.kind == kFluid && M.bulk > 0.0) {
      lam = M.bulk;
      ctx->dlam_dE[m] = 0.0;
    }
    Law<float>& L = P.law[m];
    L.kind = M.kind;
    L.mu = (float)mu;
    L.lam = (float)lam;
    L.cy = (float)(M.wide_yield ? M.yield_stress / mu : M.yield_stress / (2.0 * mu));
    L.visc = (float)M.viscosity;
    L.act_k = (float)M.act_strength;
    L.mass = (float)(M.density * M.volume);
    L.vol = (float)M.volume;
    L.dmu_dE = (float)ctx->dmu_dE[m];
    L.dlam_dE = (float)ctx->dlam_dE[m];
    P.dmu_dE[m] = ctx->dmu_dE[m];
    P.dlam_dE[m] = ctx->dlam_dE[m];
    ctx->law_kind[m] = M.kind;
  }
  ctx->law = mats[0].kind;
  for (int m = 1; m < num_materials; ++m)
    if (mats[m].kind != ctx->law) ctx->law = -1;
  for (int c = 0; c < P.K; ++c) {
    ColShape& s = P.shape[c];
    s.kind = shapes[c].kind;
    for (int a = 0; a < 3; ++a) {
      s.nrm[a] = (float)shapes[c].normal[a];
      s.half[a] = (float)shapes[c].half[a];
    }
    s.radius = (float)shapes[c].radius;
    s.length = (float)shapes[c].length;
    s.thickness = (float)shapes[c].thickness;
  }
  {
#define DM_SMEM_ATTR1(LW, CO, CG)                                                                                 \
  cudaFuncSetAttribute(k_p2g<LW, CO, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kP2gSmem);            \
  cudaFuncSetAttribute(k_g2p_adj<LW, 1, CO, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kG2pAdjSmem); \
  cudaFuncSetAttribute(k_g2p_adj<LW, 4, CO, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kG2pAdjSmem)
#define DM_SMEM_ATTR(LW)        \
  DM_SMEM_ATTR1(LW, false, 4);  \
  DM_SMEM_ATTR1(LW, true, 2);   \
  DM_SMEM_ATTR1(LW, true, 4)
    DM_SMEM_ATTR(0);
    DM_SMEM_ATTR(1);
    DM_SMEM_ATTR(2);
    DM_SMEM_ATTR(3);
    DM_SMEM_ATTR(-1);
#undef DM_SMEM_ATTR
#undef DM_SMEM_ATTR1
  }
  ctx->Ntot = (size_t)P.E * P.N;
  const size_t N = ctx->Ntot;
  const size_t TT = (size_t)P.E * P.Tn;
  const int Kc = P.K > 0 ? P.K : 1, Gc = P.G > 0 ? P.G : 1;
  ctx->n_store = cfg->max_steps * cfg->substeps / ck + 1;
  bool ok = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && dalloc(ctx, &ctx->store, (size_t)ctx->n_store * state_floats(ctx)) &&
       dalloc(ctx, &ctx->store_attr, (size_t)ctx->n_store * N);
  if (ck > 1) ok = ok && dalloc(ctx, &ctx->seg, (size_t)(ck - 1) * state_floats(ctx)) && dalloc(ctx, &ctx->seg_attr, (size_t)(ck - 1) * N);

  if (ck > 1)
    for (int i = 0; i < 2; ++i)
      ok = ok && dalloc(ctx, &ctx->scratch[i], state_floats(ctx)) && dalloc(ctx, &ctx->scratch_attr[i], N);
  ok = ok && dalloc(ctx, &ctx->adj[0], state_floats(ctx)) && dalloc(ctx, &ctx->adj[1], state_floats(ctx)) &&
       dalloc(ctx, &ctx->part, state_floats(ctx) / 2);
  ok = ok && dalloc(ctx, &ctx->keys, N) && dalloc(ctx, &ctx->ptile, N) &&
       dalloc(ctx, &ctx->perm_all, (size_t)ck * N) && dalloc(ctx, &ctx->tstart_all, (size_t)ck * TT) &&
       dalloc(ctx, &ctx->tcount_all, (size_t)ck * TT) && dalloc(ctx, &ctx->active_all, (size_t)ck * TT) &&
       dalloc(ctx, &ctx->work_all, (size_t)ck * TT) && dalloc(ctx, &ctx->ord_all, (size_t)ck * 2 * kOrdBuckets) &&
       dalloc(ctx, &ctx->vref_all, (size_t)ck * P.E) &&
       dalloc(ctx, &ctx->abase_all, (size_t)ck * P.E) && dalloc(ctx, &ctx->acount_all, (size_t)ck * P.E) &&
       dalloc(ctx, &ctx->nact_all, (size_t)ck) && dalloc(ctx, &ctx->tail, state_floats(ctx)) && dalloc(ctx, &ctx->tail_attr, N);
  const size_t NN = (size_t)P.E * P.dims[0] * P.dims[1] * P.dims[2];
  ok = ok && dalloc(ctx, &ctx->gmp, NN) && dalloc(ctx, &ctx->gv, NN) && dalloc(ctx, &ctx->gmb, NN);
  ok = ok && dalloc(ctx, &ctx->blocks, TT * kExt3) && dalloc(ctx, &ctx->ablocks, TT * kExt3) &&
       dalloc(ctx, &ctx->tile_acc, TT * kNacc) && dalloc(ctx, &ctx->flags, 1) && dalloc(ctx, &ctx->wq_ring, kWqRing);
  ok = ok && dalloc(ctx, &ctx->cvo_tape, (size_t)cfg->max_steps * P.E * Kc * 9) &&
       dalloc(ctx, &ctx->act_tape, (size_t)cfg->max_steps * P.E * Gc) &&
       dalloc(ctx, &ctx->obs_tape, (size_t)cfg->max_steps * P.E * ctx->od) &&
       dalloc(ctx, &ctx->dobs_buf, (size_t)P.E * ctx->od) &&
       dalloc(ctx, &ctx->gcvo, (size_t)cfg->max_steps * P.E * Kc * 9) &&
       dalloc(ctx, &ctx->gact, (size_t)cfg->max_steps * P.E * Gc) && dalloc(ctx, &ctx->gmu, (size_t)P.E * 4) &&
       dalloc(ctx, &ctx->glam, (size_t)P.E * 4);
  ok = ok && dalloc(ctx, &ctx->obs_cvo, (size_t)P.E * Kc * 9) && dalloc(ctx, &ctx->obs_out, (size_t)P.E * ctx->od) &&
       dalloc(ctx, &ctx->f32_stage, (size_t)P.E * (Kc * 9 > Gc ? Kc * 9 : Gc)) &&
       dalloc(ctx, &ctx->dE_dev, (size_t)P.E * num_materials) && dalloc(ctx, &ctx->vmax_hist, (size_t)cfg->max_steps) &&
       dalloc(ctx, &ctx->replay_bad, 1);
  ok = ok && cudaMallocHost(reinterpret_cast<void**>(&ctx->h_flags), sizeof(DevFlags)) == cudaSuccess;
  if (!ok) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "dm_create: device allocation failed (%.2f GB requested so far)",
                  ctx->bytes / 1e9);
    return fail(buf);
  }
  if (!make_grid_tmap(&ctx->tm_gv, ctx->gv, P) || !make_grid_tmap(&ctx->tm_gmb, ctx->gmb, P))
    return fail("dm_create: TMA descriptor encoding failed (cuTensorMapEncodeTiled)");
  if (ctx->law == kElastoplastic && !std::getenv("DIFFMPM_NO_TAU_CACHE")) {
    // the stress cache (+25 % of the state memory), when it leaves room for the rest
    const size_t want = ((size_t)ctx->n_store + (ck > 1 ? ck + 1 : 0)) * tau_floats(ctx) * sizeof(float);
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (want + (size_t)(8ull << 30) < free_b) {
      bool r = dalloc(ctx, &ctx->tau_store, (size_t)ctx->n_store * tau_floats(ctx));
      if (ck > 1)
        r = r && dalloc(ctx, &ctx->tau_seg, (size_t)(ck - 1) * tau_floats(ctx)) &&
            dalloc(ctx, &ctx->tau_scratch[0], tau_floats(ctx)) && dalloc(ctx, &ctx->tau_scratch[1], tau_floats(ctx));
      ctx->tau_on = r;
      if (!r)
        for (float** q : {&ctx->tau_store, &ctx->tau_seg, &ctx->tau_scratch[0], &ctx->tau_scratch[1]})
          if (*q) cudaFree(*q), *q = nullptr;
    }
  }
  cudaMemsetAsync(ctx->store_attr, 0, N * sizeof(uint32_t), ctx->stream);
  cudaMemsetAsync(ctx->tile_acc, 0, TT * kNacc * sizeof(float), ctx->stream);
  cudaMemsetAsync(ctx->wq_ring, 0, kWqRing * sizeof(int), ctx->stream);
  {
    // sort records for every substep of the tape, when device memory allows
    // (DIFFMPM_NO_SORT_RECORDS=1 disables them)
    const size_t n_sub = (size_t)cfg->max_steps * cfg->substeps;
    ctx->rec_cap = (int)std::min<size_t>(TT, std::max<size_t>(1024, N / 32));
    const size_t per = N * 4 + TT * 4 + 2 * (size_t)ctx->rec_cap * 16 + (size_t)P.E * (4 + 4 + 16) + 8;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if (!std::getenv("DIFFMPM_NO_SORT_RECORDS") && cfg->substeps > 1 && n_sub * per + (size_t)(6ull << 30) < free_b) {
      bool r = dalloc(ctx, &ctx->rec.perm, n_sub * N) && dalloc(ctx, &ctx->rec.tile_count, n_sub * TT) &&
               dalloc(ctx, &ctx->rec.active, n_sub * ctx->rec_cap) && dalloc(ctx, &ctx->rec.work, n_sub * ctx->rec_cap) &&
               dalloc(ctx, &ctx->rec.abase, n_sub * P.E) && dalloc(ctx, &ctx->rec.acount, n_sub * P.E) &&
               dalloc(ctx, &ctx->rec.nact, n_sub) && dalloc(ctx, &ctx->rec.vref, n_sub * P.E) &&
               dalloc(ctx, &ctx->rec.ovf, n_sub);
      void* m[9] = {ctx->rec.perm, ctx->rec.tile_count, ctx->rec.active, ctx->rec.work, ctx->rec.abase,
                    ctx->rec.acount, ctx->rec.nact, ctx->rec.vref, ctx->rec.ovf};
      for (int i = 0; i < 9; ++i) ctx->rec_mem[i] = m[i];
      if (!r) {  // not enough after all: no records (the replay bins)
        for (void*& q : ctx->rec_mem)
          if (q) cudaFree(q), q = nullptr;
        ctx->rec = SortRec{};
      } else {
        cudaMemsetAsync(ctx->rec.ovf, 0xFF, n_sub * sizeof(int), ctx->stream);  // nothing recorded yet
      }
    }
  }
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, cfg->device);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_p2g_adj<-1, 16, 4, false, 4>, kWarps * 32, 0);
  if (occ < 1) occ = 1;
  ctx->grid_tiles = dev_sms * (occ < 8 ? 8 : occ);
  ctx->dev_sms = dev_sms;
  // CTA-cooperative tiles when the batch gives each resident warp only a few
  // chunks (DIFFMPM_COOP=0/1 forces the mode)
  ctx->coop = N < (size_t)kCoopParticlesPerWarp * ctx->grid_tiles * kWarps;
  ctx->coop_p2g = N < (size_t)kCoopP2gParticlesPerWarp * ctx->grid_tiles * kWarps;
  if (const char* f = std::getenv("DIFFMPM_COOP")) ctx->coop = ctx->coop_p2g = f[0] == '1';
  // the grid kernels' tiles are short (owned nodes): sharing them pays only
  // when there are fewer tiles than warps (r02 A/B: cfg1 grid -25 %, grid_adj
  // -32 %; neutral at 32 envs; +5 / +11 % at 128 envs)
  ctx->grid_coop = N < (size_t)kGridCoopParticlesPerWarp * ctx->grid_tiles * kWarps;
  if (const char* f = std::getenv("DIFFMPM_GRID_COOP")) ctx->grid_coop = f[0] == '1';
  // two-warp tile groups unless the batch is tiny (a tile's chunk chain is
  // then the critical path); DIFFMPM_COOP_CG=2/4 forces it
  ctx->coop_cg = N < (size_t)kGridCoopParticlesPerWarp * ctx->grid_tiles * kWarps ? 4 : 2;
  if (const char* f = std::getenv("DIFFMPM_COOP_CG")) ctx->coop_cg = f[0] == '2' ? 2 : 4;
  // launch chaining for small batches (r02 A/B: cfg1 +18 %, cfg2 +5 %, 128 envs
  // neutral, 1,024 envs -2 %)
  ctx->pdl = ctx->coop;
  if (const char* f = std::getenv("DIFFMPM_PDL")) ctx->pdl = f[0] == '1';
  if (reset_flags(ctx) != DM_OK) return ctx;
  return ctx;
}

void dm_destroy(DmContext* ctx) {
  if (!ctx) return;
  void* ptrs[] = {ctx->tau_store, ctx->tau_seg, ctx->tau_scratch[0], ctx->tau_scratch[1],
                  ctx->store,     ctx->store_attr, ctx->seg,       ctx->seg_attr,   ctx->scratch[0], ctx->scratch[1],
                  ctx->scratch_attr[0], ctx->scratch_attr[1], ctx->adj[0], ctx->adj[1], ctx->part, ctx->keys,
                  ctx->perm_all,  ctx->ptile, ctx->tstart_all, ctx->tcount_all, ctx->abase_all, ctx->acount_all,
                  ctx->active_all, ctx->work_all, ctx->ord_all, ctx->nact_all, ctx->tail, ctx->tail_attr, ctx->gvb_pool, ctx->gmpb_pool,
                  ctx->blocks,    ctx->ablocks,    ctx->tile_acc,   ctx->gmp, ctx->gv, ctx->gmb,   ctx->flags, ctx->wq_ring, ctx->cvo_tape,  ctx->act_tape,
                  ctx->obs_tape,  ctx->dobs_buf, ctx->gcvo,       ctx->gact,       ctx->gmu,        ctx->glam,
                  ctx->obs_cvo,   ctx->obs_out,  ctx->f32_stage,  ctx->dE_dev,     ctx->vmax_hist,  ctx->replay_bad,
                  ctx->vref_all,  ctx->spc_tape, ctx->gspc,       ctx->cut_tape,   ctx->dcloud_buf};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (void* p : ctx->rec_mem)
    if (p) cudaFree(p);
  if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int dm_last_error(const DmContext* ctx, char* buf, int len) {
  if (!ctx) return DM_ERR_ARG;
  if (buf && len > 0) std::snprintf(buf, (size_t)len, "%s", ctx->err.c_str());
  return ctx->poisoned ? DM_ERR_RUNTIME : DM_OK;
}

void* dm_stream(DmContext* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
unsigned long long dm_device_bytes(const DmContext* ctx) { return ctx ? ctx->bytes : 0; }
int dm_tape_steps(const DmContext* ctx) { return ctx ? ctx->steps : 0; }
unsigned long long dm_launch_count(const DmContext* ctx) { return ctx ? ctx->launches : 0; }

int dm_set_state(DmContext* ctx, const float* x, const float* v, const float* F, const float* C, const int* material,
                 const int* group) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return set_state_impl(ctx, x, v, F, C, material, group, cudaMemcpyHostToDevice);
}
int dm_set_state_device(DmContext* ctx, const float* x, const float* v, const float* F, const float* C,
                        const int* material, const int* group) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return set_state_impl(ctx, x, v, F, C, material, group, cudaMemcpyDeviceToDevice);
}
namespace {
// Device-side reset (dm_reset_lattice): masked envs regenerated on the GPU,
// the others keep their current state; the tape restarts at step 0.
int reset_lattice_impl(DmContext* ctx, const DmLatticeReset* spec, unsigned long long seed, int env_offset,
                       const unsigned char* mask, const int* pgroup, double* odelta, bool dev) {
  if (!ctx || !ctx->store || !spec) return DM_ERR_ARG;
  const int E = ctx->P.E, N = ctx->P.N;
  if ((long long)spec->counts[0] * spec->counts[1] * spec->counts[2] != N || spec->counts[0] < 1 ||
      spec->counts[1] < 1 || spec->counts[2] < 1) {
    ctx->err = "dm_reset_lattice: counts[0] * counts[1] * counts[2] must equal particles_per_env";
    return DM_ERR_ARG;
  }
  if (spec->origin_draws < 0 || spec->origin_draws > 3 || spec->material < 0 || spec->material >= ctx->nmat ||
      spec->group < 0 || (ctx->P.G > 0 ? spec->group >= ctx->P.G : spec->group > 0)) {
    ctx->err = "dm_reset_lattice: origin_draws must be 0..3 and material / group in range";
    return DM_ERR_ARG;
  }
  if (ctx->poisoned && ctx->h_flags->err_key == ~0ull) ctx->poisoned = false;
  // scratch in the (idle) particle-cotangent buffer: mask, groups, deltas, flags
  unsigned char* base = reinterpret_cast<unsigned char*>(ctx->part);
  double* d_delta = reinterpret_cast<double*>(base);
  int* d_flag = reinterpret_cast<int*>(base + (size_t)E * 3 * sizeof(double));
  int* d_group = d_flag + E;
  unsigned char* d_mask = reinterpret_cast<unsigned char*>(d_group + N);
  const unsigned char* m = mask;
  const int* g = pgroup;
  if (!dev) {
    if (mask) DM_CUDA(cudaMemcpyAsync(d_mask, mask, E, cudaMemcpyHostToDevice, ctx->stream));
    if (pgroup) DM_CUDA(cudaMemcpyAsync(d_group, pgroup, (size_t)N * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    m = mask ? d_mask : nullptr;
    g = pgroup ? d_group : nullptr;
  }
  DM_CUDA(cudaMemsetAsync(d_flag, 0, (size_t)E * sizeof(int), ctx->stream));
  DM_CUDA(cudaMemsetAsync(d_delta, 0, (size_t)E * 3 * sizeof(double), ctx->stream));
  // the unmasked envs' current state becomes the new initial state
  const StateView S0 = store_view(ctx, 0);
  const StateView cur = fwd_state(ctx, ctx->steps * ctx->cfg.substeps);
  if (mask && cur.f != S0.f) {
    DM_CUDA(cudaMemcpyAsync(S0.f, cur.f, state_floats(ctx) * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    DM_CUDA(cudaMemcpyAsync(S0.attr, cur.attr, ctx->Ntot * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    if (ctx->law == kFluid) {  // the kept envs' F becomes a general initial state
      dm_launch(ctx->grid_tiles, 256, 0, ctx->stream, ctx->pdl, k_fiso_expand, ctx->Ntot, S0);
      ++ctx->launches;
    }
  }
  ResetSpec R;
  for (int a = 0; a < 3; ++a) {
    R.org[a] = spec->origin[a];
    R.sp[a] = spec->spacing[a];
    R.size[a] = spec->size[a];
    R.cnt[a] = spec->counts[a];
  }
  R.odraws = spec->origin_draws;
  R.olo = spec->origin_lo;
  R.ohi = spec->origin_hi;
  R.jlo = spec->jitter_lo;
  R.jhi = spec->jitter_hi;
  R.sigma = spec->velocity_sigma;
  R.material = spec->material;
  R.group = spec->group;
  double* od = odelta ? (dev ? odelta : d_delta) : nullptr;
  dm_launch(ctx->grid_tiles, 256, 0, ctx->stream, ctx->pdl, k_reset_lattice, R, E, N, seed, env_offset, m, g, od, d_flag, S0);
  dm_launch((E + 127) / 128, 128, 0, ctx->stream, ctx->pdl, k_reset_normals_seq, R, E, N, seed, env_offset, d_flag, S0);
  ctx->launches += 2;
  if (odelta && !dev)
    DM_CUDA(cudaMemcpyAsync(odelta, d_delta, (size_t)E * 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->steps = 0;
  ctx->cfl_checked = 0;
  ctx->bwd_t = -1;
  ctx->kept_t = -1;
  ctx->kept_ok = false;
  ctx->poisoned = false;
  const int rc = reset_flags(ctx);  // synchronises the stream
  if (rc != DM_OK) return rc;
  DM_CUDA(cudaGetLastError());
  return DM_OK;
}
}  // namespace

int dm_reset_lattice(DmContext* ctx, const DmLatticeReset* spec, unsigned long long seed, int env_offset,
                     const unsigned char* env_mask, const int* particle_group, double* origin_delta) {
  return reset_lattice_impl(ctx, spec, seed, env_offset, env_mask, particle_group, origin_delta, false);
}
int dm_reset_lattice_device(DmContext* ctx, const DmLatticeReset* spec, unsigned long long seed, int env_offset,
                            const unsigned char* env_mask, const int* particle_group, double* origin_delta) {
  return reset_lattice_impl(ctx, spec, seed, env_offset, env_mask, particle_group, origin_delta, true);
}

int dm_get_state(DmContext* ctx, float* x, float* v, float* F, float* C) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return get_state_impl(ctx, x, v, F, C, cudaMemcpyDeviceToHost);
}
int dm_get_state_device(DmContext* ctx, float* x, float* v, float* F, float* C) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return get_state_impl(ctx, x, v, F, C, cudaMemcpyDeviceToDevice);
}
int dm_step(DmContext* ctx, const float* cvo, const float* act, float* obs) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return step_impl(ctx, cvo, act, obs, cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost);
}
int dm_step_device(DmContext* ctx, const float* cvo, const float* act, float* obs) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return step_impl(ctx, cvo, act, obs, cudaMemcpyDeviceToDevice, cudaMemcpyDeviceToDevice);
}
int dm_backward(DmContext* ctx, const float* dobs, const float* dfx, const float* dfv, const float* dfF,
                const float* dfC, float* dx0, float* dv0, float* dF0, float* dC0, float* dcvo, float* dact, double* dE) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return backward_impl(ctx, dobs, dfx, dfv, dfF, dfC, dx0, dv0, dF0, dC0, dcvo, dact, dE, cudaMemcpyHostToDevice,
                       cudaMemcpyDeviceToHost);
}
int dm_backward_device(DmContext* ctx, const float* dobs, const float* dfx, const float* dfv, const float* dfF,
                       const float* dfC, float* dx0, float* dv0, float* dF0, float* dC0, float* dcvo, float* dact,
                       double* dE) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return backward_impl(ctx, dobs, dfx, dfv, dfF, dfC, dx0, dv0, dF0, dC0, dcvo, dact, dE, cudaMemcpyDeviceToDevice,
                       cudaMemcpyDeviceToDevice);
}

int dm_profile(DmContext* ctx, int enable, double* ms, long long* counts) {
  if (!ctx) return DM_ERR_ARG;
  prof_flush(ctx);
  for (int i = 0; i < kProfClasses; ++i) {
    if (ms) ms[i] = ctx->prof_ms[i];
    if (counts) counts[i] = ctx->prof_n[i];
    ctx->prof_ms[i] = 0.0;
    ctx->prof_n[i] = 0;
  }
  ctx->prof = enable != 0;
  return DM_OK;
}

int dm_backward_begin(DmContext* ctx, const float* dfx, const float* dfv, const float* dfF, const float* dfC) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return backward_begin(ctx, dfx, dfv, dfF, dfC, cudaMemcpyHostToDevice);
}
int dm_backward_begin_device(DmContext* ctx, const float* dfx, const float* dfv, const float* dfF, const float* dfC) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return backward_begin(ctx, dfx, dfv, dfF, dfC, cudaMemcpyDeviceToDevice);
}
int dm_backward_step(DmContext* ctx, const float* dobs_t, float* dcvo_t, float* dact_t) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return backward_step(ctx, dobs_t, dcvo_t, dact_t, cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost);
}
int dm_backward_step_device(DmContext* ctx, const float* dobs_t, float* dcvo_t, float* dact_t) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return backward_step(ctx, dobs_t, dcvo_t, dact_t, cudaMemcpyDeviceToDevice, cudaMemcpyDeviceToDevice);
}
int dm_backward_end(DmContext* ctx, float* dx0, float* dv0, float* dF0, float* dC0, double* dE) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return backward_end(ctx, dx0, dv0, dF0, dC0, dE, cudaMemcpyDeviceToHost);
}
int dm_backward_end_device(DmContext* ctx, float* dx0, float* dv0, float* dF0, float* dC0, double* dE) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  return backward_end(ctx, dx0, dv0, dF0, dC0, dE, cudaMemcpyDeviceToDevice);
}
int dm_obs_dim(const DmContext* ctx) { return ctx ? ctx->od : DM_OBS_DIM; }

int dm_sync(DmContext* ctx) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  if (ctx->poisoned) return DM_ERR_RUNTIME;
  return check_flags(ctx);
}

int dm_debug_inject(DmContext* ctx, int step, int env, int particle) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  if (env < 0 || env >= ctx->P.E || particle < 0 || particle >= ctx->P.N) {
    ctx->err = "dm_debug_inject: env / particle out of range";
    return DM_ERR_ARG;
  }
  ctx->inj_step = step;
  ctx->inj_env = env;
  ctx->inj_particle = particle;
  return DM_OK;
}

static int observe_impl(DmContext* ctx, const float* cvo, float* obs, cudaMemcpyKind kin, cudaMemcpyKind kout) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  if (ctx->poisoned) return DM_ERR_RUNTIME;
  const int E = ctx->P.E, K = ctx->P.K;
  // the pose and the output have their own buffers: the tape's recorded
  // poses and observables stay untouched (a later backward reads the poses)
  DevParams P = ctx->P;
  if (K > 0 && cvo)
    DM_CUDA(cudaMemcpyAsync(ctx->obs_cvo, cvo, (size_t)E * K * 9 * sizeof(float), kin, ctx->stream));
  else
    P.K = 0;  // no pose: no spill statistic
  float* o = ctx->obs_out;
  dm_launch(E, 256, 0, ctx->stream, ctx->pdl, k_obs, P, fwd_state(ctx, ctx->steps * ctx->cfg.substeps), ctx->obs_cvo,
                                    (float)ctx->cfg.spill_half, (float)ctx->cfg.spill_temp, ctx->cfg.obs_groups, o,
                                    ctx->od, (const float*)nullptr);
  ++ctx->launches;
  DM_CUDA(cudaMemcpyAsync(obs, o, (size_t)E * ctx->od * sizeof(float), kout, ctx->stream));
  if (kout != cudaMemcpyDeviceToDevice) DM_CUDA(cudaStreamSynchronize(ctx->stream));
  return DM_OK;
}
int dm_observe(DmContext* ctx, const float* cvo, float* obs) {
  return observe_impl(ctx, cvo, obs, cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost);
}
int dm_observe_device(DmContext* ctx, const float* cvo, float* obs) {
  return observe_impl(ctx, cvo, obs, cudaMemcpyDeviceToDevice, cudaMemcpyDeviceToDevice);
}

int dm_debug_sort(DmContext* ctx, int* keys, int* perm) {
  if (!ctx || !ctx->store) return DM_ERR_ARG;
  const int s = ctx->steps * ctx->cfg.substeps;
  ctx->kept_ok = false;  // slot 0 is overwritten
  launch_bin(ctx, fwd_state(ctx, s), slot(ctx, 0), 0, 0);
  const size_t N = ctx->Ntot;
  std::vector<int> p(N);
  DM_CUDA(cudaMemcpyAsync(keys, ctx->keys, N * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  DM_CUDA(cudaMemcpyAsync(p.data(), slot(ctx, 0).perm, N * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  DM_CUDA(cudaStreamSynchronize(ctx->stream));
  for (size_t i = 0; i < N; ++i) perm[i] = p[i] - (int)((i / ctx->P.N) * ctx->P.N);
  return check_flags(ctx);
}

}  // extern "C"

#include "dm_task.cuh"
