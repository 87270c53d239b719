// cbx_device.cuh -- device-side state layout and kernel parameter block.
#pragma once

#include <cuda_runtime.h>

#include "../../include/cascade_b200.h"
#include "cbx_internal.h"

namespace cbx {

// spline table on the device: the reference's 7-coefficient segments
// (spline.h:19-22) plus the evaluation constants
// fast-path spline records: 32-byte aligned, normalised s = (r - x0)/h - i,
// segment nseg padded with the last segment re-expanded at s + 1
struct FastTab {
  const double* rec;  // density: 4 doubles/segment (A B C D); force: 8 (z A-D, rho A-D)
  double ih, c0;      // u = r*ih + c0
  int nseg;
};

struct Tab {
  const double* seg;  // 7 doubles per segment
  double x0, h, ih, xl;
  int nseg;
};

// clash list: records sorted by (key, bucket order); interior records and
// their ghost images (gf = 1) share one array.  head[dev] -> first record.
struct Clash {
  long long* key;      // reference site id of the bucket
  long long* hkey;     // new hash computed by k_clash_kick_drift
  unsigned char* gf;   // ghost image?
  int* src;            // ghost image: index of its interior source record
  double *px, *py, *pz, *vx, *vy, *vz, *fx, *fy, *fz;
  double *rho, *df;
  double *e_emb, *e_pair, *v2;  // per-record partials (deterministic sums)
  unsigned long long* tag;
};

// pass-1 evictees of update_hash (store.cpp:46-54)
// rehash items: key = new hash (local id); (walk, cls, sub) = the record's
// position in the reference's pass-2 walk (store.cpp:59-75): walk key of the
// bucket it is visited in, class 0 = earlier bucket member / 1 = pass-1
// evictee, sub = bucket order or old site id
struct Movers {
  long long *key, *walk, *sub;
  int* cls;
  double *px, *py, *pz, *vx, *vy, *vz;
  unsigned long long* tag;
  int* dir;  // outbound list only: -1 / +1 neighbour rank
};

// single-block sort scratch
struct Scratch {
  long long *k1, *k2, *k3;
  int *pl, *flag, *pos;
};

struct DevStatus {
  int err;  // cbx_status of the first store error (domain / logic / capacity)
  int n_ovl;
  unsigned long long ovl_key[kMaxOverlapRecords];
  unsigned long long ovl_a[kMaxOverlapRecords], ovl_b[kMaxOverlapRecords];
  double ovl_r2[kMaxOverlapRecords];
  double err_pos[3];
  unsigned long long r_underflow, rho_clamp;
  int n_clash, n_mov, n_out, n_remote;
  // StepState mirror (sim.h:11-21)
  long long step;
  double t, dt, kinetic, pair, embedding, max_speed;
  double dt_next;  // dt of the next step (fixed, or adaptive_dt from max_speed)
  int adaptive;
  double dt_max, max_disp;
  unsigned long long cnt_cand, cnt_pair;
  unsigned fin_count;  // blocks of k_kick2 done (the last one runs the finalize)
  // deferred finalize: the StepState sums of the last k_kick2 run later, in
  // an otherwise idle block of the next step's k_kick_drift (fixed dt) or
  // before the host reads the status (k_finalize_pending)
  int fin_pending, fin_stepping, fin_energies;
  int fin_nemb, fin_npp, fin_nke;  // partial counts of the pending sums
  int fin_clash;  // > 0: the clash records' sums are in that many reserved slots
  int fin_bad;    // err | n_ovl when the sums were deferred (their step's outcome)
  int fin_reduce; // slab ranks (peer memory): the cross-rank reduction follows the sums
  // a step of the current multi-step replay failed (set by k_rehash_images of
  // the next step from the stable status words): the passes of the remaining
  // steps are no-ops, so the store stays at the failing step (sim.cpp:303-315)
  int halt;
  // merged kick: the step's second half kick is pending and runs in the next
  // step's k_kick_drift (set by the force pass, consumed by k_rehash_images)
  int k2_pending;
};

// clash blocks of k_kick_drift / k_kick2, and the reserved partial slots
// (the last kClashSlots of each partial array) of the merged kick
constexpr int kClashSlots = 8;

struct P2PLinks;

// Reverse halo fused into the passes (z-slab ranks on the peer-memory
// transport, Newton-3 stencil): a density / force partial for a site of my
// halo planes is added straight into the owning neighbour's boundary site
// (peer memory over NVLink) instead of being staged and sent by the RHO / FRC
// exchanges.  Index 0: the neighbour below, 1: above.
struct RevHalo {
  double* rho[2];
  double* frc[2];    // 3 planes of S[q]
  long long S[2], NC[2];
  long long lo, hi;  // my halo cells: cell < lo (below) or cell >= hi (above)
  // cell shift of my halo block into the neighbour's frame (the halo planes'
  // x/y images are already folded by tgt, so a partial's target is an owner
  // column of the plane)
  long long delta[2];
  int on;
};

// records of the density spline staged in shared memory by the density pass
// (x 32 B = 105,600 B; x 24 B compressed), and the first staged record of the
// compressed window: even, so the fp32 [A B] pairs (8 B each) start 16-byte
// aligned for the bulk copy (host: the fp32 guard covers exactly this window)
constexpr int kDensTabRecords = 3300;
__host__ __device__ __forceinline__ int dens_window_lo_cmp(int nseg) {
  const int lo = nseg + 2 - kDensTabRecords;
  return ((lo > 0 ? lo : 0) + 1) & ~1;
}

// records of the force spline window staged in shared memory by the force
// pass (contiguous: the top kLeanTabRecords records).  Split-3 layout (24 B
// per record): when the lattice leaves a stretch of r between two neighbour
// shells that no pair visits short of a cascade core, the window skips it and
// fits kLeanTabRecordsGap records -- 62.4 KB, inside the 64 KB shared-memory
// carveout instead of the 100 KB one, i.e. 36 KB more L1 for the partner
// gathers and the texture fetches (capi.cu force_window_setup)
constexpr int kLeanTabRecords = 3300;
constexpr int kLeanTabRecordsGap = 2600;

// Regional displacement bound (density-pass skin pruning).  One entry per
// chunk of 32 interior cells of an x row (both sublattices), written by
// k_kick_drift: (stamp << kUbShift) | q, q >= |u| * kUbScale for every atom of
// the chunk, u = its position minus its own site's lattice position.  A chunk
// whose atom left the fast hash (wrap / new site) or received an atom in
// update_hash pass 2 carries kUbQMax ("unbounded").  ustamp[0] is the stamp
// the density pass accepts (0: no valid bounds), ustamp[1] the stamp of the
// next k_kick_drift; k_rehash(_images) publishes it after pass 2.
constexpr int kUbShift = 24;
constexpr unsigned long long kUbQMax = (1ull << kUbShift) - 1;
constexpr double kUbScale = 65536.0;  // q in units of 2^-16 A
constexpr double kUbDirty = 1e300;    // per-site marker: no bound
// skin shells of an offset list: offsets [nin, end[0]) have lattice
// distance len[0] (A), [end[0], end[1]) at least len[1], ... (ascending)
struct SkinGroups {
  double len[4];
  int end[4];
  int n;
};

struct KP {
  Geo G;
  unsigned long long* ub;      // regional displacement bounds (null: off)
  unsigned long long* ustamp;  // [2]
  SkinGroups skh[2], skf[2];   // half / full lists per sublattice
  int skin_reach[2];           // cells a skin offset reaches per axis (half, full lists)
  // [3]: skin candidates examined / listed by the density pass, counting on
  // (cbx_skin_stats; a device word, so captured step graphs see it)
  unsigned long long* skin_cnt;
  RevHalo rev;
  P2PLinks* lk;  // device copy of the peer links (fused reverse halo signals)
  int rev_wait;  // per launch: wait for the neighbours' flags of this exchange first
  float4* uf;      // fp32 shadow (x, y, z, owner-or--1) for the candidate filter
  int* work;       // persistent-kernel work counters (zeroed per launch)
  FastTab fd, ff;  // density / force fast tables
  // force-table chunks staged in shared memory by the force pass (fp64):
  // [zA zB zC zD] per record (32 B); [zC zD] (16 B) and qC (8 B) per record
  // (split-3); the full 64-byte records ff.rec are also bound to the texture
  // tex_ff (int4 texels, 4 per record) for the chunks fetched through TEX
  const double *ffz, *ffzc, *ffqc;
  unsigned long long tex_ff;  // cudaTextureObject_t
  const double* ffab;         // [zA zB qA qB] per segment (32 B), bound to tex_fab (int4 texels, 2 per segment)
  unsigned long long tex_fab;
  unsigned long long tex_fd;  // the compressed density records' [D C] (int4 texels)
  // compressed density records: [D C] (16 B) then, after the last record,
  // [A B as fp32] (8 B) per record; null when the fp32 rounding bound fails
  const double* fdc;
  // fp64 density records for the density pass: [A B] pairs (16 B per
  // record, staged in shared memory) and the [C D] pairs bound to a texture
  // (one int4 texel per record); nin64: every inner list fits one 64-bit
  // mask word
  const double* fdab;
  unsigned long long tex_fd4;
  int nin64;
  FastTab fe;      // embedding F(rho): 4 doubles/segment (A B C D), padded
  float band_hi, band_lo;  // fp32 r^2 filter: reject above hi, exact test in [lo, hi]
  double guard_r2;         // below: overlap / short-range guard path
  double cut2_lo, cut2_hi; // fp64 (FMA) r^2 decides outside [lo, hi]; exact r^2 inside
  struct KP* dself;        // this parameter block in device memory (guard paths)
  unsigned long long* pmask;  // [S][2] pair masks from the density pass (or null)
  int use_mask;               // force pass replays pmask (set per launch by the host)
  int mark_k2;                // force pass: mark the second half kick pending (merged kick)
  int offs_const;             // force pass: stencil offsets from the constant cache (else smem)
  int unit_rr;                // stencil passes: round-robin unit batches (0: contiguous ranges)
  int idle_pred;              // force pass: idle lanes of the union walk issue no gather
  // force pass, split-3 table: the shared-memory window holds records
  // [fw_lo, nseg] minus [fw_gap_lo, fw_gap_lo + fw_gap_n) (fw_gap_n == 0:
  // contiguous, fw_gap_lo = INT_MAX); fw_cap records of capacity
  int fw_lo, fw_gap_lo, fw_gap_n, fw_cap;
  int tab_packed;             // force pass: the TEX-fetched chunks from the packed [zA zB qA qB] array
  int skin_lane;              // force pass: each lane walks its own skin bits after the inner union
  // fast hash: an atom closer than sqrt(hash_r2) to its own site (the
  // half nearest-neighbour distance sqrt(3)/4 a0 less a margin far above
  // rounding) hashes to that site and needs no periodic wrap (0: off)
  double hash_r2;
  int n_pair_part;         // partials written by the force pass
  double accel, mv2;  // units::accel_factor, units::mv2_to_ev (units.h:17-24)
  long long S;  // 2*NC sites
  double4* pdf;  // x y z dF
  double* rho;
  double* vel;  // 3 planes of S
  double* frc;  // 3 planes of S
  unsigned long long* tag;
  int* tgt;  // owner of a site: itself (interior) or its periodic source (ghost)
  int *gh_dst, *gh_src;
  signed char* gh_k;  // 3 per ghost: box shifts (store.cpp:166-169)
  long long n_gh;
  int* head;
  Clash cl, cl2;
  int cap_clash;
  Movers mv;
  Movers out;      // outbound migrants (z-slab decomposition)
  int cap_mov;
  Clash rem;       // remote clash sources received with the position halo
  int cap_rem;
  Scratch sc;
  int cap_items;  // power of two
  Tab dens, zr, emb;
  double cutoff, cut2, mass;
  double *part_emb, *part_pair, *part_ke, *part_vmax;

  int n_part;
  int count_pairs;
  DevStatus* st;
};

#if defined(__CUDACC__)
// thread -> (parity, interior cell): blocks of 8 warps cover 128 cells,
// warps 0-3 the even sublattice, 4-7 the odd one (warp-uniform offset lists)
__device__ __forceinline__ bool map_site(const KP& P, int& par, long long& d, int vb = -1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  par = warp >> 2;
  const long long e = (long long)(vb < 0 ? (int)blockIdx.x : vb) * 128 + (warp & 3) * 32 + lane;
  if (e >= P.G.NI) return false;
  d = par * P.G.NC + interior_cell(e, P.G);
  return true;
}

// map_site that also returns the ghost-inclusive cell coordinates of the
// site (one magic-number division pair, reused by the caller)
__device__ __forceinline__ bool map_site_xyz(const KP& P, int vb, int& par, long long& d,
                                             int& cx, int& cy, int& cz) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  par = warp >> 2;
  const long long e = (long long)vb * 128 + (warp & 3) * 32 + lane;
  if (e >= P.G.NI) return false;
  const Geo& G = P.G;
  if (e < (1ll << 31)) {
    const unsigned u = (unsigned)e, r = magic_div(u, G.mbx, G.sbx);
    const unsigned q = magic_div(r, G.mby, G.sby);
    cx = (int)(u - r * (unsigned)G.bx) + G.g;
    cy = (int)(r - q * (unsigned)G.by) + G.g;
    cz = (int)q + G.g;
  } else {
    const long long r = e / G.bx;
    cx = (int)(e - r * G.bx) + G.g;
    cy = (int)(r % G.by) + G.g;
    cz = (int)(r / G.by) + G.g;
  }
  d = par * G.NC + cell_of(cx, cy, cz, G);
  return true;
}

// read-only 32-byte record load through the non-coherent path
__device__ __forceinline__ double4 ldg4(const double4* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// deterministic block reduction (fixed tree); result valid in thread 0
template <int N>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < N / 32; ++i) s += sh[i];
  __syncthreads();
  return s;
}
template <int N>
__device__ __forceinline__ double block_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < N / 32; ++i) s = fmax(s, sh[i]);
  __syncthreads();
  return s;
}

__device__ __forceinline__ void set_error(DevStatus* st, int code) { atomicCAS(&st->err, 0, code); }

// zero the pair-energy partials no block of this launch writes (entries
// [written, n_pair_part)), so the finalize sums a fixed range without a
// memset before every force pass
// where a partial for site t goes: locally, or (fused reverse halo, halo
// plane) into the neighbour's boundary site
template <int A>
__device__ __forceinline__ double* acc_ptr(const KP& P, long long t) {
  if (P.rev.on) {
    const int par = t >= P.G.NC;
    const long long c = par ? t - P.G.NC : t;
    if (c < P.rev.lo || c >= P.rev.hi) {
      const int up = c >= P.rev.hi;
      const long long d = (up ? P.rev.NC[1] : P.rev.NC[0]) * par + c +
                          (up ? P.rev.delta[1] : P.rev.delta[0]);
      if (A < 0) return (up ? P.rev.rho[1] : P.rev.rho[0]) + d;
      return (up ? P.rev.frc[1] : P.rev.frc[0]) + A * (up ? P.rev.S[1] : P.rev.S[0]) + d;
    }
  }
  return A < 0 ? P.rho + t : P.frc + (long long)A * P.S + t;
}

// the hot-loop form for the Newton-3 slot passes, whose half-list partners
// lie at dz >= 0: only the upper halo can be hit; 32-bit site arithmetic
__device__ __forceinline__ double* acc_ptr_up(const KP& P, int t, int A) {
  const int NC = (int)P.G.NC;
  const int par = t >= NC;
  const int c = t - (par ? NC : 0);
  if (c >= (int)P.rev.hi) {
    const long long d = par * P.rev.NC[1] + c + P.rev.delta[1];
    return A < 0 ? P.rev.rho[1] + d : P.rev.frc[1] + d;
  }
  return A < 0 ? P.rho + t : P.frc + t;
}

__device__ __forceinline__ void zero_pair_tail(const KP& P, int written) {
  if (blockIdx.x == 0)
    for (int i = written + threadIdx.x; i < P.n_pair_part; i += blockDim.x) P.part_pair[i] = 0.0;
}

// Programmatic dependent launch (PDL) on the step path: a kernel launched by
// launch_pdl may start while its predecessor in the stream drains (its CTAs
// take SMs as the predecessor's leave, its launch latency and constant-table
// staging overlap the predecessor's tail).  Every such kernel executes
// pdl_wait() -- which returns once the predecessor grid has completed and its
// writes are visible -- before it reads or writes anything the stream's
// earlier work touches, then pdl_trigger() to let its own successor launch.
// Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();  // CBX_PDL (default on)
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, args...);
}
#endif

#if defined(__CUDACC__)
// shared-memory loads through a 32-bit shared address held in a register
// (the generic-to-shared conversion is done once per kernel, not per load)
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// ---- bulk (TMA engine) staging of a constant table into shared memory:
// one thread arms an mbarrier with the byte count and issues 1-D bulk
// copies; every thread waits on the barrier's phase 0.  Spares the per-thread
// load/store round trips of a copy loop at kernel start.
__device__ __forceinline__ void mbar_init(unsigned mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned mbar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes,
                                         unsigned mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait0(unsigned mbar) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra WAIT%=;\n}" ::"r"(mbar)
      : "memory");
}
// bytes (multiple of 16, both addresses 16-byte aligned) in chunks of 32 KB;
// called by one thread after mbar_init
__device__ __forceinline__ void bulk_stage(unsigned dst, const void* src, unsigned bytes,
                                           unsigned mbar) {
  const char* s = static_cast<const char*>(src);
  for (unsigned o = 0; o < bytes; o += 32768u)
    bulk_g2s(dst + o, s + o, min(32768u, bytes - o), mbar);
}

// wait for the phase of parity `ph` of an mbarrier (multi-stage pipelines)
__device__ __forceinline__ void mbar_wait(unsigned mbar, unsigned ph) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT%=;\n}" ::"r"(mbar), "r"(ph)
      : "memory");
}
#endif

// device entry points (launch wrappers), implemented in the .cu files
bool launch_density(const KP& P, int mode, cudaStream_t s);  // true: clash pass fused
void launch_clash_density(const KP& P, cudaStream_t s);
// literal: the reference arithmetic of spline_eval (stencil mode 2)
void launch_embed(const KP& P, cudaStream_t s, bool literal = false);
bool launch_force(const KP& P, int mode, cudaStream_t s);
int force_table_mode();  // the force pass's table source (kTabSplit, ...)
void launch_clash_force(const KP& P, cudaStream_t s);
// zero_acc: clear the interior sites' rho / force accumulators as well;
// images: write each site's ghost images too (the step path, no ghost fill)
void launch_kick_drift(const KP& P, int move, cudaStream_t s, int zero_acc = 0, int images = 0,
                       int n_pairp = 0);
// update_hash pass 2 + ghost clash images in one single-block launch
void launch_clash_zero(const KP& P, int what, cudaStream_t s);
void launch_rehash(const KP& P, cudaStream_t s, int merge = 0, int n_emb = 0, int n_pairp = 0,
                   int n_ke = 0);
void launch_ghost_fill(const KP& P, cudaStream_t s);
// zero_rho: also zero the records' density accumulators (density follows)
void launch_clash_images(const KP& P, cudaStream_t s, int zero_rho = 0);
// second half kick; stepping > -2 also runs the finalize (last block)
// fin: 1 the StepState finalize in the last block, 2 deferred (fin_pending);
// n_pairp: pair-energy partials written by the preceding force pass
void launch_kick2(const KP& P, int kick, int stepping, int energies, cudaStream_t s, int fin = 1,
                  int n_pairp = -1);
void launch_finalize_pending(const KP& P, cudaStream_t s);
// merge != 0: a pending second half kick found by k_kick_drift is marked
// consumed here and the previous step's StepState sums are marked pending
// (for the density pass's idle block), with these partial counts
void launch_rehash_images(const KP& P, cudaStream_t s, int merge, int n_emb, int n_pairp,
                          int n_ke);
int force_partials(const KP& P, int mode);  // partials the force launch writes
int kick_drift_grid(const KP& P);           // KE partials of a merged-kick k_kick_drift
bool kd_bulk(const KP& P);                  // k_kick_drift_bulk (bx % 128 == 0)

void launch_count_defects(const KP& P, unsigned long long* out, cudaStream_t s);
void upload_offsets(const int* half_dev[2], const int half_n[2], const int* full_dev[2],
                    const int full_n[2], const long long* full_flat[2], const int half_nin[2],
                    const int full_nin[2], cudaStream_t s);
int eam_blocks(const KP& P);
int pair_partials(const KP& P, int mode);
void launch_uf_refresh(const KP& P, cudaStream_t s);
long long slab_buffer_bytes(const KP& P, int kind);
constexpr long long kMsgRecords = 8192;  // clash / migrant records per in-graph message

// peer-memory links of one slab rank (P2P transport).  Exchange kinds 0-4;
// index 5 of epoch/done is the StepState reduction.  [k][0] is the packet
// toward / from the rank below, [k][1] toward / from the rank above.
struct P2PLinks {
  unsigned char* dst[5][2];               // neighbours' receive buffers for my packets
  const unsigned char* src[5][2];         // my receive buffers
  unsigned long long* flag_dst[5][2];     // neighbours' flags raised after my packets
  const unsigned long long* flag_src[5][2];
  unsigned long long* epoch;              // [6] exchanges completed (this rank)
  unsigned* done;                         // [6] block arrival counters of k_p2p_send
  long long msg[5], plane_bytes[5];
  double* red_dst[8];                     // every rank's reduction slots [8][4]
  unsigned long long* red_flag_dst[8];    // every rank's reduction flags [8]
  const double* red_src;
  const unsigned long long* red_flag_src;
  int rank, nranks;
};
constexpr int kMaxP2PRanks = 8;
// links (device copy): slab rank on the P2P transport -- the cross-rank
// reduction runs in the same kernel
void launch_finalize(const KP& P, int stepping, int energies, cudaStream_t s,
                     const P2PLinks* links = nullptr);
int launch_p2p_exchange(const KP& P, const P2PLinks& L, int kind, long long gs_lo,
                         long long gs_hi, int* rem_base, cudaStream_t s);
void launch_p2p_send(const KP& P, const P2PLinks& L, int kind, cudaStream_t s);
void launch_p2p_recv(const KP& P, const P2PLinks& L, int kind, long long gs_lo, long long gs_hi,
                     int* rem_base, cudaStream_t s);
void launch_p2p_reduce(const KP& P, const P2PLinks& L, int energies, int kinetic,
                       cudaStream_t s);
// fused reverse halo: raise the neighbours' flags of exchange `kind` (2 RHO,
// 4 FRC) once the pass that added into their memory has completed
void launch_rev_signal(const KP& P, int kind, cudaStream_t s);
// wait for both neighbours' flags of exchange `kind` (a consumer that is not
// k_embed / k_kick2, e.g. the evaluation's finalize)
void launch_rev_wait(const KP& P, int kind, cudaStream_t s);
long long slab_msg_bytes(const KP& P, int kind);
long long slab_plane_bytes(const KP& P, int kind);
void launch_slab_red_in(const KP& P, double* red, cudaStream_t s);
void launch_slab_red_out(const KP& P, const double* red, int energies, int kinetic, cudaStream_t s);
void launch_pack(const KP& P, int kind, int dir, unsigned char* buf, long long cap,
                 cudaStream_t s);
void launch_unpack(const KP& P, int kind, int from, const unsigned char* buf, long long gshift,
                   int* rem_base, cudaStream_t s);
void launch_remote_df(const KP& P, cudaStream_t s);

int embed_blocks(const KP& P);
int embed_grid(const KP& P);  // energy partials of the embed pass
int kick_grid(const KP& P);   // KE partials of the kick2 pass

}  // namespace cbx
