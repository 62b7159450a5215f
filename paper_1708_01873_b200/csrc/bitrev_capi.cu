// bitrev_capi.cu -- extern "C" entry points of libbitrev_sm100a.so (declared in
// include/bitrev_b200.h): argument checks, kernel selection, launch geometry.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <map>
#include <memory>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "bitrev_b200.h"
#include "bitrev_kernels.cuh"

using namespace bitrev_b200;

namespace {

constexpr int kMaxBits = 48;  // src/bits.py:15-18 MAX_BITS
constexpr int kMaxDevices = 64;

std::atomic<int64_t> g_launches{0};

// Tile bits in use per (element size, kernel family); 0 = default.
// Defaults chosen by measurement on B200 (see DESIGN.md / profiles/).
std::atomic<int> g_q_oop[17];
std::atomic<int> g_q_ip[17];

// Large-size defaults, measured on B200 with interleaved rounds (tools/
// tune_all.py, rect_qz.py, sweep.py; profiles/tune_r01*, r01_rect_qz*,
// r01_inplace_cluster_ab): tile bits Q and staging path per (E, family).
// Smaller launches are re-routed by mid_tier and by the short-row kernels.
int default_q(int E, bool inplace) {
  switch (E) {
    case 4: return inplace ? 6 : 8;   // out of place: rectangular QX = 8 (path 3)
    case 8: return inplace ? 6 : 7;   // out of place: rectangular QX = 7 (path 3)
    case 16: return 6;                // 1 KB rows: square tiles / in place 2-CTA cluster pairs
    default: return 0;
  }
}

bool q_supported(int E, int q) {
  switch (E) {
    case 4: return q >= 5 && q <= 8;
    case 8: return q >= 4 && q <= 8;
    case 16: return q >= 3 && q <= 7;
    default: return false;
  }
}

int current_q(int E, bool inplace) {
  if (E != 4 && E != 8 && E != 16) return 0;
  const int v = inplace ? g_q_ip[E].load() : g_q_oop[E].load();
  return v ? v : default_q(E, inplace);
}

// Tile visit order (work_to_y in bitrev_kernels.cuh).  Defaults chosen by
// measurement; BITREV_B200_ORDER_OOP / BITREV_B200_ORDER_IP override them.
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

std::atomic<int> g_order_oop{-1}, g_order_ip{-1};

// Staging path per (element size, family): 0 = register tiles (LDG/STS),
// 1 = TMA bulk ring, 2 = TMA tensor ring, 3 = rectangular tiles (out of
// place), 4 = cp.async pairs, 5 = TMA-store pairs, 6 = 2-CTA cluster pairs
// (in place).  -1 = not yet read from the environment (BITREV_B200_PATH_OOP /
// BITREV_B200_PATH_IP), else default.
std::atomic<int> g_path_oop[17] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
std::atomic<int> g_path_ip[17] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};

int default_path(int E, bool inplace) {
  // in place: register tile pairs (compact pair enumeration); complex128 pairs
  // of 1 KB-row tiles split over 2-CTA clusters (profiles/r01_inplace_cluster_ab.jsonl)
  if (inplace) return E == 16 ? 6 : 0;
  switch (E) {
    case 4:
    case 8: return 3;     // rectangular register tiles (1 KB destination rows)
    default: return 0;    // square register tiles (E=16: 1 KB rows both sides)
  }
}

int tile_path(int E, bool inplace) {
  if (E != 4 && E != 8 && E != 16) return 0;
  std::atomic<int>& p = inplace ? g_path_ip[E] : g_path_oop[E];
  int v = p.load();
  if (v < 0) {
    v = env_int(inplace ? "BITREV_B200_PATH_IP" : "BITREV_B200_PATH_OOP", default_path(E, inplace));
    p.store(v);
  }
  return v;
}

int tile_order(bool inplace) {
  std::atomic<int>& o = inplace ? g_order_ip : g_order_oop;
  int v = o.load();
  if (v < 0) {
    // in place: compact pair enumeration (2); out of place: y = work index (0)
    v = env_int(inplace ? "BITREV_B200_ORDER_IP" : "BITREV_B200_ORDER_OOP", inplace ? 2 : 0);
    o.store(v);
  }
  return v;
}

struct DevInfo {
  int sms = 0;
};
DevInfo g_dev[kMaxDevices];
std::mutex g_dev_mu;

int device_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (g_dev[dev].sms == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_dev[dev].sms = v > 0 ? v : 148;
  }
  return g_dev[dev].sms;
}

bool valid_elem(int E) { return E == 1 || E == 2 || E == 4 || E == 8 || E == 16; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int finish_launch() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BITREV_OK : (int)e;
}

int grid_for(uint64_t work, int per_sm, int threads_hint = 0) {
  (void)threads_hint;
  const uint64_t cap = (uint64_t)device_sms() * (uint64_t)(per_sm > 0 ? per_sm : 1);
  const uint64_t g = work < cap ? work : cap;
  return (int)(g > 0 ? g : 1);
}

// Streaming (evict-first) stores for launches whose working set is far beyond
// the 126 MB L2 (>= 64 MiB per side); the default large-array shapes have a
// CS = true kernel instantiation for it (bitrev_kernels.cuh, st_vec).
bool stream_stores(int E, int b, int64_t batch) {
  return ((uint64_t)E << b) * (uint64_t)batch >= (64ull << 20);
}

// In-place work items: tile order 2 = compact pair enumeration
// (pair_from_index: one item per unordered pair, walked with a division-free
// cursor); other orders visit every y and skip items with rev(y) < y.
bool compact_pairs() { return tile_order(true) == 2; }

int grid_for_pairs(uint64_t work, int per_sm);

// Fills the work fields of an in-place launch; returns the grid size.
int set_pair_work(TileArgs& a, int64_t batch, bool compact, int per_sm) {
  a.batch = batch;
  if (!compact) {
    a.npairs = 0;
    a.step_b = a.step_w = 0;
    a.ntiles = (uint64_t)batch << a.m;
    return grid_for_pairs(a.ntiles, per_sm);
  }
  a.npairs = pair_count(a.m);
  a.ntiles = (uint64_t)batch * a.npairs;
  // BITREV_B200_IP_GRID_MULT: launch that many times the resident CTAs (A/B runs)
  static const int mult = env_int("BITREV_B200_IP_GRID_MULT", 1);
  const int grid = grid_for(a.ntiles, per_sm * (mult > 0 ? mult : 1));  // every item is real work
  a.step_b = (uint64_t)grid / a.npairs;
  a.step_w = (uint64_t)grid % a.npairs;
  return grid;
}

// Persistent grid for the in-place pair kernels.  CTA j visits work items
// j, j+G, j+2G, ...; an item is skipped when rev(y) < y, and that depends on
// y's low bits.  With an even G every CTA sees a fixed residue of y's low
// bits, so skip rates (and CTA run times) differ by up to ~2x -- ncu showed
// SMs active 61 % of the elapsed cycles.  An odd G cycles every CTA through
// all residues.
int grid_for_pairs(uint64_t work, int per_sm) {
  int g = grid_for(work, per_sm);
  if (g > 1 && (g & 1) == 0) --g;
  return g;
}

// Resident CTAs per SM of a kernel at a dynamic smem size.
template <typename K>
int occupancy(K kernel, int threads, size_t smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess)
    n = 1;
  return n > 0 ? n : 1;
}

// Per-device launch setup of one kernel instantiation: raises its dynamic
// shared-memory limit on the current device (an attribute is per device, so
// a process driving several GPUs needs it on each) and caches its occupancy.
std::mutex g_prep_mu;
std::map<std::pair<const void*, int>, int> g_prep;  // (kernel, device) -> CTAs per SM

template <typename K>
int prepare_kernel(K kernel, int threads, int smem_bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  std::lock_guard<std::mutex> lk(g_prep_mu);
  auto it = g_prep.find(key);
  if (it != g_prep.end()) return it->second;
  if (smem_bytes > 48 * 1024)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  const int v = occupancy(kernel, threads, smem_bytes);
  g_prep.emplace(key, v);
  return v;
}

// Programmatic dependent launch for the hot tile kernels: each kernel
// triggers its dependents when a CTA reaches its last work item and waits
// (griddepcontrol.wait) for its predecessor before its first load, so a
// back-to-back call's launch and CTA start overlap the previous call's tail.
// BITREV_B200_PDL=0 launches plainly (A/B runs).
bool pdl_enabled() {
  static const int v = env_int("BITREV_B200_PDL", 1);
  return v != 0;
}

template <typename K, typename... Args>
int launch_tiles(K kern, int grid, int threads, size_t smem, cudaStream_t st, Args... args) {
  if (!pdl_enabled()) {
    kern<<<grid, threads, smem, st>>>(args...);
    return finish_launch();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess) return (int)e;
  return finish_launch();
}

// ---------------------------------------------------------------------------
// tile launches

// Out-of-place tile grids: not one persistent CTA per SM slot but about
// kOopTilesPerCta tiles per CTA, so the resident CTAs start on tiles far
// apart and the block scheduler keeps refilling SMs with new CTAs.  Each CTA
// still prefetches its next tile into registers.  cfg3-16 6529 -> 6712
// GB/s (~7 tiles per CTA), cfg3-8 6320 -> 6677 (~3.5), cfg4 6370 -> 6545
// (~3.5), cfg5 on one GPU 6308 -> 6610 (~7); float32 (the 1-CTA/SM (8,6)
// tiles) and the in-place pairs lose, so they stay persistent
// (tools/grid_mult_sweep.sh -> profiles/r02_grid_mult_sweep.jsonl).  Only
// launches with at least 16 such grids' worth of waves take it: at 1.4-5.5
// waves the last wave's idle SMs cost up to 15 % (complex128 at 64 MiB,
// float64 at 32-64 MiB; tools/oop_tpc_ab.sh -> profiles/r02_oop_tpc_ab.jsonl).
// BITREV_B200_OOP_TILES_PER_CTA overrides the target (0 = persistent).
int spread_grid(uint64_t ntiles, int per_sm, int tpc) {
  const int resident = grid_for(ntiles, per_sm);
  if (tpc <= 0) return resident;
  const uint64_t want = ntiles / (uint64_t)tpc;
  if (want < 16ull * (uint64_t)resident) return resident;
  return (int)(want < (1ull << 31) - 1 ? want : (1ull << 31) - 1);
}

int oop_grid(int E, uint64_t ntiles, int per_sm) {
  static const int env = env_int("BITREV_B200_OOP_TILES_PER_CTA", -1);
  return spread_grid(ntiles, per_sm, env >= 0 ? env : (E == 4 ? 0 : 5));
}

// The same for the sharded pack / fused scatter and the FFT pre-pass tiles
// (tools/spread_grid_ab.sh -> profiles/r02_spread_grid_ab.*): the pack and
// scatter move by -1 to +0.6 %, so they stay persistent; the complex128
// square-tile FFT takes it at 1-3 stages (+2 to +6.5 %; -14 % at 4-5), the
// complex64 FFT tiles keep persistent grids (-1 to -8 % at 1-5 stages,
// within 1.5 % at 6-7).  BITREV_B200_PACK_TILES_PER_CTA /
// BITREV_B200_FFT_TILES_PER_CTA override (A/B runs).
int pack_grid(uint64_t ntiles, int per_sm) {
  static const int env = env_int("BITREV_B200_PACK_TILES_PER_CTA", 0);
  return spread_grid(ntiles, per_sm, env);
}
int fft_grid(uint64_t ntiles, int per_sm, int dflt = 0) {
  static const int env = env_int("BITREV_B200_FFT_TILES_PER_CTA", -1);
  return spread_grid(ntiles, per_sm, env >= 0 ? env : dflt);
}


template <int E, int Q, int NT = BITREV_TILE_THREADS>
int launch_oop_tile(const void* src, void* dst, int b, int64_t batch, int64_t sbs, int64_t dbs,
                    cudaStream_t st) {
  using T = Tile<E, Q, NT>;
  auto kern = bitrev_oop_tile_kernel<E, Q, NT, false>;
  if constexpr ((E == 16 && Q == 6 && NT == BITREV_TILE_THREADS) || (E == 8 && Q == 7 && NT == 512))
    if (stream_stores(E, b, batch)) kern = bitrev_oop_tile_kernel<E, Q, NT, true>;
  if constexpr (E == 16 && Q == 5 && NT == BITREV_TILE_THREADS) {
    // complex128 up to 32 MiB per side (the Q5 tier): 4 CTAs/SM (63
    // registers) instead of 2 puts every tile of a 2^20 array in flight at
    // once: L2-hot cfg1 6860 -> 7250 GB/s, L2-flushed unchanged (at the
    // copy_ floor, profiles/r02_cfg1_minb_ab.jsonl, r02_minb_sizes_ab.jsonl).
    // BITREV_B200_SMALL_MINB=1|3 selects the other forms (A/B runs).
    static const int minb = env_int("BITREV_B200_SMALL_MINB", 4);
    if (minb == 4) kern = bitrev_oop_tile_kernel<E, Q, NT, false, 4>;
    if (minb == 3) kern = bitrev_oop_tile_kernel<E, Q, NT, false, 3>;
  }
  const int per_sm = prepare_kernel(kern, T::THREADS, T::BYTES);
  TileArgs a;
  a.src = static_cast<const char*>(src);
  a.dst = static_cast<char*>(dst);
  a.b = b;
  a.m = b - 2 * Q;
  a.ntiles = (uint64_t)batch << a.m;
  a.src_bstride = sbs * E;
  a.dst_bstride = dbs * E;
  a.order = tile_order(false);
  a.npairs = 0;
  a.batch = batch;
  const int grid = oop_grid(E, a.ntiles, per_sm);
  return launch_tiles(kern, grid, T::THREADS, T::BYTES, st, a);
}

template <int E, int Q, bool COMPACT>
int launch_ip_tile_mode(void* buf, int b, int64_t batch, int64_t bs, cudaStream_t st) {
  using T = Tile<E, Q>;
  auto kern = bitrev_inplace_tile_kernel<E, Q, COMPACT, false>;
  if constexpr (COMPACT && Q == 6 && (E == 4 || E == 8))
    if (stream_stores(E, b, batch)) kern = bitrev_inplace_tile_kernel<E, Q, COMPACT, true>;
  const int per_sm = prepare_kernel(kern, T::THREADS, 2 * T::BYTES);
  TileArgs a;
  a.src = static_cast<const char*>(buf);
  a.dst = static_cast<char*>(buf);
  a.b = b;
  a.m = b - 2 * Q;
  a.src_bstride = bs * E;
  a.dst_bstride = bs * E;
  a.order = tile_order(true);
  const int grid = set_pair_work(a, batch, COMPACT, per_sm);
  return launch_tiles(kern, grid, T::THREADS, 2 * T::BYTES, st, a);  // PDL: cfg2 +1.0 %
}

template <int E, int Q>
int launch_ip_tile(void* buf, int b, int64_t batch, int64_t bs, cudaStream_t st) {
  return compact_pairs() ? launch_ip_tile_mode<E, Q, true>(buf, b, batch, bs, st)
                         : launch_ip_tile_mode<E, Q, false>(buf, b, batch, bs, st);
}

// ---------------------------------------------------------------------------
// in-place cp.async path (4): compact pairs only

template <int E, int Q>
int launch_ip_cpa(void* buf, int b, int64_t batch, int64_t bs, cudaStream_t st) {
  using T = CpaTile<E, Q>;
  if (T::SMEM > 227 * 1024) return BITREV_ETILE;
  auto kern = bitrev_inplace_cpa_kernel<E, Q>;
  const int per_sm = prepare_kernel(kern, T::THREADS, T::SMEM);
  TileArgs a;
  memset(&a, 0, sizeof a);
  a.src = static_cast<const char*>(buf);
  a.dst = static_cast<char*>(buf);
  a.b = b;
  a.m = b - 2 * Q;
  a.src_bstride = bs * E;
  a.dst_bstride = bs * E;
  a.order = 2;
  const int grid = set_pair_work(a, batch, true, per_sm);
  kern<<<grid, T::THREADS, T::SMEM, st>>>(a);
  return finish_launch();
}

int dispatch_ip_cpa(int E, int q, void* buf, int b, int64_t batch, int64_t bs, cudaStream_t st) {
  if (E == 4 && q == 6) return launch_ip_cpa<4, 6>(buf, b, batch, bs, st);
  if (E == 4 && q == 7) return launch_ip_cpa<4, 7>(buf, b, batch, bs, st);
  if (E == 8 && q == 5) return launch_ip_cpa<8, 5>(buf, b, batch, bs, st);
  if (E == 8 && q == 6) return launch_ip_cpa<8, 6>(buf, b, batch, bs, st);
  if (E == 16 && q == 5) return launch_ip_cpa<16, 5>(buf, b, batch, bs, st);
  if (E == 16 && q == 6) return launch_ip_cpa<16, 6>(buf, b, batch, bs, st);
  return BITREV_ETILE;
}

// ---------------------------------------------------------------------------
// TMA ring paths (1 = per-row bulk copies, 2 = tensor-map tiles)

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 5-D view of the kTensor mode (bitrev_kernels.cuh).  Returns false if the
// driver rejects it; the caller then takes the register path.
bool encode_tile_map(CUtensorMap* map, const void* base, int b, int E, int q, int64_t batch,
                     int64_t bstride_elems) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int unit = E == 4 ? 4 : 8;
  const uint64_t row = (uint64_t)E << q;
  const int m = b - 2 * q;
  if (m > 31 || batch > (int64_t(1) << 31) || row % 128 != 0) return false;
  cuuint64_t dims[5] = {128u / unit, (cuuint64_t)1 << q, row / 128, (cuuint64_t)1 << m,
                        (cuuint64_t)batch};
  cuuint64_t strides[4] = {(cuuint64_t)E << (b - q), 128, row,
                           (cuuint64_t)(batch > 1 ? bstride_elems : (int64_t(1) << b)) * E};
  cuuint32_t box[5] = {128u / unit, 1u << q, (cuuint32_t)(row / 128), 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = fn(map, unit == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64,
                        5, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// In-place tile pairs split over 2-CTA clusters (path 6): compact pairs only.
template <int E, int Q, int NT, int MINB = 1>
int launch_ip_cluster(void* buf, int b, int64_t batch, int64_t bs, cudaStream_t st) {
  using T = Tile<E, Q, NT>;
  if (2 * Q > b) return BITREV_ETILE;
  auto kern = bitrev_inplace_cluster_kernel<E, Q, NT, MINB, false>;
  if constexpr (E == 16 && Q == 6)
    if (stream_stores(E, b, batch)) kern = bitrev_inplace_cluster_kernel<E, Q, NT, MINB, true>;
  const int per_sm = prepare_kernel(kern, T::THREADS, T::BYTES);
  TileArgs a;
  memset(&a, 0, sizeof a);
  a.src = static_cast<const char*>(buf);
  a.dst = static_cast<char*>(buf);
  a.b = b;
  a.m = b - 2 * Q;
  a.src_bstride = bs * E;
  a.dst_bstride = bs * E;
  a.order = 2;
  a.batch = batch;
  a.npairs = pair_count(a.m);
  a.ntiles = (uint64_t)batch * a.npairs;
  // co-resident clusters: both CTAs of a cluster sit in one GPC, so a GPC with
  // an odd number of free SMs strands one; a persistent grid larger than this
  // would run its last clusters as a second wave
  uint64_t clusters = (uint64_t)device_sms() * (uint64_t)per_sm / 2;
  {
    static std::atomic<int> cached[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    int c = (dev >= 0 && dev < kMaxDevices) ? cached[dev].load() : 0;
    if (c == 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(2 * clusters));
      cfg.blockDim = dim3(T::THREADS);
      cfg.dynamicSmemBytes = T::BYTES;
      if (cudaOccupancyMaxActiveClusters(&c, kern, &cfg) != cudaSuccess || c <= 0) {
        cudaGetLastError();
        c = (int)clusters;
      }
      if (dev >= 0 && dev < kMaxDevices) cached[dev].store(c);
    }
    if ((uint64_t)c < clusters) clusters = (uint64_t)c;
  }
  if (clusters > a.ntiles) clusters = a.ntiles;
  if (clusters < 1) clusters = 1;
  a.step_b = clusters / a.npairs;
  a.step_w = clusters % a.npairs;
  kern<<<(unsigned)(2 * clusters), T::THREADS, T::BYTES, st>>>(a);
  return finish_launch();
}

int dispatch_ip_cluster(int E, int q, void* buf, int b, int64_t batch, int64_t bs,
                        cudaStream_t st) {
  if (E == 4 && q == 7) return launch_ip_cluster<4, 7, 256>(buf, b, batch, bs, st);
  if (E == 8 && q == 6) return launch_ip_cluster<8, 6, 256, 2>(buf, b, batch, bs, st);  // 2 CTAs/SM
  if (E == 8 && q == 7) return launch_ip_cluster<8, 7, 512>(buf, b, batch, bs, st);  // 128 KB tile
  if (E == 16 && q == 5) return launch_ip_cluster<16, 5, 256>(buf, b, batch, bs, st);
  if (E == 16 && q == 6) return launch_ip_cluster<16, 6, 256>(buf, b, batch, bs, st);
  return BITREV_ETILE;
}

// In-place tile pairs with TMA tensor stores (path 5): compact pairs only.
template <int E, int Q>
int launch_ip_tstore(void* buf, int b, int64_t batch, int64_t bs, cudaStream_t st) {
  using S = TsTile<E, Q>;
  if (S::SMEM > 227 * 1024) return BITREV_ETILE;
  CUtensorMap map;
  memset(&map, 0, sizeof map);
  if (!encode_tile_map(&map, buf, b, E, Q, batch, bs)) return BITREV_ETILE;
  auto kern = bitrev_inplace_tstore_kernel<E, Q>;
  const int per_sm = prepare_kernel(kern, Tile<E, Q>::THREADS, S::SMEM);
  TileArgs a;
  memset(&a, 0, sizeof a);
  a.src = static_cast<const char*>(buf);
  a.dst = static_cast<char*>(buf);
  a.b = b;
  a.m = b - 2 * Q;
  a.src_bstride = bs * E;
  a.dst_bstride = bs * E;
  a.order = 2;
  const int grid = set_pair_work(a, batch, true, per_sm);
  kern<<<grid, Tile<E, Q>::THREADS, S::SMEM, st>>>(map, a);
  return finish_launch();
}

int dispatch_ip_tstore(int E, int q, void* buf, int b, int64_t batch, int64_t bs,
                       cudaStream_t st) {
  if (2 * q > b) return BITREV_ETILE;
  if (E == 4 && q == 6) return launch_ip_tstore<4, 6>(buf, b, batch, bs, st);
  if (E == 8 && q == 5) return launch_ip_tstore<8, 5>(buf, b, batch, bs, st);
  if (E == 8 && q == 6) return launch_ip_tstore<8, 6>(buf, b, batch, bs, st);
  if (E == 16 && q == 4) return launch_ip_tstore<16, 4>(buf, b, batch, bs, st);
  if (E == 16 && q == 5) return launch_ip_tstore<16, 5>(buf, b, batch, bs, st);
  return BITREV_ETILE;
}

template <int E, int Q, bool INPLACE, int MODE, bool COMPACT>
int launch_ring_mode(const void* src, void* dst, int b, int64_t batch, int64_t sbs, int64_t dbs,
                     cudaStream_t st) {
  using R = Ring<E, Q, INPLACE, MODE>;
  static_assert(R::SMEM <= 227 * 1024, "ring exceeds shared memory");
  CUtensorMap map;
  memset(&map, 0, sizeof map);
  if (MODE == kTensor && !encode_tile_map(&map, src, b, E, Q, batch, sbs)) return BITREV_ETILE;
  auto kern = bitrev_ring_kernel<E, Q, INPLACE, MODE, COMPACT>;
  const int per_sm = prepare_kernel(kern, R::THREADS, R::SMEM);
  TileArgs a;
  a.src = static_cast<const char*>(src);
  a.dst = static_cast<char*>(dst);
  a.b = b;
  a.m = b - 2 * Q;
  a.ntiles = (uint64_t)batch << a.m;
  a.src_bstride = sbs * E;
  a.dst_bstride = dbs * E;
  a.order = tile_order(INPLACE);
  a.npairs = 0;
  a.batch = batch;
  int grid;
  if (INPLACE) {
    grid = set_pair_work(a, batch, COMPACT, per_sm);
  } else {
    grid = grid_for(a.ntiles, per_sm);
  }
  kern<<<grid, R::THREADS, R::SMEM, st>>>(map, a);
  return finish_launch();
}

template <int E, int Q, bool INPLACE, int MODE>
int launch_ring(const void* src, void* dst, int b, int64_t batch, int64_t sbs, int64_t dbs,
                cudaStream_t st) {
  if (INPLACE && compact_pairs())
    return launch_ring_mode<E, Q, INPLACE, MODE, true>(src, dst, b, batch, sbs, dbs, st);
  return launch_ring_mode<E, Q, INPLACE, MODE, false>(src, dst, b, batch, sbs, dbs, st);
}

// Instantiated (E, Q) per ring mode and family; anything else -> BITREV_ETILE.
int dispatch_ring(int mode, int E, int q, bool inplace, const void* src, void* dst, int b,
                  int64_t batch, int64_t sbs, int64_t dbs, cudaStream_t st) {
#define RING(M_, E_, Q_, IP_)                                                      \
  if (mode == M_ && E == E_ && q == Q_ && inplace == IP_)                          \
    return launch_ring<E_, Q_, IP_, M_>(src, dst, b, batch, sbs, dbs, st);
#define RING_BOTH(M_, E_, Q_) RING(M_, E_, Q_, false) RING(M_, E_, Q_, true)
  RING_BOTH(kTensor, 4, 5) RING_BOTH(kTensor, 4, 6) RING_BOTH(kTensor, 8, 4)
  RING_BOTH(kTensor, 8, 5) RING_BOTH(kTensor, 8, 6) RING_BOTH(kTensor, 16, 3)
  RING_BOTH(kTensor, 16, 4) RING_BOTH(kTensor, 16, 5)
  RING(kTensor, 4, 7, false) RING(kTensor, 16, 6, false)
  RING_BOTH(kBulkRows, 4, 6) RING_BOTH(kBulkRows, 8, 5) RING_BOTH(kBulkRows, 8, 6)
  RING_BOTH(kBulkRows, 16, 4) RING_BOTH(kBulkRows, 16, 5)
  RING(kBulkRows, 4, 7, false) RING(kBulkRows, 16, 6, false)
#undef RING_BOTH
#undef RING
  return BITREV_ETILE;
}

// Rectangular out-of-place tiles: path 3 (QX = long destination side).
template <int E, int QX, int QZ>
int launch_oop_rect(const void* src, void* dst, int b, int64_t batch, int64_t sbs, int64_t dbs,
                    cudaStream_t st) {
  using T = Rect<E, QX, QZ>;
  if (b < QX + QZ) return BITREV_ETILE;
  auto kern = bitrev_oop_rect_kernel<E, QX, QZ, false>;
  if constexpr ((E == 4 && QX == 8 && QZ == 6) || (E == 8 && QX == 7 && QZ == 5))
    if (stream_stores(E, b, batch)) kern = bitrev_oop_rect_kernel<E, QX, QZ, true>;
  static const int pad_kb = env_int("BITREV_B200_RECT_SMEM_KB", 0);  // A/B runs: cap CTAs/SM
  const int smem = pad_kb * 1024 > T::BYTES ? pad_kb * 1024 : T::BYTES;
  const int per_sm = prepare_kernel(kern, T::THREADS, smem);
  TileArgs a;
  a.src = static_cast<const char*>(src);
  a.dst = static_cast<char*>(dst);
  a.b = b;
  a.m = b - QX - QZ;
  a.ntiles = (uint64_t)batch << a.m;
  a.src_bstride = sbs * E;
  a.dst_bstride = dbs * E;
  a.order = tile_order(false);
  a.npairs = 0;
  a.batch = batch;
  const int grid = oop_grid(E, a.ntiles, per_sm);
  return launch_tiles(kern, grid, T::THREADS, smem, st, a);
}

// Rectangular tiles: q selects the destination run (QX elements), rect_qz the
// source piece (QZ elements).  Measured on B200 (tools/rect_qz.py ->
// profiles/r01_rect_qz.jsonl, b = 26/28/30): 1 KB destination rows with
// 256-byte source pieces win -- E=8 (7,5) 6.17 TB/s vs (7,4) 5.91; E=4 (8,6)
// 6.22 vs square Q7 6.00.  BITREV_B200_RECT_QZ overrides QZ for every QX
// (experiments; shapes outside the table below fall back to square tiles).
int rect_qz(int E, int qx) {
  static const int env = env_int("BITREV_B200_RECT_QZ", 0);
  if (env) return env;
  switch (E) {
    case 4: return qx >= 7 ? 6 : 5;
    case 8: return qx >= 6 ? 5 : 4;
    case 16: return qx >= 6 ? 4 : 3;
  }
  return 0;
}

int dispatch_oop_rect(int E, int q, const void* src, void* dst, int b, int64_t batch, int64_t sbs,
                      int64_t dbs, cudaStream_t st) {
  const int qz = rect_qz(E, q);
#define RECT(EE, QX, QZ)                                                       \
  if (E == EE && q == QX && qz == QZ)                                          \
    return launch_oop_rect<EE, QX, QZ>(src, dst, b, batch, sbs, dbs, st);
  RECT(4, 6, 5) RECT(4, 7, 6) RECT(4, 8, 6)
  RECT(8, 5, 4) RECT(8, 6, 5) RECT(8, 7, 5) RECT(8, 8, 5)
  RECT(16, 4, 3) RECT(16, 5, 3) RECT(16, 6, 4) RECT(16, 7, 4)
#undef RECT
  return BITREV_ETILE;
}

int dispatch_oop_tile(int E, int q, const void* src, void* dst, int b, int64_t batch, int64_t sbs,
                      int64_t dbs, cudaStream_t st) {
  switch (E) {
    case 4:
      switch (q) {
        case 5: return launch_oop_tile<4, 5>(src, dst, b, batch, sbs, dbs, st);
        case 6: return launch_oop_tile<4, 6>(src, dst, b, batch, sbs, dbs, st);
        case 7: return launch_oop_tile<4, 7>(src, dst, b, batch, sbs, dbs, st);
      }
      break;
    case 8:
      switch (q) {
        case 4: return launch_oop_tile<8, 4>(src, dst, b, batch, sbs, dbs, st);
        case 5: return launch_oop_tile<8, 5>(src, dst, b, batch, sbs, dbs, st);
        case 6: return launch_oop_tile<8, 6>(src, dst, b, batch, sbs, dbs, st);
        case 7: return launch_oop_tile<8, 7, 512>(src, dst, b, batch, sbs, dbs, st);  // 128 KB
      }
      break;
    case 16:
      switch (q) {
        case 3: return launch_oop_tile<16, 3>(src, dst, b, batch, sbs, dbs, st);
        case 4: return launch_oop_tile<16, 4>(src, dst, b, batch, sbs, dbs, st);
        case 5: return launch_oop_tile<16, 5>(src, dst, b, batch, sbs, dbs, st);
        case 6: return launch_oop_tile<16, 6>(src, dst, b, batch, sbs, dbs, st);
      }
      break;
  }
  return BITREV_ETILE;
}

int dispatch_ip_tile(int E, int q, void* buf, int b, int64_t batch, int64_t bs, cudaStream_t st) {
  switch (E) {
    case 4:
      switch (q) {
        case 5: return launch_ip_tile<4, 5>(buf, b, batch, bs, st);
        case 6: return launch_ip_tile<4, 6>(buf, b, batch, bs, st);
        case 7: return launch_ip_tile<4, 7>(buf, b, batch, bs, st);
      }
      break;
    case 8:
      switch (q) {
        case 4: return launch_ip_tile<8, 4>(buf, b, batch, bs, st);
        case 5: return launch_ip_tile<8, 5>(buf, b, batch, bs, st);
        case 6: return launch_ip_tile<8, 6>(buf, b, batch, bs, st);
      }
      break;
    case 16:
      switch (q) {
        case 3: return launch_ip_tile<16, 3>(buf, b, batch, bs, st);
        case 4: return launch_ip_tile<16, 4>(buf, b, batch, bs, st);
        case 5: return launch_ip_tile<16, 5>(buf, b, batch, bs, st);
        case 6: return launch_ip_tile<16, 6>(buf, b, batch, bs, st);
      }
      break;
  }
  return BITREV_ETILE;
}

// ---------------------------------------------------------------------------
// small / element-wise launches

template <int E>
int launch_small(const void* src, void* dst, int b, int64_t batch, int64_t sbs, int64_t dbs,
                 cudaStream_t st) {
  const int bytes = (1 << b) * E;
  auto kern = bitrev_small_kernel<E>;
  const int per_sm = prepare_kernel(kern, 256, kSmallBytes);
  const int threads = (1 << b) < 256 ? ((1 << b) < 32 ? 32 : (1 << b)) : 256;
  const int grid = grid_for((uint64_t)batch, per_sm * (256 / threads));
  kern<<<grid, threads, bytes, st>>>(static_cast<const char*>(src), static_cast<char*>(dst), b,
                                     batch, sbs * E, dbs * E);
  return finish_launch();
}

// Short rows (n*E <= 32 KB) of 4/8/16-byte elements on 16-byte aligned rows:
// many rows per CTA (bitrev_rows_kernel).  sbs/dbs in elements.
template <int E, int KB>
int launch_rows(const void* src, void* dst, int b, int64_t batch, int64_t sbs, int64_t dbs,
                cudaStream_t st) {
  using R = Rows<E, KB>;
  const int vb = b - R::LV;
  if (vb < 0) return BITREV_ETILE;
  const int rb = const_log2(R::BYTES / 16) - vb;
  if (rb < 0) return BITREV_ETILE;
  const int64_t nblocks = (batch + (int64_t(1) << rb) - 1) >> rb;
  const int sh = vb - R::LV - 3 > 3 ? vb - R::LV - 3 : 3;
  const bool ip = src == dst;
  auto kern = ip ? bitrev_rows_kernel<E, true, KB> : bitrev_rows_kernel<E, false, KB>;
  const int per_sm = prepare_kernel(kern, R::THREADS, R::BYTES);
  // ~2 blocks per CTA instead of a persistent grid (see oop_grid) for 8- and
  // 16-byte rows: batches of 2^26 elements as rows of 2^6..2^12, in and out
  // of place, 6.0-6.4 -> 6.6-6.9 TB/s; float32 rows unchanged
  // (tools/small_rows_probe.py -> profiles/r02_rows_tpc_ab.jsonl).
  // BITREV_B200_ROWS_TILES_PER_CTA overrides it (A/B runs).
  static const int rows_env = env_int("BITREV_B200_ROWS_TILES_PER_CTA", -1);
  const int grid = spread_grid((uint64_t)nblocks, per_sm, rows_env >= 0 ? rows_env : (E == 4 ? 0 : 2));
  kern<<<grid, R::THREADS, R::BYTES, st>>>(static_cast<const char*>(src), static_cast<char*>(dst),
                                            b, batch, sbs * E, dbs * E, sh);
  return finish_launch();
}

int dispatch_rows(int E, const void* src, void* dst, int b, int64_t batch, int64_t sbs,
                  int64_t dbs, cudaStream_t st) {
  const int64_t row = (int64_t)E << b;
  // block: 16 KB for 8/16-byte elements, 32 KB for 4-byte ones (measured,
  // profiles/r01_short_rows_blocks.txt: +3-5 % and best respectively), or one
  // whole row when it is longer; float32 rows of 128 KB would spill (unused)
#define ROWS_E(EE, MAXKB)                                                                 \
  if (E == EE) {                                                                          \
    if (EE != 4 && row <= 16 * 1024) return launch_rows<EE, 16>(src, dst, b, batch, sbs, dbs, st); \
    if (row <= 32 * 1024) return launch_rows<EE, 32>(src, dst, b, batch, sbs, dbs, st);   \
    if (row <= 64 * 1024) return launch_rows<EE, 64>(src, dst, b, batch, sbs, dbs, st);   \
    if constexpr (MAXKB >= 128)                                                           \
      if (row <= 128 * 1024) return launch_rows<EE, 128>(src, dst, b, batch, sbs, dbs, st); \
  }
  ROWS_E(4, 64) ROWS_E(8, 128) ROWS_E(16, 128)
#undef ROWS_E
  return BITREV_ETILE;
}


int dispatch_small(int E, const void* src, void* dst, int b, int64_t batch, int64_t sbs,
                   int64_t dbs, cudaStream_t st) {
  switch (E) {
    case 1: return launch_small<1>(src, dst, b, batch, sbs, dbs, st);
    case 2: return launch_small<2>(src, dst, b, batch, sbs, dbs, st);
    case 4: return launch_small<4>(src, dst, b, batch, sbs, dbs, st);
    case 8: return launch_small<8>(src, dst, b, batch, sbs, dbs, st);
    case 16: return launch_small<16>(src, dst, b, batch, sbs, dbs, st);
  }
  return BITREV_EELEM;
}

uint64_t elementwise_grid(uint64_t total) {
  const uint64_t blocks = (total + 255) / 256;
  const uint64_t cap = (uint64_t)device_sms() * 8;
  return blocks < cap ? (blocks ? blocks : 1) : cap;
}

template <int E>
int launch_gather(const void* src, void* dst, int b, int64_t batch, int64_t sbs, int64_t dbs,
                  cudaStream_t st) {
  const uint64_t total = (1ull << b) * (uint64_t)batch;
  bitrev_gather_kernel<E><<<(unsigned)elementwise_grid(total), 256, 0, st>>>(
      static_cast<const char*>(src), static_cast<char*>(dst), b, batch, sbs * E, dbs * E);
  return finish_launch();
}

int dispatch_gather(int E, const void* src, void* dst, int b, int64_t batch, int64_t sbs,
                    int64_t dbs, cudaStream_t st) {
  switch (E) {
    case 1: return launch_gather<1>(src, dst, b, batch, sbs, dbs, st);
    case 2: return launch_gather<2>(src, dst, b, batch, sbs, dbs, st);
    case 4: return launch_gather<4>(src, dst, b, batch, sbs, dbs, st);
    case 8: return launch_gather<8>(src, dst, b, batch, sbs, dbs, st);
    case 16: return launch_gather<16>(src, dst, b, batch, sbs, dbs, st);
  }
  return BITREV_EELEM;
}

template <int E>
int launch_swap(void* a, int b, int64_t batch, int64_t bs, cudaStream_t st) {
  const uint64_t total = (1ull << b) * (uint64_t)batch;
  bitrev_swap_kernel<E><<<(unsigned)elementwise_grid(total), 256, 0, st>>>(
      static_cast<char*>(a), b, batch, bs * E);
  return finish_launch();
}

int dispatch_swap(int E, void* a, int b, int64_t batch, int64_t bs, cudaStream_t st) {
  switch (E) {
    case 1: return launch_swap<1>(a, b, batch, bs, st);
    case 2: return launch_swap<2>(a, b, batch, bs, st);
    case 4: return launch_swap<4>(a, b, batch, bs, st);
    case 8: return launch_swap<8>(a, b, batch, bs, st);
    case 16: return launch_swap<16>(a, b, batch, bs, st);
  }
  return BITREV_EELEM;
}

int check_common(int b, int E, int64_t batch) {
  if (b < 1 || b > kMaxBits) return BITREV_EWIDTH;
  if (!valid_elem(E)) return BITREV_EELEM;
  if (batch < 1) return BITREV_EBATCH;
  return BITREV_OK;
}

// Mid-size tile tiers, measured on B200 (tools/mid_sizes.py ->
// profiles/r01_mid_sizes.jsonl, event means over 80 flushed launches): up to
// a per-side byte budget a persistent grid of one default tile per SM gets
// only a few hundred tiles (1.7-3.5 waves), and smaller tiles with more
// resident CTAs per SM balance it -- up to 1.28x (E=4, b=19, out of place),
// 1.23x (E=8 in place, b=20), 1.16x (E=16 out of place, b=20), 1.07x (E=8
// out of place, b=22), 1.2-1.5x (E=16 in place against the cluster default,
// b = 19..25).  Above the last budget the defaults win.
struct Tier {
  int q = 0, path = 0;  // q = 0: no tier applies
};

Tier mid_tier(int E, bool inplace, uint64_t side_bytes) {
  Tier t;
  if (E != 4 && E != 8 && E != 16) return t;
  // Knobs compare by value, so saving a knob and setting it back keeps the
  // tiers; any other value switches them off.
  if (current_q(E, inplace) != default_q(E, inplace)) return t;
  if (tile_path(E, inplace) != default_path(E, inplace)) return t;
  const uint64_t mib = side_bytes >> 20, exact = side_bytes & ((1u << 20) - 1);
  auto within = [&](uint64_t budget_mib) { return mib < budget_mib || (mib == budget_mib && !exact); };
  if (E == 4 && !inplace) {
    if (within(32)) t = {5, 0};       // square Q5 up to b = 23
    else if (within(64)) t = {7, 3};  // rectangular QX = 7 (512 B rows) at b = 24
  } else if (E == 4 && inplace) {
    if (within(64)) t = {5, 0};
  } else if (E == 8 && !inplace) {
    if (within(32)) t = {4, 0};       // square Q4 up to b = 22
  } else if (E == 8 && inplace) {
    if (within(64)) t = {4, 0};
  } else if (E == 16 && !inplace) {
    // 8-32 MiB per side: Q4 tiles through the TMA tensor ring (96 KB, 2
    // CTAs/SM).  From DRAM it ties the Q5 register tiles (b = 20: 3264-3282
    // vs 3256-3280 GB/s; b = 21: -0.9 %); with the array L2-resident it is
    // +7.5 % (b = 20) / +23 % (b = 21): one TMA instruction per tile instead
    // of the register path's LDG/STS issue (tools/small_ring_e16_ab.sh ->
    // profiles/r02_small_ring_e16_ab.jsonl).  Up to 8 MiB the register tiles
    // stay ahead L2-resident (b = 17/18: -12 % / -4 % for the ring).
    if (within(8)) t = {5, 0};
    else if (within(32)) t = {4, 2};
  } else if (E == 16 && inplace) {
    if (within(512)) t = {5, 0};  // single-CTA pairs up to b = 25; clusters from b = 26
  }
  return t;
}

uint64_t side_bytes(int E, int b, int64_t batch) { return ((uint64_t)E << b) * (uint64_t)batch; }

// Batched 8-byte rows out of place, rows of 2^13..2^22 elements past the
// mid-size budget: rectangular tiles with 2 KB destination rows (QX = 8, 64
// KB tiles) beat the 1 KB default by 1-4 % (cfg4's 4096 x 2^16: +1.5 %);
// single arrays of 2^23 and up are neutral to 0.3 % either way
// (tools/rect_e8_rows_sweep.py -> profiles/r02_rect_e8_rows.jsonl,
// tools/rect_e8_q8_ab.sh -> profiles/r02_rect_e8_q8_ab.jsonl).
Tier batched_rows_tier(int E, bool inplace, int b, int64_t batch) {
  Tier t;
  if (E != 8 || inplace || batch < 2 || b < 13 || b > 22) return t;
  if (current_q(E, inplace) != default_q(E, inplace)) return t;
  if (tile_path(E, inplace) != default_path(E, inplace)) return t;
  if (side_bytes(E, b, batch) <= (32ull << 20)) return t;
  t.q = 8;
  t.path = 3;
  return t;
}

// In place, rows of 32-128 KB in large batches also take the short-row
// kernel (a whole row staged in one CTA, 64/128 KB blocks): +6 % (float32,
// 64 KB rows), +10-15 % (float64), +19-20 % (complex128) over tile pairs
// (profiles/r01_short_rows.jsonl).  Out of place the tiles stay 2-6 % ahead,
// float32 rows of 128 KB spill, and small batches would leave SMs idle (one
// CTA per block), hence the limits.
bool rows_inplace_ok(int E, int b, int64_t batch) {
  if (E != 4 && E != 8 && E != 16) return false;
  const int64_t row = (int64_t)E << b;
  const int64_t cap = E == 4 ? 64 * 1024 : 128 * 1024;
  return row > kSmallBytes && row <= cap && side_bytes(E, b, batch) >= (64ull << 20);
}

// Tile bits for the square kernels: the configured q, reduced so that
// 2q <= b.  The dispatchers then walk further down to the largest
// instantiated width.
int clamp_q(int q, int b) {
  while (q > 0 && 2 * q > b) --q;
  return q;
}

// The calling thread's most recent launch choice (bitrev_last_tile).
thread_local int t_last_q = 0;
thread_local int t_last_path = 0;

int note(int rc, int q, int path) {
  if (rc == BITREV_OK) {
    t_last_q = q;
    t_last_path = path;
  }
  return rc;
}


// Steps 1(+2) of the sharded plan: the local (b_local)-bit reversal with each
// destination row stored at peer[d] + ((c << (sb + g)) | (rank << sb) | k') * E
// for local output index u = d * C + c * 2^sb + k'.
int launch_scatter(const void* local, char* const* peer, int b_local, int g, int rank, int sb,
                   int E, cudaStream_t st) {
  const int q = E == 4 ? 6 : 5;  // 256 / 256 / 512-byte rows
  if (sb < q || 2 * q > b_local) return BITREV_ESHARD;  // rows inside one sub-chunk
  if (!aligned16(local)) return BITREV_EALIGN;
  ScatterArgs sa;
  memset(&sa, 0, sizeof sa);
  for (int d = 0; d < (1 << g); ++d) {
    if (!peer[d] || !aligned16(peer[d])) return BITREV_ENULL;
    sa.peer[d] = peer[d];
  }
  sa.g = g;
  sa.rank = rank;
  sa.sb = sb;
  TileArgs& a = sa.t;
  a.src = static_cast<const char*>(local);
  a.b = b_local;
  a.m = b_local - 2 * q;
  a.ntiles = 1ull << a.m;
  a.batch = 1;
#define SCATTER(E_, Q_)                                                                   \
  if (E == E_ && q == Q_) {                                                               \
    using T = Tile<E_, Q_>;                                                               \
    auto kern = bitrev_scatter_tile_kernel<E_, Q_>;                                       \
    const int per_sm = prepare_kernel(kern, T::THREADS, T::BYTES);                        \
    kern<<<grid_for(a.ntiles, per_sm), T::THREADS, T::BYTES, st>>>(sa);                   \
    return finish_launch();                                                               \
  }
  SCATTER(4, 6) SCATTER(8, 5) SCATTER(16, 5)
#undef SCATTER
  return BITREV_ETILE;
}

// Streams and events of the host-buffer entry points, created on a thread's
// first call per device and kept for the thread's lifetime (round 1 created
// and destroyed 3 streams and 10 events on every call).  Per thread, so calls
// from several host threads never share them; never destroyed, because a
// thread_local destructor may run after the CUDA runtime has shut down.
//
// Host <-> device copies are split into 256 MiB chunks alternating over two
// streams per direction: with 16 GiB pinned buffers the concurrent H2D + D2H
// of whole arrays reached 88 GB/s, the same bytes in 256 MiB chunks 98-99
// (tools/pcie_probe2.py -> profiles/r02_pcie_probe2.jsonl).
constexpr int kPipeSlots = 3;
constexpr size_t kCopyChunk = size_t(256) << 20;
struct PipeRes {
  bool ok = false;
  cudaStream_t sin[2] = {}, sk = nullptr, sout[2] = {}, aux = nullptr;
  cudaEvent_t ev_start = nullptr, ev_a = nullptr, ev_b = nullptr;
  cudaEvent_t ev_in[kPipeSlots][2] = {}, ev_k[kPipeSlots] = {}, ev_out[kPipeSlots][2] = {};
};

cudaError_t pipe_resources(PipeRes** out) {
  thread_local PipeRes res[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  PipeRes& r = res[dev];
  if (!r.ok) {
    auto stream = [&](cudaStream_t* s) { return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking); };
    auto event = [&](cudaEvent_t* v) { return cudaEventCreateWithFlags(v, cudaEventDisableTiming); };
    for (int i = 0; i < 2; ++i) {
      if ((e = stream(&r.sin[i])) != cudaSuccess) return e;
      if ((e = stream(&r.sout[i])) != cudaSuccess) return e;
    }
    if ((e = stream(&r.sk)) != cudaSuccess) return e;
    if ((e = stream(&r.aux)) != cudaSuccess) return e;
    if ((e = event(&r.ev_start)) != cudaSuccess) return e;
    if ((e = event(&r.ev_a)) != cudaSuccess) return e;
    if ((e = event(&r.ev_b)) != cudaSuccess) return e;
    for (int i = 0; i < kPipeSlots; ++i) {
      if ((e = event(&r.ev_k[i])) != cudaSuccess) return e;
      for (int j = 0; j < 2; ++j) {
        if ((e = event(&r.ev_in[i][j])) != cudaSuccess) return e;
        if ((e = event(&r.ev_out[i][j])) != cudaSuccess) return e;
      }
    }
    r.ok = true;
  }
  *out = &r;
  return cudaSuccess;
}

// bytes from src to dst as kCopyChunk pieces alternating over s[0] / s[1]
cudaError_t copy_split(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                       const cudaStream_t (&s)[2]) {
  for (size_t off = 0, i = 0; off < bytes; off += kCopyChunk, ++i) {
    const size_t n = bytes - off < kCopyChunk ? bytes - off : kCopyChunk;
    const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + off,
                                          static_cast<const char*>(src) + off, n, kind, s[i & 1]);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Pageable host memory (numpy arrays): the runtime's own pageable copies run
// ~15 GB/s for the whole round trip (tools/numpy_path_probe.py).  Instead the
// bytes are staged through a small ring of pinned bounce buffers: host
// threads copy chunk k+1 into a bounce slot while the DMA engine moves chunk
// k, in both directions.

// Fixed pool of host threads for parallel memcpy (never destroyed: its
// threads are detached and live as long as the process).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool();
    return *pool;
  }
  void copy(void* dst, const void* src, size_t n) {
    if (n < (size_t(4) << 20) || nworkers_ == 0) {
      memcpy(dst, src, n);
      return;
    }
    auto j = std::make_shared<Job>();
    j->dst = static_cast<char*>(dst);
    j->src = static_cast<const char*>(src);
    j->n = n;
    const size_t parts = size_t(nworkers_ + 1) * 2;
    j->piece = ((n + parts - 1) / parts + 4095) & ~size_t(4095);
    j->npieces = (n + j->piece - 1) / j->piece;
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = j;
      ++gen_;
    }
    cv_.notify_all();
    work(*j);  // the caller takes pieces too
    while (j->done.load(std::memory_order_acquire) < j->npieces) std::this_thread::yield();
  }

 private:
  struct Job {
    char* dst = nullptr;
    const char* src = nullptr;
    size_t n = 0, piece = 0, npieces = 0;
    std::atomic<size_t> next{0}, done{0};
  };
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    nworkers_ = (int)std::min(7u, hw > 1 ? hw - 1 : 0u);
    for (int i = 0; i < nworkers_; ++i) std::thread([this] { loop(); }).detach();
  }
  static void work(Job& j) {
    for (size_t k; (k = j.next.fetch_add(1, std::memory_order_relaxed)) < j.npieces;) {
      const size_t off = k * j.piece, len = std::min(j.piece, j.n - off);
      memcpy(j.dst + off, j.src + off, len);
      j.done.fetch_add(1, std::memory_order_release);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::shared_ptr<Job> j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        j = job_;
      }
      work(*j);
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::shared_ptr<Job> job_;
  uint64_t gen_ = 0;
  int nworkers_ = 0;
};

// Pinned bounce ring of the calling thread (per device, lazily allocated,
// never freed: see PipeRes).
constexpr int kBounceSlots = 3;
constexpr size_t kBounceBytes = size_t(64) << 20;
struct Bounce {
  bool ok = false;
  char* slot[kBounceSlots] = {};
  cudaEvent_t ev[kBounceSlots] = {};
};

cudaError_t bounce_ring(Bounce** out) {
  thread_local Bounce rings[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  Bounce& r = rings[dev];
  if (!r.ok) {
    for (int i = 0; i < kBounceSlots; ++i) {
      void* p = nullptr;
      if ((e = cudaHostAlloc(&p, kBounceBytes, cudaHostAllocPortable)) != cudaSuccess) return e;
      r.slot[i] = static_cast<char*>(p);
      if ((e = cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    r.ok = true;
  }
  *out = &r;
  return cudaSuccess;
}

bool pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // older drivers report unregistered memory as an error
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// host (pageable) -> device on st through the bounce ring; returns once the
// last chunk's DMA is enqueued (the slots are guarded by their events)
cudaError_t h2d_staged(void* dev, const void* host, size_t bytes, cudaStream_t st) {
  Bounce* r = nullptr;
  cudaError_t e = bounce_ring(&r);
  if (e != cudaSuccess) return e;
  for (size_t off = 0, i = 0; off < bytes; off += kBounceBytes, ++i) {
    const int s = (int)(i % kBounceSlots);
    const size_t n = std::min(kBounceBytes, bytes - off);
    if ((e = cudaEventSynchronize(r->ev[s])) != cudaSuccess) return e;  // slot's last DMA done
    CopyPool::get().copy(r->slot[s], static_cast<const char*>(host) + off, n);
    if ((e = cudaMemcpyAsync(static_cast<char*>(dev) + off, r->slot[s], n, cudaMemcpyHostToDevice,
                             st)) != cudaSuccess)
      return e;
    if ((e = cudaEventRecord(r->ev[s], st)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// device -> host (pageable) after st's prior work, through the bounce ring;
// returns when every byte is in host memory
cudaError_t d2h_staged(void* host, const void* dev, size_t bytes, cudaStream_t st) {
  Bounce* r = nullptr;
  cudaError_t e = bounce_ring(&r);
  if (e != cudaSuccess) return e;
  const size_t nchunks = (bytes + kBounceBytes - 1) / kBounceBytes;
  auto issue = [&](size_t i) -> cudaError_t {
    const int s = (int)(i % kBounceSlots);
    const size_t off = i * kBounceBytes, n = std::min(kBounceBytes, bytes - off);
    cudaError_t r2 = cudaMemcpyAsync(r->slot[s], static_cast<const char*>(dev) + off, n,
                                     cudaMemcpyDeviceToHost, st);
    return r2 != cudaSuccess ? r2 : cudaEventRecord(r->ev[s], st);
  };
  for (size_t i = 0; i < nchunks && i < (size_t)kBounceSlots; ++i)
    if ((e = issue(i)) != cudaSuccess) return e;
  for (size_t i = 0; i < nchunks; ++i) {
    const int s = (int)(i % kBounceSlots);
    const size_t off = i * kBounceBytes, n = std::min(kBounceBytes, bytes - off);
    if ((e = cudaEventSynchronize(r->ev[s])) != cudaSuccess) return e;
    CopyPool::get().copy(static_cast<char*>(host) + off, r->slot[s], n);
    if (i + kBounceSlots < nchunks && (e = issue(i + kBounceSlots)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// A blocking host-buffer call's copy on stream st, split over st and the
// thread's aux stream; st continues only after both halves.
cudaError_t copy_split_on(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                          cudaStream_t st) {
  PipeRes* pr = nullptr;
  cudaError_t e = pipe_resources(&pr);
  if (e != cudaSuccess) return e;
  if ((e = cudaEventRecord(pr->ev_a, st)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(pr->aux, pr->ev_a, 0)) != cudaSuccess) return e;
  const cudaStream_t s[2] = {st, pr->aux};
  if ((e = copy_split(dst, src, bytes, kind, s)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(pr->ev_b, pr->aux)) != cudaSuccess) return e;
  return cudaStreamWaitEvent(st, pr->ev_b, 0);
}

cudaStream_t st_of(void* stream) { return static_cast<cudaStream_t>(stream); }

template <int E, int QX, int QZ>
int launch_pack_rect(const void* src, char* const* peer, int rank, int b, int g, int sb,
                     cudaStream_t st);

// Rectangular pack tiles per element size (1 KB destination rows): E=4
// (8,6), E=8 (7,5), E=16 (6,6); BITREV_ETILE when the shape does not fit.
int dispatch_pack_rect(int E, const void* src, char* const* peer, int rank, int b, int g, int sb,
                       cudaStream_t st) {
  if (!aligned16(src)) return BITREV_ETILE;
  for (int d = 0; d < (1 << g); ++d)
    if (!aligned16(peer[d])) return BITREV_ETILE;
  if (E == 4) return launch_pack_rect<4, 8, 6>(src, peer, rank, b, g, sb, st);
  if (E == 8) return launch_pack_rect<8, 7, 5>(src, peer, rank, b, g, sb, st);
  if (E == 16) return launch_pack_rect<16, 6, 6>(src, peer, rank, b, g, sb, st);
  return BITREV_ETILE;
}

template <int E, int QX, int QZ>
int launch_pack_rect(const void* src, char* const* peer, int rank, int b, int g, int sb,
                     cudaStream_t st) {
  using T = Rect<E, QX, QZ>;
  if (b < QX + QZ || sb < QX) return BITREV_ETILE;
  auto kern = bitrev_pack_rect_kernel<E, QX, QZ>;
  // Dynamic shared memory padded to 80 KB caps the pack at 2 CTAs/SM: the E=8
  // (7,5) tiles would otherwise run 3 (80 registers) and measured 0.92-0.94
  // of the peak against 0.95-0.97 at 2 (profiles/r02_pack_smem_ab.jsonl).
  // BITREV_B200_PACK_SMEM_KB overrides the pad (A/B runs; 0 = none).
  static const int pad_kb = env_int("BITREV_B200_PACK_SMEM_KB", 80);
  const int smem = pad_kb * 1024 > T::BYTES ? pad_kb * 1024 : T::BYTES;
  const int per_sm = prepare_kernel(kern, T::THREADS, smem);
  PackArgs pa;
  memset(&pa, 0, sizeof pa);
  TileArgs& a = pa.t;
  a.src = static_cast<const char*>(src);
  a.b = b;
  a.m = b - QX - QZ;
  a.ntiles = 1ull << a.m;
  a.batch = 1;
  for (int d = 0; d < (1 << g); ++d) pa.peer[d] = peer[d];
  pa.g = g;
  pa.sb = sb;
  pa.rank = rank;
  kern<<<pack_grid(a.ntiles, per_sm), T::THREADS, smem, st>>>(pa);
  return finish_launch();
}

// swap_count (src/schedule.py:23-37) in closed form: (2^b - 2^ceil(b/2)) / 2
uint64_t swap_count_dev_host(int b) {
  return ((1ull << b) - (1ull << ((b + 1) >> 1))) >> 1;
}

}  // namespace

extern "C" {

const char* bitrev_version(void) { return "bitrev_b200 0.1.0 sm_100a"; }

const char* bitrev_strerror(int code) {
  switch (code) {
    case BITREV_OK: return "ok";
    case BITREV_EWIDTH: return "bit width must be in 1..48";
    case BITREV_EELEM: return "element size must be 1, 2, 4, 8 or 16 bytes";
    case BITREV_ENULL: return "null data pointer";
    case BITREV_EBATCH: return "batch must be >= 1 and batch strides >= 2**b";
    case BITREV_EOVERLAP: return "source and dest must not overlap";
    case BITREV_ESHARD: return "sharded plan needs 2g <= b (global width)";
    case BITREV_ETILE: return "tile bits not instantiated for this element size";
    case BITREV_ESTAGES: return "stages must be in 0..b (fused tiles: at most 7 for complex64, 6 for complex128)";
    case BITREV_EALIGN: return "fused FFT tiles need 16-byte aligned rows";
  }
  if (code > 0) return cudaGetErrorString(static_cast<cudaError_t>(code));
  return "unknown bitrev error";
}

int bitrev_oop(const void* src, void* dst, int b, int elem_bytes, int64_t batch,
               int64_t src_batch_stride, int64_t dst_batch_stride, void* stream) {
  const int E = elem_bytes;
  int rc = check_common(b, E, batch);
  if (rc) return rc;
  if (!src || !dst) return BITREV_ENULL;
  const int64_t n = int64_t(1) << b;
  if (batch > 1 && (src_batch_stride < n || dst_batch_stride < n)) return BITREV_EBATCH;
  if (batch == 1) src_batch_stride = dst_batch_stride = n;
  {
    const uintptr_t s0 = (uintptr_t)src, d0 = (uintptr_t)dst;
    const uintptr_t s1 = s0 + (uintptr_t)((batch - 1) * src_batch_stride + n) * E;
    const uintptr_t d1 = d0 + (uintptr_t)((batch - 1) * dst_batch_stride + n) * E;
    if (s0 < d1 && d0 < s1) return BITREV_EOVERLAP;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec_ok = aligned16(src) && aligned16(dst) && ((src_batch_stride * E) % 16 == 0) &&
                      ((dst_batch_stride * E) % 16 == 0);
  if (n * E <= kSmallBytes) {
    // short rows: many rows per CTA (5.9-6.3 TB/s for every b measured, up to
    // 8.8x the one-row-per-CTA kernel and above the tile kernels in place;
    // tools/small_rows_probe.py -> profiles/r01_short_rows.jsonl)
    if (vec_ok && (E == 4 || E == 8 || E == 16)) {
      rc = dispatch_rows(E, src, dst, b, batch, src_batch_stride, dst_batch_stride, st);
      if (rc != BITREV_ETILE) return note(rc, 0, -3);
    }
    return note(dispatch_small(E, src, dst, b, batch, src_batch_stride, dst_batch_stride, st), 0,
                -1);
  }
  if (vec_ok && (E == 4 || E == 8 || E == 16)) {
    // configured path first; every miss (shape not instantiated, b too small)
    // falls through to the square register tiles, then to the gather kernel
    int path = tile_path(E, false), q0 = current_q(E, false);
    Tier t = mid_tier(E, false, side_bytes(E, b, batch));
    if (!t.q) t = batched_rows_tier(E, false, b, batch);
    if (t.q) {
      q0 = t.q;
      path = t.path;
    }
    if (path == 3) {
      rc = dispatch_oop_rect(E, q0, src, dst, b, batch, src_batch_stride, dst_batch_stride, st);
      if (rc != BITREV_ETILE) return note(rc, q0, 3);
    }
    for (int q = clamp_q(q0, b); q >= 3; --q) {
      if (path == 1 || path == 2) {
        rc = dispatch_ring(path, E, q, false, src, dst, b, batch, src_batch_stride,
                           dst_batch_stride, st);
        if (rc != BITREV_ETILE) return note(rc, q, path);
      }
      rc = dispatch_oop_tile(E, q, src, dst, b, batch, src_batch_stride, dst_batch_stride, st);
      if (rc != BITREV_ETILE) return note(rc, q, 0);
    }
  }
  return note(dispatch_gather(E, src, dst, b, batch, src_batch_stride, dst_batch_stride, st), 0,
              -2);
}

int bitrev_inplace(void* a, int b, int elem_bytes, int64_t batch, int64_t batch_stride,
                   void* stream) {
  const int E = elem_bytes;
  int rc = check_common(b, E, batch);
  if (rc) return rc;
  if (!a) return BITREV_ENULL;
  const int64_t n = int64_t(1) << b;
  if (batch > 1 && batch_stride < n) return BITREV_EBATCH;
  if (batch == 1) batch_stride = n;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec_ok = aligned16(a) && ((batch_stride * E) % 16 == 0);
  if (vec_ok && rows_inplace_ok(E, b, batch)) {
    rc = dispatch_rows(E, a, a, b, batch, batch_stride, batch_stride, st);
    if (rc != BITREV_ETILE) return note(rc, 0, -3);
  }
  if (n * E <= kSmallBytes) {  // short rows: see bitrev_oop
    if (vec_ok && (E == 4 || E == 8 || E == 16)) {
      rc = dispatch_rows(E, a, a, b, batch, batch_stride, batch_stride, st);
      if (rc != BITREV_ETILE) return note(rc, 0, -3);
    }
    return note(dispatch_small(E, a, a, b, batch, batch_stride, batch_stride, st), 0, -1);
  }
  if (vec_ok && (E == 4 || E == 8 || E == 16)) {
    int path = tile_path(E, true);
    const Tier t = mid_tier(E, true, side_bytes(E, b, batch));
    if (t.q) path = t.path;
    for (int q = clamp_q(t.q ? t.q : current_q(E, true), b); q >= 3; --q) {
      if (path == 4) {
        rc = dispatch_ip_cpa(E, q, a, b, batch, batch_stride, st);
        if (rc != BITREV_ETILE) return note(rc, q, 4);
      }
      if (path == 5) {
        rc = dispatch_ip_tstore(E, q, a, b, batch, batch_stride, st);
        if (rc != BITREV_ETILE) return note(rc, q, 5);
      }
      if (path == 6) {
        rc = dispatch_ip_cluster(E, q, a, b, batch, batch_stride, st);
        if (rc != BITREV_ETILE) return note(rc, q, 6);
      }
      if (path == 1 || path == 2) {
        rc = dispatch_ring(path, E, q, true, a, a, b, batch, batch_stride, batch_stride, st);
        if (rc != BITREV_ETILE) return note(rc, q, path);
      }
      rc = dispatch_ip_tile(E, q, a, b, batch, batch_stride, st);
      if (rc != BITREV_ETILE) return note(rc, q, 0);
    }
  }
  return note(dispatch_swap(E, a, b, batch, batch_stride, st), 0, -2);
}

int bitrev_oop_host(const void* host_src, void* host_dst, int b, int elem_bytes, int64_t batch,
                    void* dev_src, void* dev_dst, void* stream) {
  int rc = check_common(b, elem_bytes, batch);
  if (rc) return rc;
  if (!host_src || !host_dst) return BITREV_ENULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = ((size_t)1 << b) * (size_t)elem_bytes * (size_t)batch;
  // NULL scratch: stream-ordered allocation from the device's default pool
  void* own = nullptr;
  if (!dev_src || !dev_dst) {
    cudaError_t e = cudaMallocAsync(&own, 2 * bytes, st);
    if (e != cudaSuccess) return (int)e;
    dev_src = own;
    dev_dst = static_cast<char*>(own) + bytes;
  }
  const int64_t n = int64_t(1) << b;
  cudaError_t e = pageable(host_src) ? h2d_staged(dev_src, host_src, bytes, st)
                                     : copy_split_on(dev_src, host_src, bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    rc = bitrev_oop(dev_src, dev_dst, b, elem_bytes, batch, n, n, stream);
    if (rc == BITREV_OK) {
      e = pageable(host_dst) ? d2h_staged(host_dst, dev_dst, bytes, st)
                             : copy_split_on(host_dst, dev_dst, bytes, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) rc = (int)e;
    }
  } else {
    rc = (int)e;
  }
  if (own) cudaFreeAsync(own, st);
  e = cudaStreamSynchronize(st);
  if (rc == BITREV_OK && e != cudaSuccess) rc = (int)e;
  return rc;
}

int bitrev_inplace_host(void* host_a, int b, int elem_bytes, int64_t batch, void* dev_buf,
                        void* stream) {
  int rc = check_common(b, elem_bytes, batch);
  if (rc) return rc;
  if (!host_a) return BITREV_ENULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = ((size_t)1 << b) * (size_t)elem_bytes * (size_t)batch;
  void* own = nullptr;
  if (!dev_buf) {
    cudaError_t e = cudaMallocAsync(&own, bytes, st);
    if (e != cudaSuccess) return (int)e;
    dev_buf = own;
  }
  const int64_t n = int64_t(1) << b;
  const bool pg = pageable(host_a);
  cudaError_t e = pg ? h2d_staged(dev_buf, host_a, bytes, st)
                     : copy_split_on(dev_buf, host_a, bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    rc = bitrev_inplace(dev_buf, b, elem_bytes, batch, n, stream);
    if (rc == BITREV_OK) {
      e = pg ? d2h_staged(host_a, dev_buf, bytes, st)
             : copy_split_on(host_a, dev_buf, bytes, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) rc = (int)e;
    }
  } else {
    rc = (int)e;
  }
  if (own) cudaFreeAsync(own, st);
  e = cudaStreamSynchronize(st);
  if (rc == BITREV_OK && e != cudaSuccess) rc = (int)e;
  return rc;
}

}  // extern "C"

namespace {

// The pinned-memory pipeline shared by bitrev_host_pipeline (permutation in
// place in each slot) and bitrev_dit_prepass_host_pipeline (FFT pre-pass out
// of place: two buffers per slot): array k's H2D (sin[0..1]) overlaps array
// k-1's kernel (sk) and array k-2's D2H (sout[0..1]), over kPipeSlots device
// slots of `bufs` * bytes.  op(in, out, stream) runs the kernel(s) of one
// array; out == in when bufs == 1.  Synchronous.
template <typename Op>
int pipeline_run(const void* const* host_src, void* const* host_dst, int64_t count, size_t bytes,
                 int bufs, Op op, void* dev_scratch, cudaStream_t user) {
  constexpr int kSlots = kPipeSlots;
  const size_t slot_bytes = bytes * (size_t)bufs;
  void* own = nullptr;
  char* slots = static_cast<char*>(dev_scratch);
  cudaError_t e = cudaSuccess;
  int rc = BITREV_OK;
  PipeRes* pr = nullptr;
#define PIPE_TRY(x)              \
  do {                           \
    e = (x);                     \
    if (e != cudaSuccess) goto done; \
  } while (0)
  PIPE_TRY(pipe_resources(&pr));
  // order after the caller's prior work
  PIPE_TRY(cudaEventRecord(pr->ev_start, user));
  for (int i = 0; i < 2; ++i) PIPE_TRY(cudaStreamWaitEvent(pr->sin[i], pr->ev_start, 0));
  if (!slots) {
    PIPE_TRY(cudaMallocAsync(&own, kSlots * slot_bytes, pr->sin[0]));
    slots = static_cast<char*>(own);
    PIPE_TRY(cudaEventRecord(pr->ev_a, pr->sin[0]));  // the allocation, for sin[1]
    PIPE_TRY(cudaStreamWaitEvent(pr->sin[1], pr->ev_a, 0));
  }
  for (int64_t k = 0; k < count; ++k) {
    const int s = (int)(k % kSlots);
    char* buf = slots + (size_t)s * slot_bytes;
    char* obuf = bufs > 1 ? buf + bytes : buf;
    auto wait_out = [&](int slot) -> cudaError_t {  // both in-streams after slot's D2H
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
          const cudaError_t r = cudaStreamWaitEvent(pr->sin[i], pr->ev_out[slot][j], 0);
          if (r != cudaSuccess) return r;
        }
      return cudaSuccess;
    };
    if (k >= kSlots) PIPE_TRY(wait_out(s));  // slot drained
    // the host source may be the destination of a step still in flight
    for (int64_t j = k - 1; j >= 0 && j > k - kSlots; --j) {
      const uintptr_t a0 = (uintptr_t)host_src[k], d0 = (uintptr_t)host_dst[j];
      if (a0 < d0 + bytes && d0 < a0 + bytes) PIPE_TRY(wait_out((int)(j % kSlots)));
    }
    PIPE_TRY(copy_split(buf, host_src[k], bytes, cudaMemcpyHostToDevice, pr->sin));
    for (int i = 0; i < 2; ++i) {
      PIPE_TRY(cudaEventRecord(pr->ev_in[s][i], pr->sin[i]));
      PIPE_TRY(cudaStreamWaitEvent(pr->sk, pr->ev_in[s][i], 0));
    }
    rc = op(buf, obuf, pr->sk);
    if (rc != BITREV_OK) goto done;
    PIPE_TRY(cudaEventRecord(pr->ev_k[s], pr->sk));
    for (int i = 0; i < 2; ++i) PIPE_TRY(cudaStreamWaitEvent(pr->sout[i], pr->ev_k[s], 0));
    PIPE_TRY(copy_split(host_dst[k], obuf, bytes, cudaMemcpyDeviceToHost, pr->sout));
    for (int i = 0; i < 2; ++i) PIPE_TRY(cudaEventRecord(pr->ev_out[s][i], pr->sout[i]));
  }
  // sout[0] after every D2H (each D2H after its kernel, each kernel after its H2D)
  PIPE_TRY(cudaEventRecord(pr->ev_b, pr->sout[1]));
  PIPE_TRY(cudaStreamWaitEvent(pr->sout[0], pr->ev_b, 0));
  if (own) {
    PIPE_TRY(cudaFreeAsync(own, pr->sout[0]));
    own = nullptr;
  }
  PIPE_TRY(cudaStreamSynchronize(pr->sout[0]));
done:
#undef PIPE_TRY
  // error or not, nothing may still be using the slots when this returns
  if (pr) {
    for (int i = 0; i < 2; ++i) {
      cudaStreamSynchronize(pr->sin[i]);
      cudaStreamSynchronize(pr->sout[i]);
    }
    cudaStreamSynchronize(pr->sk);
  }
  if (own) cudaFree(own);  // only on an error path: the normal path frees stream-ordered
  if (rc != BITREV_OK) return rc;
  return e == cudaSuccess ? BITREV_OK : (int)e;
}

int check_pipeline_args(const void* const* host_src, void* const* host_dst, int64_t count) {
  if (count < 0) return BITREV_EBATCH;
  if (count == 0) return BITREV_OK;
  if (!host_src || !host_dst) return BITREV_ENULL;
  for (int64_t k = 0; k < count; ++k)
    if (!host_src[k] || !host_dst[k]) return BITREV_ENULL;
  return BITREV_OK;
}

bool any_pageable(const void* const* host_src, void* const* host_dst, int64_t count) {
  for (int64_t k = 0; k < count; ++k)
    if (pageable(host_src[k]) || pageable(host_dst[k])) return true;
  return false;
}

}  // namespace

extern "C" {

int bitrev_host_pipeline(const void* const* host_src, void* const* host_dst, int64_t count, int b,
                         int elem_bytes, int64_t batch, void* dev_scratch, void* stream) {
  int rc = check_common(b, elem_bytes, batch);
  if (rc) return rc;
  if ((rc = check_pipeline_args(host_src, host_dst, count)) != BITREV_OK || count == 0) return rc;
  const size_t bytes = ((size_t)1 << b) * (size_t)elem_bytes * (size_t)batch;
  const int64_t n = int64_t(1) << b;
  if (any_pageable(host_src, host_dst, count)) {
    // pageable arrays cannot overlap their copies (the runtime stages them
    // synchronously): run each through the bounce-ring single call instead
    for (int64_t k = 0; k < count; ++k) {
      if (host_src[k] != host_dst[k]) {
        rc = bitrev_oop_host(host_src[k], host_dst[k], b, elem_bytes, batch, dev_scratch,
                             dev_scratch ? static_cast<char*>(dev_scratch) + bytes : nullptr,
                             stream);
      } else {
        rc = bitrev_inplace_host(host_dst[k], b, elem_bytes, batch, dev_scratch, stream);
      }
      if (rc != BITREV_OK) return rc;
    }
    return BITREV_OK;
  }
  auto op = [&](char* in, char*, cudaStream_t st) {
    return bitrev_inplace(in, b, elem_bytes, batch, n, st);
  };
  return pipeline_run(host_src, host_dst, count, bytes, 1, op, dev_scratch,
                      static_cast<cudaStream_t>(stream));
}

int bitrev_dit_prepass_host_pipeline(const void* const* host_src, void* const* host_dst,
                                     int64_t count, int b, int elem_bytes, int64_t batch,
                                     int stages, int inverse, void* dev_scratch, void* stream) {
  if (elem_bytes != 8 && elem_bytes != 16) return BITREV_EELEM;
  int rc = check_common(b, elem_bytes, batch);
  if (rc) return rc;
  if (stages < 0 || stages > b) return BITREV_ESTAGES;
  if ((rc = check_pipeline_args(host_src, host_dst, count)) != BITREV_OK || count == 0) return rc;
  const size_t bytes = ((size_t)1 << b) * (size_t)elem_bytes * (size_t)batch;
  const int64_t n = int64_t(1) << b;
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  auto op = [&](char* in, char* out, cudaStream_t st) {
    return bitrev_dit_prepass(in, out, b, elem_bytes, batch, n, n, stages, inverse, st);
  };
  if (any_pageable(host_src, host_dst, count)) {
    // one array at a time through the pinned bounce ring (see bitrev_oop_host)
    void* own = nullptr;
    char* buf = static_cast<char*>(dev_scratch);
    cudaError_t e = cudaSuccess;
    if (!buf) {
      if ((e = cudaMallocAsync(&own, 2 * bytes, user)) != cudaSuccess) return (int)e;
      buf = static_cast<char*>(own);
    }
    for (int64_t k = 0; k < count && rc == BITREV_OK && e == cudaSuccess; ++k) {
      if ((e = h2d_staged(buf, host_src[k], bytes, user)) != cudaSuccess) break;
      if ((rc = op(buf, buf + bytes, user)) != BITREV_OK) break;
      e = d2h_staged(host_dst[k], buf + bytes, bytes, user);
    }
    if (own) {
      const cudaError_t f = cudaFreeAsync(own, user);
      const cudaError_t s2 = cudaStreamSynchronize(user);
      if (e == cudaSuccess) e = f != cudaSuccess ? f : s2;
    }
    if (rc != BITREV_OK) return rc;
    return e == cudaSuccess ? BITREV_OK : (int)e;
  }
  return pipeline_run(host_src, host_dst, count, bytes, 2, op, dev_scratch, user);
}

int bitrev_transpose_square(void* a, int h, int elem_bytes, int64_t batch, int64_t batch_stride,
                            void* stream) {
  if (h < 0 || 2 * h > kMaxBits) return BITREV_EWIDTH;
  if (!valid_elem(elem_bytes)) return BITREV_EELEM;
  if (batch < 1) return BITREV_EBATCH;
  if (!a) return BITREV_ENULL;
  const int64_t n = int64_t(1) << (2 * h);
  if (batch > 1 && batch_stride < n) return BITREV_EBATCH;
  if (batch == 1) batch_stride = n;
  if (h == 0) return BITREV_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec_ok = aligned16(a) && ((batch_stride * elem_bytes) % 16 == 0);
  // vectorised tile pairs: 256-byte rows (512 for complex128)
  const int tq = elem_bytes == 4 ? 6 : 5;
  if (vec_ok && (elem_bytes == 4 || elem_bytes == 8 || elem_bytes == 16) && h >= tq) {
    const uint64_t nt = 1ull << (h - tq);
    const uint64_t work = nt * (nt + 1) / 2 * (uint64_t)batch;
#define TRT_CASE(E_, Q_)                                                                   \
  if (elem_bytes == E_) {                                                                  \
    using T = TrTile<E_, Q_>;                                                              \
    auto kern = transpose_tile_kernel<E_, Q_>;                                             \
    const int per_sm = prepare_kernel(kern, T::THREADS, 2 * T::BYTES);                    \
    kern<<<grid_for(work, per_sm), T::THREADS, 2 * T::BYTES, st>>>(static_cast<char*>(a), h, \
                                                                   batch, batch_stride * E_); \
    return finish_launch();                                                                \
  }
    TRT_CASE(4, 6) TRT_CASE(8, 5) TRT_CASE(16, 5)
#undef TRT_CASE
  }
  const int side = 1 << h;
  const int ts = side < kTT ? side : kTT;
  const uint64_t nt = (uint64_t)(side / ts);
  const uint64_t work = nt * nt * (uint64_t)batch;
  const int grid = grid_for(work, 6);
  switch (elem_bytes) {
#define TR_CASE(E)                                                                        \
  case E:                                                                                 \
    transpose_square_kernel<E><<<grid, 256, 0, st>>>(static_cast<char*>(a), h, batch,     \
                                                     batch_stride * E);                   \
    return finish_launch();
    TR_CASE(1) TR_CASE(2) TR_CASE(4) TR_CASE(8) TR_CASE(16)
#undef TR_CASE
  }
  return BITREV_EELEM;
}

int bitrev_stockham_scratch(const void* a, void* scratch, int b, int elem_bytes, void* stream) {
  const int E = elem_bytes;
  if (b < 1 || b > kMaxBits) return BITREV_EWIDTH;
  if (!valid_elem(E)) return BITREV_EELEM;
  if (!a || !scratch) return BITREV_ENULL;
  const uint64_t n = 1ull << b;
  {
    const uintptr_t a0 = (uintptr_t)a, s0 = (uintptr_t)scratch;
    if (a0 < s0 + n * E && s0 < a0 + n * E) return BITREV_EOVERLAP;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned grid = (unsigned)elementwise_grid(n);
  switch (E) {
#define SS_CASE(E_)                                                                          \
  case E_:                                                                                   \
    stockham_scratch_kernel<E_><<<grid, 256, 0, st>>>(static_cast<const char*>(a),            \
                                                      static_cast<char*>(scratch), b);        \
    return finish_launch();
    SS_CASE(1) SS_CASE(2) SS_CASE(4) SS_CASE(8) SS_CASE(16)
#undef SS_CASE
  }
  return BITREV_EELEM;
}

int bitrev_even_odd(const void* src, void* dst, int b, int elem_bytes, int64_t batch,
                    int64_t src_batch_stride, int64_t dst_batch_stride, void* stream) {
  const int E = elem_bytes;
  int rc = check_common(b, E, batch);
  if (rc) return rc;
  if (!src || !dst) return BITREV_ENULL;
  const int64_t n = int64_t(1) << b;
  if (batch > 1 && (src_batch_stride < n || dst_batch_stride < n)) return BITREV_EBATCH;
  if (batch == 1) src_batch_stride = dst_batch_stride = n;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t total = (uint64_t)(n / 2) * (uint64_t)batch;
  const unsigned grid = (unsigned)elementwise_grid(total);
  switch (E) {
#define EO_CASE(E_)                                                                          \
  case E_:                                                                                   \
    even_odd_kernel<E_><<<grid, 256, 0, st>>>(static_cast<const char*>(src),                  \
                                              static_cast<char*>(dst), b, batch,              \
                                              src_batch_stride * E_, dst_batch_stride * E_); \
    return finish_launch();
    EO_CASE(1) EO_CASE(2) EO_CASE(4) EO_CASE(8) EO_CASE(16)
#undef EO_CASE
  }
  return BITREV_EELEM;
}

int bitrev_apply_pairs(void* a, const void* pairs, int64_t npairs, int elem_bytes, void* stream) {
  if (!valid_elem(elem_bytes)) return BITREV_EELEM;
  if (npairs < 0) return BITREV_EBATCH;
  if (npairs == 0) return BITREV_OK;
  if (!a || !pairs) return BITREV_ENULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned grid = (unsigned)elementwise_grid((uint64_t)npairs);
  const long long* pr = static_cast<const long long*>(pairs);
  switch (elem_bytes) {
#define AP_CASE(E_)                                                                  \
  case E_:                                                                           \
    apply_pairs_kernel<E_><<<grid, 256, 0, st>>>(static_cast<char*>(a), pr, npairs); \
    return finish_launch();
    AP_CASE(1) AP_CASE(2) AP_CASE(4) AP_CASE(8) AP_CASE(16)
#undef AP_CASE
  }
  return BITREV_EELEM;
}

int bitrev_apply_pairs_ordered(void* a, const void* pairs, int64_t npairs, int elem_bytes,
                               void* stream) {
  if (!valid_elem(elem_bytes)) return BITREV_EELEM;
  if (npairs < 0) return BITREV_EBATCH;
  if (npairs == 0) return BITREV_OK;
  if (!a || !pairs) return BITREV_ENULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long* pr = static_cast<const long long*>(pairs);
  switch (elem_bytes) {
#define APO_CASE(E_)                                                                    \
  case E_:                                                                              \
    apply_pairs_ordered_kernel<E_><<<1, 32, 0, st>>>(static_cast<char*>(a), pr, npairs); \
    return finish_launch();
    APO_CASE(1) APO_CASE(2) APO_CASE(4) APO_CASE(8) APO_CASE(16)
#undef APO_CASE
  }
  return BITREV_EELEM;
}

int bitrev_swap_schedule(int b, void* pairs_out, void* stream) {
  if (b < 1 || b > kMaxBits) return BITREV_EWIDTH;
  if (!pairs_out) return BITREV_ENULL;
  const uint64_t count = b <= 2 ? (uint64_t)(b - 1) : swap_count_dev_host(b);
  if (count == 0) return BITREV_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  swap_schedule_kernel<<<(unsigned)elementwise_grid(count), 256, 0, st>>>(
      static_cast<long long*>(pairs_out), b, count);
  return finish_launch();
}

int bitrev_dit_prepass(const void* src, void* dst, int b, int elem_bytes, int64_t batch,
                       int64_t src_batch_stride, int64_t dst_batch_stride, int stages,
                       int inverse, void* stream) {
  const int E = elem_bytes;
  int rc = check_common(b, E, batch);
  if (rc) return rc;
  if (E != 8 && E != 16) return BITREV_EELEM;
  if (!src || !dst) return BITREV_ENULL;
  const int64_t n = int64_t(1) << b;
  if (batch > 1 && (src_batch_stride < n || dst_batch_stride < n)) return BITREV_EBATCH;
  if (batch == 1) src_batch_stride = dst_batch_stride = n;
  {
    const uintptr_t s0 = (uintptr_t)src, d0 = (uintptr_t)dst;
    const uintptr_t s1 = s0 + (uintptr_t)((batch - 1) * src_batch_stride + n) * E;
    const uintptr_t d1 = d0 + (uintptr_t)((batch - 1) * dst_batch_stride + n) * E;
    if (s0 < d1 && d0 < s1) return BITREV_EOVERLAP;
  }
  if (stages < 0 || stages > b) return BITREV_ESTAGES;
  // No butterflies: the plain permutation kernels are faster than the
  // butterfly tiles with zero stages (6.43 vs 5.32 TB/s complex128, 6.32 vs
  // 6.02 complex64, profiles/r01_fft_qz_ab.txt).
  if (stages == 0)
    return bitrev_oop(src, dst, b, E, batch, src_batch_stride, dst_batch_stride, stream);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  FftArgs fa;
  memset(&fa, 0, sizeof fa);
  fa.stages = stages;
  fa.inverse = inverse ? 1 : 0;
  TileArgs& a = fa.t;
  a.src = static_cast<const char*>(src);
  a.dst = static_cast<char*>(dst);
  a.b = b;
  a.batch = batch;
  a.src_bstride = src_batch_stride * E;
  a.dst_bstride = dst_batch_stride * E;
  const bool rows_ok = aligned16(src) && aligned16(dst) && ((src_batch_stride * E) % 16 == 0) &&
                       ((dst_batch_stride * E) % 16 == 0) && b >= (E == 8 ? 1 : 0);
  // rows of 64 KB take the staged-row kernel only for more stages than the
  // tiles fuse (a complete FFT of the row): for <= 7 / 6 stages the tiles run
  // 6.1-6.4 TB/s against 1.7-5.2 (tools/fft64_probe.py)
  const int tile_stages = E == 8 ? 7 : 6;
  if (rows_ok && (n * E <= kSmallBytes || (n * E <= 2 * kSmallBytes && stages > tile_stages))) {
    // many short rows per CTA (one row per CTA for 64 KB rows); the stages run
    // on the staged block in shared memory (fft_rows_kernel)
    const int lv = E == 8 ? 1 : 0;
    const int vb = b - lv;
    const int sh = vb - lv - 3 > 3 ? vb - lv - 3 : 3;
    const bool big = n * E > kSmallBytes;
    // 16 KB blocks for rows up to 16 KB: +1-6 % over 32 KB blocks
    // (profiles/r01_short_row_fft.jsonl history in DESIGN.md)
    const bool small16 = n * E <= kSmallBytes / 2;
    const int lblk = big ? 12 : (small16 ? 10 : 11);  // log2(block bytes / 16)
    const int64_t nblocks = (batch + (int64_t(1) << (lblk - vb)) - 1) >> (lblk - vb);
    const int blk_bytes = big ? 2 * kSmallBytes : (small16 ? kSmallBytes / 2 : kSmallBytes);
    const int smem = blk_bytes + (int)((n / 2) * E);
    // rotated quad order for longer rows (profiles/r01_short_row_fft.jsonl)
    const bool rot = E == 8 ? b >= 10 : b >= 8;
    auto kern = big ? (E == 8 ? fft_rows_kernel<8, true, 64> : fft_rows_kernel<16, true, 64>)
              : small16 ? (E == 8 ? (rot ? fft_rows_kernel<8, true, 16> : fft_rows_kernel<8, false, 16>)
                                  : (rot ? fft_rows_kernel<16, true, 16> : fft_rows_kernel<16, false, 16>))
                    : (E == 8 ? (rot ? fft_rows_kernel<8, true> : fft_rows_kernel<8, false>)
                              : (rot ? fft_rows_kernel<16, true> : fft_rows_kernel<16, false>));
    const int per_sm = prepare_kernel(kern, 256, blk_bytes + blk_bytes / 2);
    kern<<<grid_for((uint64_t)nblocks, per_sm), 256, smem, st>>>(fa, sh);
    return finish_launch();
  }
  if (n * E <= kSmallBytes) {
    const int bytes = (int)(n * E);
    const int grid = grid_for((uint64_t)batch, 8);
    if (E == 8) {
      prepare_kernel(fft_prepass_small_kernel<8>, 256, kSmallBytes);
      fft_prepass_small_kernel<8><<<grid, 256, bytes, st>>>(fa);
    } else {
      prepare_kernel(fft_prepass_small_kernel<16>, 256, kSmallBytes);
      fft_prepass_small_kernel<16><<<grid, 256, bytes, st>>>(fa);
    }
    return finish_launch();
  }
  // complex128 with 1-5 stages: the square Q6 tiles of the out-of-place
  // kernel (1 KB rows on both sides) with the stages on warp shuffles in the
  // drain (bitrev_fft_tile16_kernel, select-free butterflies): 2048 x 2^16,
  // 1 / 2 / 3 / 4 / 5 stages 5988 / 5698 / 6401 / 6330 / 5987 ->
  // 6494 / 6425 / 6405 / 6758 / 6100 GB/s against the rectangular radix-4
  // drain (tools/fft_c128_tile_ab.sh, fft_c128_tile2_ab.sh ->
  // profiles/r02_fft_c128_tile*_ab.txt; the first form, with selects, lost
  // 15 / 30 % at 4 / 5 stages).  BITREV_B200_FFT_C128_TILE=0 keeps the
  // rectangular tiles, BITREV_B200_FFT_C128_TILE_MAX caps the stage count
  // (A/B runs).
  static const int c128_tile = env_int("BITREV_B200_FFT_C128_TILE", 1);
  static const int c128_tile_max = env_int("BITREV_B200_FFT_C128_TILE_MAX", 5);
  if (E == 16 && c128_tile && stages <= c128_tile_max && b >= 12 && aligned16(src) &&
      aligned16(dst)) {
    a.m = b - 12;
    a.ntiles = (uint64_t)batch << a.m;
    constexpr int kBytes = 64 * 64 * 16;
#define FFT16_LAUNCH(S_)                                                                 \
  case S_: {                                                                             \
    auto kern = stream_stores(16, b, batch) ? bitrev_fft_tile16_kernel<S_, true>         \
                                            : bitrev_fft_tile16_kernel<S_, false>;       \
    const int per_sm = prepare_kernel(kern, 256, kBytes);                                \
    return launch_tiles(kern, fft_grid(a.ntiles, per_sm, S_ <= 3 ? 5 : 0), 256, kBytes, st, fa); \
  }
    switch (stages) { FFT16_LAUNCH(1) FFT16_LAUNCH(2) FFT16_LAUNCH(3) FFT16_LAUNCH(4) FFT16_LAUNCH(5) }
#undef FFT16_LAUNCH
  }
  // Fused path: rectangular tiles whose destination rows are the FFT blocks
  // (complex64: QX = 7, 128-element rows, up to 7 stages; complex128: QX = 6,
  // 64-element rows, up to 6 stages).  Rows too big for the small kernel are
  // always wide enough (b >= 13 resp. 12 >= QX + QZ).
  // QZ = 4 source-piece bits for both types (tools/fft_stage_sweep.py,
  // profiles/r01_fft_qz_ab.txt): complex128 with QZ = 3 has 8 rows per tile,
  // and with 2 rows per warp pass half the warps idled in the butterfly drain
  // (16 rows: +29 % at 4 stages); complex64 with QZ = 5 needs ~170 registers
  // (1 CTA/SM) and trails QZ = 4 once the drain's shared-memory conflicts are
  // gone.
  // complex64: 256-byte source pieces (QZ = 5, 32 KB tiles, 2 CTAs/SM) for 2-7
  // fused stages, 128-byte pieces (QZ = 4, 3 CTAs/SM) for 1: measured A/B
  // (profiles/r02_fft_qz_ab.txt): QZ = 5 +1 % / +3 % / +3 % / +5 % / +7 % at
  // 2 / 3 / 4 / 5 / 6 stages, -0.4 % at 1 stage; with the radix-8 drain also
  // +2-4 % at 7 (cfg4-fft7 5646 vs 5493-5564 GB/s, same box).
  // BITREV_B200_FFT_QZ=4|5 forces one shape (A/B runs).
  static const int qz_env = env_int("BITREV_B200_FFT_QZ", 0);
  // complex64: 256-element destination rows (QX = 8: two 128-element FFT
  // blocks per row, radix-8 drain, 64 KB tiles at 1 CTA/SM) against 128-element
  // rows (QX = 7, 2 CTAs/SM), tools/fft_qx8_ab.sh / fft_qx8_low_ab.sh /
  // fft_qx8_sizes.py -> profiles/r02_fft_qx8_*: 1 stage +6-14 % at every
  // shape, 2-5 stages +3-7 % on rows up to 2^18 and neutral (0.997-1.03) on
  // longer rows and single arrays; 6-7 stages lose 1-3 % (the drain is
  // issue-bound at one CTA/SM) except on rows of 2^13-2^14 (+7 %).  Launches
  // below 16 MiB per side keep the smaller tiles (wave quantisation).
  // BITREV_B200_FFT_QX=7|8 forces a width (A/B runs).
  static const int qx_env = env_int("BITREV_B200_FFT_QX", 0);
  const bool wide_ok = E == 8 && stages >= 1 && stages <= 7 && b >= 13;
  const bool wide_rule = (stages <= 5 || b <= 14) && side_bytes(E, b, batch) >= (16ull << 20);
  const bool wide = wide_ok && (qx_env == 8 || (qx_env == 0 && wide_rule));
  const int qx = wide ? 8 : E == 8 ? 7 : 6;
  int qz = 4;
  if (E == 8) qz = qz_env == 4 || qz_env == 5 ? qz_env : (stages >= 2 ? 5 : 4);
  if (wide) qz = 5;  // the 256-element rows are instantiated with 256-byte source pieces only
  if (stages > qx || b < qx + qz) return BITREV_ESTAGES;
  const bool vec_ok = aligned16(src) && aligned16(dst) && ((src_batch_stride * E) % 16 == 0) &&
                      ((dst_batch_stride * E) % 16 == 0);
  if (!vec_ok) return BITREV_EALIGN;
  a.m = b - qx - qz;
  a.ntiles = (uint64_t)batch << a.m;
#define FFT_LAUNCH(E_, QX_, QZ_, S_)                                                       \
  case S_: {                                                                                 \
    using T = Rect<E_, QX_, QZ_>;                                                            \
    auto kern = bitrev_fft_rect_kernel<E_, QX_, QZ_, S_>;                                    \
    const int per_sm = prepare_kernel(kern, T::THREADS, T::BYTES);                           \
    return launch_tiles(kern, fft_grid(a.ntiles, per_sm), T::THREADS, T::BYTES, st, fa);     \
  }
  if (wide && qz == 5) {
    switch (stages) {
      FFT_LAUNCH(8, 8, 5, 1) FFT_LAUNCH(8, 8, 5, 2) FFT_LAUNCH(8, 8, 5, 3)
      FFT_LAUNCH(8, 8, 5, 4) FFT_LAUNCH(8, 8, 5, 5) FFT_LAUNCH(8, 8, 5, 6)
      FFT_LAUNCH(8, 8, 5, 7)
    }
  } else if (E == 8 && qz == 5) {
    switch (stages) {
      FFT_LAUNCH(8, 7, 5, 1) FFT_LAUNCH(8, 7, 5, 2) FFT_LAUNCH(8, 7, 5, 3)
      FFT_LAUNCH(8, 7, 5, 4) FFT_LAUNCH(8, 7, 5, 5) FFT_LAUNCH(8, 7, 5, 6)
      FFT_LAUNCH(8, 7, 5, 7)
    }
  } else if (E == 8) {
    switch (stages) {
      FFT_LAUNCH(8, 7, 4, 1) FFT_LAUNCH(8, 7, 4, 2) FFT_LAUNCH(8, 7, 4, 3)
      FFT_LAUNCH(8, 7, 4, 4) FFT_LAUNCH(8, 7, 4, 5) FFT_LAUNCH(8, 7, 4, 6)
      FFT_LAUNCH(8, 7, 4, 7)
    }
  } else {
    switch (stages) {
      FFT_LAUNCH(16, 6, 4, 1) FFT_LAUNCH(16, 6, 4, 2) FFT_LAUNCH(16, 6, 4, 3)
      FFT_LAUNCH(16, 6, 4, 4) FFT_LAUNCH(16, 6, 4, 5) FFT_LAUNCH(16, 6, 4, 6)
    }
  }
#undef FFT_LAUNCH
  return BITREV_ETILE;
}

int bitrev_sharded_scatter(const void* local, void* const* peer_recv, int b_local, int g, int rank,
                           int elem_bytes, void* stream) {
  const int E = elem_bytes;
  if (b_local < 1 || b_local > kMaxBits) return BITREV_EWIDTH;
  if (E != 4 && E != 8 && E != 16) return BITREV_EELEM;
  if (g < 0 || (1 << g) > kMaxPeers || rank < 0 || rank >= (1 << g)) return BITREV_ESHARD;
  if (!local || !peer_recv) return BITREV_ENULL;
  if (b_local < 2 * g) return BITREV_ESHARD;
  char* peer[kMaxPeers] = {};
  for (int d = 0; d < (1 << g); ++d) {
    if (!peer_recv[d]) return BITREV_ENULL;
    peer[d] = static_cast<char*>(peer_recv[d]);
  }
  const int rc = dispatch_pack_rect(E, local, peer, rank, b_local, g, b_local - g, st_of(stream));
  if (rc != BITREV_ETILE) return rc;
  return launch_scatter(local, peer, b_local, g, rank, b_local - g, E, st_of(stream));
}

int bitrev_sharded_pack(const void* local, void* send, int b_local, int g, int chunk_bits,
                        int elem_bytes, void* stream) {
  const int E = elem_bytes;
  if (b_local < 1 || b_local > kMaxBits) return BITREV_EWIDTH;
  if (E != 4 && E != 8 && E != 16) return BITREV_EELEM;
  if (g < 0 || (1 << g) > kMaxPeers || chunk_bits < 0 || b_local < 2 * g + chunk_bits)
    return BITREV_ESHARD;
  if (!local || !send) return BITREV_ENULL;
  const uintptr_t l0 = (uintptr_t)local, s0 = (uintptr_t)send;
  const uintptr_t bytes = (uintptr_t)E << b_local;
  if (l0 < s0 + bytes && s0 < l0 + bytes) return BITREV_EOVERLAP;
  if (chunk_bits == 0)  // one chunk: the send layout is the plain reversal
    return bitrev_oop(local, send, b_local, E, 1, 0, 0, stream);
  const int sb = b_local - g - chunk_bits;
  char* peer[kMaxPeers] = {};
  for (int d = 0; d < (1 << g); ++d) peer[d] = static_cast<char*>(send) + ((uint64_t)E << sb) * d;
  // rectangular tiles with re-addressed rows (1 KB destination rows), else
  // the square scatter tiles (shorter rows fit shorter sub-chunks)
  const int rc = dispatch_pack_rect(E, local, peer, 0, b_local, g, sb, st_of(stream));
  if (rc != BITREV_ETILE) return rc;
  return launch_scatter(local, peer, b_local, g, 0, sb, E, st_of(stream));
}

int bitrev_sharded_unpack(const void* recv, void* dst, int b_local, int g, int elem_bytes,
                          void* stream) {
  const int E = elem_bytes;
  if (b_local < 1 || b_local > kMaxBits) return BITREV_EWIDTH;
  if (!valid_elem(E)) return BITREV_EELEM;
  if (g < 0 || g > b_local) return BITREV_ESHARD;
  if (!recv || !dst) return BITREV_ENULL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t C = 1ull << (b_local - g);
  const char* r = static_cast<const char*>(recv);
  char* d = static_cast<char*>(dst);
  // vector kernel: 16-byte aligned, at least 16 bytes per source chunk, G <= 8
  const bool vec = aligned16(recv) && aligned16(dst) && C * (uint64_t)E >= 16 && g <= 3 &&
                   (E == 4 || E == 8 || E == 16);
  if (vec) {
    const uint64_t threads = C / (16 / E);
    // A grid of up to 256 CTAs per SM (2-4 resident by registers, the rest
    // queued; each CTA strides over few blocks) against 8 per SM: G = 2 / 4 /
    // 8 at the cfg5 shard sizes 6357 / 6132 / 6245 -> 6446 / 6650 / 6688 GB/s
    // (tools/unpack_grid_ab.py -> profiles/r02_unpack_grid_ab*.jsonl).  Short
    // grid-stride loops also let CTAs retire throughout the kernel, which
    // frees SM slots for NCCL's CTAs while later rounds are on the wire.
    // BITREV_B200_UNPACK_PER_SM overrides it (A/B runs).
    static const int per_sm = env_int("BITREV_B200_UNPACK_PER_SM", 256);
    const unsigned grid = (unsigned)grid_for((threads + 255) / 256, per_sm > 0 ? per_sm : 256);
#define UNPACK_G(E_, G_)                                                  \
  case G_:                                                                \
    sharded_unpack_kernel<E_, G_><<<grid, 256, 0, st>>>(r, d, C);         \
    return finish_launch();
#define UNPACK_E(E_)                                                            \
  case E_:                                                                      \
    switch (1 << g) { UNPACK_G(E_, 1) UNPACK_G(E_, 2) UNPACK_G(E_, 4) UNPACK_G(E_, 8) } \
    break;
    switch (E) { UNPACK_E(4) UNPACK_E(8) UNPACK_E(16) }
#undef UNPACK_E
#undef UNPACK_G
  }
  switch (E) {
#define UNPACK_GEN(E_)                                                                    \
  case E_:                                                                                \
    sharded_unpack_generic_kernel<E_><<<(unsigned)elementwise_grid(C << g), 256, 0, st>>>( \
        r, d, C, g);                                                                      \
    return finish_launch();
    UNPACK_GEN(1) UNPACK_GEN(2) UNPACK_GEN(4) UNPACK_GEN(8) UNPACK_GEN(16)
#undef UNPACK_GEN
  }
  return BITREV_EELEM;
}

int bitrev_get_tile_bits(int elem_bytes, int inplace) { return current_q(elem_bytes, inplace != 0); }

int bitrev_set_tile_bits(int elem_bytes, int inplace, int q) {
  if (elem_bytes != 4 && elem_bytes != 8 && elem_bytes != 16) return BITREV_ETILE;
  if (q != 0 && !q_supported(elem_bytes, q)) return BITREV_ETILE;
  (inplace ? g_q_ip : g_q_oop)[elem_bytes].store(q);
  return BITREV_OK;
}

int bitrev_get_tile_path(int elem_bytes, int inplace) { return tile_path(elem_bytes, inplace != 0); }

int bitrev_set_tile_path(int elem_bytes, int inplace, int path) {
  if (elem_bytes != 4 && elem_bytes != 8 && elem_bytes != 16) return BITREV_ETILE;
  if (path < 0 || path > 6 || (path == 3 && inplace) || (path >= 4 && !inplace))
    return BITREV_ETILE;
  (inplace ? g_path_ip : g_path_oop)[elem_bytes].store(path);
  return BITREV_OK;
}

int bitrev_last_tile(int* q, int* path) {
  if (!q || !path) return BITREV_ENULL;
  *q = t_last_q;
  *path = t_last_path;
  return BITREV_OK;
}

int bitrev_get_tile_order(int inplace) { return tile_order(inplace != 0); }

int bitrev_set_tile_order(int inplace, int order) {
  if (order < 0 || (order > 2 && (order & ~0x1ff) != 0) || (order > 2 && order < 0x100))
    return BITREV_ETILE;
  (inplace ? g_order_ip : g_order_oop).store(order);
  return BITREV_OK;
}

int64_t bitrev_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
