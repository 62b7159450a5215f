// Tile-pattern probe with TMA TENSOR copies on both sides (measurement only,
// not product code): as tilebulk.cu, but a whole tile (64 rows x R bytes at
// stride `stride`) moves with ONE cp.async.bulk.tensor.2d load and ONE store
// through a 2-D tensor map {stride/8 units, 64 rows}, box {R/8, 64}.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tiletma tiletma.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t rev(uint64_t v, int w) { return w ? __brevll(v) >> (64 - w) : 0; }
__device__ __forceinline__ void g2s(uint32_t dst, const void* src, uint32_t n, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(n), "r"(bar) : "memory");
}
__device__ __forceinline__ void s2g(void* dst, uint32_t src, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}"
               ::"r"(bar), "r"(ph) : "memory");
}

// SWAP: unit = pair list entry y (tiles y and rev y, exchanged);
// !SWAP: unit = tile y -> tile rev(y) of dst.  Persistent, CTA stride over units.
__device__ __forceinline__ void tload(uint32_t dst, const void* map, int c0, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(map), "r"(c0), "r"(0), "r"(bar) : "memory");
}
__device__ __forceinline__ void tstore(const void* map, int c0, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(map), "r"(c0), "r"(0), "r"(src) : "memory");
}

template <int R, int ROWS, bool SWAP>
__global__ void __launch_bounds__(32) tile_bulk(const __grid_constant__ CUtensorMap mi,
                                                const __grid_constant__ CUtensorMap mo,
                                                const uint32_t* ys, int nunits, int m, int ns) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int TILE = ROWS * R;
  constexpr int SLOT = (SWAP ? 2 : 1) * TILE;
  if (threadIdx.x != 0) return;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bars = base + ns * SLOT;
  for (int i = 0; i < ns; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * i));
  asm volatile("fence.mbarrier_init.release.cluster;");
  uint32_t phase = 0;  // bit i = parity of slot i
  auto unit = [&](int j, uint64_t& y) {
    const int u = blockIdx.x + j * gridDim.x;
    if (u >= nunits) return false;
    y = SWAP ? ys[u] : (uint64_t)u;
    return true;
  };
  auto load = [&](int j) {
    uint64_t y;
    if (!unit(j, y)) return;
    const int slot = j % ns;
    const uint32_t sb = base + slot * SLOT, bb = bars + 8 * slot;
    const uint64_t ry = rev(y, m);
    const bool two = SWAP && ry != y;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb),
                 "r"((two ? 2 : 1) * TILE) : "memory");
    tload(sb, &mi, (int)(y * (R / 8)), bb);
    if (two) tload(sb + TILE, &mi, (int)(ry * (R / 8)), bb);
  };
  for (int j = 0; j < ns - 1; ++j) load(j);
  for (int j = 0;; ++j) {
    uint64_t y;
    if (!unit(j, y)) break;
    const int slot = j % ns;
    const uint32_t sb = base + slot * SLOT, bb = bars + 8 * slot;
    wait_bar(bb, (phase >> slot) & 1);
    phase ^= 1u << slot;
    const uint64_t ry = rev(y, m);
    tstore(&mo, (int)(ry * (R / 8)), sb);
    if (SWAP && ry != y) tstore(&mo, (int)(y * (R / 8)), sb + TILE);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the slot loaded next was last used by unit j-1: its store group must
    // have read shared memory (only unit j's group may stay pending)
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    load(j + ns - 1);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static uint32_t revb(uint32_t v, int m) {
  uint32_t r = 0;
  for (int i = 0; i < m; ++i) r |= ((v >> i) & 1u) << (m - 1 - i);
  return r;
}

template <int R, bool SWAP>
void run(char* a, char* b, uint32_t* d_ys, uint64_t total, int sms, int ns, int cps) {
  constexpr int ROWS = 64;
  const uint64_t stride = total / ROWS;
  int m = 0;
  while (((uint64_t)R << (m + 1)) <= stride) ++m;
  const uint64_t n = 1ull << m;
  std::vector<uint32_t> ys;
  for (uint32_t y = 0; y < n; ++y)
    if (y <= revb(y, m)) ys.push_back(y);
  cudaMemcpy(d_ys, ys.data(), ys.size() * 4, cudaMemcpyHostToDevice);
  const int nunits = SWAP ? (int)ys.size() : (int)n;
  const int smem = ns * (SWAP ? 2 : 1) * ROWS * R + 8 * ns;
  auto k = tile_bulk<R, ROWS, SWAP>;
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  CUtensorMap mi, mo;
  auto make = [&](CUtensorMap* mp, void* base) {
    cuuint64_t dims[2] = {stride / 8, (cuuint64_t)ROWS};
    cuuint64_t strides[1] = {stride};
    cuuint32_t box[2] = {R / 8, ROWS};
    cuuint32_t es[2] = {1, 1};
    return enc(mp, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  char* dst = SWAP ? a : b;
  if (make(&mi, a) != CUDA_SUCCESS || make(&mo, dst) != CUDA_SUCCESS) {
    printf("{\"R\": %d, \"error\": \"tensor map encode failed\"}\n", R);
    return;
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem + 1024);
  const int grid = sms * cps;
  for (int w = 0; w < 3; ++w) k<<<grid, 32, smem + 1024>>>(mi, mo, d_ys, nunits, m, ns);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ts;
  for (int r = 0; r < 15; ++r) {
    cudaEventRecord(e0);
    k<<<grid, 32, smem + 1024>>>(mi, mo, d_ys, nunits, m, ns);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  const uint64_t moved = 2 * (uint64_t)ROWS * R * n;
  printf("{\"bytes\": %llu, \"R\": %d, \"swap\": %d, \"ns\": %d, \"cps\": %d, \"gbs\": %.1f, "
         "\"best_gbs\": %.1f, \"err\": \"%s\"}\n",
         (unsigned long long)total, R, (int)SWAP, ns, cps, moved / ts[ts.size() / 2] / 1e6,
         moved / ts[0] / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (uint64_t total : {512ull << 20, 4096ull << 20}) {
    char *a, *b;
    uint32_t* ys;
    cudaMalloc(&a, total);
    cudaMalloc(&b, total);
    cudaMalloc(&ys, (total / 64 / 256) * 4 + 1024);
    cudaMemset(a, 3, total);
    // out of place: 32 KB per slot
    run<512, false>(a, b, ys, total, sms, 3, 2);
    run<512, false>(a, b, ys, total, sms, 6, 1);
    run<512, false>(a, b, ys, total, sms, 2, 3);
    // in place: 64 KB per pair slot
    run<512, true>(a, b, ys, total, sms, 3, 1);
    run<512, true>(a, b, ys, total, sms, 2, 1);
    run<256, true>(a, b, ys, total, sms, 3, 2);
    run<256, true>(a, b, ys, total, sms, 6, 1);
    run<1024, false>(a, b, ys, total, sms, 3, 1);
    cudaFree(a);
    cudaFree(b);
    cudaFree(ys);
  }
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
