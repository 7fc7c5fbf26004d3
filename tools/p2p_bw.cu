// NVLink peer-access microbenchmark (diagnostic, not part of the product):
// one process, G GPUs with peer access; every GPU runs the same kernel
// simultaneously.  Patterns (rows of 512 B):
//   store_rows   : constant rows stored at random slots of the right neighbour
//   load_rows    : rows loaded from random slots of the right neighbour
//   gather_store : random LOCAL row loaded, stored at a random slot of peer
//                  (r % (G-1)) -- the serve / gradient-push pattern, all-to-all
//   local_rows   : random local read + local write (reference)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/p2p_bw.cu -o tools/p2p_bw
//   (__graft_entry__.build() does this).
// Usage: p2p_bw [G] [--json]: --json measures only the exchange patterns
// (gather_store, store_rows) and prints one JSON line with the best grid's
// GB/s per GPU per direction -- the NVLink ceiling bench.py reports against.
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

struct Peers { float4* p[8]; int n; };

template <int MODE, int INFLIGHT>
__global__ void kern(float4* __restrict__ local, float4* __restrict__ scratch, Peers peers, uint64_t rows,
                     uint32_t slots) {
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31;
  float4 acc = make_float4(0, 0, 0, 0);
  for (uint64_t r0 = gw * INFLIGHT; r0 < rows; r0 += nw * INFLIGHT) {
    float4 v[INFLIGHT];
#pragma unroll
    for (int k = 0; k < INFLIGHT; ++k) {
      const uint32_t r = (uint32_t)(r0 + k);
      const uint32_t slot = hash32(r) % slots;
      if (MODE == 0) v[k] = make_float4(r, lane, 0, 1);
      if (MODE == 1) v[k] = peers.p[0][(uint64_t)slot * 32 + lane];
      if (MODE == 2 || MODE == 3) v[k] = local[(uint64_t)slot * 32 + lane];
    }
#pragma unroll
    for (int k = 0; k < INFLIGHT; ++k) {
      const uint32_t r = (uint32_t)(r0 + k);
      const uint32_t slot2 = hash32(r ^ 0x5bd1e995u) % slots;
      if (MODE == 0) peers.p[0][(uint64_t)slot2 * 32 + lane] = v[k];
      if (MODE == 1) { acc.x += v[k].x; acc.y += v[k].y; }
      if (MODE == 2) peers.p[r % peers.n][(uint64_t)slot2 * 32 + lane] = v[k];
      if (MODE == 3) scratch[(uint64_t)slot2 * 32 + lane] = v[k];
    }
  }
  if (acc.x == 12345.f) scratch[0] = acc;
}

int main(int argc, char** argv) {
  int G = 0; CK(cudaGetDeviceCount(&G));
  if (argc > 1) G = std::min(G, atoi(argv[1]));
  const uint32_t slots = 1u << 21;  // 2M rows x 512 B = 1 GiB per buffer
  const uint64_t rows = 1u << 22;   // rows moved per GPU (2 GiB)
  std::vector<float4*> buf(G), scratch(G);
  std::vector<cudaStream_t> st(G);
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < G; ++p) if (p != g) { cudaDeviceEnablePeerAccess(p, 0); cudaGetLastError(); }
    CK(cudaMalloc(&buf[g], (size_t)slots * 512));
    CK(cudaMalloc(&scratch[g], (size_t)slots * 512));
    CK(cudaMemset(buf[g], 0, (size_t)slots * 512));
    CK(cudaStreamCreate(&st[g]));
  }
  const bool json = argc > 2 && std::string(argv[2]) == "--json";
  const char* names[] = {"store_rows", "load_rows", "gather_store", "local_rows"};
  float best[4] = {0, 0, 0, 0};
  for (int mode = 0; mode < 4; ++mode) {
    if (json && mode != 0 && mode != 2) continue;
    for (int bps : {1, 2, 4, 8}) {
      for (int infl : {4, 8}) {
        std::vector<cudaEvent_t> e0(G), e1(G);
        float worst = 0;
        for (int rep = 0; rep < 3; ++rep) {
          for (int g = 0; g < G; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventCreate(&e0[g])); CK(cudaEventCreate(&e1[g]));
            Peers pr{}; pr.n = 0;
            if (mode == 2) { for (int p = 0; p < G; ++p) if (p != g) pr.p[pr.n++] = buf[p]; }
            else { pr.p[0] = buf[(g + 1) % G]; pr.n = 1; }
            dim3 grid(148 * bps), block(256);
            CK(cudaEventRecord(e0[g], st[g]));
#define L(M, I) kern<M, I><<<grid, block, 0, st[g]>>>(buf[g], scratch[g], pr, rows, slots)
            if (infl == 4) { switch (mode) { case 0: L(0,4); break; case 1: L(1,4); break; case 2: L(2,4); break; case 3: L(3,4); break; } }
            else { switch (mode) { case 0: L(0,8); break; case 1: L(1,8); break; case 2: L(2,8); break; case 3: L(3,8); break; } }
            CK(cudaEventRecord(e1[g], st[g]));
          }
          worst = 0;
          for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaEventSynchronize(e1[g])); float ms; CK(cudaEventElapsedTime(&ms, e0[g], e1[g])); worst = std::max(worst, ms); }
        }
        const float gbs = rows * 512.0 / worst / 1e6;
        best[mode] = std::max(best[mode], gbs);
        for (int g = 0; g < G; ++g) { CK(cudaEventDestroy(e0[g])); CK(cudaEventDestroy(e1[g])); }
        if (!json) printf("G=%d %-12s blocks/SM=%d inflight=%d: %.3f ms  %.1f GB/s per GPU (one direction)\n", G, names[mode], bps, infl, worst, gbs);
      }
    }
  }
  if (json) {
    printf("{\"gpus\": %d, \"gather_store_gbs\": %.1f, \"store_rows_gbs\": %.1f, \"rows_bytes\": 512, "
           "\"what\": \"best over grids of 1-8 blocks/SM, every GPU at once, per GPU per direction\"}\n",
           G, best[2], best[0]);
  }
  return 0;
}
