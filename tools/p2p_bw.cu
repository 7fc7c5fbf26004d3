// NVLink peer-access microbenchmark (diagnostic, not part of the product):
// one process, G GPUs with peer access; every GPU runs the same kernel
// against its right neighbour simultaneously.  Patterns:
//   store_seq  : coalesced contiguous float4 stores into the peer
//   store_rows : 512 B rows stored at random row slots of the peer
//   load_rows  : 512 B rows loaded from random row slots of the peer
//   local_rows : 512 B rows random local read + local write (reference)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/p2p_bw.cu -o tools/p2p_bw
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void kern(float4* __restrict__ dst, const float4* __restrict__ src, uint64_t rows, uint32_t row_slots,
                     int rows_in_flight) {
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31;
  float4 acc = make_float4(0, 0, 0, 0);
  for (uint64_t r = gw; r < rows; r += nw) {
    if (MODE == 0) {  // seq stores: row r -> slot r
      dst[r * 32 + lane] = make_float4(r, lane, 0, 1);
    } else {
      const uint32_t slot = hash32((uint32_t)r) % row_slots;
      if (MODE == 1) dst[(uint64_t)slot * 32 + lane] = make_float4(r, lane, 0, 1);
      if (MODE == 2) { float4 v = src[(uint64_t)slot * 32 + lane]; acc.x += v.x; acc.y += v.y; }
      if (MODE == 3) { float4 v = src[(uint64_t)slot * 32 + lane]; dst[(uint64_t)hash32(slot) % row_slots * 32 + lane] = v; }
    }
  }
  if (acc.x == 12345.f) dst[0] = acc;
}

int main(int argc, char** argv) {
  int G = 0; CK(cudaGetDeviceCount(&G));
  if (argc > 1) G = std::min(G, atoi(argv[1]));
  const uint32_t slots = 1u << 21;  // 2M rows x 512 B = 1 GiB per buffer
  const uint64_t rows = 1u << 21;   // rows moved per GPU
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
  const char* names[] = {"store_seq", "store_rows", "load_rows", "local_rows"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int grid_mult : {1, 4, 16}) {
      std::vector<cudaEvent_t> e0(G), e1(G);
      for (int rep = 0; rep < 3; ++rep) {
        for (int g = 0; g < G; ++g) {
          CK(cudaSetDevice(g));
          CK(cudaEventCreate(&e0[g])); CK(cudaEventCreate(&e1[g]));
          const int peer = (g + 1) % G;
          float4* dst = mode == 3 ? scratch[g] : (mode == 2 ? scratch[g] : buf[peer]);
          const float4* src = mode == 3 ? buf[g] : buf[peer];
          dim3 grid(148 * grid_mult), block(256);
          CK(cudaEventRecord(e0[g], st[g]));
          switch (mode) {
            case 0: kern<0><<<grid, block, 0, st[g]>>>(dst, src, rows, slots, 1); break;
            case 1: kern<1><<<grid, block, 0, st[g]>>>(dst, src, rows, slots, 1); break;
            case 2: kern<2><<<grid, block, 0, st[g]>>>(dst, src, rows, slots, 1); break;
            case 3: kern<3><<<grid, block, 0, st[g]>>>(dst, src, rows, slots, 1); break;
          }
          CK(cudaEventRecord(e1[g], st[g]));
        }
        float worst = 0;
        for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaEventSynchronize(e1[g])); float ms; CK(cudaEventElapsedTime(&ms, e0[g], e1[g])); worst = std::max(worst, ms); }
        if (rep == 2) printf("G=%d %-11s grid=%4d blocks: %.3f ms  %.1f GB/s per GPU (one direction)\n", G, names[mode], 148 * grid_mult, worst, rows * 512.0 / worst / 1e6);
      }
    }
  }
  return 0;
}
