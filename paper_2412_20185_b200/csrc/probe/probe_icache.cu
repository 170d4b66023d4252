// Cold-code probe: cycles to execute N straight-line (fully unrolled, executed once) ALU
// instructions vs the same work as a small loop, in a fresh launch; 148 CTAs x 256 threads.
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

template <int N, bool UNROLL>
__global__ void k_code(unsigned* out, unsigned seed) {
  unsigned a = seed ^ threadIdx.x, b = a * 3u, c = a * 5u, d = a * 7u;
  long long t0 = clock64();
  if (UNROLL) {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      a = a * 1664525u + 1013904223u + i; b = (b ^ (b >> 3)) + i; c = c * 69069u + i; d = (d << 1) ^ (d + i);
    }
  } else {
#pragma unroll 1
    for (int i = 0; i < N / 4; ++i) {
      a = a * 1664525u + 1013904223u + i; b = (b ^ (b >> 3)) + i; c = c * 69069u + i; d = (d << 1) ^ (d + i);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned)(t1 - t0);
  if ((a ^ b ^ c ^ d) == 0x12345u) out[4095] = 1;
}

int main() {
  unsigned* o; CK(cudaMalloc(&o, 4096 * 4));
  unsigned h[148];
  auto run = [&](auto kern, const char* name) {
    for (int rep = 0; rep < 3; ++rep) {
      kern<<<148, 256>>>(o, rep);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(h, o, 148 * 4, cudaMemcpyDeviceToHost));
      unsigned mx = 0; double avg = 0;
      for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; avg += h[i]; }
      printf("{\"kernel\": \"%s\", \"rep\": %d, \"avg_cycles\": %.0f, \"max_cycles\": %u}\n", name, rep, avg / 148, mx);
    }
    return 0;
  };
  run(k_code<512, true>, "unrolled_512");
  run(k_code<512, false>, "loop_512");
  run(k_code<2048, true>, "unrolled_2048");
  run(k_code<2048, false>, "loop_2048");
  return 0;
}
