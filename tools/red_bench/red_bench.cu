// microbenchmark: fp32 vector reductions into a token-major [T, d] buffer in the FFN2 epilogue's
// access pattern (8 lanes x 16 B per row, 4 rows per warp instruction), rows in expert-major order
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
__global__ void red_kernel(float* out, const int* tok, int rows, int d, int mode) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  // each warp: 32-row block x 256 columns (one epilogue warp's tile share)
  const int nblk = (rows / 32) * (d / 256);
  for (int b = gw; b < nblk; b += nw) {
    const int rb = b / (d / 256), cb = b % (d / 256);
    for (int c0 = 0; c0 < 256; c0 += 32) {
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int r = rb * 32 + it * 8 + (lane >> 3);
        const int piece = lane & 7;
        const int t = tok[r];
        float* p = out + (int64_t)t * d + cb * 256 + c0 + piece * 4;
        const float v = 1.0f;
        if (mode == 0)
          asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
        else
          asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
      }
    }
  }
}
extern "C" int red_launch(float* out, const int* tok, int rows, int d, int mode, int blocks, void* stream) {
  red_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, tok, rows, d, mode);
  return (int)cudaGetLastError();
}
