/* Polar Express from plain C through the C ABI (include/pe.h): no Python, no
 * PyTorch.  Builds one 256 x 768 bf16 Gaussian-like matrix, runs pe_polar
 * (T = 5) on the GPU and checks that the rows of the result are close to
 * orthonormal (polar(M) has orthonormal rows for a full-rank wide M).
 *
 *   gcc -std=c99 -O2 -I include -I /usr/local/cuda/include examples/polar_c.c \
 *       -L paper_2505_16932_b200 -l:libpe.so -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,paper_2505_16932_b200 -lm -o polar_c && ./polar_c
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pe.h"

static uint16_t to_bf16(float f) {             /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main(void) {
  enum { R = 256, C = 768 };
  uint16_t* h = (uint16_t*)malloc(sizeof(uint16_t) * R * C);
  uint64_t s = 0x9E3779B97F4A7C15ull;
  for (int i = 0; i < R * C; ++i) {           /* sum of 4 uniforms: roughly Gaussian */
    float acc = 0.f;
    for (int k = 0; k < 4; ++k) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      acc += (float)((s >> 40) & 0xFFFFFF) / 16777216.0f - 0.5f;
    }
    h[i] = to_bf16(0.02f * acc);
  }
  void* d = NULL;
  if (cudaMalloc(&d, sizeof(uint16_t) * R * C) != cudaSuccess) return 2;
  cudaMemcpy(d, h, sizeof(uint16_t) * R * C, cudaMemcpyHostToDevice);
  pe_ctx ctx;
  pe_status st = pe_create(&ctx, 0);
  if (st != PE_OK) { fprintf(stderr, "pe_create: %s\n", pe_status_string(st)); return 3; }
  const int64_t shape[2] = {R, C};
  const void* in[1] = {d};
  void* out[1] = {d};                          /* in place */
  st = pe_polar(ctx, in, out, shape, 1, 5, PE_BF16, NULL);
  if (st != PE_OK) { fprintf(stderr, "pe_polar: %s\n", pe_status_string(st)); return 4; }
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(uint16_t) * R * C, cudaMemcpyDeviceToHost);
  double worst = 0.0;
  for (int i = 0; i < R; i += 17)
    for (int j = i; j < R; j += 23) {
      double dot = 0.0;
      for (int k = 0; k < C; ++k) dot += (double)from_bf16(h[i * C + k]) * from_bf16(h[j * C + k]);
      const double e = fabs(dot - (i == j ? 1.0 : 0.0));
      if (e > worst) worst = e;
    }
  pe_destroy(ctx);
  cudaFree(d);
  free(h);
  printf("max |(X X^T - I)_ij| over sampled pairs: %.4f\n", worst);
  return worst < 0.15 ? 0 : 5;
}
