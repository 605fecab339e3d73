/* Calling the B200 hot path from C through the C ABI alone (no Python, no
 * torch): two 8-bit volumes with a folded z-score, the oct fast-path layout,
 * and the squared NCC of three particles (identity, a one-voxel shift along
 * k, and a transform that maps the target outside the source).
 *
 *   gcc -O2 examples/measure_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2504_19930_b200/_lib -lechoreg_sm100 -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2504_19930_b200/_lib -o measure_demo && ./measure_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "echoreg_b200.h"

#define CHECK(x)                                                          \
  do {                                                                    \
    int rc_ = (x);                                                        \
    if (rc_ != 0) {                                                       \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, er_last_error());    \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main(void) {
  enum { NX = 24, NY = 20, NZ = 28, P = 3 };
  const size_t n = (size_t)NX * NY * NZ;
  unsigned char* host = (unsigned char*)malloc(n);
  double mean = 0.0, sq = 0.0;
  for (size_t q = 0; q < n; ++q) {
    const int i = (int)(q / (NY * NZ)), j = (int)(q / NZ % NY), k = (int)(q % NZ);
    host[q] = (unsigned char)(128 + 60 * sin(0.5 * i) * cos(0.4 * j) + 40 * sin(0.7 * k));
    mean += host[q];
  }
  mean /= (double)n;
  for (size_t q = 0; q < n; ++q) sq += (host[q] - mean) * (host[q] - mean);
  const double sd = sqrt(sq / (double)n);

  void *vol, *oct, *mom, *A, *B, *ncc, *deg, *nin, *ws;
  if (cudaMalloc(&vol, n) != cudaSuccess) return 1;
  cudaMemcpy(vol, host, n, cudaMemcpyHostToDevice);
  er_volume v = {vol, ER_U8, NX, NY, NZ, 1.0 / sd, -mean / sd, NULL, NULL, NULL};

  cudaMalloc(&mom, ER_MOMENTS_DOUBLES * sizeof(double));
  CHECK(er_volume_moments(&v, (double*)mom, NULL));
  cudaMalloc(&oct, er_oct_bytes(&v));
  CHECK(er_build_oct(&v, oct, NULL));
  er_volume src = v;
  src.oct_dev = oct;

  /* index affines A (P x 9, row-major) and b (P x 3): source index = A * target index + b */
  double a[P * 9] = {0}, b[P * 3] = {0};
  for (int p = 0; p < P; ++p) a[9 * p + 0] = a[9 * p + 4] = a[9 * p + 8] = 1.0;
  b[3 * 1 + 2] = 1.0;     /* particle 1: one voxel along k */
  b[3 * 2 + 0] = 1000.0;  /* particle 2: entirely outside the source */
  cudaMalloc(&A, sizeof a);
  cudaMalloc(&B, sizeof b);
  cudaMemcpy(A, a, sizeof a, cudaMemcpyHostToDevice);
  cudaMemcpy(B, b, sizeof b, cudaMemcpyHostToDevice);
  cudaMalloc(&ncc, P * sizeof(double));
  cudaMalloc(&deg, P);
  cudaMalloc(&nin, P * sizeof(int64_t));
  const size_t wsb = er_measure_workspace_bytes(&v, P);
  cudaMalloc(&ws, wsb);
  CHECK(er_measure_ncc(&v, &src, (const double*)mom, (const double*)A, (const double*)B, P, 0,
                       ER_LERP_F32, (double*)ncc, (uint8_t*)deg, (int64_t*)nin, ws, wsb,
                       NULL));
  double z[P];
  unsigned char d[P];
  int64_t cnt[P];
  cudaMemcpy(z, ncc, sizeof z, cudaMemcpyDeviceToHost);
  cudaMemcpy(d, deg, sizeof d, cudaMemcpyDeviceToHost);
  cudaMemcpy(cnt, nin, sizeof cnt, cudaMemcpyDeviceToHost);
  for (int p = 0; p < P; ++p) printf("particle %d: ncc %.9f degenerate %d in-bounds %lld\n", p, z[p], d[p], (long long)cnt[p]);
  printf("abi %d\n", er_abi_version());
  return 0;
}
