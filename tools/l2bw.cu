// L2 read-bandwidth probe (tool, not product): every SM streams an
// L2-resident buffer with 8- or 16-byte lane loads (4 independent loads in
// flight per thread); reports achieved TB/s.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void rd(const T* __restrict__ p, long long n, int reps, unsigned long long* out) {
  unsigned long long acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
      T a = __ldcg(p + i), b = __ldcg(p + i + stride), c = __ldcg(p + i + 2 * stride),
        d = __ldcg(p + i + 3 * stride);
      acc += *(const unsigned*)&a + *(const unsigned*)&b + *(const unsigned*)&c +
             *(const unsigned*)&d;
    }
    for (; i < n; i += stride) { T a = __ldcg(p + i); acc += *(const unsigned*)&a; }
  }
  if (acc == 0x12345) *out = acc;
}
int main() {
  for (int mb : {16, 52, 96, 400}) {
    long long bytes = (long long)mb << 20;
    char* buf; unsigned long long* o;
    cudaMalloc(&buf, bytes); cudaMalloc(&o, 8); cudaMemset(buf, 1, bytes);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w : {8, 16}) {
      long long n = bytes / w; int reps = 10;
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        if (w == 8) rd<uint2><<<148 * 8, 256>>>((const uint2*)buf, n, reps, o);
        else rd<uint4><<<148 * 8, 256>>>((const uint4*)buf, n, reps, o);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (it) printf("buffer %4d MB, %2d-byte lanes: %.2f TB/s\n", mb, w, bytes * (double)reps / (ms * 1e-3) / 1e12);
      }
    }
    cudaFree(buf); cudaFree(o);
  }
}
