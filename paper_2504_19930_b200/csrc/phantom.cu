// Device phantom generator: the reference's speckled
// LV shell sequence (E/phantom.py:61-91) and the echo-like 8-bit pairs built
// from it, generated on the GPU with the reference's exact arithmetic.
//
// Speckle: numpy's Generator(Philox(key=seed)).standard_normal(n) consumes a
// variable number of 64-bit stream words per normal (1 on the ziggurat's
// fast path, more after a wedge/tail rejection), so normal i starts at a
// word position only known after normals 0..i-1.  The stream is parsed in
// parallel instead of sequentially:
//   1. words_kernel   : all M stream words (Philox4x64-10, ctr b+1, key seed)
//   2. draw_kernel    : for EVERY word q, the normal a draw starting at q
//                       would return and how many words it would consume
//   3. chunk_kernel   : per 1024-word chunk and per entry offset e < 16
//                       (where the chain enters the chunk), the exit offset
//                       into the next chunk and the number of draws started
//   4. resolve_kernel : one CTA walks the chunk tables (shared-memory batches)
//                       from chunk 0 / offset 0: each chunk's real entry and
//                       the index of its first normal
//   5. emit_kernel    : per chunk, the chain positions -> normals in order,
//                       speckle = np.exp(sigma * z) (npexp.cuh, bit-exact)
// Frames: base intensities from the two ellipsoid radii in numpy's fp64
// operation order, times the speckle; cavity masks as bytes.
#include "common.cuh"
#include "npexp.cuh"
#include "rng.cuh"

namespace {

constexpr int kChunk = 1024;   // stream words per chain chunk
constexpr int kEntries = 16;   // entry offsets per chunk (max words per draw)
constexpr int kBatch = 512;    // chunks per shared-memory batch in resolve
constexpr uint8_t kBad = 0xFF;

__global__ void words_kernel(uint64_t seed, long long nblocks, uint64_t* __restrict__ w) {
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nblocks;
       b += (long long)gridDim.x * blockDim.x) {
    ErPhilox s;
    er_stream_init(&s, seed, 0, 0, 0);  // Philox(key=seed): counter 0, pre-incremented
    er_stream_seek_block(&s, (uint64_t)b);
    uint64_t out[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = er_next_u64(&s);
    reinterpret_cast<ulonglong2*>(w)[2 * b] = make_ulonglong2(out[0], out[1]);
    reinterpret_cast<ulonglong2*>(w)[2 * b + 1] = make_ulonglong2(out[2], out[3]);
  }
}

__global__ void draw_kernel(const uint64_t* __restrict__ w, long long M, double* __restrict__ val,
                            uint8_t* __restrict__ len) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < M;
       q += (long long)gridDim.x * blockDim.x) {
    ErArrayWords a{w, q, M};
    const double v = er_standard_normal_from(a);
    const long long used = a.pos - q;
    val[q] = v;
    len[q] = (a.exhausted() || used >= kEntries) ? 0 : (uint8_t)used;  // 0 = unusable
  }
}

// one CTA per chunk: walks from every entry offset
__global__ void chunk_kernel(const uint8_t* __restrict__ len, long long M,
                             uint8_t* __restrict__ exit_off, uint16_t* __restrict__ count) {
  __shared__ uint8_t sl[kChunk];
  const long long base = (long long)blockIdx.x * kChunk;
  for (int i = threadIdx.x; i < kChunk; i += blockDim.x)
    sl[i] = base + i < M ? len[base + i] : 0;
  __syncthreads();
  if (threadIdx.x < kEntries) {
    int p = threadIdx.x, n = 0;
    bool ok = true;
    while (p < kChunk) {
      const int L = sl[p];
      if (L == 0) {
        ok = false;
        break;
      }
      p += L;
      ++n;
    }
    const int ex = p - kChunk;
    exit_off[blockIdx.x * kEntries + threadIdx.x] = (ok && ex < kEntries) ? (uint8_t)ex : kBad;
    count[blockIdx.x * kEntries + threadIdx.x] = (uint16_t)n;
  }
}

// single CTA: chunk c's real entry offset and first normal index
__global__ void resolve_kernel(const uint8_t* __restrict__ exit_off,
                               const uint16_t* __restrict__ count, long long nchunks,
                               long long n_needed, uint8_t* __restrict__ entry,
                               long long* __restrict__ first, int* __restrict__ status) {
  __shared__ uint8_t se[kBatch * kEntries];
  __shared__ uint16_t sc[kBatch * kEntries];
  __shared__ int e_sh, bad_sh;
  __shared__ long long total_sh;
  if (threadIdx.x == 0) {
    e_sh = 0;
    bad_sh = 0;
    total_sh = 0;
  }
  for (long long c0 = 0; c0 < nchunks; c0 += kBatch) {
    const int nb = (int)min((long long)kBatch, nchunks - c0);
    __syncthreads();
    if (bad_sh || total_sh >= n_needed) break;  // shared, read after the barrier: uniform
    for (int i = threadIdx.x; i < nb * kEntries; i += blockDim.x) {
      se[i] = exit_off[c0 * kEntries + i];
      sc[i] = count[c0 * kEntries + i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int e = e_sh;
      long long total = total_sh;
      for (int c = 0; c < nb && total < n_needed; ++c) {
        entry[c0 + c] = (uint8_t)e;
        first[c0 + c] = total;
        const uint8_t ex = se[c * kEntries + e];
        total += sc[c * kEntries + e];
        if (ex == kBad) {  // an unusable draw on the chain (stream end / > 15 words)
          bad_sh = 1;
          break;
        }
        e = ex;
      }
      e_sh = e;
      total_sh = total;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *status = bad_sh ? 1 : (total_sh < n_needed ? 2 : 0);
}

// one CTA per chunk: chain positions in order -> normals n [first, first+m)
__global__ void emit_kernel(const uint8_t* __restrict__ len, const double* __restrict__ val,
                            long long M, const uint8_t* __restrict__ entry,
                            const long long* __restrict__ first, long long n, double sigma,
                            double* __restrict__ speckle, double* __restrict__ normals) {
  __shared__ uint8_t sl[kChunk];
  __shared__ uint16_t pos[kChunk];
  __shared__ int m_sh;
  const long long base = (long long)blockIdx.x * kChunk;
  const long long f0 = first[blockIdx.x];
  if (f0 >= n) return;  // chunks past the last needed normal (uniform per CTA)
  for (int i = threadIdx.x; i < kChunk; i += blockDim.x)
    sl[i] = base + i < M ? len[base + i] : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int p = entry[blockIdx.x], m = 0;
    while (p < kChunk && sl[p] != 0) {
      pos[m++] = (uint16_t)p;
      p += sl[p];
    }
    m_sh = m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m_sh; i += blockDim.x) {
    const long long idx = f0 + i;
    if (idx >= n) break;
    const double z = val[base + pos[i]];
    if (normals) normals[idx] = z;
    speckle[idx] = npexp::exp_svml_ha(rn_mul(sigma, z));  // np.exp(sigma * z)
  }
}

struct FrameGeom {
  int nx, ny, nz;
  double sp[3], c[3], outer[3], inner[3];
};

__device__ __forceinline__ double ell_radius(double x, double y, double z, const double* a) {
  // ((x/ax)**2 + (y/ay)**2) + (z/az)**2, phantom.py:94-96 (numpy broadcast order)
  const double u = rn_div(x, a[0]), v = rn_div(y, a[1]), w = rn_div(z, a[2]);
  return rn_add(rn_add(rn_mul(u, u), rn_mul(v, v)), rn_mul(w, w));
}

__global__ void frame_kernel(const double* __restrict__ speckle, FrameGeom g,
                             double* __restrict__ frame, uint8_t* __restrict__ mask) {
  const long long n = (long long)g.nx * g.ny * g.nz;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const long long row = q / g.nz;
    const int k = (int)(q - row * g.nz);
    const int i = (int)(row / g.ny);
    const int j = (int)(row - (long long)i * g.ny);
    // xs = np.arange(nx) * sx - center[0] (phantom.py:72-74)
    const double x = rn_sub(rn_mul((double)i, g.sp[0]), g.c[0]);
    const double y = rn_sub(rn_mul((double)j, g.sp[1]), g.c[1]);
    const double z = rn_sub(rn_mul((double)k, g.sp[2]), g.c[2]);
    const bool cavity = ell_radius(x, y, z, g.inner) <= 1.0;
    double base = ell_radius(x, y, z, g.outer) <= 1.0 ? 1.0 : 0.2;  // INTENSITY_*
    if (cavity) base = 0.1;
    if (frame) frame[q] = rn_mul(base, speckle[q]);
    if (mask) mask[q] = cavity ? 1 : 0;
  }
}

// clip(round(v * scale), 0, 255) as uint8 (round half to even = np.round);
// entries at index >= keep_before are zeroed (make_pair's overlap crop)
__global__ void quantize_kernel(const double* __restrict__ v, long long n, double scale,
                                long long keep_before, uint8_t* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    double r = rint(q < keep_before ? rn_mul(v[q], scale) : 0.0);
    r = fmin(fmax(r, 0.0), 255.0);
    out[q] = (uint8_t)r;
  }
}

// (v > threshold) as bytes (volume.py:133-135), zeroed at index >= keep_before
__global__ void binarize_kernel(const double* __restrict__ v, long long n, double threshold,
                                long long keep_before, uint8_t* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    out[q] = (q < keep_before && v[q] > threshold) ? 1 : 0;
}

int grid_for(long long n, int threads) {
  const long long b = (n + threads - 1) / threads;
  return (int)min(b, (long long)ER_NUM_SMS_B200 * 16);
}

struct SpeckleLayout {
  long long M, nchunks;
  size_t o_words, o_val, o_len, o_exit, o_cnt, o_entry, o_first, o_status, total;
};

SpeckleLayout speckle_layout(long long n) {
  SpeckleLayout L;
  // ~1.013 words per normal on average; 1/8 + 4 chunks of slack
  long long M = n + n / 8 + 4 * kChunk;
  M = (M + kChunk - 1) / kChunk * kChunk;  // whole chunks, whole Philox blocks
  L.M = M;
  L.nchunks = M / kChunk;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t o = 0;
  L.o_words = o;
  o = al(o + (size_t)M * 8);
  L.o_val = o;
  o = al(o + (size_t)M * 8);
  L.o_len = o;
  o = al(o + (size_t)M);
  L.o_exit = o;
  o = al(o + (size_t)L.nchunks * kEntries);
  L.o_cnt = o;
  o = al(o + (size_t)L.nchunks * kEntries * 2);
  L.o_entry = o;
  o = al(o + (size_t)L.nchunks);
  L.o_first = o;
  o = al(o + (size_t)L.nchunks * 8);
  L.o_status = o;
  o = al(o + 8);
  L.total = o;
  return L;
}

}  // namespace

extern "C" size_t er_phantom_scratch_bytes(int64_t n) {
  return n > 0 ? speckle_layout(n).total : 0;
}

extern "C" int er_phantom_speckle(uint64_t seed, int64_t n, double sigma, void* scratch,
                                  size_t scratch_bytes, double* speckle_out, double* normals_out,
                                  void* stream) {
  if (n <= 0 || !scratch || !speckle_out)
    return er_set_error(ER_EINVAL, "er_phantom_speckle: bad arguments");
  const SpeckleLayout L = speckle_layout(n);
  if (scratch_bytes < L.total)
    return er_set_error(ER_EINVAL, "er_phantom_speckle: scratch smaller than "
                                   "er_phantom_scratch_bytes(n)");
  cudaStream_t s = as_stream(stream);
  char* b = static_cast<char*>(scratch);
  uint64_t* w = reinterpret_cast<uint64_t*>(b + L.o_words);
  double* val = reinterpret_cast<double*>(b + L.o_val);
  uint8_t* len = reinterpret_cast<uint8_t*>(b + L.o_len);
  uint8_t* ex = reinterpret_cast<uint8_t*>(b + L.o_exit);
  uint16_t* cnt = reinterpret_cast<uint16_t*>(b + L.o_cnt);
  uint8_t* entry = reinterpret_cast<uint8_t*>(b + L.o_entry);
  long long* first = reinterpret_cast<long long*>(b + L.o_first);
  int* status = reinterpret_cast<int*>(b + L.o_status);
  const long long nblocks = L.M / 4;
  words_kernel<<<grid_for(nblocks, 256), 256, 0, s>>>(seed, nblocks, w);
  draw_kernel<<<grid_for(L.M, 256), 256, 0, s>>>(w, L.M, val, len);
  chunk_kernel<<<(unsigned)L.nchunks, 256, 0, s>>>(len, L.M, ex, cnt);
  // chunks the chain never reaches keep first = n (emit skips them)
  cudaMemsetAsync(first, 0x7F, (size_t)L.nchunks * 8, s);
  resolve_kernel<<<1, 1024, 0, s>>>(ex, cnt, L.nchunks, n, entry, first, status);
  emit_kernel<<<(unsigned)L.nchunks, 256, 0, s>>>(len, val, L.M, entry, first, n, sigma,
                                                  speckle_out, normals_out);
  ER_CHECK_LAUNCH();
  int st = 0;
  cudaMemcpyAsync(&st, status, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return er_set_cuda_error(e, "er_phantom_speckle");
  if (st != 0)
    return er_set_error(ER_ECUDA, st == 1 ? "er_phantom_speckle: a draw on the chain used "
                                            "more than 15 stream words"
                                          : "er_phantom_speckle: stream words exhausted");
  return ER_OK;
}

extern "C" int er_phantom_frame(const double* speckle, int32_t nx, int32_t ny, int32_t nz,
                                const double spacing[3], const double center[3],
                                const double outer[3], const double inner[3], double* frame_out,
                                uint8_t* mask_out, void* stream) {
  if (nx < 1 || ny < 1 || nz < 1 || (frame_out && !speckle) || (!frame_out && !mask_out))
    return er_set_error(ER_EINVAL, "er_phantom_frame: bad arguments");
  FrameGeom g;
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  for (int d = 0; d < 3; ++d) {
    g.sp[d] = spacing[d];
    g.c[d] = center[d];
    g.outer[d] = outer[d];
    g.inner[d] = inner[d];
  }
  const long long n = (long long)nx * ny * nz;
  frame_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(speckle, g, frame_out, mask_out);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_quantize_u8(const double* v, int64_t n, double scale, int64_t keep_before,
                              uint8_t* out, void* stream) {
  if (n < 0 || (n && (!v || !out))) return er_set_error(ER_EINVAL, "er_quantize_u8: bad arguments");
  if (n == 0) return ER_OK;
  quantize_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(v, n, scale, keep_before, out);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

extern "C" int er_binarize_u8(const double* v, int64_t n, double threshold, int64_t keep_before,
                              uint8_t* out, void* stream) {
  if (n < 0 || (n && (!v || !out))) return er_set_error(ER_EINVAL, "er_binarize_u8: bad arguments");
  if (n == 0) return ER_OK;
  binarize_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(v, n, threshold, keep_before,
                                                                  out);
  ER_CHECK_LAUNCH();
  return ER_OK;
}

ER_DEFINE_FAULT_READER(er_faults_phantom)
