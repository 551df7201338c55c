// Throughput probe for the attention softmax inner loop on one SM: per thread,
// 128 scores -> exp2 (MUFU.EX2 or the FMA-pipe cubic for POLY of every 8
// pairs) -> fp32 row sum (FADD2) + bf16x2 packs, as in attn_fwd.cu.  Reports
// cycles per 128-column row per warp at 1 and 2 warps per SMSP.
#include <cstdio>
#include <cstdlib>
#include "sm100.cuh"

using namespace rcp;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t f2(float a, float b) {
  uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ float2 unf2(uint64_t v) {
  float2 r; asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.0f);
  const float t = __fadd_rn(x, 12582912.0f);
  const float f = __fsub_rn(x, __fsub_rn(t, 12582912.0f));
  const float p = fmaf(fmaf(fmaf(0.05500893f, f, 0.24221097f), f, 0.69328290f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Packed (f32x2) variant of ex2_poly: the rounding split and Horner steps on
// FADD2/FFMA2, clamp and exponent add per element on the ALU pipe.
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x2) {
  float2 x = unf2(x2);
  x2 = f2(fmaxf(x.x, -126.0f), fmaxf(x.y, -126.0f));
  const uint64_t magic = f2(12582912.0f, 12582912.0f), nmagic = f2(-12582912.0f, -12582912.0f);
  const uint64_t t = fadd2(x2, magic);
  uint64_t r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x2), "l"(fadd2(t, nmagic)));
  uint64_t pp = ffma2(f2(0.05500893f, 0.05500893f), r, f2(0.24221097f, 0.24221097f));
  pp = ffma2(pp, r, f2(0.69328290f, 0.69328290f));
  pp = ffma2(pp, r, f2(1.0f, 1.0f));
  const float2 pf = unf2(pp), tf = unf2(t);
  return f2(__int_as_float(__float_as_int(pf.x) + (__float_as_int(tf.x) << 23)),
            __int_as_float(__float_as_int(pf.y) + (__float_as_int(tf.y) << 23)));
}

constexpr int kRows = 64;

// PACK: 0 = cvt.rn.bf16x2.f32 (F2FP), 1 = no pack (xor of the fp32 bits),
//       2 = truncating pack (PRMT of the high halves)
template <int POLY, int PACK>
__global__ void __launch_bounds__(256, 1) sm_probe(const float* in, float sl2, unsigned long long* out, uint32_t* sink) {
  float s[128];
  for (int c = 0; c < 128; ++c) s[c] = in[(threadIdx.x * 7 + c) & 1023];
  const uint64_t sl2x2 = f2(sl2, sl2);
  uint32_t x_or = 0;
  float l = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < kRows; ++r) {
    float m8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) m8[k] = fmaxf(s[k], s[8 + k]);
#pragma unroll
    for (int c = 16; c < 128; c += 8)
#pragma unroll
      for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[c + k]);
    const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                           fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
    const uint64_t negm2 = f2(-mx * sl2, -mx * sl2);
    uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int ip = 0; ip < 64; ++ip) {
      const float2 x = unf2(ffma2(f2(s[2 * ip], s[2 * ip + 1]), sl2x2, negm2));
      float p0, p1;
      if (PACK == 3 && (ip & 7) < POLY) {
        const float2 pp = unf2(ex2_poly2(f2(x.x, x.y)));
        p0 = pp.x; p1 = pp.y;
      } else if (PACK == 4 && (ip & 7) >= POLY) {
        // MUFU on f16x2: two exps per instruction, widened back to f32
        uint32_t h, e2;
        asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x.y), "f"(x.x));
        asm("ex2.approx.f16x2 %0, %1;" : "=r"(e2) : "r"(h));
        asm("{\n.reg .f16 lo, hi;\nmov.b32 {lo, hi}, %2;\ncvt.f32.f16 %0, lo;\ncvt.f32.f16 %1, hi;\n}" : "=f"(p0), "=f"(p1) : "r"(e2));
      } else if (PACK != 4 && (ip & 7) < POLY) { p0 = ex2_poly(x.x); p1 = ex2_poly(x.y); }
      else { p0 = ex2_approx(x.x); p1 = ex2_approx(x.y); }
      acc2[ip & 3] = fadd2(acc2[ip & 3], f2(p0, p1));
      if (PACK == 0 || PACK >= 3) x_or ^= pack_bf16x2(p0, p1);
      else if (PACK == 1) x_or ^= __float_as_uint(p0) ^ __float_as_uint(p1);
      else {
        uint32_t r;
        asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(p0)), "r"(__float_as_uint(p1)));
        x_or ^= r;
      }
    }
    const float2 a01 = unf2(fadd2(acc2[0], acc2[1])), a23 = unf2(fadd2(acc2[2], acc2[3]));
    l += (a01.x + a01.y) + (a23.x + a23.y);
    // perturb the scores so the loop is not hoisted
    s[r & 127] += l * 1e-30f;
  }
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = x_or ^ __float_as_uint(l);
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + (threadIdx.x >> 5)] = (unsigned long long)(t1 - t0);
}

// Instruction-form variants of the same loop (poly = 2 of 8 pairs, scalar cubic):
//   XF 0: x = FFMA2(s, scale, -m)      1: x = FFMA(s, imm scale, -m) per element
//   SF 0: row sum FADD2 (4 partials)   1: scalar FADD (8 partials)
template <int XF, int SF>
__global__ void __launch_bounds__(256, 1) form_probe(const float* in, float sl2, unsigned long long* out, uint32_t* sink) {
  float s[128];
  for (int c = 0; c < 128; ++c) s[c] = in[(threadIdx.x * 7 + c) & 1023];
  const uint64_t sl2x2 = f2(sl2, sl2);
  uint32_t x_or = 0;
  float l = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < kRows; ++r) {
    float m8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) m8[k] = fmaxf(s[k], s[8 + k]);
#pragma unroll
    for (int c = 16; c < 128; c += 8)
#pragma unroll
      for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[c + k]);
    const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                           fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
    const float negm = -mx * 0.12751743f;
    const uint64_t negm2 = f2(negm, negm);
    uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ip = 0; ip < 64; ++ip) {
      float2 x;
      if (XF == 0) x = unf2(ffma2(f2(s[2 * ip], s[2 * ip + 1]), sl2x2, negm2));
      else { x.x = fmaf(s[2 * ip], 0.12751743f, negm); x.y = fmaf(s[2 * ip + 1], 0.12751743f, negm); }
      float p0, p1;
      if ((ip & 7) < 2) { p0 = ex2_poly(x.x); p1 = ex2_poly(x.y); }
      else { p0 = ex2_approx(x.x); p1 = ex2_approx(x.y); }
      if (SF == 0) acc2[ip & 3] = fadd2(acc2[ip & 3], f2(p0, p1));
      else { acc[(2 * ip) & 7] += p0; acc[(2 * ip + 1) & 7] += p1; }
      x_or ^= pack_bf16x2(p0, p1);
    }
    if (SF == 0) {
      const float2 a01 = unf2(fadd2(acc2[0], acc2[1])), a23 = unf2(fadd2(acc2[2], acc2[3]));
      l += (a01.x + a01.y) + (a23.x + a23.y);
    } else {
      l += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    }
    s[r & 127] += l * 1e-30f;
  }
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = x_or ^ __float_as_uint(l);
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + (threadIdx.x >> 5)] = (unsigned long long)(t1 - t0);
}

int main() {
  float* d_in; unsigned long long* d_out; uint32_t* d_sink;
  CK(cudaMalloc(&d_in, 1024 * 4)); CK(cudaMalloc(&d_out, 148 * 8 * 8)); CK(cudaMalloc(&d_sink, 148 * 256 * 4));
  float h[1024]; for (int i = 0; i < 1024; ++i) h[i] = (float)((i * 37) % 101) * 0.05f - 2.5f;
  CK(cudaMemcpy(d_in, h, sizeof(h), cudaMemcpyHostToDevice));
  auto report = [&](const char* name, int threads) {
    unsigned long long c[8]; CK(cudaMemcpy(c, d_out, 64, cudaMemcpyDeviceToHost));
    unsigned long long lo = c[0], hi = c[0];
    for (int w = 1; w < threads / 32; ++w) { lo = c[w] < lo ? c[w] : lo; hi = c[w] > hi ? c[w] : hi; }
    printf("%-28s warps/SMSP %d : first warp %6.0f, last warp %6.0f cycles per row-block -> %6.1f SMSP cycles per 128-col row-warp\n",
           name, threads / 128, (double)lo / kRows, (double)hi / kRows, (double)hi / kRows / (threads / 128));
  };
#define RUN(P, K, name)                                                              \
  for (int threads : {128, 256}) {                                                   \
    for (int rep = 0; rep < 2; ++rep) {                                              \
      sm_probe<P, K><<<148, threads>>>(d_in, 0.127f, d_out, d_sink);                 \
      CK(cudaGetLastError()); CK(cudaDeviceSynchronize());                           \
    }                                                                                \
    report(name, threads);                                                           \
  }
  RUN(2, 0, "poly2 F2FP (current)")
#define RUNF(X, S, name)                                                             \
  for (int threads : {128, 256}) {                                                   \
    for (int rep = 0; rep < 2; ++rep) {                                              \
      form_probe<X, S><<<148, threads>>>(d_in, 0.127f, d_out, d_sink);               \
      CK(cudaGetLastError()); CK(cudaDeviceSynchronize());                           \
    }                                                                                \
    report(name, threads);                                                           \
  }
  RUNF(0, 0, "FFMA2 x, FADD2 sum")
  RUNF(1, 0, "imm FFMA x, FADD2 sum")
  RUNF(0, 1, "FFMA2 x, FADD sum")
  RUNF(1, 1, "imm FFMA x, FADD sum")
  return 0;
}
