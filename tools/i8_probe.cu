// Descriptor probe (diagnostics, not product) for the packed-V value path on
// the int8 tensor pipe: D[128 cols x 16] (s32) = C^T x P with
//   C^T : u8 codes, MN-major SW128 (token row = 128 B = 128 columns, 16-B
//         chunk c of row r at (c ^ (r & 7)), 8-row groups 1024 B apart),
//   P   : s8 digits, K-major SW128 (16 rows x 128 tokens, 1 KB per 8 rows),
// four tcgen05.mma.kind::i8 (K = 32) over 128 tokens.  Checked exactly
// against a CPU integer product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2407_21118_b200/csrc \
//        -I include -o tools/i8_probe tools/i8_probe.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "palu_sm100.cuh"

using namespace palu::tc;

constexpr uint32_t IDESC_Q = (2u << 4) | (0u << 7) | (1u << 10) | (1u << 15) |
                             ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}

__global__ void probe(const uint8_t* C, const int8_t* P, int* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = sm;            // 16 KB: 128 tokens x 128 B
  uint8_t* Bp = sm + 16384;   // 2 KB: 16 rows x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 2048);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // codes: token t (K), column m (M): row t, chunk (m / 16) ^ (t & 7), byte m % 16
  for (int i = tid; i < 128 * 128; i += blockDim.x) {
    const int t = i / 128, m = i % 128;
    A[t * 128 + ((((m >> 4) ^ t) & 7) << 4) + (m & 15)] = C[t * 128 + m];
  }
  // digits: row n (N), token t (K): group n / 8, row n % 8, chunk (t / 16) ^ (n & 7)
  for (int i = tid; i < 16 * 128; i += blockDim.x) {
    const int n = i / 128, t = i % 128;
    Bp[(n >> 3) * 1024 + (n & 7) * 128 + ((((t >> 4) ^ n) & 7) << 4) + (t & 15)] = (uint8_t)P[n * 128 + t];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    for (int kk = 0; kk < 4; ++kk)
      umma_i8(tmem, sdesc_mn(smem_u32(A) + kk * 4096, 16384, 1024), sdesc(smem_u32(Bp) + kk * 32),
              IDESC_Q, kk > 0);
    umma_commit(&bar[0]);
  }
  mbar_wait(&bar[0], 0);
  fence_after();
  float v[16];
  tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  tmem_wait_ld();
  const int m = warp * 32 + (tid & 31);
  for (int n = 0; n < 16; ++n) out[m * 16 + n] = __float_as_int(v[n]);
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  }
}

// back-to-back MMA issue rate: ITERS x 4 MMAs on fixed operands, one CTA per SM
template <int KIND, int N>  // KIND 0: kind::i8 (K 32), 1: kind::f16 bf16 (K 16)
__global__ void rate(int iters, float* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01020304u * (i & 7);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (KIND == 0) {
          constexpr uint32_t ID = (2u << 4) | (0u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(sdesc_mn(a + kk * 4096, 16384, 1024)), "l"(sdesc(b + kk * 32)), "r"(ID), "r"(1)
                       : "memory");
        } else {
          constexpr uint32_t ID = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(sdesc_mn(a + kk * 2048, 16384, 1024)), "l"(sdesc(b + kk * 32)), "r"(ID), "r"(1)
                       : "memory");
        }
      }
    }
    umma_commit(&bar[0]);
    mbar_wait(&bar[0], 0);
    if (blockIdx.x == 0) out[0] = (float)(clock64() - c0) / (4.f * iters);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

template <int KIND, int N>
static void run_rate(const char* name) {
  float* d;
  cudaMalloc(&d, 4);
  cudaFuncSetAttribute(rate<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  rate<KIND, N><<<148, 128, 70 * 1024>>>(2000, d);
  cudaDeviceSynchronize();
  rate<KIND, N><<<148, 128, 70 * 1024>>>(20000, d);
  cudaError_t e = cudaDeviceSynchronize();
  float h = 0;
  cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("rate %-22s N %3d: %6.1f SM clocks per MMA (%s)\n", name, N, h, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run_rate<0, 8>("i8 M128 K32");
  run_rate<0, 16>("i8 M128 K32");
  run_rate<0, 32>("i8 M128 K32");
  run_rate<0, 64>("i8 M128 K32");
  run_rate<0, 128>("i8 M128 K32");
  run_rate<1, 16>("bf16 M128 K16 (MN A)");
  run_rate<1, 64>("bf16 M128 K16 (MN A)");
  run_rate<1, 256>("bf16 M128 K16 (MN A)");
  std::vector<uint8_t> C(128 * 128);
  std::vector<int8_t> P(16 * 128);
  srand(7);
  for (auto& c : C) c = rand() % 256;
  for (auto& p : P) p = (int8_t)(rand() % 256 - 128);
  uint8_t* dC;
  int8_t* dP;
  int* dO;
  cudaMalloc(&dC, C.size());
  cudaMalloc(&dP, P.size());
  cudaMalloc(&dO, 128 * 16 * 4);
  cudaMemcpy(dC, C.data(), C.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 32 * 1024>>>(dC, dP, dO);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("i8_probe: CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<int> O(128 * 16);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      long ref = 0;
      for (int t = 0; t < 128; ++t) ref += (long)C[t * 128 + m] * P[n * 128 + t];
      if (ref != O[m * 16 + n]) {
        if (bad < 5) printf("mismatch m %d n %d: gpu %d ref %ld\n", m, n, O[m * 16 + n], ref);
        ++bad;
      }
    }
  printf("i8_probe: %s (%d mismatches of %d)\n", bad ? "FAIL" : "OK", bad, 128 * 16);
  return bad != 0;
}
