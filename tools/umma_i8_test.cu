// Stage-1 check of the tcgen05 INT8 path used by the emulated-FP64 contraction:
// one CTA computes C[128×N] = A[128×K] · B[N×K]ᵀ (int8 → int32) with tcgen05.mma.cta_group::1.kind::i8,
// operands in shared memory in the K-major SWIZZLE_NONE canonical layout (8-row × 16-byte core
// matrices; LBO = stride between K-adjacent core matrices, SBO = stride between 8-row groups),
// accumulator in TMEM, read back with tcgen05.ld.32x32b. Compared bit-exactly with a CPU GEMM.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int M = 128;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// smem matrix descriptor (cute::UMMA::SmemDescriptor): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), base_offset [49,52), lbo_mode [52], layout_type [61,64) (0 = SWIZZLE_NONE)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// instruction descriptor (cute::UMMA::InstrDescriptor): c_format S32=2 [4,6), a/b format signed 1
// [7,10)/[10,13), a/b K-major 0 [15]/[16], n_dim N>>3 [17,23), m_dim M>>4 [24,29)
__host__ __device__ constexpr uint32_t make_idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// byte offset of element (r, k) of a rows×K int8 tile in the canonical K-major no-swizzle layout
__host__ __device__ inline int canon_off(int r, int k, int K) {
  return (r >> 3) * (K / 16) * 128 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}

template <int N, int K>
__global__ void umma_i8(const int8_t* __restrict__ Ag, const int8_t* __restrict__ Bg, int32_t* __restrict__ C) {
  __shared__ __align__(1024) int8_t As[M * K];
  __shared__ __align__(1024) int8_t Bs[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) As[i] = Ag[i];  // already in canonical order
  for (int i = tid; i < N * K; i += blockDim.x) Bs[i] = Bg[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "r"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes → async proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_i8(M, N);
    for (int k = 0; k < K / 32; ++k) {
      const uint64_t da = make_desc(su32(As) + k * 256, 128, (K / 16) * 128);
      const uint64_t db = make_desc(su32(Bs) + k * 256, 128, (K / 16) * 128);
      const uint32_t acc = k > 0;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                 : "memory");
  }
  // wait for the MMAs
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(&mbar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads TMEM lanes 32w..32w+31 (= rows), N columns, 8 at a time
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) C[row * N + c0 + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N < 32 ? 32 : N));
}

template <int N, int K>
int run() {
  std::vector<int8_t> A(M * K), B(N * K), Ac(M * K), Bc(N * K);
  srand(1234 + N + K);
  for (auto& x : A) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : B) x = (int8_t)(rand() % 255 - 127);
  for (int r = 0; r < M; ++r) for (int k = 0; k < K; ++k) Ac[canon_off(r, k, K)] = A[r * K + k];
  for (int r = 0; r < N; ++r) for (int k = 0; k < K; ++k) Bc[canon_off(r, k, K)] = B[r * K + k];
  int8_t *dA, *dB; int32_t* dC;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dC, M * N * 4));
  CK(cudaMemcpy(dA, Ac.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bc.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0, M * N * 4));
  umma_i8<N, K><<<1, 128>>>(dA, dB, dC);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> C(M * N);
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += (int32_t)A[i * K + k] * (int32_t)B[j * K + k];
      if (ref != C[i * N + j]) {
        if (bad < 5) printf("  mismatch (%d,%d): got %d want %d\n", i, j, C[i * N + j], ref);
        ++bad;
      }
    }
  printf("{\"test\": \"umma_i8\", \"N\": %d, \"K\": %d, \"mismatches\": %ld}\n", N, K, bad);
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  return bad != 0;
}

// Throughput: every SM issues ITER × 56 back-to-back M=128×N×K=32 int8 MMAs on resident smem operands
template <int N>
__global__ void umma_rate(int iters, int32_t* sink) {
  constexpr int K = 32;
  __shared__ __align__(1024) int8_t As[4][M * K];
  __shared__ __align__(1024) int8_t Bs[2][N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4 * M * K; i += blockDim.x) (&As[0][0])[i] = (int8_t)(i * 7);
  for (int i = tid; i < 2 * N * K; i += blockDim.x) (&Bs[0][0])[i] = (int8_t)(i * 3);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_i8(M, N);
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < 56; ++j) {
        const uint64_t da = make_desc(su32(As[j & 3]), 128, 256);
        const uint64_t db = make_desc(su32(Bs[(j >> 2) & 1]), 128, 256);
        const uint32_t d = tmem + (uint32_t)((j % (512 / N)) * N);
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                     " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                     "l"(da), "l"(db), "r"(idesc), "r"(1u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                   : "memory");
      if (it >= 2) {  // keep ≤ 2 commit groups in flight
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                       : "=r"(done) : "r"(su32(&mbar)), "r"(phase) : "memory");
        phase ^= 1;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) sink[blockIdx.x] = 1;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N>
void rate() {
  int32_t* sink; cudaMalloc(&sink, 1024 * 4);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  umma_rate<N><<<sms, 128>>>(10, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  cudaEventRecord(e0);
  umma_rate<N><<<sms, 128>>>(iters, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double macs = (double)sms * iters * 56 * M * N * 32;
  printf("{\"test\": \"umma_i8_rate\", \"N\": %d, \"ms\": %.3f, \"TOPS\": %.1f, \"err\": \"%s\"}\n", N, ms,
         2 * macs / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

int main() {
  int fails = 0;
  fails += run<64, 64>();
  fails += run<64, 224>();
  fails += run<128, 96>();
  fails += run<16, 32>();
  printf("{\"umma_i8_all_ok\": %s}\n", fails ? "false" : "true");
  rate<64>();
  rate<128>();
  rate<256>();
  return fails;
}
