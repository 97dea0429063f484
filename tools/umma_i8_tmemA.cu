// Can the INT8 UMMA read its A operand from TMEM? C[128×N] = A[128×K]·B[N×K]ᵀ with A placed in TMEM by
// (1) tcgen05.st from registers (lane = row, column j = k 4j..4j+3, little-endian bytes) or (2) tcgen05.cp
// 128x256b from the canonical K-major shared-memory layout; compared bit-exactly with a CPU GEMM. Then the
// back-to-back rate with A in TMEM vs in shared memory (N = 64).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int M = 128;
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t make_idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__host__ __device__ inline int canon_off(int r, int k, int K) {
  return (r >> 3) * (K / 16) * 128 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}

template <int N, int K, int MODE>  // MODE 1: tcgen05.st, 2: tcgen05.cp
__global__ void umma_tmemA(const int8_t* __restrict__ Ag /* row-major */, const int8_t* __restrict__ Acan,
                           const int8_t* __restrict__ Bg /* canonical */, int32_t* __restrict__ C) {
  __shared__ __align__(1024) int8_t As[M * K];
  __shared__ __align__(1024) int8_t Bs[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += blockDim.x) As[i] = Acan[i];
  for (int i = tid; i < N * K; i += blockDim.x) Bs[i] = Bg[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t tA = tmem + 128;  // A at columns 128.. (K/4 columns), D at columns 0..N−1
  if (MODE == 1) {
    const int row = warp * 32 + lane;
    for (int k0 = 0; k0 < K; k0 += 32) {
      uint32_t w[8];
      for (int j = 0; j < 8; ++j) {
        uint32_t v = 0;
        for (int b = 0; b < 4; ++b) v |= ((uint32_t)(uint8_t)Ag[row * K + k0 + 4 * j + b]) << (8 * b);
        w[j] = v;
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                       tA + ((uint32_t)(warp * 32) << 16) + k0 / 4),
                   "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t idesc = make_idesc_i8(M, N);
    for (int k = 0; k < K / 32; ++k) {
      if (MODE == 2) {
        const uint64_t sa = make_desc(su32(As) + k * 256, 128, (K / 16) * 128);
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tA + k * 8), "l"(sa));
      }
      const uint64_t db = make_desc(su32(Bs) + k * 256, 128, (K / 16) * 128);
      const uint32_t acc = k > 0;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                   "r"(tA + k * 8), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                 : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(&mbar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) C[row * N + c0 + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int N, int K, int MODE>
int run() {
  std::vector<int8_t> A(M * K), B(N * K), Ac(M * K), Bc(N * K);
  srand(77 + N + K + MODE);
  for (auto& x : A) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : B) x = (int8_t)(rand() % 255 - 127);
  for (int r = 0; r < M; ++r) for (int k = 0; k < K; ++k) Ac[canon_off(r, k, K)] = A[r * K + k];
  for (int r = 0; r < N; ++r) for (int k = 0; k < K; ++k) Bc[canon_off(r, k, K)] = B[r * K + k];
  int8_t *dA, *dAc, *dB; int32_t* dC;
  CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dAc, A.size())); CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dC, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dAc, Ac.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bc.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0, M * N * 4));
  umma_tmemA<N, K, MODE><<<1, 128>>>(dA, dAc, dB, dC);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("{\"test\": \"tmemA\", \"mode\": %d, \"error\": \"%s\"}\n", MODE, cudaGetErrorString(e)); exit(2); }
  std::vector<int32_t> C(M * N);
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t ref = 0;
      for (int k = 0; k < K; ++k) ref += (int32_t)A[i * K + k] * (int32_t)B[j * K + k];
      if (ref != C[i * N + j]) { if (bad < 3) printf("  (%d,%d) got %d want %d\n", i, j, C[i * N + j], ref); ++bad; }
    }
  printf("{\"test\": \"tmemA\", \"mode\": %d, \"N\": %d, \"K\": %d, \"mismatches\": %ld}\n", MODE, N, K, bad);
  cudaFree(dA); cudaFree(dAc); cudaFree(dB); cudaFree(dC);
  return bad != 0;
}

// rate: 56 back-to-back MMAs per commit, A from TMEM (cp'd once) or from shared memory
template <int N, bool TMEM_A>
__global__ void rate(int iters, int32_t* sink) {
  __shared__ __align__(1024) int8_t As[4][M * 32];
  __shared__ __align__(1024) int8_t Bs[2][N * 32];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4 * M * 32; i += blockDim.x) (&As[0][0])[i] = (int8_t)(i * 7);
  for (int i = tid; i < 2 * N * 32; i += blockDim.x) (&Bs[0][0])[i] = (int8_t)(i * 3);
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
    const uint32_t tA = tmem + 448;  // 4 A tiles × 8 columns at columns 448..479
    if (TMEM_A)
      for (int j = 0; j < 4; ++j)
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tA + j * 8), "l"(make_desc(su32(As[j]), 128, 256)));
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < 56; ++j) {
        const uint64_t db = make_desc(su32(Bs[(j >> 2) & 1]), 128, 256);
        const uint32_t d = tmem + (uint32_t)((j % (448 / N)) * N);
        if (TMEM_A)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                       " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(tA + (j & 3) * 8),
                       "l"(db), "r"(idesc), "r"(1u));
        else
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                       " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(make_desc(su32(As[j & 3]), 128, 256)), "l"(db), "r"(idesc), "r"(1u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                   : "memory");
      if (it >= 2) {
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

template <int N, bool TA>
void time_rate() {
  int32_t* sink; CK(cudaMalloc(&sink, 4096));
  int sms = 148; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  rate<N, TA><<<sms, 128>>>(10, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  cudaEventRecord(e0);
  rate<N, TA><<<sms, 128>>>(iters, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double macs = (double)sms * iters * 56 * M * N * 32;
  printf("{\"test\": \"rate\", \"N\": %d, \"A_in_tmem\": %d, \"ms\": %.3f, \"TOPS\": %.1f, \"err\": \"%s\"}\n", N, (int)TA, ms,
         2 * macs / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

int main() {
  int f = 0;
  f += run<64, 32, 1>();
  f += run<64, 64, 1>();
  f += run<64, 32, 2>();
  f += run<64, 96, 2>();
  printf("{\"tmemA_all_ok\": %s}\n", f ? "false" : "true");
  time_rate<64, false>();
  time_rate<64, true>();
  time_rate<128, true>();
  return f;
}
