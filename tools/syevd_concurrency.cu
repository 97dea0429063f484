// Does cuSOLVER's Hermitian eigensolver (Xsyevd) overlap across streams / host threads on one B200?
// n×n random Hermitian (complex128), timings in ms (host wall around the calls + a device sync):
//   single, 4 sequential on one stream, 4 concurrent (4 threads, 4 handles + streams, own params),
//   and 4 concurrent sharing one cusolverDnParams_t.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void fill(double2* a, int n, unsigned seed) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < (long)n * n; i += (long)gridDim.x * blockDim.x) {
    const int r = i % n, c = i / n;
    const int lo = r < c ? r : c, hi = r < c ? c : r;
    unsigned h = seed ^ (lo * 2654435761u) ^ (hi * 40503u);
    h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
    const double x = (h & 0xffff) / 65536.0 - 0.5, y = ((h >> 16) & 0xffff) / 65536.0 - 0.5;
    a[i] = make_double2(x + (r == c ? n * 0.01 : 0.0), r == c ? 0.0 : (r < c ? y : -y));
  }
}

static bool use_j = false;
struct Job {
  syevjInfo_t jp = nullptr;
  int lwj = 0;
  double2* wj = nullptr;
  cusolverDnHandle_t h;
  cudaStream_t s;
  cusolverDnParams_t prm;
  double2 *A, *A0;
  double* W;
  void* work;
  size_t wd, wh;
  std::vector<char> hw;
  int* info;
};

static double now() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 2000, J = 4;
  use_j = argc > 2 && argv[2][0] == 'j';
  std::vector<Job> jobs(J);
  cusolverDnParams_t shared;
  cusolverDnCreateParams(&shared);
  for (int j = 0; j < J; ++j) {
    Job& b = jobs[j];
    cusolverDnCreate(&b.h);
    CK(cudaStreamCreateWithFlags(&b.s, cudaStreamNonBlocking));
    cusolverDnSetStream(b.h, b.s);
    cusolverDnCreateParams(&b.prm);
    CK(cudaMalloc(&b.A, (size_t)n * n * 16));
    CK(cudaMalloc(&b.A0, (size_t)n * n * 16));
    CK(cudaMalloc(&b.W, n * 8));
    CK(cudaMalloc(&b.info, 4));
    fill<<<1024, 256>>>(b.A0, n, 77 + j);
    cusolverDnXsyevd_bufferSize(b.h, b.prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, b.A, n,
                                CUDA_R_64F, b.W, CUDA_C_64F, &b.wd, &b.wh);
    CK(cudaMalloc(&b.work, b.wd + 16));
    b.hw.resize(b.wh + 16);
    cusolverDnCreateSyevjInfo(&b.jp);
    cusolverDnXsyevjSetTolerance(b.jp, 0.0);
    cusolverDnXsyevjSetMaxSweeps(b.jp, 100);
    cusolverDnZheevj_bufferSize(b.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, (cuDoubleComplex*)b.A, n, b.W, &b.lwj, b.jp);
    CK(cudaMalloc(&b.wj, (size_t)b.lwj * 16 + 16));
  }
  CK(cudaDeviceSynchronize());
  auto run = [&](int j, cusolverDnParams_t p) {
    Job& b = jobs[j];
    cudaMemcpyAsync(b.A, b.A0, (size_t)n * n * 16, cudaMemcpyDeviceToDevice, b.s);
    if (use_j)
      cusolverDnZheevj(b.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, (cuDoubleComplex*)b.A, n, b.W,
                       (cuDoubleComplex*)b.wj, b.lwj, b.info, b.jp);
    else
      cusolverDnXsyevd(b.h, p, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_C_64F, b.A, n, CUDA_R_64F, b.W,
                       CUDA_C_64F, b.work, b.wd, b.hw.data(), b.wh, b.info);
  };
  run(0, jobs[0].prm);
  CK(cudaDeviceSynchronize());
  double t = now();
  run(0, jobs[0].prm);
  CK(cudaDeviceSynchronize());
  printf("{\"n\": %d, \"solver\": \"%s\", \"single_ms\": %.1f", n, use_j ? "heevj" : "syevd", now() - t);
  t = now();
  for (int j = 0; j < J; ++j) { Job& b = jobs[j]; cusolverDnSetStream(b.h, jobs[0].s); run(j, b.prm); cusolverDnSetStream(b.h, b.s); }
  CK(cudaDeviceSynchronize());
  printf(", \"seq4_ms\": %.1f", now() - t);
  for (int shared_p = 0; shared_p < 2; ++shared_p) {
    t = now();
    std::vector<std::thread> th;
    for (int j = 0; j < J; ++j) th.emplace_back([&, j] { run(j, shared_p ? shared : jobs[j].prm); cudaStreamSynchronize(jobs[j].s); });
    for (auto& x : th) x.join();
    CK(cudaDeviceSynchronize());
    printf(", \"conc4_%s_ms\": %.1f", shared_p ? "shared_params" : "own_params", now() - t);
  }
  // concurrent, all from ONE host thread (async calls back to back)
  t = now();
  for (int j = 0; j < J; ++j) run(j, jobs[j].prm);
  CK(cudaDeviceSynchronize());
  printf(", \"conc4_one_thread_ms\": %.1f}\n", now() - t);
  return 0;
}
