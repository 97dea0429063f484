// Bandwidth probe for the K5 access pattern at config-3 sector shapes (d = N+1 = 32, χ = 4096):
// pure load → store of every Θ element's L-vector (no math), in three orders:
//   (a) linear copy of all sector buffers (reference HBM rate)
//   (b) tile order: warp = 8 consecutive columns of one (c_l, c_r) block, all L sectors (current K5)
//   (c) row order: a CTA streams ONE row α through every sector c ≤ c_l (contiguous sector rows)
// Reads per-charge counts from tools/config3_counts.txt. Prints GB/s of (read+write) traffic.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int NQ = 32;
struct Sec { double2* p[NQ]; int ld[NQ]; int off_l[NQ + 1]; int off_r[NQ + 1]; };

__global__ void copy_lin(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = __ldcs(a + i);
}

// (b): one warp per 8-group of a (cl, cr) block; blocks enumerated by a flat table
struct Grp { int cl, cr, row, col0, w; };
__global__ void tile_order(Sec s, const Grp* __restrict__ g, int ng) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= ng) return;
  const Grp G = g[warp];
  const int e = lane & 7, q = lane >> 3;  // 8 elements × 4 sectors per instruction
  if (e >= G.w) return;
  const int L = G.cl - G.cr + 1;
  double2 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int u = k * 4 + q;
    const int c = G.cr + u;
    if (u < L) v[k] = __ldcs(s.p[c] + (size_t)(G.row - s.off_l[c]) * s.ld[c] + (G.col0 + e));
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int u = k * 4 + q;
    const int c = G.cr + u;
    if (u < L) __stcs(s.p[c] + (size_t)(G.row - s.off_l[c]) * s.ld[c] + (G.col0 + e), make_double2(v[k].x * 1.0000001, v[k].y));
  }
}

// (c): one CTA per row α (charge cl): for each sector c ≤ cl, stream its full row (cols [0, off_r[c+1]))
__global__ void row_order(Sec s, const int* __restrict__ rowcl) {
  const int row = blockIdx.x;
  const int cl = rowcl[row];
  for (int c = 0; c <= cl; ++c) {
    double2* r = s.p[c] + (size_t)(row - s.off_l[c]) * s.ld[c];
    const int n = s.off_r[c + 1];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double2 x = __ldcs(r + i);
      __stcs(r + i, make_double2(x.x * 1.0000001, x.y));
    }
  }
}

// (d): item order: a CTA handles (row, c_r block, W-column chunk) and streams the L sector runs of
// W×16 B each (the TMA-item K5 design); items ordered row-major so neighbours share DRAM pages
struct Item { int row, cl, cr, j0, w; };
__global__ void item_order(Sec s, const Item* __restrict__ it, int n) {
  const Item I = it[blockIdx.x];
  const int L = I.cl - I.cr + 1;
  for (int idx = threadIdx.x; idx < L * I.w; idx += blockDim.x) {
    const int u = idx / I.w, col = idx - u * I.w;
    const int c = I.cr + u;
    double2* p = s.p[c] + (size_t)(I.row - s.off_l[c]) * s.ld[c] + (s.off_r[I.cr] + I.j0 + col);
    double2 x = __ldcs(p);
    __stcs(p, make_double2(x.x * 1.0000001, x.y));
  }
}

// (e): like (b) but a warp owns 32 consecutive columns of one row and moves ONE sector per
// instruction (lane = column); (f) 16 columns × 2 sectors per instruction
template <int EPW>
__global__ void warp_rows(Sec s, const Grp* __restrict__ g, int ng) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= ng) return;
  const Grp G = g[warp];
  constexpr int SPI = 32 / EPW;  // sectors per instruction
  const int e = lane % EPW, q = lane / EPW;
  if (e >= G.w) return;
  const int L = G.cl - G.cr + 1;
  double2 v[32 / SPI];
#pragma unroll
  for (int k = 0; k < 32 / SPI; ++k) {
    const int u = k * SPI + q, c = G.cr + u;
    if (u < L) v[k] = __ldcs(s.p[c] + (size_t)(G.row - s.off_l[c]) * s.ld[c] + (G.col0 + e));
  }
#pragma unroll
  for (int k = 0; k < 32 / SPI; ++k) {
    const int u = k * SPI + q, c = G.cr + u;
    if (u < L) __stcs(s.p[c] + (size_t)(G.row - s.off_l[c]) * s.ld[c] + (G.col0 + e), make_double2(v[k].x * 1.0000001, v[k].y));
  }
}

int main() {
  FILE* f = fopen("tools/config3_counts.txt", "r");
  int nl[NQ], nc[NQ], nr[NQ];
  for (int i = 0; i < NQ; ++i) fscanf(f, "%d", &nl[i]);
  for (int i = 0; i < NQ; ++i) fscanf(f, "%d", &nc[i]);
  for (int i = 0; i < NQ; ++i) fscanf(f, "%d", &nr[i]);
  Sec s;
  int ol[NQ + 1], orr[NQ + 1];
  ol[0] = orr[0] = 0;
  for (int i = 0; i < NQ; ++i) { ol[i + 1] = ol[i] + nl[i]; orr[i + 1] = orr[i] + nr[i]; }
  size_t tot = 0;
  for (int c = 0; c < NQ; ++c) {
    const int R = ol[NQ] - ol[c], C = orr[c + 1];
    s.ld[c] = C; s.off_l[c] = ol[c];
    CK(cudaMalloc(&s.p[c], (size_t)R * C * 16));
    CK(cudaMemset(s.p[c], 0, (size_t)R * C * 16));
    tot += (size_t)R * C;
  }
  for (int i = 0; i <= NQ; ++i) s.off_r[i] = orr[i];
  s.off_l[0] = 0;
  printf("{\"theta_elems\": %zu, \"bytes_rw\": %zu}\n", tot, tot * 32);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // (a)
  double2 *a, *b; CK(cudaMalloc(&a, tot * 16)); CK(cudaMalloc(&b, tot * 16)); CK(cudaMemset(a, 0, tot * 16));
  for (int r = 0; r < 3; ++r) copy_lin<<<148 * 8, 256>>>(a, b, tot);
  cudaEventRecord(e0); for (int r = 0; r < 5; ++r) copy_lin<<<148 * 8, 256>>>(a, b, tot); cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  printf("{\"probe\": \"linear_copy\", \"ms\": %.4f, \"GBps\": %.1f}\n", ms, tot * 32 / ms / 1e6);
  // (b)
  std::vector<Grp> gs;
  for (int cl = 0; cl < NQ; ++cl) for (int cr = 0; cr <= cl; ++cr) for (int row = ol[cl]; row < ol[cl + 1]; ++row)
    for (int c0 = 0; c0 < nr[cr]; c0 += 8) gs.push_back(Grp{cl, cr, row, orr[cr] + c0, nr[cr] - c0 < 8 ? nr[cr] - c0 : 8});
  Grp* dg; CK(cudaMalloc(&dg, gs.size() * sizeof(Grp)));
  CK(cudaMemcpy(dg, gs.data(), gs.size() * sizeof(Grp), cudaMemcpyHostToDevice));
  const int ng = (int)gs.size();
  for (int r = 0; r < 3; ++r) tile_order<<<(ng + 7) / 8, 256>>>(s, dg, ng);
  cudaEventRecord(e0); for (int r = 0; r < 5; ++r) tile_order<<<(ng + 7) / 8, 256>>>(s, dg, ng); cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  printf("{\"probe\": \"tile_order\", \"groups\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", ng, ms, tot * 32 / ms / 1e6);
  // (c)
  std::vector<int> rowcl(ol[NQ]);
  for (int cl = 0; cl < NQ; ++cl) for (int r = ol[cl]; r < ol[cl + 1]; ++r) rowcl[r] = cl;
  int* drc; CK(cudaMalloc(&drc, rowcl.size() * 4)); CK(cudaMemcpy(drc, rowcl.data(), rowcl.size() * 4, cudaMemcpyHostToDevice));
  for (int bs : {256, 512, 1024}) {
    for (int r = 0; r < 3; ++r) row_order<<<ol[NQ], bs>>>(s, drc);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) row_order<<<ol[NQ], bs>>>(s, drc); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("{\"probe\": \"row_order\", \"block\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", bs, ms, tot * 32 / ms / 1e6);
  }
  // (d)
  for (int W : {64, 128, 256}) {
    std::vector<Item> items;
    for (int cl = 0; cl < NQ; ++cl) for (int row = ol[cl]; row < ol[cl + 1]; ++row) for (int cr = 0; cr <= cl; ++cr)
      for (int j0 = 0; j0 < nr[cr]; j0 += W) items.push_back(Item{row, cl, cr, j0, nr[cr] - j0 < W ? nr[cr] - j0 : W});
    Item* di; CK(cudaMalloc(&di, items.size() * sizeof(Item)));
    CK(cudaMemcpy(di, items.data(), items.size() * sizeof(Item), cudaMemcpyHostToDevice));
    const int n = (int)items.size();
    for (int r = 0; r < 3; ++r) item_order<<<n, 256>>>(s, di, n);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) item_order<<<n, 256>>>(s, di, n); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("{\"probe\": \"item_order\", \"W\": %d, \"items\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", W, n, ms, tot * 32 / ms / 1e6);
    cudaFree(di);
  }
  // (e)/(f)
  for (int EPW : {32, 16, 8}) {
    std::vector<Grp> g2;
    for (int cl = 0; cl < NQ; ++cl) for (int cr = 0; cr <= cl; ++cr) for (int row = ol[cl]; row < ol[cl + 1]; ++row)
      for (int c0 = 0; c0 < nr[cr]; c0 += EPW) g2.push_back(Grp{cl, cr, row, orr[cr] + c0, nr[cr] - c0 < EPW ? nr[cr] - c0 : EPW});
    Grp* dg2; CK(cudaMalloc(&dg2, g2.size() * sizeof(Grp)));
    CK(cudaMemcpy(dg2, g2.data(), g2.size() * sizeof(Grp), cudaMemcpyHostToDevice));
    const int n2 = (int)g2.size();
    auto run = [&]() {
      if (EPW == 32) warp_rows<32><<<(n2 + 7) / 8, 256>>>(s, dg2, n2);
      else if (EPW == 16) warp_rows<16><<<(n2 + 7) / 8, 256>>>(s, dg2, n2);
      else warp_rows<8><<<(n2 + 7) / 8, 256>>>(s, dg2, n2);
    };
    for (int r = 0; r < 3; ++r) run();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) run(); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("{\"probe\": \"warp_rows\", \"elems_per_instr\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", EPW, ms, tot * 32 / ms / 1e6);
    cudaFree(dg2);
  }
  return 0;
}
