// dram_pattern.cu -- DRAM over-fetch of strided interior-row reads (layout experiment).
// Copies, per "row" of RS doubles, the first RL doubles (16-byte accesses), over a buffer >> L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dram_pattern tools/dram_pattern.cu
//   ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum tools/dram_pattern
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_rows(const double* __restrict__ src, double* __restrict__ dst, long rows, int rs, int rl,
                       int off) {
  const int h = rl / 2;
  const long tot = rows * h;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < tot; t += (long)gridDim.x * blockDim.x) {
    const long r = t / h;
    const int c = (int)(t - r * h);
    const double2 v = __ldcs(reinterpret_cast<const double2*>(src + r * rs + off) + c);
    __stcs(reinterpret_cast<double2*>(dst + r * rs + off) + c, v);
  }
}

int main() {
  const long total = 400l * 1000 * 1000;   // doubles per buffer (3.2 GB)
  double *a, *b;
  if (cudaMalloc(&a, total * 8) || cudaMalloc(&b, total * 8)) return 1;
  cudaMemset(a, 0, total * 8);
  cudaMemset(b, 0, total * 8);
  struct Case { int rs, rl, off; const char* name; } cs[] = {
      {20, 16, 0, "m16 rows: 16 of 20 (rotated interior-first)"},
      {20, 16, 2, "m16 rows: 16 of 20 at +2 (natural layout)"},
      {20, 20, 0, "m16 rows: whole 20"},
      {16, 16, 0, "dense 16 of 16"},
      {36, 32, 0, "m32 rows: 32 of 36"},
  };
  for (auto& c : cs) {
    const long rows = total / c.rs;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_rows<<<148 * 8, 256>>>(a, b, rows, c.rs, c.rl, c.off);
    cudaEventRecord(e0);
    k_rows<<<148 * 8, 256>>>(a, b, rows, c.rs, c.rl, c.off);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double useful = 2.0 * rows * c.rl * 8;
    printf("%-45s useful %.2f GB  %.3f ms  %.0f GB/s useful\n", c.name, useful / 1e9, ms, useful / ms / 1e6);
  }
  return 0;
}
