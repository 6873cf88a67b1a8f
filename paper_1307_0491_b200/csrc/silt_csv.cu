// silt_csv.cu — snapshot CSV on the device: write_snapshot / snapshot_to_string
// (src/snapshot.cpp:50-93) byte for byte.  Compiled with -fmad=false: the
// derived columns (x = (i + 0.5) dx, u = hu / h, eta = h + zb) are single
// IEEE operations, as in the reference.
//
// Three kernels per chunk of rows: format every cell's CSV row into a
// fixed-stride stage (one thread per cell), exclusive-scan the row lengths
// (CUB), compact the rows into contiguous bytes (one warp per 32 rows).
#include <cub/device/device_scan.cuh>

#include "silt_csv_launch.h"

namespace {

__device__ __forceinline__ int put_num(char* out, double v, const silt_csv::Pow5Table* T) {
    return silt_csv::format_g17(v, out, T);
}

__global__ void __launch_bounds__(128) csv_format_kernel(CsvField F, CsvGeom G,
                                                         const silt_csv::Pow5Table* T, char* stage,
                                                         int* len) {
    const long long n = (long long)G.nx * G.rows;
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int i = (int)(k % G.nx), j = (int)(k / G.nx);
    const long long at = (long long)j * F.row_stride + (long long)i * F.col_stride;
    const double h = F.f[0][at], hu = F.f[1][at], hv = F.f[2][at], zb = F.f[3][at];
    // primitives (src/grid.cpp:47-59)
    const bool wet = h > G.h_dry;
    const double u = wet ? hu / h : 0.0;
    const double v = wet ? hv / h : 0.0;
    char buf[kCsvRowMax];
    int p = 0;
    p += put_num(buf + p, (i + 0.5) * G.dx, T);  // Grid::x_center
    buf[p++] = ',';
    if (G.dim == 2) {
        p += put_num(buf + p, (G.j0 + j + 0.5) * G.dy, T);  // Grid::y_center
        buf[p++] = ',';
    }
    p += put_num(buf + p, h, T);
    buf[p++] = ',';
    p += put_num(buf + p, u, T);
    buf[p++] = ',';
    if (G.dim == 2) {
        p += put_num(buf + p, v, T);
        buf[p++] = ',';
    }
    p += put_num(buf + p, zb, T);
    buf[p++] = ',';
    p += put_num(buf + p, h + zb, T);
    buf[p++] = ',';
    p += put_num(buf + p, G.time, T);
    buf[p++] = '\n';
    char* dst = stage + k * kCsvRowMax;
    for (int q = 0; q < p; ++q) dst[q] = buf[q];
    len[k] = p;
}

// One warp per group of 32 rows; lanes copy each row's bytes cooperatively.
__global__ void __launch_bounds__(256) csv_compact_kernel(const char* stage, const int* len,
                                                          const int* off, int n, char* out) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long r0 = warp * 32;
    if (r0 >= n) return;
    const int rn = (int)((n - r0) < 32 ? (n - r0) : 32);
    for (int r = 0; r < rn; ++r) {
        const long long row = r0 + r;
        const int L = len[row];
        const char* src = stage + row * kCsvRowMax;
        char* dst = out + off[row];
        for (int q = lane; q < L; q += 32) dst[q] = src[q];
    }
}

}  // namespace

void silt_csv_format_launch(const CsvField& F, const CsvGeom& G, const silt_csv::Pow5Table* T,
                            char* stage, int* len, cudaStream_t st) {
    const long long n = (long long)G.nx * G.rows;
    if (n <= 0) return;
    csv_format_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(F, G, T, stage, len);
}

size_t silt_csv_scan_temp_bytes(int n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int*)nullptr, (int*)nullptr, n);
    return bytes;
}

void silt_csv_scan(const int* len, int* off, int n, void* temp, size_t temp_bytes,
                   cudaStream_t st) {
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, len, off, n, st);
}

void silt_csv_compact_launch(const char* stage, const int* len, const int* off, int n, char* out,
                             cudaStream_t st) {
    if (n <= 0) return;
    const long long threads = ((long long)n + 31) / 32 * 32;
    csv_compact_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(stage, len, off, n, out);
}
