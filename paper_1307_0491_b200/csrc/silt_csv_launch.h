// silt_csv_launch.h — device CSV snapshot formatting (kernels in silt_csv.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "silt_csv.cuh"

// Field accessor: value c of local cell (i, j) is f[c][j * row_stride + i * col_stride]
// (AoS: f[c] = base + c, strides 4 nx / 4; solver planes: strides pitch / 1).
struct CsvField {
    const double* f[4];
    long long row_stride, col_stride;
};

// Geometry of the rows being formatted (snapshot_to_string, src/snapshot.cpp:50-84).
struct CsvGeom {
    int nx, rows, j0, dim;  // rows of this chunk; j0 = global index of its first row
    double dx, dy, h_dry, time;
};

// Longest row: 8 numbers of at most 25 characters plus 8 separators.
constexpr int kCsvRowMax = 8 * silt_csv::kMaxNum + 8;

void silt_csv_format_launch(const CsvField& F, const CsvGeom& G, const silt_csv::Pow5Table* T,
                            char* stage, int* len, cudaStream_t st);
size_t silt_csv_scan_temp_bytes(int n);
void silt_csv_scan(const int* len, int* off, int n, void* temp, size_t temp_bytes,
                   cudaStream_t st);
void silt_csv_compact_launch(const char* stage, const int* len, const int* off, int n, char* out,
                             cudaStream_t st);
