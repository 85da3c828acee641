// mg_sort.cuh -- scan / radix sort / CSR primitives (host-callable).
#pragma once
#include "mg_common.cuh"

namespace mg {
size_t scan_workspace_bytes(int64_t n);
void excl_scan(const int* in, int* out, int64_t n, void* ws, cudaStream_t st);
size_t radix_workspace_bytes(int64_t n);
void radix_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, int* vals_out, int64_t n, int bits, void* ws,
                      cudaStream_t st);
size_t csr_workspace_bytes(int64_t ncell);
size_t counting_workspace_bytes(int64_t n, int64_t ncell);
void counting_sort_pairs(const uint32_t* keys, uint32_t* keys_out, int* vals_out, int* starts, int64_t n,
                         int64_t ncell, void* ws, cudaStream_t st);
void csr_starts(const uint32_t* keys, int64_t n, int64_t ncell, int* starts, void* ws, cudaStream_t st);
int bits_for(int64_t maxval);
}  // namespace mg
