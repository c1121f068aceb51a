// aiwc_util.cuh -- device-wide scan / radix sort / run-length reduce.
#pragma once
#include "aiwc_internal.cuh"

namespace aiwc {

enum { RLE_ONES = 0, RLE_RW = 1, RLE_SUM = 2 };

size_t scan_scratch_elems(uint64_t n);
void scan_exclusive_u32(uint32_t* d, uint64_t n, uint32_t* scratch, uint32_t* total_out, cudaStream_t s,
                        int* kernels);
// same over u64 (scratch: scan_scratch_elems(n) u64s)
void scan_exclusive_u64(unsigned long long* d, uint64_t n, unsigned long long* scratch, unsigned long long* total_out,
                        cudaStream_t s, int* kernels);
size_t rle_scratch_elems(uint64_t n);
uint64_t rle_reduce(const uint64_t* keys, const unsigned long long* wts, uint64_t n, int shift, int mode,
                    uint64_t* out_key, unsigned long long* out_a, unsigned long long* out_b, uint32_t* scratch,
                    cudaStream_t s, int* kernels);

}  // namespace aiwc
