// hs_pool.cu -- device frame pool gather for online training.
//
// The online stream (S/stream.py:27-86) keeps every pooled frame resident in HBM
// (u8 RGBA image + theta per slot); a training step's batch is a list of slot
// ids drawn on the host by the reference's sampling rule, and this gather turns
// them into the step's contiguous target / theta buffers without any H2D copy of
// frame data.  One CTA row-chunk per (row, 16 KiB piece), 16-byte vector copies.
#include "hs_common.cuh"

namespace hs {

constexpr int kGatherThreads = 256;
constexpr int64_t kGatherChunk = 16 * 1024;   // bytes per CTA

__global__ void __launch_bounds__(kGatherThreads) gather_rows_kernel(int64_t row_bytes, int64_t chunks_per_row,
                                                                    const int32_t *__restrict__ idx,
                                                                    const unsigned char *__restrict__ src,
                                                                    unsigned char *__restrict__ dst, bool vec) {
    pdl_prologue();
    const int64_t r = blockIdx.y;
    const int64_t c0 = (int64_t)blockIdx.x * kGatherChunk;
    const int64_t n = min(kGatherChunk, row_bytes - c0);
    if (n <= 0) return;
    const unsigned char *s = src + (int64_t)idx[r] * row_bytes + c0;
    unsigned char *d = dst + r * row_bytes + c0;
    if (vec) {
        const int64_t n16 = n / 16;
        for (int64_t i = threadIdx.x; i < n16; i += blockDim.x)
            __stcs(reinterpret_cast<uint4 *>(d) + i, __ldcs(reinterpret_cast<const uint4 *>(s) + i));
        for (int64_t i = n16 * 16 + threadIdx.x; i < n; i += blockDim.x) d[i] = s[i];
    } else {
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) d[i] = s[i];
    }
}

}  // namespace hs

using namespace hs;

extern "C" {

int hs_gather_rows(int num_rows, int64_t row_bytes, const int32_t *slots, const void *pool, void *out,
                   void *stream) {
    if (num_rows < 0 || row_bytes < 0) {
        set_error("hs_gather_rows: bad sizes rows=%d row_bytes=%lld", num_rows, (long long)row_bytes);
        return HS_ERR_SHAPE;
    }
    if (num_rows == 0 || row_bytes == 0) return HS_OK;
    const bool vec = row_bytes % 16 == 0 && (uintptr_t)pool % 16 == 0 && (uintptr_t)out % 16 == 0;
    const int64_t chunks = (row_bytes + kGatherChunk - 1) / kGatherChunk;
    const dim3 grid((unsigned)chunks, (unsigned)num_rows);
    launch_k(gather_rows_kernel, grid, kGatherThreads, 0, HS_CHECK_STREAM(stream), 
        row_bytes, chunks, slots, reinterpret_cast<const unsigned char *>(pool), reinterpret_cast<unsigned char *>(out),
        vec);
    return check_launch("hs_gather_rows");
}

// Page-lock a caller's host buffer in place (end-to-end inputs DMA'd without a staging
// copy).  A failure (e.g. the range overlaps a registered one) is reported and the
// runtime error state cleared, so the caller can fall back to staging.
int hs_host_register(void *ptr, size_t bytes) {
    const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("hs_host_register: %s", cudaGetErrorString(e));
        return HS_ERR_CUDA;
    }
    return HS_OK;
}

int hs_host_unregister(void *ptr) {
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("hs_host_unregister: %s", cudaGetErrorString(e));
        return HS_ERR_CUDA;
    }
    return HS_OK;
}

}  // extern "C"
