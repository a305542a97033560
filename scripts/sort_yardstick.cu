// Yardstick: our hs_sort_pairs32 / hs_depth_order against CUB's DeviceRadixSort on the
// binning sizes (2M tile keys of 14 bits, 800k depth keys of 32 bits). Not part of the
// product; CUB only sets the bar.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/sort_yardstick.cu -o /tmp/sy -ldl
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

// keeps the GPU busy while the host enqueues the timed launches, so the events see
// device time only
__global__ void spin(long long ns) {
    const long long t0 = clock64();
    while (clock64() - t0 < ns * 2) {}
}

typedef int (*sort32_t)(int64_t, uint32_t, uint32_t *, uint32_t *, uint32_t *, uint32_t *, void *, size_t, int *, void *);
typedef size_t (*wsz_t)(int64_t);

int main(int argc, char **argv) {
    const char *lib = argc > 1 ? argv[1] : "paper_2503_12886_b200/lib/libhs_b200.so";
    void *h = dlopen(lib, RTLD_NOW);
    if (!h) { printf("dlopen: %s\n", dlerror()); return 1; }
    auto sort32 = (sort32_t)dlsym(h, "hs_sort_pairs32");
    auto wsz = (wsz_t)dlsym(h, "hs_sort_workspace_size");
    struct Case { int64_t n; int bits; bool clustered; const char *name; };
    Case cases[] = {{2037984, 14, true, "tile keys 2.04M x 14 bits"}, {802816, 32, false, "depth keys 0.80M x 32 bits"}};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (auto &c : cases) {
        std::mt19937 rng(1);
        std::vector<uint32_t> hk(c.n);
        const uint32_t mask = c.bits == 32 ? 0xFFFFFFFFu : ((1u << c.bits) - 1);
        for (int64_t i = 0; i < c.n; ++i) {
            if (c.clustered) {   // runs of ~3 adjacent tiles per item, like the emission
                uint32_t base = rng() & mask;
                int r = 1 + (rng() % 4);
                for (int k = 0; k < r && i < c.n; ++k, ++i) hk[i] = (base + k) & mask;
                --i;
            } else {
                hk[i] = 0x3f000000u | (rng() & 0x00ffffffu);
            }
        }
        uint32_t *k0, *k1, *v0, *v1, *kin;
        cudaMalloc(&k0, c.n * 4); cudaMalloc(&k1, c.n * 4); cudaMalloc(&v0, c.n * 4); cudaMalloc(&v1, c.n * 4);
        cudaMalloc(&kin, c.n * 4);
        cudaMemcpy(kin, hk.data(), c.n * 4, cudaMemcpyHostToDevice);
        size_t ws = wsz(c.n);
        void *w;
        cudaMalloc(&w, ws);
        const int reps = 50;
        float ours = 0, cubt = 0;
        for (int r = 0; r < reps + 5; ++r) {
            cudaMemcpyAsync(k0, kin, c.n * 4, cudaMemcpyDeviceToDevice);
            spin<<<1, 1>>>(300000);
            cudaEventRecord(e0);
            int alt = 0;
            sort32(c.n, mask, k0, v0, k1, v1, w, ws, &alt, nullptr);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 5) ours += ms;
        }
        size_t cws = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, cws, k0, k1, v0, v1, (int)c.n, 0, c.bits);
        void *cw;
        cudaMalloc(&cw, cws);
        for (int r = 0; r < reps + 5; ++r) {
            cudaMemcpyAsync(k0, kin, c.n * 4, cudaMemcpyDeviceToDevice);
            spin<<<1, 1>>>(300000);
            cudaEventRecord(e0);
            cub::DeviceRadixSort::SortPairs(cw, cws, k0, k1, v0, v1, (int)c.n, 0, c.bits);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 5) cubt += ms;
        }
        printf("%s: ours %.1f us, cub %.1f us\n", c.name, ours / reps * 1000, cubt / reps * 1000);
        cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(kin); cudaFree(w); cudaFree(cw);
    }
    return 0;
}
