// Microbenchmark: shared-memory throughput of the CX access mix (4 LDS.128 + 2 STS.128 per
// lane-item) when a warp's 16-byte lane accesses are scattered over rows of RB bytes
// (RB/16 lanes per row), rows drawn at random (optionally made bank-conflict-free per
// quarter-warp).  Prints bytes/clk/SM for each pattern; the sequential pattern is the
// roofline probe of libpfs (pfs_measure_smem_bandwidth).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o smem_scatter smem_scatter.cu && ./smem_scatter
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

__global__ void __launch_bounds__(512) k(const uint32_t* __restrict__ offs, int iters, int items, uint32_t* sink, long long* cyc) {
    extern __shared__ __align__(16) uint4 sb[];
    const int t = threadIdx.x;
    for (int i = t; i < 160 * 1024 / 16; i += blockDim.x) sb[i] = make_uint4(i, i * 3, i * 5, i * 7);
    __syncthreads();
    const uint32_t zoff = 80 * 1024 / 16;  // z plane 80 KB above the x plane (uint4 units)
    uint4 acc = make_uint4(0, 0, 0, 0);
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        for (int i = t; i < items; i += blockDim.x) {
            const uint32_t w = __ldg(offs + i);
            const uint32_t a = w & 0xFFFFu, b = w >> 16;  // uint4 indices in the x plane
            uint4 x0 = sb[a], x1 = sb[b], z0 = sb[a + zoff], z1 = sb[b + zoff];
            x1.x ^= x0.x; x1.y ^= x0.y; x1.z ^= x0.z; x1.w ^= x0.w;
            z0.x ^= z1.x; z0.y ^= z1.y; z0.z ^= z1.z; z0.w ^= z1.w;
            sb[b] = x1;
            sb[a + zoff] = z0;
            acc.x ^= x1.x;
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    if (t == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    if (acc.x == 0x12345678u) sink[0] = acc.x;
}

int main() {
    const int threads = 512, iters = 200;
    const int items = 512 * 16;  // lane-items per iteration per CTA
    uint32_t *d_offs, *d_sink; long long* d_cyc;
    cudaMalloc(&d_offs, items * 4); cudaMalloc(&d_sink, 4); cudaMalloc(&d_cyc, 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mode = 0; mode < 6; mode++) {
        // mode 0: sequential; 1..4: random rows of RB = 16, 32, 64, 128 bytes (bank-balanced per
        // quarter-warp); 5: RB = 32 fully random rows (conflicts as they fall)
        const int RB = mode == 0 ? 0 : mode == 5 ? 32 : (16 << (mode - 1));
        std::vector<uint32_t> offs(items);
        const int plane16 = 80 * 1024 / 16;  // uint4 per plane
        srand(1234 + mode);
        for (int i0 = 0; i0 < items; i0 += 8) {  // one quarter-warp phase: 8 lanes
            if (mode == 0) { for (int l = 0; l < 8; l++) { uint32_t a = (i0 + l) % (plane16 / 2), b = a + plane16 / 2; offs[i0 + l] = a | (b << 16); } continue; }
            const int lpr = RB / 16;            // lanes per row
            const int rows_per_phase = 8 / lpr; // rows a phase touches
            const int nrows = 80 * 1024 / RB;
            const int classes = 128 / RB;       // bank classes of a row (row index mod classes)
            for (int op = 0; op < 2; op++) {
                std::vector<int> rows;
                for (int j = 0; j < rows_per_phase; j++) {
                    int r;
                    if (mode == 5 || classes <= 1) r = rand() % (nrows / 2);
                    else { r = (rand() % (nrows / 2 / classes)) * classes + (j % classes); }  // distinct bank class
                    rows.push_back(r + (op ? nrows / 2 : 0));
                }
                for (int l = 0; l < 8; l++) {
                    const uint32_t idx = (uint32_t)rows[l / lpr] * lpr + (l % lpr);
                    if (op == 0) offs[i0 + l] = idx; else offs[i0 + l] |= idx << 16;
                }
            }
        }
        cudaMemcpy(d_offs, offs.data(), items * 4, cudaMemcpyHostToDevice);
        for (int grid_mul = 1; grid_mul <= 1; grid_mul++) {
            k<<<sms, threads, 160 * 1024>>>(d_offs, 5, items, d_sink, d_cyc);
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            k<<<sms, threads, 160 * 1024>>>(d_offs, iters, items, d_sink, d_cyc);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            long long cyc; cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
            const double bytes = (double)items * iters * 6 * 16;
            printf("mode %d RB %3d: %.1f B/clk/SM (cycles %lld), %.2f TB/s chip, err=%s\n", mode, RB, bytes / cyc, cyc,
                   bytes * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
