// On-device output writers: shot-major b8 tables ->
// the reference's text / sparse formats, byte-exact with
// stabsim/io_formats.py:66-187:
//   01   — one ASCII '0'/'1' per result, '\n' per shot (io_formats.py:66-72);
//   hits — ascending set-bit indices, comma separated, '\n' per shot (114-124);
//   r8   — run lengths between ones, 255 = 255 zeros without a one, a virtual
//          one at index R closing each shot (145-166).
// 01 has a fixed length per shot.  hits / r8 are variable: pass 1 counts each
// shot's bytes (a warp per shot), an exclusive scan gives the offsets, pass 2
// writes (a warp per shot, lanes own 32-bit words of the row; a warp scan of
// per-lane byte counts places every lane's output).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>
#include <cstdint>

#include "pfs_internal.h"

namespace pfs {

namespace {

__device__ __forceinline__ uint32_t row_word(const uint8_t* row, int64_t nbytes, int64_t w) {
    uint32_t v = 0;
    const int64_t b0 = w * 4;
#pragma unroll
    for (int j = 0; j < 4; j++)
        if (b0 + j < nbytes) v |= (uint32_t)row[b0 + j] << (8 * j);
    return v;
}

__device__ __forceinline__ uint32_t ndigits(uint32_t v) {
    uint32_t d = 1;
    while (v >= 10) { v /= 10; d++; }
    return d;
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, int lane, uint32_t& total) {
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
        if (lane >= d) x += y;
    }
    total = __shfl_sync(0xFFFFFFFFu, x, 31);
    return x - v;
}

__global__ void __launch_bounds__(256) write01_kernel(const uint8_t* __restrict__ in, int64_t pitch,
                                                      int64_t shots, int64_t R, uint8_t* __restrict__ out) {
    const int64_t line = R + 1;
    const int64_t total = shots * line;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / line, r = i - s * line;
        out[i] = r == R ? (uint8_t)'\n' : (uint8_t)('0' + ((in[s * pitch + (r >> 3)] >> (r & 7)) & 1));
    }
}

// pass 1 (fmt 2 hits / 3 r8): bytes of each shot's output
template <int FMT>
__global__ void __launch_bounds__(256) sparse_len_kernel(const uint8_t* __restrict__ in, int64_t pitch,
                                                         int64_t shots, int64_t R, uint64_t* __restrict__ len) {
    const int lane = threadIdx.x & 31;
    const int64_t nbytes = (R + 7) >> 3, nwords = (nbytes + 3) >> 2;
    for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < shots;
         s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint8_t* row = in + s * pitch;
        uint64_t acc = 0;
        int64_t prev = -1;  // r8: last one before this chunk
        for (int64_t w0 = 0; w0 < nwords; w0 += 32) {
            const int64_t w = w0 + lane;
            const uint32_t v = w < nwords ? row_word(row, nbytes, w) : 0u;
            uint64_t mine = 0;
            if (FMT == 2) {
                uint32_t b = v;
                while (b) { mine += ndigits((uint32_t)(w * 32 + __ffs(b) - 1)) + 1; b &= b - 1; }  // digits + comma
            } else {
                // r8: one byte per one, plus a 255 per whole 255 zeros of its gap
                const int last = v ? (int)(w * 32 + 31 - __clz(v)) : -1;
                // previous one before this lane: max over lower lanes' last, else prev
                int pl = last;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(0xFFFFFFFFu, pl, d);
                    if (lane >= d) pl = max(pl, y);
                }
                int before = __shfl_up_sync(0xFFFFFFFFu, pl, 1);
                if (lane == 0) before = -1;
                int64_t p = max((int64_t)before, prev);
                uint32_t b = v;
                while (b) {
                    const int64_t pos = w * 32 + __ffs(b) - 1;
                    mine += 1 + (uint64_t)((pos - p - 1) / 255);
                    p = pos;
                    b &= b - 1;
                }
                const int lastall = __shfl_sync(0xFFFFFFFFu, pl, 31);
                prev = max(prev, (int64_t)lastall);
            }
            for (int d = 16; d > 0; d >>= 1) mine += __shfl_xor_sync(0xFFFFFFFFu, mine, d);
            acc += mine;
        }
        if (lane == 0) {
            if (FMT == 2) len[s] = (acc ? acc - 1 : 0) + 1;  // no trailing comma, newline
            else len[s] = acc + 1 + (uint64_t)((R - prev - 1) / 255);  // closing virtual one
        }
    }
}

// pass 2: write each shot's bytes at off[s]
template <int FMT>
__global__ void __launch_bounds__(256) sparse_write_kernel(const uint8_t* __restrict__ in, int64_t pitch,
                                                           int64_t shots, int64_t R, const uint64_t* __restrict__ off,
                                                           uint8_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nbytes = (R + 7) >> 3, nwords = (nbytes + 3) >> 2;
    for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < shots;
         s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint8_t* row = in + s * pitch;
        uint8_t* o = out + off[s];
        uint64_t pos0 = 0;       // bytes written by earlier chunks
        int64_t prev = -1;       // r8
        for (int64_t w0 = 0; w0 < nwords; w0 += 32) {
            const int64_t w = w0 + lane;
            const uint32_t v = w < nwords ? row_word(row, nbytes, w) : 0u;
            if (FMT == 2) {
                // the line is ",i1,i2,...,ik" without its first byte: write every
                // token at its virtual position minus one, dropping position 0
                uint32_t mine = 0, b = v;
                while (b) { mine += ndigits((uint32_t)(w * 32 + __ffs(b) - 1)) + 1; b &= b - 1; }
                uint32_t tot;
                const uint32_t ex = warp_excl_scan(mine, lane, tot);
                uint64_t vp = pos0 + ex;
                b = v;
                while (b) {
                    const uint32_t idx = (uint32_t)(w * 32 + __ffs(b) - 1);
                    if (vp > 0) o[vp - 1] = ',';
                    vp++;
                    const uint32_t nd = ndigits(idx);
                    uint32_t t = idx;
                    for (uint32_t k = 0; k < nd; k++) {
                        o[vp - 1 + (nd - 1 - k)] = (uint8_t)('0' + t % 10);
                        t /= 10;
                    }
                    vp += nd;
                    b &= b - 1;
                }
                pos0 += tot;
            } else {
                const int last = v ? (int)(w * 32 + 31 - __clz(v)) : -1;
                int pl = last;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(0xFFFFFFFFu, pl, d);
                    if (lane >= d) pl = max(pl, y);
                }
                int before = __shfl_up_sync(0xFFFFFFFFu, pl, 1);
                if (lane == 0) before = -1;
                int64_t p = max((int64_t)before, prev);
                uint32_t mine = 0, b = v;
                int64_t q = p;
                while (b) {
                    const int64_t pos = w * 32 + __ffs(b) - 1;
                    mine += 1 + (uint32_t)((pos - q - 1) / 255);
                    q = pos;
                    b &= b - 1;
                }
                uint32_t tot;
                const uint32_t ex = warp_excl_scan(mine, lane, tot);
                uint64_t at = pos0 + ex;
                b = v;
                q = p;
                while (b) {
                    const int64_t pos = w * 32 + __ffs(b) - 1;
                    int64_t gap = pos - q - 1;
                    while (gap >= 255) { o[at++] = 255; gap -= 255; }
                    o[at++] = (uint8_t)gap;
                    q = pos;
                    b &= b - 1;
                }
                pos0 += tot;
                prev = max(prev, (int64_t)__shfl_sync(0xFFFFFFFFu, pl, 31));
            }
        }
        if (lane == 0) {
            if (FMT == 2) {
                o[pos0 ? pos0 - 1 : 0] = '\n';
            } else {
                int64_t gap = R - prev - 1;
                uint64_t at = pos0;
                while (gap >= 255) { o[at++] = 255; gap -= 255; }
                o[at] = (uint8_t)gap;
            }
        }
    }
}

}  // namespace

// fmt: 0 = 01, 2 = hits, 3 = r8 (b8 is the input itself).  Device pointers.
// out == nullptr: only *out_len is computed.  scratch: 2 x shots uint64 +
// the scan's temporary storage, allocated here.
cudaError_t write_format(const uint8_t* in, int64_t pitch, int64_t shots, int64_t R, int fmt, uint8_t* out,
                         int64_t capacity, int64_t* out_len, cudaStream_t st) {
    *out_len = 0;
    if (shots <= 0) return cudaSuccess;
    const int grid = 148 * 8;
    if (fmt == 0) {
        *out_len = shots * (R + 1);
        if (out && capacity >= *out_len) write01_kernel<<<grid, 256, 0, st>>>(in, pitch, shots, R, out);
        return cudaGetLastError();
    }
    uint64_t* len = nullptr;
    uint64_t* off = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t e = cudaMallocAsync(&len, (size_t)(shots + 1) * 8, st);
    if (e != cudaSuccess) return e;
    e = cudaMallocAsync(&off, (size_t)(shots + 1) * 8, st);
    if (e == cudaSuccess) {
        if (fmt == 2) sparse_len_kernel<2><<<grid, 256, 0, st>>>(in, pitch, shots, R, len);
        else sparse_len_kernel<3><<<grid, 256, 0, st>>>(in, pitch, shots, R, len);
        e = cudaMemsetAsync(len + shots, 0, 8, st);
    }
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, len, off, shots + 1, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&tmp, tmp_bytes, st);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, len, off, shots + 1, st);
    uint64_t total = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&total, off + shots, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
        *out_len = (int64_t)total;
        if (out && capacity >= *out_len) {
            if (fmt == 2) sparse_write_kernel<2><<<grid, 256, 0, st>>>(in, pitch, shots, R, off, out);
            else sparse_write_kernel<3><<<grid, 256, 0, st>>>(in, pitch, shots, R, off, out);
            e = cudaGetLastError();
        }
    }
    cudaFreeAsync(tmp, st);
    cudaFreeAsync(off, st);
    cudaFreeAsync(len, st);
    return e;
}

}  // namespace pfs
