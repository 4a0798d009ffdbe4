// Roofline microbenchmarks for the force kernel's denominators (SURVEY B-15):
//   fp64_fma:     FP64 pipe issue rate (independent DFMA chains)
//   gather_replay: the force kernel's exact access pattern with no math --
//                  G lanes per row, index load + one 32-B record gather per
//                  entry, summed into registers (achieved gather bandwidth)
//   stream_list:  sequential read of the CSR index array (HBM stream)
// Built as tools/libljmicro.so, driven by tools/microbench.py.
#include <cuda_runtime.h>
#include <stdint.h>

struct __align__(32) rec4 {
    double x, y, z, w;
};

__device__ __forceinline__ rec4 ldrec(const rec4* p) {
    rec4 r;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}

__global__ void k_fp64_fma(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
           x7 = x0 + 7;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
            x0 = fma(x0, a, b);
            x1 = fma(x1, a, b);
            x2 = fma(x2, a, b);
            x3 = fma(x3, a, b);
            x4 = fma(x4, a, b);
            x5 = fma(x5, a, b);
            x6 = fma(x6, a, b);
            x7 = fma(x7, a, b);
        }
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[0] = s;
}

template <int G>
__global__ void k_gather(const rec4* __restrict__ q, int64_t rows, const int32_t* __restrict__ npart,
                         const int64_t* __restrict__ ptr, const int32_t* __restrict__ list, double* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t r = t / G;
    int g = threadIdx.x % G;
    double s = 0;
    if (r < rows) {
        const int32_t* l = list + ptr[r];
        int n = npart[r];
        int k = g;
        for (; k + G < n; k += 2 * G) {
            int j0 = __ldg(l + k), j1 = __ldg(l + k + G);
            rec4 a = ldrec(q + j0), b = ldrec(q + j1);
            s += a.x + a.y + a.z + b.x + b.y + b.z;
        }
        if (k < n) {
            rec4 a = ldrec(q + __ldg(l + k));
            s += a.x + a.y + a.z;
        }
    }
    if (s == 12345.678) out[0] = s;
}


// G=1 rows per thread, the CTA's CSR segment staged in shared memory first
__global__ void k_gather_smem(const rec4* __restrict__ q, int64_t rows, const int32_t* __restrict__ npart,
                              const int64_t* __restrict__ ptr, const int32_t* __restrict__ list, double* out,
                              int cap) {
    extern __shared__ int sidx[];
    const int64_t r0 = blockIdx.x * (int64_t)blockDim.x;
    const int64_t r = r0 + threadIdx.x;
    const int64_t rl = min(rows, r0 + (int64_t)blockDim.x);
    const int64_t b = ptr[r0], e = ptr[rl];
    const int64_t len = e - b;
    double s = 0;
    if (len <= cap) {
        for (int64_t k = threadIdx.x; k < len; k += blockDim.x) sidx[k] = list[b + k];
        __syncthreads();
        if (r < rows) {
            const int* l = sidx + (ptr[r] - b);
            const int n = npart[r];
            int k = 0;
            for (; k + 4 <= n; k += 4) {
                int j0 = l[k], j1 = l[k + 1], j2 = l[k + 2], j3 = l[k + 3];
                rec4 a0 = ldrec(q + j0), a1 = ldrec(q + j1), a2 = ldrec(q + j2), a3 = ldrec(q + j3);
                s += a0.x + a0.y + a0.z + a1.x + a1.y + a1.z + a2.x + a2.y + a2.z + a3.x + a3.y + a3.z;
            }
            for (; k < n; k++) {
                rec4 a = ldrec(q + l[k]);
                s += a.x + a.y + a.z;
            }
        }
    }
    if (s == 12345.678) out[0] = s;
}

// G lanes per row, indices loaded 4 at a time (int4 from the 16-B aligned base)
template <int G>
__global__ void k_gather_vec(const rec4* __restrict__ q, int64_t rows, const int32_t* __restrict__ npart,
                             const int64_t* __restrict__ ptr, const int32_t* __restrict__ list, double* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t r = t / G;
    int g = threadIdx.x % G;
    double s = 0;
    if (r < rows) {
        const int64_t p0 = ptr[r];
        const int n = npart[r];
        const int64_t base = p0 & ~3ll;
        const int off = (int)(p0 - base);
        for (int c = 4 * g; c < off + n; c += 4 * G) {
            int4 v = __ldg(reinterpret_cast<const int4*>(list + base + c));
            int jj[4] = {v.x, v.y, v.z, v.w};
            rec4 a[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                int k = c + u - off;
                if (k >= 0 && k < n) a[u] = ldrec(q + jj[u]);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                int k = c + u - off;
                if (k >= 0 && k < n) s += a[u].x + a[u].y + a[u].z;
            }
        }
    }
    if (s == 12345.678) out[0] = s;
}

__global__ void k_stream(const int4* __restrict__ a, int64_t n4, int* out) {
    int acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        int4 v = __ldg(a + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678) out[0] = acc;
}

extern "C" {

int mb_fp64_fma(double* out, int blocks, int threads, int iters, void* stream) {
    k_fp64_fma<<<blocks, threads, 0, (cudaStream_t)stream>>>(out, iters, 0.999999, 1e-7);
    return (int)cudaGetLastError();
}

int mb_gather(const double* q, int64_t rows, const int32_t* npart, const int64_t* ptr, const int32_t* list,
              double* out, int G, void* stream) {
    int64_t threads = rows * G;
    unsigned grid = (unsigned)((threads + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    const rec4* qq = (const rec4*)q;
    switch (G) {
        case 1: k_gather<1><<<grid, 256, 0, s>>>(qq, rows, npart, ptr, list, out); break;
        case 2: k_gather<2><<<grid, 256, 0, s>>>(qq, rows, npart, ptr, list, out); break;
        case 4: k_gather<4><<<grid, 256, 0, s>>>(qq, rows, npart, ptr, list, out); break;
        case 8: k_gather<8><<<grid, 256, 0, s>>>(qq, rows, npart, ptr, list, out); break;
        case 16: k_gather<16><<<grid, 256, 0, s>>>(qq, rows, npart, ptr, list, out); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}

int mb_gather_smem(const double* q, int64_t rows, const int32_t* npart, const int64_t* ptr, const int32_t* list,
                   double* out, int rows_per_cta, int cap, void* stream) {
    unsigned grid = (unsigned)((rows + rows_per_cta - 1) / rows_per_cta);
    cudaFuncSetAttribute(k_gather_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, cap * 4);
    k_gather_smem<<<grid, rows_per_cta, cap * 4, (cudaStream_t)stream>>>((const rec4*)q, rows, npart, ptr, list, out,
                                                                       cap);
    return (int)cudaGetLastError();
}

int mb_gather_vec(const double* q, int64_t rows, const int32_t* npart, const int64_t* ptr, const int32_t* list,
                  double* out, int G, void* stream) {
    int64_t threads = rows * G;
    unsigned grid = (unsigned)((threads + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    const rec4* qq = (const rec4*)q;
    switch (G) {
        case 1: k_gather_vec<1><<<grid, 256, 0, s>>>(qq, rows, npart, ptr, list, out); break;
        case 2: k_gather_vec<2><<<grid, 256, 0, s>>>(qq, rows, npart, ptr, list, out); break;
        case 4: k_gather_vec<4><<<grid, 256, 0, s>>>(qq, rows, npart, ptr, list, out); break;
        case 8: k_gather_vec<8><<<grid, 256, 0, s>>>(qq, rows, npart, ptr, list, out); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}

int mb_stream(const void* a, int64_t bytes, int* out, void* stream) {
    k_stream<<<148 * 16, 256, 0, (cudaStream_t)stream>>>((const int4*)a, bytes / 16, out);
    return (int)cudaGetLastError();
}
}

// ---- B-15 (round 2): uniform random 32-B gathers and fp64 RED throughput ----------
// Random gathers: record index = hash(thread, k) mod n (integer ALU, no index
// stream), 8 independent gathers in flight per thread; bytes = 32 per gather.
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

__global__ void k_random_gather(const rec4* __restrict__ q, uint32_t n, int iters, double* out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double s = 0;
    for (int it = 0; it < iters; it++) {
        rec4 a[8];
#pragma unroll
        for (int u = 0; u < 8; u++) a[u] = ldrec(q + (hash32(t * 131u + (uint32_t)(it * 8 + u) * 0x9e3779b9u) % n));
#pragma unroll
        for (int u = 0; u < 8; u++) s += a[u].x + a[u].y + a[u].z;
    }
    if (s == 12345.678) out[0] = s;
}

// fp64 RED throughput: each thread adds to the x, y, z of random records (the half
// list's 24-B p_j read-modify-write per entry: 3 RED.E.ADD.F64), 4 records per
// iteration.
__global__ void k_random_red(double* p, uint32_t n, int iters) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t j = hash32(t * 977u + (uint32_t)(it * 4 + u) * 0x9e3779b9u) % n;
            atomicAdd(p + 4 * (size_t)j + 0, 1e-30);
            atomicAdd(p + 4 * (size_t)j + 1, 1e-30);
            atomicAdd(p + 4 * (size_t)j + 2, 1e-30);
        }
    }
}

// The half list's RED pattern on its own: for every entry of every row, 3 REDs
// to p_j (G lanes per row, as k_force), and 3 REDs to p_i per row -- no gathers,
// no arithmetic (the atomics floor of the half-list kernel).
template <int G>
__global__ void k_half_red_replay(double* p, int64_t rows, const int32_t* __restrict__ npart,
                                  const int64_t* __restrict__ ptr, const int32_t* __restrict__ list) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = t / G;
    const int g = threadIdx.x % G;
    if (r >= rows) return;
    const int32_t* l = list + ptr[r];
    const int n = npart[r];
    for (int k = g; k < n; k += G) {
        const int j = __ldg(l + k);
        atomicAdd(p + 4 * (size_t)j + 0, 1e-30);
        atomicAdd(p + 4 * (size_t)j + 1, 1e-30);
        atomicAdd(p + 4 * (size_t)j + 2, 1e-30);
    }
    if (g == 0) {
        atomicAdd(p + 4 * r + 0, 1e-30);
        atomicAdd(p + 4 * r + 1, 1e-30);
        atomicAdd(p + 4 * r + 2, 1e-30);
    }
}

extern "C" {
int mb_random_gather(const double* q, int64_t n, int blocks, int threads, int iters, double* out, void* stream) {
    k_random_gather<<<blocks, threads, 0, (cudaStream_t)stream>>>((const rec4*)q, (uint32_t)n, iters, out);
    return (int)cudaGetLastError();
}
int mb_random_red(double* p, int64_t n, int blocks, int threads, int iters, void* stream) {
    k_random_red<<<blocks, threads, 0, (cudaStream_t)stream>>>(p, (uint32_t)n, iters);
    return (int)cudaGetLastError();
}
int mb_half_red_replay(double* p, int64_t rows, const int32_t* npart, const int64_t* ptr, const int32_t* list, int G,
                       void* stream) {
    const unsigned grid = (unsigned)((rows * G + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    switch (G) {
        case 4: k_half_red_replay<4><<<grid, 256, 0, s>>>(p, rows, npart, ptr, list); break;
        case 8: k_half_red_replay<8><<<grid, 256, 0, s>>>(p, rows, npart, ptr, list); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}
}

// ---- index-stream layout probe (round 2): row-major padded list vs a warp-tiled copy ----
// Warp-tiled: for warp w (rows w*R .. w*R+R-1, R = 32/G), chunk c, unroll slot u, lane l =
// (r % R)*G + g, the index of entry e = c*U*G + u*G + g of row r sits at
// tiled[w*C*U*32 + (c*U + u)*32 + l]: each index load of a warp is one coalesced 128-B line.
template <int G, int U>
__global__ void k_tile_list(const int32_t* __restrict__ npart, const int32_t* __restrict__ list, int stride,
                            int64_t rows, int C, int32_t* __restrict__ tiled) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = t / G;
    if (r >= rows) return;
    const int g = (int)(t % G), l = (int)(t % 32);
    const int64_t w = t / 32;
    const int n = npart[r];
    for (int c = 0; c < C; c++)
        for (int u = 0; u < U; u++) {
            const int e = c * U * G + u * G + g;
            tiled[w * C * U * 32 + (c * U + u) * 32 + l] = e < n ? list[r * stride + e] : -1;
        }
}

// MODE bit 0: index loads only (no record gathers); bit 1: tiled index layout
template <int G, int U, int MODE>
__global__ void __launch_bounds__(256, 4)
    k_probe_layout(const rec4* __restrict__ q, int64_t rows, const int32_t* __restrict__ npart,
                   const int32_t* __restrict__ list, int stride, const int32_t* __restrict__ tiled, int C,
                   double* sink) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = t / G;
    const int g = threadIdx.x % G, l = threadIdx.x % 32;
    const bool active = r < rows;
    const int n = active ? npart[r] : 0;
    const int32_t* __restrict__ lst = list + (active ? r : 0) * stride;
    const int32_t* __restrict__ til = tiled + (t / 32) * (int64_t)C * U * 32 + l;
    double s = 0.0;
    int acc = 0;
    int jn[U];
#pragma unroll
    for (int u = 0; u < U; u++)
        jn[u] = (g + u * G < n) ? ((MODE & 2) ? __ldg(til + u * 32) : __ldg(lst + g + u * G)) : -1;
    int c = 0;
    for (int k0 = g; __any_sync(0xffffffffu, k0 < n); k0 += U * G, c++) {
        int j[U];
#pragma unroll
        for (int u = 0; u < U; u++) j[u] = jn[u];
        rec4 qj[U];
        if (!(MODE & 1)) {
#pragma unroll
            for (int u = 0; u < U; u++) qj[u] = ldrec(q + (j[u] >= 0 ? j[u] : 0));
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int kn = k0 + U * G + u * G;
            jn[u] = kn < n ? ((MODE & 2) ? __ldg(til + ((c + 1) * U + u) * 32) : __ldg(lst + kn)) : -1;
        }
        if (!(MODE & 1)) {
#pragma unroll
            for (int u = 0; u < U; u++) s += j[u] >= 0 ? qj[u].x + qj[u].y + qj[u].z : 0.0;
        } else {
#pragma unroll
            for (int u = 0; u < U; u++) acc += j[u];
        }
    }
    if (s == 1.2345678e300 || acc == 0x7fffffff) sink[0] = s + acc;   // never true: keeps the loads alive
}

extern "C" {
int mb_tile_list(const int32_t* npart, const int32_t* list, int stride, int64_t rows, int C, int32_t* tiled, int G,
                 int U, void* stream) {
    const unsigned grid = (unsigned)((rows * G + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
#define TL(g, u) \
    if (G == g && U == u) { k_tile_list<g, u><<<grid, 256, 0, s>>>(npart, list, stride, rows, C, tiled); return (int)cudaGetLastError(); }
    TL(4, 3) TL(4, 2) TL(8, 2) TL(8, 3) TL(16, 2)
#undef TL
    return -1;
}

int mb_probe_layout(const double* q, int64_t rows, const int32_t* npart, const int32_t* list, int stride,
                    const int32_t* tiled, int C, double* sink, int G, int U, int mode, void* stream) {
    const unsigned grid = (unsigned)((rows * G + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    const rec4* qq = (const rec4*)q;
#define PL(g, u, m) \
    if (G == g && U == u && mode == m) { k_probe_layout<g, u, m><<<grid, 256, 0, s>>>(qq, rows, npart, list, stride, tiled, C, sink); return (int)cudaGetLastError(); }
#define PL4(g, u) PL(g, u, 0) PL(g, u, 1) PL(g, u, 2) PL(g, u, 3)
    PL4(4, 3) PL4(4, 2) PL4(8, 2) PL4(8, 3) PL4(16, 2)
#undef PL4
#undef PL
    return -1;
}
}
