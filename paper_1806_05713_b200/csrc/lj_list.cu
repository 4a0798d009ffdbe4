// Neighbour-list construction on the GPU:
//   linked-cell index -> cell-order permutation ->
//   Verlet list with search length r_s, grouped per i-atom into
//   the "sorted list" CSR of PAPER.md:214-219 (Fig. sorted_list).
//
// B200 design (not the paper's CPU linked list):
//   * cells by counting sort (histogram atomics -> exclusive scan -> scatter),
//     each cell's atoms then sorted ascending so the cell order is the stable
//     sort of the atoms by cell id (deterministic, = config 3's reorder);
//   * positions copied into cell order (q_cell) so that the candidate scan
//     reads each neighbour cell as one coalesced run of 32-B records;
//   * one CTA per cell, one warp per row: the 8 warps of a CTA scan the same 27
//     cells, so after the first warp the candidates come from L1;
//   * two passes (count -> int64 scan -> fill); the fill pass compacts accepted
//     j with a warp ballot into a per-warp shared-memory row buffer, sorts it
//     with a warp bitonic sort and writes the row once, coalesced.
//   The accept test is bit-identical to the oracle's: minimum image by the
//   same branches, r2 = (dx*dx + dy*dy) + dz*dz with explicit _rn intrinsics
//   (no FMA contraction), strict r2 < rs2 with rs2 = rs*rs computed on the host.
#include <climits>

#include "lj_internal.cuh"

namespace lj {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr int kRowBuf = 512;     // per-warp row buffer (entries); longer rows take the slow path
constexpr int kCellBuf = 256;    // per-warp cell buffer for the in-cell sort
constexpr int kListWarps = 8;

__device__ __forceinline__ double min_image(double d, double L, double halfL) {
    if (L > 0.0) {
        if (d > halfL)
            d = __dsub_rn(d, L);
        else if (d < -halfL)
            d = __dadd_rn(d, L);
    }
    return d;
}

// r^2 exactly as the oracle evaluates it (reading O3).
__device__ __forceinline__ double dist2_exact(const rec4& a, const rec4& b, double L, double halfL) {
    double dx = min_image(__dsub_rn(b.x, a.x), L, halfL);
    double dy = min_image(__dsub_rn(b.y, a.y), L, halfL);
    double dz = min_image(__dsub_rn(b.z, a.z), L, halfL);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

__device__ __forceinline__ int cell_coord(double x, const CellGrid& cg) {
    // wrap into [0,L) (reading C-3), then floor(xw * (nc/L)), clamped
    double xw = __dsub_rn(x, __dmul_rn(cg.L, floor(__ddiv_rn(x, cg.L))));
    if (xw >= cg.L) xw = __dsub_rn(xw, cg.L);
    double f = floor(__dmul_rn(xw, cg.inv_w));
    int c = (int)f;
    if (c > cg.nc - 1) c = cg.nc - 1;
    if (c < 0) c = 0;
    return c;
}

// Bitonic sort of buf[0..P) (P a power of two <= capacity) by one warp.
__device__ void warp_bitonic_sort(int* buf, int P, int lane) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int idx = lane; idx < P; idx += 32) {
                int ixj = idx ^ j;
                if (ixj > idx) {
                    int a = buf[idx], b = buf[ixj];
                    bool up = (idx & k) == 0;
                    if ((a > b) == up) {
                        buf[idx] = b;
                        buf[ixj] = a;
                    }
                }
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// ---- cells ---------------------------------------------------------------

__global__ void k_cell_assign(const rec4* __restrict__ q, int64_t n, CellGrid cg, int32_t* __restrict__ cell_of,
                              int32_t* __restrict__ count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        rec4 r = q[i];
        int cx = cell_coord(r.x, cg), cy = cell_coord(r.y, cg), cz = cell_coord(r.z, cg);
        int c = (cx * cg.nc + cy) * cg.nc + cz;
        cell_of[i] = c;
        atomicAdd(&count[c], 1);
    }
}

__global__ void k_cell_scatter(int64_t n, const int32_t* __restrict__ cell_of, const int64_t* __restrict__ start,
                               int32_t* __restrict__ cursor, int32_t* __restrict__ atoms) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int c = cell_of[i];
        int pos = atomicAdd(&cursor[c], 1);
        atoms[start[c] + pos] = (int32_t)i;
    }
}

// One warp per cell: sort the cell's atoms ascending, then gather q into cell order.
__global__ void k_cell_sort_gather(const rec4* __restrict__ q, int64_t ncell, const int64_t* __restrict__ start,
                                   int32_t* __restrict__ atoms, rec4* __restrict__ q_cell) {
    __shared__ int buf[kListWarps][kCellBuf];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t c = blockIdx.x * (int64_t)kListWarps + w; c < ncell; c += (int64_t)gridDim.x * kListWarps) {
        int64_t s = start[c];
        int cnt = (int)(start[c + 1] - s);
        if (cnt <= kCellBuf) {
            int P = next_pow2(cnt);
            for (int k = lane; k < P; k += 32) buf[w][k] = k < cnt ? atoms[s + k] : INT_MAX;
            __syncwarp();
            warp_bitonic_sort(buf[w], P, lane);
            for (int k = lane; k < cnt; k += 32) atoms[s + k] = buf[w][k];
            __syncwarp();
        } else if (lane == 0) {   // pathological cell occupancy: insertion sort in place
            for (int a = 1; a < cnt; a++) {
                int v = atoms[s + a], b = a - 1;
                while (b >= 0 && atoms[s + b] > v) {
                    atoms[s + b + 1] = atoms[s + b];
                    b--;
                }
                atoms[s + b + 1] = v;
            }
        }
        __syncwarp();
        for (int k = lane; k < cnt; k += 32) q_cell[s + k] = q[atoms[s + k]];
    }
}

// ---- list ----------------------------------------------------------------

struct Stencil {
    int64_t s[27];
    int n[27];
};

__device__ __forceinline__ void neighbour_cells(int c, const CellGrid& cg, const int64_t* __restrict__ start,
                                                int64_t* s, int* cnt) {
    int nc = cg.nc;
    int cz = c % nc, cy = (c / nc) % nc, cx = c / (nc * nc);
    int t = 0;
    for (int dx = -1; dx <= 1; dx++)
        for (int dy = -1; dy <= 1; dy++)
            for (int dz = -1; dz <= 1; dz++) {
                int x = cx + dx, y = cy + dy, z = cz + dz;
                x += (x < 0) ? nc : 0;
                x -= (x >= nc) ? nc : 0;
                y += (y < 0) ? nc : 0;
                y -= (y >= nc) ? nc : 0;
                z += (z < 0) ? nc : 0;
                z -= (z >= nc) ? nc : 0;
                int cc = (x * nc + y) * nc + z;
                s[t] = start[cc];
                cnt[t] = (int)(start[cc + 1] - s[t]);
                t++;
            }
}

template <bool FILL>
__global__ void __launch_bounds__(kListWarps * 32)
    k_list(const rec4* __restrict__ q_cell, const int32_t* __restrict__ atoms, const int64_t* __restrict__ start,
           int64_t ncell, CellGrid cg, double rs2, int half, int64_t row_begin, int64_t row_end,
           int32_t* __restrict__ npart, const int64_t* __restrict__ ptr, int32_t* __restrict__ list) {
    __shared__ int64_t s_start[27];
    __shared__ int s_cnt[27];
    __shared__ int rowbuf[FILL ? kListWarps : 1][FILL ? kRowBuf : 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double L = cg.L, halfL = 0.5 * cg.L;
    for (int64_t c = blockIdx.x; c < ncell; c += gridDim.x) {
        int64_t cs = start[c];
        int ccnt = (int)(start[c + 1] - cs);
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t s[27];
            int cn[27];
            neighbour_cells((int)c, cg, start, s, cn);
            for (int t = 0; t < 27; t++) {
                s_start[t] = s[t];
                s_cnt[t] = cn[t];
            }
        }
        __syncthreads();
        for (int t = w; t < ccnt; t += kListWarps) {
            int i = atoms[cs + t];
            if (i < row_begin || i >= row_end) continue;
            rec4 qi = q_cell[cs + t];
            int64_t r = i - row_begin;
            if (!FILL) {
                int count = 0;
                for (int nb = 0; nb < 27; nb++) {
                    int64_t s2 = s_start[nb];
                    int n2 = s_cnt[nb];
                    for (int k = lane; k < n2; k += 32) {
                        int j = atoms[s2 + k];
                        rec4 qj = q_cell[s2 + k];
                        bool ok = half ? (j > i) : (j != i);
                        if (ok && dist2_exact(qi, qj, L, halfL) < rs2) count++;
                    }
                }
                for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
                if (lane == 0) npart[r] = count;
            } else {
                int cnt = npart[r];
                int64_t base = ptr[r];
                int* buf = rowbuf[w];
                bool fits = cnt <= kRowBuf;
                int cursor = 0;
                for (int nb = 0; nb < 27; nb++) {
                    int64_t s2 = s_start[nb];
                    int n2 = s_cnt[nb];
                    for (int k0 = 0; k0 < n2; k0 += 32) {
                        int k = k0 + lane;
                        bool acc = false;
                        int j = -1;
                        if (k < n2) {
                            j = atoms[s2 + k];
                            rec4 qj = q_cell[s2 + k];
                            bool ok = half ? (j > i) : (j != i);
                            acc = ok && dist2_exact(qi, qj, L, halfL) < rs2;
                        }
                        unsigned m = __ballot_sync(0xffffffffu, acc);
                        int pos = cursor + __popc(m & ((1u << lane) - 1u));
                        if (acc) {
                            if (fits)
                                buf[pos] = j;
                            else
                                list[base + pos] = j;
                        }
                        cursor += __popc(m);
                    }
                }
                __syncwarp();
                if (fits) {
                    int P = next_pow2(cnt);
                    for (int k = cnt + lane; k < P; k += 32) buf[k] = INT_MAX;
                    __syncwarp();
                    warp_bitonic_sort(buf, P, lane);
                    for (int k = lane; k < cnt; k += 32) list[base + k] = buf[k];
                    __syncwarp();
                } else if (lane == 0) {   // very long row: insertion sort in global memory
                    for (int a = 1; a < cnt; a++) {
                        int v = list[base + a], b = a - 1;
                        while (b >= 0 && list[base + b] > v) {
                            list[base + b + 1] = list[base + b];
                            b--;
                        }
                        list[base + b + 1] = v;
                    }
                }
                __syncwarp();
            }
        }
    }
}

// ---- exclusive scan int32 -> int64 (3 phases) -------------------------------

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
    __shared__ int64_t warp_sums[32];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t s = lane < nw ? warp_sums[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        warp_sums[lane] = s;
    }
    __syncthreads();
    int64_t off = w > 0 ? warp_sums[w - 1] : 0;
    *total = warp_sums[nw - 1];
    return off + x - v;
}

__global__ void k_scan_reduce(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ block_sums) {
    int64_t base = blockIdx.x * (int64_t)kScanTile;
    int64_t s = 0;
    for (int k = 0; k < kScanItems; k++) {
        int64_t idx = base + k * kScanThreads + threadIdx.x;
        if (idx < n) s += in[idx];
    }
    int64_t tot;
    block_exclusive_scan(s, &tot);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

__global__ void k_scan_top(int64_t* block_sums, int64_t nblocks) {
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nblocks; b0 += blockDim.x) {
        int64_t b = b0 + threadIdx.x;
        int64_t v = b < nblocks ? block_sums[b] : 0;
        int64_t tot;
        int64_t ex = block_exclusive_scan(v, &tot);
        int64_t c = carry;
        __syncthreads();
        if (b < nblocks) block_sums[b] = c + ex;
        if (threadIdx.x == 0) carry = c + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) block_sums[nblocks] = carry;
}

__global__ void k_scan_down(const int32_t* __restrict__ in, int64_t n, const int64_t* __restrict__ block_sums,
                            int64_t* __restrict__ out) {
    // each thread owns kScanItems consecutive elements of the tile
    int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * (int64_t)kScanItems;
    int64_t v[kScanItems];
    int64_t s = 0;
    for (int k = 0; k < kScanItems; k++) {
        int64_t idx = base + k;
        v[k] = idx < n ? in[idx] : 0;
        s += v[k];
    }
    int64_t tot;
    int64_t ex = block_exclusive_scan(s, &tot) + block_sums[blockIdx.x];
    for (int k = 0; k < kScanItems; k++) {
        int64_t idx = base + k;
        if (idx < n) out[idx] = ex;
        ex += v[k];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = block_sums[gridDim.x];
}

__global__ void k_perm_from_atoms(const int32_t* __restrict__ atoms, int64_t n, int64_t* __restrict__ perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        perm[i] = atoms[i];
}

__global__ void k_permute(const rec4* __restrict__ in, rec4* __restrict__ out, const int64_t* __restrict__ perm,
                          int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[perm[i]];
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

BuildWorkspace build_workspace_layout(int64_t n, int64_t ncell, int64_t rows) {
    BuildWorkspace W;
    int64_t m = n > ncell ? n : ncell;
    if (rows > m) m = rows;
    W.scan_blocks = (m + 1 + kScanTile - 1) / kScanTile;
    size_t o = 0;
    W.off_cell_of = o;
    o = align256(o + sizeof(int32_t) * (size_t)n);
    W.off_count = o;   // int32 counts per cell (ncell)
    o = align256(o + sizeof(int32_t) * (size_t)(ncell + 1));
    W.off_start = o;   // int64 exclusive scan (ncell + 1)
    o = align256(o + sizeof(int64_t) * (size_t)(ncell + 1));
    W.off_cursor = o;
    o = align256(o + sizeof(int32_t) * (size_t)ncell);
    W.off_atoms = o;
    o = align256(o + sizeof(int32_t) * (size_t)n);
    W.off_qcell = o;
    o = align256(o + sizeof(rec4) * (size_t)n);
    W.off_scan = o;
    o = align256(o + sizeof(int64_t) * (size_t)(W.scan_blocks + 1));
    W.off_misc = o;
    o = align256(o + 64);
    W.total = o;
    return W;
}

cudaError_t launch_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, int64_t* block_sums,
                                   int64_t nblocks_cap, cudaStream_t s) {
    if (n == 0) return cudaMemsetAsync(out, 0, sizeof(int64_t), s);
    int64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb > nblocks_cap) return cudaErrorInvalidValue;
    k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, block_sums);
    k_scan_top<<<1, 1024, 0, s>>>(block_sums, nb);
    k_scan_down<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, block_sums, out);
    g_launches += 3;
    return cudaGetLastError();
}

cudaError_t launch_cells(const double* q, int64_t n, const CellGrid& cg, char* ws, const BuildWorkspace& W,
                         cudaStream_t s) {
    int32_t* cell_of = (int32_t*)(ws + W.off_cell_of);
    int32_t* count = (int32_t*)(ws + W.off_count);
    int64_t* start = (int64_t*)(ws + W.off_start);
    int32_t* cursor = (int32_t*)(ws + W.off_cursor);
    int32_t* atoms = (int32_t*)(ws + W.off_atoms);
    rec4* q_cell = (rec4*)(ws + W.off_qcell);
    int64_t* scan = (int64_t*)(ws + W.off_scan);
    cudaError_t e;
    if ((e = cudaMemsetAsync(count, 0, sizeof(int32_t) * (size_t)cg.ncell, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (size_t)cg.ncell, s)) != cudaSuccess) return e;
    if (n > 0) {
        k_cell_assign<<<grid_for(n, 256), 256, 0, s>>>((const rec4*)q, n, cg, cell_of, count);
        g_launches++;
    }
    if ((e = launch_scan_i32_to_i64(count, start, cg.ncell, scan, W.scan_blocks, s)) != cudaSuccess) return e;
    if (n > 0) {
        k_cell_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, cell_of, start, cursor, atoms);
        k_cell_sort_gather<<<grid_for(cg.ncell, kListWarps), kListWarps * 32, 0, s>>>((const rec4*)q, cg.ncell, start,
                                                                                     atoms, q_cell);
        g_launches += 2;
    }
    return cudaGetLastError();
}

cudaError_t launch_list_count(const double* q, int64_t n, const CellGrid& cg, double rs2, int half,
                              int64_t row_begin, int64_t row_end, int32_t* npart, char* ws,
                              const BuildWorkspace& W, cudaStream_t s) {
    (void)q;
    (void)n;
    const int32_t* atoms = (const int32_t*)(ws + W.off_atoms);
    const rec4* q_cell = (const rec4*)(ws + W.off_qcell);
    const int64_t* start = (const int64_t*)(ws + W.off_start);
    int grid = (int)(cg.ncell < 148 * 16 ? cg.ncell : 148 * 16);
    k_list<false><<<grid, kListWarps * 32, 0, s>>>(q_cell, atoms, start, cg.ncell, cg, rs2, half, row_begin, row_end,
                                                   npart, nullptr, nullptr);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_list_fill(const double* q, int64_t n, const CellGrid& cg, double rs2, int half,
                             int64_t row_begin, int64_t row_end, const int32_t* npart, const int64_t* ptr,
                             int32_t* list, char* ws, const BuildWorkspace& W, cudaStream_t s) {
    (void)q;
    (void)n;
    const int32_t* atoms = (const int32_t*)(ws + W.off_atoms);
    const rec4* q_cell = (const rec4*)(ws + W.off_qcell);
    const int64_t* start = (const int64_t*)(ws + W.off_start);
    int grid = (int)(cg.ncell < 148 * 16 ? cg.ncell : 148 * 16);
    k_list<true><<<grid, kListWarps * 32, 0, s>>>(q_cell, atoms, start, cg.ncell, cg, rs2, half, row_begin, row_end,
                                                  const_cast<int32_t*>(npart), ptr, list);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_perm_from_cells(int64_t* perm, int64_t n, char* ws, const BuildWorkspace& W, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_perm_from_atoms<<<grid_for(n, 256), 256, 0, s>>>((const int32_t*)(ws + W.off_atoms), n, perm);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_permute(const double* in, double* out, const int64_t* perm, int64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_permute<<<grid_for(n, 256), 256, 0, s>>>((const rec4*)in, (rec4*)out, perm, n);
    g_launches++;
    return cudaGetLastError();
}

}  // namespace lj
