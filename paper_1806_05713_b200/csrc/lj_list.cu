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
}  // namespace
constexpr int kRowCap = 192;     // v2: scratch entries per row (longer rows -> direct second pass)
namespace {
constexpr int kRowBuf = 512;     // fallback: per-warp row buffer (entries)
constexpr int kCellBuf = 256;    // per-warp cell buffer for the in-cell sort
constexpr int kListWarps = 8;
constexpr int kMaxCand = 1344;   // v3: candidates staged per cell in shared memory (4 CTAs/SM)

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

__device__ __forceinline__ bool half_ok(int half, int i, int j) { return half ? (j > i) : (j != i); }

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
__device__ __forceinline__ double wrap_exact(double x, double L) {
    double xw = __dsub_rn(x, __dmul_rn(L, floor(__ddiv_rn(x, L))));
    if (xw >= L) xw = __dsub_rn(xw, L);
    return xw;
}

__global__ void k_cell_sort_gather(const rec4* __restrict__ q, CellGrid cg, const int64_t* __restrict__ start,
                                   int32_t* __restrict__ atoms, rec4* __restrict__ q_cell,
                                   float4* __restrict__ qf_cell) {
    const int64_t ncell = cg.ncell;
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
        for (int k = lane; k < cnt; k += 32) {
            const rec4 r = q[atoms[s + k]];
            q_cell[s + k] = r;
            qf_cell[s + k] = make_float4((float)wrap_exact(r.x, cg.L), (float)wrap_exact(r.y, cg.L),
                                         (float)wrap_exact(r.z, cg.L), 0.0f);
        }
    }
}

// ---- list ----------------------------------------------------------------

// Neighbour cell t (0..26) of cell c: start, count and the periodic shift that
// places its atoms (wrapped coordinates) next to cell c (float screen only).
__device__ __forceinline__ int neighbour_cell(int c, int t, const CellGrid& cg, const int64_t* __restrict__ start,
                                              int64_t& s, int& cnt, float& sx, float& sy, float& sz) {
    const int nc = cg.nc;
    const int cz = c % nc, cy = (c / nc) % nc, cx = c / (nc * nc);
    int x = cx + t / 9 - 1, y = cy + (t / 3) % 3 - 1, z = cz + t % 3 - 1;
    const float L = (float)cg.L;
    sx = x < 0 ? -L : (x >= nc ? L : 0.0f);
    sy = y < 0 ? -L : (y >= nc ? L : 0.0f);
    sz = z < 0 ? -L : (z >= nc ? L : 0.0f);
    x += (x < 0) ? nc : 0;
    x -= (x >= nc) ? nc : 0;
    y += (y < 0) ? nc : 0;
    y -= (y >= nc) ? nc : 0;
    z += (z < 0) ? nc : 0;
    z -= (z >= nc) ? nc : 0;
    const int cc = (x * nc + y) * nc + z;
    if (start) {
        s = start[cc];
        cnt = (int)(start[cc + 1] - s);
    }
    return cc;
}

struct ListArgs {
    const rec4* q_cell;       // positions in cell order (raw, for the exact test)
    const float4* qf_cell;    // wrapped positions in cell order, fp32 (screen only)
    const int32_t* atoms;     // cell order -> atom index
    const int64_t* start;     // cell -> first slot (ncell + 1)
    int64_t ncell;
    CellGrid cg;
    double rs2;               // rs*rs, the oracle's constant
    float rs2_screen;         // conservative fp32 screen radius^2 (> rs2 + max fp32 error)
    float r_screen;           // >= sqrt(rs2_screen): reach of a row for the half-cell type lists
    int half;
    int64_t row_begin, row_end;
    int32_t* npart;           // [rows]
    const int64_t* ptr;       // [rows+1] (direct mode)
    int32_t* out;             // scratch [rows * kRowCap] or list
    int32_t* overflow_cells;  // cells with more than kMaxCand candidates
    int32_t* n_overflow;      // [0] = #overflow cells, [1] = row overflow flag
};

// Exact accept test on raw fp64 coordinates, bit-identical to the oracle's
// (readings O2/O3): d = x_j - x_i (IEEE), minimum image d -/+ L when |d| > L/2,
// r2 = (dx*dx + dy*dy) + dz*dz without FMA, strict r2 < rs2.
// The image decision is taken on the high word of d (|d| compared with L/2 up
// to 2^-20 relative).  That cannot change an accept decision nor an accepted
// r2: since L >= 3 rs, an axis with |d| within 2^-20 of L/2 gives |d| > rs for
// either choice (reject both ways), and every other |d| is decided identically.
__device__ __forceinline__ bool image_needed(double d, int half_hi) {
    return (__double2hiint(d) & 0x7fffffff) > half_hi;
}
__device__ __forceinline__ double image_apply(double d, double L, bool need) {
    // need: d - L for d > 0, d + L (= d - (-L)) for d < 0, exactly as the oracle
    const double sL = __hiloint2double((__double2hiint(d) & (int)0x80000000) | __double2hiint(L), __double2loint(L));
    return need ? __dsub_rn(d, sL) : d;
}

// Builder v3: one CTA per cell.  The 27 neighbour cells' atoms (M candidates)
// are staged in shared memory in ascending atom-index order (sorted once per
// cell; no sort when the atoms are stored in cell order) as raw fp64
// coordinates + index.  Each of the 8 half-cells of the cell gets an ordered
// list of the candidates inside its reach box (~57 % of M); one warp per row
// then applies the oracle's exact test to 32 candidates of its half-cell's list
// at a time and compacts the accepted j by ballot straight into the row, which
// therefore comes out ascending.  No global loads in the inner loop.
template <int DIRECT, int HALF>
__global__ void __launch_bounds__(kListWarps * 32, 4) k_list_v2(ListArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* key = reinterpret_cast<unsigned long long*>(smem);   // staging keys, then type lists
    unsigned short* tl = reinterpret_cast<unsigned short*>(smem);
    double2* XY = reinterpret_cast<double2*>(smem + kMaxCand * 8);
    double* Z = reinterpret_cast<double*>(XY + (kMaxCand + 32));
    int* J = reinterpret_cast<int*>(Z + (kMaxCand + 32));
    unsigned char* TM = reinterpret_cast<unsigned char*>(J + (kMaxCand + 32));
    __shared__ int64_t s_start[27];
    __shared__ int s_off[28];
    __shared__ float s_shift[27][3];
    __shared__ int s_any;
    __shared__ unsigned short s_cnt[kMaxCand / 32 + 1][8];
    __shared__ int s_tbase[9];
    __shared__ int s_tlen[8];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const double L = a.cg.L;
    const int half_hi = L > 0.0 ? __double2hiint(0.5 * L) : 0x7fffffff;
    const long long rs2_bits = __double_as_longlong(a.rs2);
    const float wf = (float)(a.cg.L / a.cg.nc);
    const float R = a.r_screen;
    for (int64_t c = blockIdx.x; c < a.ncell; c += gridDim.x) {
        const int64_t cs = a.start[c];
        const int ccnt = (int)(a.start[c + 1] - cs);
        __syncthreads();   // smem of the previous cell no longer in use
        if (tid == 0) s_any = 0;
        if (tid < 27) {
            // slot of neighbour tid in ascending cell-id order (cell ids are distinct, nc >= 3)
            int64_t st;
            int cn;
            float sx, sy, sz;
            const int my = neighbour_cell((int)c, tid, a.cg, a.start, st, cn, sx, sy, sz);
            int rank = 0;
            for (int u = 0; u < 27; u++) {
                int64_t su;
                int cu;
                float fx, fy, fz;
                rank += neighbour_cell((int)c, u, a.cg, nullptr, su, cu, fx, fy, fz) < my;
            }
            s_start[rank] = st;
            s_off[rank + 1] = cn;
            s_shift[rank][0] = sx;
            s_shift[rank][1] = sy;
            s_shift[rank][2] = sz;
        }
        __syncthreads();
        for (int t = tid; t < ccnt; t += blockDim.x) {
            const int i = a.atoms[cs + t];
            if (i >= a.row_begin && i < a.row_end) s_any = 1;
        }
        if (tid == 0) {
            s_off[0] = 0;
            for (int t = 0; t < 27; t++) s_off[t + 1] += s_off[t];
        }
        __syncthreads();
        if (!s_any) continue;
        const int M = s_off[27];
        if (M > kMaxCand) {
            if (!DIRECT && tid == 0) {
                int k = atomicAdd(&a.n_overflow[0], 1);
                a.overflow_cells[k] = (int)c;
            }
            continue;
        }
        // stage the keys (j << 32 | staging slot)
        for (int m = tid; m < M; m += blockDim.x) {
            int lo = 0, hi = 27;   // largest t with s_off[t] <= m
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_off[mid] <= m) lo = mid; else hi = mid;
            }
            const int j = a.atoms[s_start[lo] + (m - s_off[lo])];
            key[m] = ((unsigned long long)(unsigned)j << 32) | (unsigned)m;
        }
        __syncthreads();
        // Adaptive: with atoms stored in cell order the staged keys are already
        // ascending (neighbour cells staged in ascending cell id) -> no sort.
        int unsorted = 0;
        for (int m = tid; m + 1 < M; m += blockDim.x) unsorted |= key[m] > key[m + 1];
        if (__syncthreads_or(unsorted)) {
            const int P = next_pow2(M);
            for (int m = M + tid; m < P; m += blockDim.x) key[m] = ~0ull;
            __syncthreads();
            for (int k = 2; k <= P; k <<= 1) {   // block bitonic sort of the staged keys
                for (int j = k >> 1; j > 0; j >>= 1) {
                    for (int idx = tid; idx < P; idx += blockDim.x) {
                        const int ixj = idx ^ j;
                        if (ixj > idx) {
                            const unsigned long long x = key[idx], y = key[ixj];
                            if ((x > y) == ((idx & k) == 0)) {
                                key[idx] = y;
                                key[ixj] = x;
                            }
                        }
                    }
                    __syncthreads();
                }
            }
        }
        // Candidates in sorted order: raw coordinates, index, and the set of
        // half-cell types whose reach box (wrapped fp32 frame, radius R) holds it.
        const int ncz = (int)(c % a.cg.nc), ncy = (int)((c / a.cg.nc) % a.cg.nc),
                  ncx = (int)(c / ((int64_t)a.cg.nc * a.cg.nc));
        const float midx = (ncx + 0.5f) * wf, midy = (ncy + 0.5f) * wf, midz = (ncz + 0.5f) * wf;
        const int M32 = (M + 31) & ~31;
        for (int s = tid; s < M32; s += blockDim.x) {
            if (s < M) {
                const unsigned long long k = key[s];
                const int m = (int)(k & 0xffffffffull);
                int lo = 0, hi = 27;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_off[mid] <= m) lo = mid; else hi = mid;
                }
                const int64_t g = s_start[lo] + (m - s_off[lo]);
                const rec4 r = a.q_cell[g];
                const float4 f = a.qf_cell[g];
                const float fx = f.x + s_shift[lo][0], fy = f.y + s_shift[lo][1], fz = f.z + s_shift[lo][2];
                XY[s] = make_double2(r.x, r.y);
                Z[s] = r.z;
                J[s] = (int)(k >> 32);
                const unsigned bx = (fx < midx + R ? 1u : 0u) | (fx >= midx - R ? 2u : 0u);
                const unsigned by = (fy < midy + R ? 1u : 0u) | (fy >= midy - R ? 2u : 0u);
                const unsigned bz = (fz < midz + R ? 1u : 0u) | (fz >= midz - R ? 2u : 0u);
                unsigned tm = 0;
#pragma unroll
                for (int tau = 0; tau < 8; tau++)
                    tm |= ((bx >> (tau >> 2)) & (by >> ((tau >> 1) & 1)) & (bz >> (tau & 1)) & 1u) << tau;
                TM[s] = (unsigned char)tm;
            } else {
                TM[s] = 0;
            }
        }
        if (tid == 0) {   // sentinel slot for the padded type lists: never accepted
            XY[kMaxCand] = make_double2(1e300, 1e300);
            Z[kMaxCand] = 1e300;
            J[kMaxCand] = -1;
        }
        __syncthreads();
        // per-type ordered slot lists
        const int nch = M32 >> 5;
        for (int ch = w; ch < nch; ch += kListWarps) {
            const unsigned tm = TM[ch * 32 + lane];
#pragma unroll
            for (int tau = 0; tau < 8; tau++) {
                const unsigned m = __ballot_sync(0xffffffffu, (tm >> tau) & 1u);
                if (lane == 0) s_cnt[ch][tau] = (unsigned short)__popc(m);
            }
        }
        __syncthreads();
        if (tid < 8) {   // exclusive scan of the chunk counts of type tid (in place)
            int acc = 0;
            for (int ch = 0; ch < nch; ch++) {
                const int v = s_cnt[ch][tid];
                s_cnt[ch][tid] = (unsigned short)acc;
                acc += v;
            }
            s_tbase[tid + 1] = (acc + 31) & ~31;   // padded length
            s_tlen[tid] = acc;
        }
        __syncthreads();
        if (tid == 0) {
            s_tbase[0] = 0;
            for (int tau = 0; tau < 8; tau++) s_tbase[tau + 1] += s_tbase[tau];
        }
        __syncthreads();
        const bool use_types = s_tbase[8] <= kMaxCand * 4;   // fits the reused key space (uint16)
        if (use_types) {
            for (int ch = w; ch < nch; ch += kListWarps) {
                const unsigned tm = TM[ch * 32 + lane];
#pragma unroll
                for (int tau = 0; tau < 8; tau++) {
                    const bool mem = (tm >> tau) & 1u;
                    const unsigned m = __ballot_sync(0xffffffffu, mem);
                    if (mem)
                        tl[s_tbase[tau] + s_cnt[ch][tau] + __popc(m & ((1u << lane) - 1u))] =
                            (unsigned short)(ch * 32 + lane);
                }
            }
            for (int tau = 0; tau < 8; tau++)   // pad each list with the sentinel slot
                for (int k = s_tbase[tau] + s_tlen[tau] + tid; k < s_tbase[tau + 1]; k += blockDim.x)
                    tl[k] = (unsigned short)kMaxCand;
        }
        __syncthreads();
        for (int t = w; t < ccnt; t += kListWarps) {
            const int i = a.atoms[cs + t];
            if (i < a.row_begin || i >= a.row_end) continue;
            const int64_t r = i - a.row_begin;
            const rec4 qi = a.q_cell[cs + t];
            const float4 fi = a.qf_cell[cs + t];
            int32_t* dst;
            int64_t cap;
            if (DIRECT) {
                dst = a.out + a.ptr[r];
                cap = LLONG_MAX;
            } else {
                dst = a.out + r * (int64_t)kRowCap;
                cap = kRowCap;
            }
            const int tau = ((fi.x >= midx) << 2) | ((fi.y >= midy) << 1) | (fi.z >= midz);
            const unsigned short* lst = use_types ? tl + s_tbase[tau] : nullptr;
            const int len32 = use_types ? s_tbase[tau + 1] - s_tbase[tau] : M32;
            const unsigned lt = (1u << lane) - 1u;
            int cursor = 0;
            for (int k = lane; k < len32; k += 32) {
                const int s = use_types ? (int)lst[k] : (k < M ? k : kMaxCand);
                const int j = J[s];
                const double2 xy = XY[s];
                double dx = __dsub_rn(xy.x, qi.x), dy = __dsub_rn(xy.y, qi.y), dz = __dsub_rn(Z[s], qi.z);
                const bool nx = image_needed(dx, half_hi), ny = image_needed(dy, half_hi), nz = image_needed(dz, half_hi);
                if (__any_sync(0xffffffffu, nx | ny | nz)) {   // warp-uniform: rows near a box face only
                    dx = image_apply(dx, L, nx);
                    dy = image_apply(dy, L, ny);
                    dz = image_apply(dz, L, nz);
                }
                const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                const bool acc = (HALF ? (j > i) : (j != i && j >= 0)) && __double_as_longlong(r2) < rs2_bits;
                const unsigned msk = __ballot_sync(0xffffffffu, acc);
                const int pos = cursor + __popc(msk & lt);
                if (acc && pos < cap) dst[pos] = j;
                cursor += __popc(msk);
            }
            if (lane == 0 && !DIRECT) {
                a.npart[r] = cursor;
                if (cursor > kRowCap) atomicOr(&a.n_overflow[1], 1);
            }
        }
    }
}

// Fallback for cells with more than kMaxCand candidates (dense or tiny boxes):
// one warp per row straight from global memory, per-row bitonic sort.
template <int DIRECT>
__global__ void __launch_bounds__(kListWarps * 32) k_list_fallback(ListArgs a) {
    __shared__ int rowbuf[kListWarps][kRowBuf];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double L = a.cg.L, halfL = 0.5 * a.cg.L;
    const int nover = a.n_overflow[0];
    for (int oc = blockIdx.x; oc < nover; oc += gridDim.x) {
        const int c = a.overflow_cells[oc];
        const int64_t cs = a.start[c];
        const int ccnt = (int)(a.start[c + 1] - cs);
        for (int t = w; t < ccnt; t += kListWarps) {
            const int i = a.atoms[cs + t];
            if (i < a.row_begin || i >= a.row_end) continue;
            const int64_t r = i - a.row_begin;
            const rec4 qi = a.q_cell[cs + t];
            int* buf = rowbuf[w];
            int cursor = 0;
            int32_t* gdst = DIRECT ? a.out + a.ptr[r] : nullptr;
            for (int nb = 0; nb < 27; nb++) {
                int64_t s2;
                int n2;
                float sx, sy, sz;
                neighbour_cell(c, nb, a.cg, a.start, s2, n2, sx, sy, sz);
                for (int k0 = 0; k0 < n2; k0 += 32) {
                    const int k = k0 + lane;
                    bool acc = false;
                    int j = -1;
                    if (k < n2) {
                        j = a.atoms[s2 + k];
                        acc = half_ok(a.half, i, j) && dist2_exact(qi, a.q_cell[s2 + k], L, halfL) < a.rs2;
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, acc);
                    const int pos = cursor + __popc(m & ((1u << lane) - 1u));
                    if (acc) {
                        if (pos < kRowBuf) buf[pos] = j;
                        if (DIRECT) gdst[pos] = j;
                    }
                    cursor += __popc(m);
                }
            }
            __syncwarp();
            if (cursor <= kRowBuf) {
                const int P = next_pow2(cursor > 0 ? cursor : 1);
                for (int k = cursor + lane; k < P; k += 32) buf[k] = INT_MAX;
                __syncwarp();
                warp_bitonic_sort(buf, P, lane);
                int32_t* dst = DIRECT ? gdst : a.out + r * (int64_t)kRowCap;
                const int lim = DIRECT ? cursor : min(cursor, kRowCap);
                for (int k = lane; k < lim; k += 32) dst[k] = buf[k];
            } else if (DIRECT && lane == 0) {   // very long row: insertion sort in place
                for (int x = 1; x < cursor; x++) {
                    int v = gdst[x], y = x - 1;
                    while (y >= 0 && gdst[y] > v) {
                        gdst[y + 1] = gdst[y];
                        y--;
                    }
                    gdst[y + 1] = v;
                }
            }
            __syncwarp();
            if (lane == 0 && !DIRECT) {
                a.npart[r] = cursor;
                if (cursor > kRowCap) atomicOr(&a.n_overflow[1], 1);
            }
        }
    }
}

// scratch rows (stride kRowCap) -> CSR, one warp per row
__global__ void k_compact(const int32_t* __restrict__ scratch, const int32_t* __restrict__ npart,
                          const int64_t* __restrict__ ptr, int64_t rows, int32_t* __restrict__ list) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int c = npart[r];
        const int32_t* src = scratch + r * (int64_t)kRowCap;
        int32_t* dst = list + ptr[r];
        for (int k = lane; k < c; k += 32) dst[k] = src[k];
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
    W.off_qf = o;
    o = align256(o + sizeof(float4) * (size_t)n);
    W.off_scan = o;
    o = align256(o + sizeof(int64_t) * (size_t)(W.scan_blocks + 1));
    W.off_over = o;    // [0] overflow cell count, [1] row overflow flag, then ncell cell ids
    o = align256(o + sizeof(int32_t) * (size_t)(ncell + 2));
    W.off_ptrtmp = o;  // rows + 1 int64 (padded layout: scan of the counts)
    o = align256(o + sizeof(int64_t) * (size_t)(rows + 1));
    W.off_scratch = o; // rows * kRowCap int32
    o = align256(o + sizeof(int32_t) * (size_t)rows * kRowCap);
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
    float4* qf_cell = (float4*)(ws + W.off_qf);
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
        k_cell_sort_gather<<<grid_for(cg.ncell, kListWarps), kListWarps * 32, 0, s>>>((const rec4*)q, cg, start,
                                                                                     atoms, q_cell, qf_cell);
        g_launches += 2;
    }
    return cudaGetLastError();
}

static ListArgs list_args(const CellGrid& cg, double rs, int half, int64_t row_begin, int64_t row_end, int32_t* npart,
                          const int64_t* ptr, int32_t* out, char* ws, const BuildWorkspace& W) {
    ListArgs a;
    a.q_cell = (const rec4*)(ws + W.off_qcell);
    a.qf_cell = (const float4*)(ws + W.off_qf);
    a.atoms = (const int32_t*)(ws + W.off_atoms);
    a.start = (const int64_t*)(ws + W.off_start);
    a.ncell = cg.ncell;
    a.cg = cg;
    a.rs2 = rs * rs;
    // fp32 screen: positions (|x| <= L) carry <= ~2 ulp(L) = 2.4e-7 L error per axis;
    // widen the radius by 8e-7 L + 1e-5 so every exact pair passes the screen.
    double rsc = rs + 8e-7 * cg.L + 1e-5;
    a.rs2_screen = (float)(rsc * rsc);
    a.r_screen = (float)(rsc * (1.0 + 1e-5));
    a.half = half;
    a.row_begin = row_begin;
    a.row_end = row_end;
    a.npart = npart;
    a.ptr = ptr;
    a.out = out;
    a.n_overflow = (int32_t*)(ws + W.off_over);
    a.overflow_cells = a.n_overflow + 2;
    return a;
}

static int list_grid(const CellGrid& cg, int per_sm) {
    int64_t g = 148 * per_sm;
    return (int)(cg.ncell < g ? cg.ncell : g);
}

constexpr size_t kListSmem = (size_t)kMaxCand * 8 + (size_t)(kMaxCand + 32) * (3 * 8 + 4 + 1);

cudaError_t launch_list_pass1(const CellGrid& cg, double rs, int half, int64_t row_begin, int64_t row_end,
                              int32_t* npart, int32_t* out, char* ws, const BuildWorkspace& W, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        void (*fns[4])(ListArgs) = {k_list_v2<0, 0>, k_list_v2<0, 1>, k_list_v2<1, 0>, k_list_v2<1, 1>};
        for (auto f : fns) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kListSmem);
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    ListArgs a = list_args(cg, rs, half, row_begin, row_end, npart, nullptr,
                           out ? out : (int32_t*)(ws + W.off_scratch), ws, W);
    cudaError_t e = cudaMemsetAsync(a.n_overflow, 0, 2 * sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    if (half)
        k_list_v2<0, 1><<<list_grid(cg, 4), kListWarps * 32, kListSmem, s>>>(a);
    else
        k_list_v2<0, 0><<<list_grid(cg, 4), kListWarps * 32, kListSmem, s>>>(a);
    k_list_fallback<0><<<148, kListWarps * 32, 0, s>>>(a);
    g_launches += 2;
    return cudaGetLastError();
}

const int32_t* list_row_overflow_flag(char* ws, const BuildWorkspace& W) { return (const int32_t*)(ws + W.off_over) + 1; }

cudaError_t launch_list_pass2(const CellGrid& cg, double rs, int half, int64_t row_begin, int64_t row_end,
                              int32_t* npart, const int64_t* ptr, int32_t* list, bool row_overflow, char* ws,
                              const BuildWorkspace& W, cudaStream_t s) {
    const int64_t rows = row_end - row_begin;
    if (!row_overflow) {
        k_compact<<<grid_for(rows * 32, 256, 148 * 32), 256, 0, s>>>((const int32_t*)(ws + W.off_scratch), npart, ptr,
                                                                     rows, list);
        g_launches++;
        return cudaGetLastError();
    }
    ListArgs a = list_args(cg, rs, half, row_begin, row_end, npart, ptr, list, ws, W);
    if (half)
        k_list_v2<1, 1><<<list_grid(cg, 4), kListWarps * 32, kListSmem, s>>>(a);
    else
        k_list_v2<1, 0><<<list_grid(cg, 4), kListWarps * 32, kListSmem, s>>>(a);
    k_list_fallback<1><<<148, kListWarps * 32, 0, s>>>(a);
    g_launches += 2;
    return cudaGetLastError();
}

__global__ void k_padded_pointer(int64_t* ptr, int64_t rows) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= rows; r += (int64_t)gridDim.x * blockDim.x)
        ptr[r] = r * (int64_t)kRowCap;
}

cudaError_t launch_padded_pointer(int64_t* ptr, int64_t rows, cudaStream_t s) {
    k_padded_pointer<<<grid_for(rows + 1, 256), 256, 0, s>>>(ptr, rows);
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
