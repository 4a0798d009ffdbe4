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
#include <cmath>

#include "lj_internal.cuh"

namespace lj {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
}  // namespace
constexpr int kRowCap = LJ_PADDED_ROW_STRIDE;   // scratch / padded entries per row (longer rows -> direct pass)
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

// Also raises flags[0] if some raw coordinate lies outside [0, L): the fast
// list kernel (k_list_v4) needs wrapped input, the exact kernel handles the rest.
__global__ void k_cell_assign(const rec4* __restrict__ q, int64_t n, CellGrid cg, int32_t* __restrict__ cell_of,
                              int32_t* __restrict__ count, int32_t* __restrict__ flags) {
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        bool outside = false;
        if (i < n) {
            rec4 r = q[i];
            int cx = cell_coord(r.x, cg), cy = cell_coord(r.y, cg), cz = cell_coord(r.z, cg);
            int c = (cx * cg.nc + cy) * cg.nc + cz;
            cell_of[i] = c;
            atomicAdd(&count[c], 1);
            outside = !(r.x >= 0.0 && r.x < cg.L && r.y >= 0.0 && r.y < cg.L && r.z >= 0.0 && r.z < cg.L);
        }
        if (__any_sync(0xffffffffu, outside) && (threadIdx.x & 31) == 0) atomicOr(&flags[0], 1);
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
                                   float4* __restrict__ qf_cell, float4* __restrict__ qr_cell, double cw) {
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
        const int cz = (int)(c % cg.nc), cy = (int)((c / cg.nc) % cg.nc), cx = (int)(c / ((int64_t)cg.nc * cg.nc));
        const double ox = cx * cw, oy = cy * cw, oz = cz * cw;
        for (int k = lane; k < cnt; k += 32) {
            const int i = atoms[s + k];
            const rec4 r = q[i];
            q_cell[s + k] = r;
            qf_cell[s + k] = make_float4((float)wrap_exact(r.x, cg.L), (float)wrap_exact(r.y, cg.L),
                                         (float)wrap_exact(r.z, cg.L), 0.0f);
            // fp32 coordinates relative to the cell's corner + atom index (k_list_v4 staging)
            qr_cell[s + k] = make_float4((float)(r.x - ox), (float)(r.y - oy), (float)(r.z - oz), __int_as_float(i));
        }
    }
}

// ---- fused rebuild (lj_rebuild): wrap + cells + cell-order permutation -------

// Wrap q into [0, L) in place (reading C-3, as lj_wrap) and assign cells.
__global__ void k_wrap_assign(rec4* __restrict__ q, int64_t n, CellGrid cg, int32_t* __restrict__ cell_of,
                              int32_t* __restrict__ count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        rec4 r = q[i];
        r.x = wrap_exact(r.x, cg.L);
        r.y = wrap_exact(r.y, cg.L);
        r.z = wrap_exact(r.z, cg.L);
        q[i] = r;
        const int cx = cell_coord(r.x, cg), cy = cell_coord(r.y, cg), cz = cell_coord(r.z, cg);
        const int c = (cx * cg.nc + cy) * cg.nc + cz;
        cell_of[i] = c;
        atomicAdd(&count[c], 1);
    }
}

// One warp per cell: sort the cell's atoms ascending (= lj_cell_order's stable
// sort by cell id), then emit the permutation and the permuted records
// (q_out, p_out, q_ref) and the builder's staging arrays for the NEW storage
// order (atoms = identity, q_cell = q_out, qr_cell), so the list kernels run
// on the permuted system without a second cell pass.
__global__ void k_cell_sort_permute(const rec4* __restrict__ q, const rec4* __restrict__ p, CellGrid cg,
                                    const int64_t* __restrict__ start, int32_t* __restrict__ atoms,
                                    int64_t* __restrict__ perm, rec4* __restrict__ q_out, rec4* __restrict__ p_out,
                                    rec4* __restrict__ q_ref, rec4* __restrict__ q_cell,
                                    float4* __restrict__ qr_cell, double cw, PeerMomenta pm) {
    const int64_t ncell = cg.ncell;
    __shared__ int buf[kListWarps][kCellBuf];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t c = blockIdx.x * (int64_t)kListWarps + w; c < ncell; c += (int64_t)gridDim.x * kListWarps) {
        const int64_t s = start[c];
        const int cnt = (int)(start[c + 1] - s);
        if (cnt <= kCellBuf) {
            const int P = next_pow2(cnt);
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
        const int cz = (int)(c % cg.nc), cy = (int)((c / cg.nc) % cg.nc), cx = (int)(c / ((int64_t)cg.nc * cg.nc));
        const double ox = cx * cw, oy = cy * cw, oz = cz * cw;
        for (int k = lane; k < cnt; k += 32) {
            const int64_t g = s + k;
            const int i = atoms[g];
            const rec4 r = q[i];
            perm[g] = i;
            q_out[g] = r;
            q_cell[g] = r;
            if (q_ref) q_ref[g] = r;
            if (pm.table) {   // own new rows only: the momenta from the rank that owned atom i
                if (g >= pm.own_lo && g < pm.own_hi)
                    p_out[g] = reinterpret_cast<const rec4*>(pm.table[i / pm.n_own])[i];   // (coherent load: peer memory)
            } else if (p) {
                p_out[g] = p[i];
            }
            qr_cell[g] = make_float4((float)(r.x - ox), (float)(r.y - oy), (float)(r.z - oz), __int_as_float((int)g));
        }
        __syncwarp();
        for (int k = lane; k < cnt; k += 32) atoms[s + k] = (int32_t)(s + k);   // new order: identity
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
    const float4* qr_cell;    // fp32 coordinates relative to the own cell's corner + atom index (v4)
    const int32_t* atoms;     // cell order -> atom index
    const int64_t* start;     // cell -> first slot (ncell + 1)
    int64_t ncell;
    CellGrid cg;
    double rs2;               // rs*rs, the oracle's constant
    float r_screen;           // reach of a row for the v3 half-cell type lists (> rs + max fp32 error)
    int half;
    int64_t row_begin, row_end;
    int32_t* npart;           // [rows]
    const int64_t* ptr;       // [rows+1] (direct mode)
    int32_t* out;             // scratch [rows * kRowCap] or list
    int32_t* overflow_cells;  // cells the first pass could not stage (-> the LARGE pass)
    int32_t* overflow_cells2; // cells the LARGE pass could not stage either, and the exact kernel's (-> fallback)
    int32_t* n_overflow;      // [0] = #overflow_cells, [1] = row overflow flag, [2] = #overflow_cells2
    int clamp;                // out is the caller's padded list: a row over kRowCap stores
                              // min(count, kRowCap) in npart (consumers stay in bounds until
                              // the overflow flag is seen); scratch mode keeps the true count
    // v4 (fast path, wrapped input only)
    const rec4* q;            // raw input positions (atom order): the exact band test
    const int32_t* flags;     // [0] != 0: some coordinate outside [0, L) -> exact kernel instead
    double w;                 // cell width L / nc
    float lo2, hi2;           // fp32 decision band around rs2: r2f < lo2 accept, r2f >= hi2 reject
    float rb2;                // squared reach of a half-cell box (rounded-box candidate screen)
    const struct CellSetup* setups;   // per-cell neighbour runs (k_cell_setup), v4 only
    int il_skip;              // kIlSkip: out is an interleaved padded list (LJ_LIST_INTERLEAVED), else 0
};

// Row rr of the non-direct output (the per-row scratch or the caller's padded list):
// stride kRowCap, or the interleaved layout (entry e of the row at il_off(e, il_skip)).
__device__ __forceinline__ int32_t* padded_row(int32_t* out, int64_t rr, int il_skip) {
    return out + (il_skip ? (rr >> 3) * (int64_t)(kIlRows * kRowCap) + (rr & (kIlRows - 1)) * kIlGran
                          : rr * (int64_t)kRowCap);
}
static_assert(kRowCap % kIlGran == 0, "interleaved rows need a stride made of whole granules");

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
    if (!a.flags[0]) return;   // wrapped input: k_list_v4 builds the list
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
            if (!DIRECT && tid == 0) {   // (the LARGE v4 pass does not run on unwrapped input)
                int k = atomicAdd(&a.n_overflow[2], 1);
                a.overflow_cells2[k] = (int)c;
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
                dst = padded_row(a.out, r, a.il_skip);
                cap = kRowCap;
            }
            const int skip = DIRECT ? 0 : a.il_skip;
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
                if (acc && pos < cap) dst[il_off(pos, skip)] = j;
                cursor += __popc(msk);
            }
            if (lane == 0 && !DIRECT) {
                a.npart[r] = (a.clamp && cursor > kRowCap) ? kRowCap : cursor;
                if (cursor > kRowCap) atomicOr(&a.n_overflow[1], 1);
            }
        }
    }
}

// Builder v4 (fast path; every raw coordinate in [0, L), i.e. wrapped input as
// the MD driver and the generators provide -- else k_list_v2 runs instead).
//
// Same cell/stencil decomposition as v3, but:
//  * candidates are staged as fp32 coordinates relative to the cell's corner:
//    u = (x - own corner) [precomputed per atom by k_cell_sort_gather] + the
//    neighbour cell's offset (-w, 0 or w per axis), plus the atom index;
//  * a half-cell's candidate list holds the candidates within the squared reach
//    rb2 of the half-cell BOX (rounded-box screen: ~382 of ~1000 candidates
//    at rho = 1, r_s = 3.3, instead of the ~570 of the v3 reach cube); warp tau
//    builds the list of type tau in one ordered pass (ballot compaction);
//  * loops swapped: a work item is (half-cell type, <= kItemRows rows of that
//    type); the rows live in registers, each lane holds two candidates of a
//    64-chunk of the type's list, and every row is tested against the chunk
//    with ballot compaction.  Warps take items dynamically (load balance);
//  * the accept decision is taken in fp32 wherever it is unambiguous: with
//    r2f the fp32 squared displacement, r2f < lo2 accepts and r2f >= hi2
//    rejects, where [lo2, hi2) brackets rs2 by more than the worst-case
//    difference between r2f and the oracle's fp64 r2 (bound in list_args()).
//    Pairs inside the band (~2e-3 per row) take the oracle's exact fp64 test
//    on the raw coordinates, so the pair SET is bit-identical to the oracle's.
// Rows come out ascending: candidates are staged in ascending atom order and a
// row's chunks are visited in order by the one warp that owns the row.
constexpr int kMaxRows = 256;   // atoms per cell handled by v4 (more -> overflow fallback)
constexpr int kItemRows = 8;    // rows per work item (8: one item per half-cell nearly always -- 8-9 items per cell, one per warp)
constexpr int kMaxItems = kMaxRows / kItemRows + 8;
constexpr int kRankPathMaxOverlaps = 40;   // overlapping neighbour-run pairs (of 351) up to which the
                                           // unsorted staging ranks atoms instead of sorting keys

__device__ __forceinline__ unsigned long long pack_f32x2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

// r2 = (dx*dx + dy*dy) + dz*dz as fmaf(dz, dz, fmaf(dy, dy, dx * dx)) for two
// candidates at once (sm_100 packed fp32x2: FADD2 / FMUL2 / FFMA2).
__device__ __forceinline__ void dist2_f32x2(unsigned long long cx, unsigned long long cy, unsigned long long cz,
                                            const float4& ri, float& r2a, float& r2b) {
    const unsigned long long rx = pack_f32x2(ri.x, ri.x), ry = pack_f32x2(ri.y, ri.y), rz = pack_f32x2(ri.z, ri.z);
    unsigned long long dx, dy, dz, r2;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(cx), "l"(rx));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(cy), "l"(ry));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dz) : "l"(cz), "l"(rz));
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(r2) : "l"(dx));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r2) : "l"(dy), "l"(r2));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r2) : "l"(dz), "l"(r2));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r2a), "=f"(r2b) : "l"(r2));
}

// Rank, in ascending wrapped coordinate, of the neighbour at offset d in {-1,0,1}
// of cell coordinate v (nc >= 3, so the three wrapped values are distinct).
__device__ __forceinline__ int axis_rank(int v, int d, int nc) {
    if (v == 0) return d == 0 ? 0 : (d == 1 ? 1 : 2);        // values 0, 1, nc-1
    if (v == nc - 1) return d == 1 ? 0 : (d == -1 ? 1 : 2);  // values 0, nc-2, nc-1
    return d + 1;
}

// bit tau set <=> the candidate lies within sqrt(rb2) of half-cell box tau
// (tau = 4 bx + 2 by + bz, b = 0: [0, w/2), b = 1: [w/2, w) along the axis)
__device__ __forceinline__ unsigned type_mask(const float4& f, float hw, float fw, float rb2) {
    const float xl = fmaxf(fmaxf(-f.x, f.x - hw), 0.f), xu = fmaxf(fmaxf(hw - f.x, f.x - fw), 0.f);
    const float yl = fmaxf(fmaxf(-f.y, f.y - hw), 0.f), yu = fmaxf(fmaxf(hw - f.y, f.y - fw), 0.f);
    const float zl = fmaxf(fmaxf(-f.z, f.z - hw), 0.f), zu = fmaxf(fmaxf(hw - f.z, f.z - fw), 0.f);
    const float ex[2] = {xl * xl, xu * xu}, ey[2] = {yl * yl, yu * yu}, ez[2] = {zl * zl, zu * zu};
    unsigned tm = 0;
#pragma unroll
    for (int tau = 0; tau < 8; tau++) tm |= ((ex[tau >> 2] + ey[(tau >> 1) & 1] + ez[tau & 1]) < rb2 ? 1u : 0u) << tau;
    return tm;
}

// The 27 neighbour runs of a cell in ascending cell id (= rank order): start,
// count (as offsets), periodic offset, first / last atom index; whether the
// storage is in cell order there; whether the cell holds own rows.  Computed for
// every cell up front by k_cell_setup (one warp per cell, no barriers), and
// copied into k_list_v4's shared memory with cp.async while the previous cell's
// work items run -- so no warp of the builder waits for a serial setup warp.
struct __align__(16) CellSetup {
    int64_t start[27];
    int off[28];
    int first[27], last[27];
    int any, unsorted;
    signed char dc[27][3];   // neighbour cell offset (-1, 0, 1) per axis
    signed char pad_[16 - (27 * 3) % 16];
};
static_assert(sizeof(CellSetup) % 16 == 0, "CellSetup is copied in 16-byte pieces");

__device__ __forceinline__ void setup_cell(const ListArgs& a, int64_t c, CellSetup& S, int lane) {
    const int nc = a.cg.nc;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t cs = a.start[c];
    const int ccnt = (int)(a.start[c + 1] - cs);
    const int ncz = (int)(c % nc), ncy = (int)((c / nc) % nc), ncx = (int)(c / ((int64_t)nc * nc));
    int cnt = 0, rank = 31, first = 0, last = 0;
    if (lane < 27) {
        const int dx = lane / 9 - 1, dy = (lane / 3) % 3 - 1, dz = lane % 3 - 1;
        int x = ncx + dx, y = ncy + dy, z = ncz + dz;
        x += x < 0 ? nc : (x >= nc ? -nc : 0);
        y += y < 0 ? nc : (y >= nc ? -nc : 0);
        z += z < 0 ? nc : (z >= nc ? -nc : 0);
        const int64_t cc = ((int64_t)x * nc + y) * nc + z;
        const int64_t st = a.start[cc];
        cnt = (int)(a.start[cc + 1] - st);
        rank = axis_rank(ncx, dx, nc) * 9 + axis_rank(ncy, dy, nc) * 3 + axis_rank(ncz, dz, nc);
        S.start[rank] = st;
        S.dc[rank][0] = (signed char)dx;
        S.dc[rank][1] = (signed char)dy;
        S.dc[rank][2] = (signed char)dz;
        if (cnt > 0) {
            first = a.atoms[st];
            last = a.atoms[st + cnt - 1];
        }
    }
    bool mine = false;   // does this cell hold rows of [row_begin, row_end)?
    for (int t = lane; t < ccnt; t += 32) {
        const int i = a.atoms[cs + t];
        mine |= i >= a.row_begin && i < a.row_end;
    }
    // in rank order: lane r handles the neighbour of rank r (lane `src` computed it)
    int src = 0;
#pragma unroll
    for (int l = 0; l < 27; l++) src = (__shfl_sync(0xffffffffu, rank, l) == lane) ? l : src;
    const int mycnt_r = __shfl_sync(0xffffffffu, cnt, src);
    const int mycnt = lane < 27 ? mycnt_r : 0;
    int incl = mycnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int rf = __shfl_sync(0xffffffffu, first, src);
    const int rl = __shfl_sync(0xffffffffu, last, src);
    if (lane < 27) S.off[lane + 1] = incl;
    if (lane == 0) S.off[0] = 0;
    // candidates already ascending (atoms stored in cell order)?  Each cell's atoms
    // are ascending (k_cell_sort_gather), so only run boundaries can break the order.
    const unsigned ne = __ballot_sync(0xffffffffu, mycnt > 0);
    const unsigned before = ne & lt;
    const int prev = before ? 31 - __clz(before) : 0;
    const int prev_last = __shfl_sync(0xffffffffu, rl, prev);
    const unsigned bad = __ballot_sync(0xffffffffu, mycnt > 0 && before != 0 && prev_last > rf);
    const unsigned any = __ballot_sync(0xffffffffu, mine);
    // how far from sorted: pairs of runs whose index intervals overlap (storage that has
    // drifted from cell order since the last sort: a few migrants per cell, few overlaps;
    // shuffled storage: nearly all 351 pairs overlap)
    int ovl = 0;
    if (bad) {
        for (int u = 0; u < 27; u++) {
            const int fu = __shfl_sync(0xffffffffu, rf, u), lu = __shfl_sync(0xffffffffu, rl, u);
            const int cu = __shfl_sync(0xffffffffu, mycnt, u);
            ovl += (lane < 27 && u > lane && mycnt > 0 && cu > 0 && !(lu < rf || fu > rl)) ? 1 : 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ovl += __shfl_xor_sync(0xffffffffu, ovl, o);
    }
    if (lane < 27) {
        S.first[lane] = mycnt > 0 ? rf : INT_MAX;
        S.last[lane] = mycnt > 0 ? rl : INT_MIN;
    }
    if (lane == 0) {
        S.unsorted = bad == 0 ? 0 : (ovl <= kRankPathMaxOverlaps ? 1 : 2);
        S.any = any != 0;
    }
}

__global__ void __launch_bounds__(256) k_cell_setup(ListArgs a, CellSetup* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < a.ncell;
         c += ((int64_t)gridDim.x * blockDim.x) >> 5)
        setup_cell(a, c, out[c], lane);
}

// 16-byte asynchronous copy global -> shared (LDGSTS): lands without registers.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// MAXC: candidates staged per cell (MAXC = 1344 for 4 CTAs/SM; the LARGE instantiation,
// MAXCLarge, takes the cells the first pass could not stage -- small or dense boxes, e.g.
// config 1's 1,687 candidates per cell -- from its overflow list; what it cannot stage either
// goes to k_list_fallback).
template <int DIRECT, int HALF, int MAXC, bool LARGE>
__global__ void __launch_bounds__(kListWarps * 32, LARGE ? 2 : 4) k_list_v4(ListArgs a) {
    if (a.flags[0]) return;   // unwrapped input: the exact kernel (k_list_v2) builds the list
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned short* tl = reinterpret_cast<unsigned short*>(smem);            // [8][MAXC + 64] slot lists
    unsigned long long* key = reinterpret_cast<unsigned long long*>(smem);   // (aliased) unsorted staging only
    // staged candidates, structure of arrays (x, y, z, atom index) so that the two
    // candidates a lane tests load straight into an fp32x2 register pair;
    // slot MAXC is the sentinel
    constexpr int kCS = MAXC + 32;
    float* CX = reinterpret_cast<float*>(smem + 8 * (MAXC + 64) * 2);
    float* CY = CX + kCS;
    float* CZ = CY + kCS;
    int* CJ = reinterpret_cast<int*>(CZ + kCS);
    unsigned char* TM = reinterpret_cast<unsigned char*>(CJ + kCS);
    __shared__ CellSetup s_set;   // this cell's neighbour runs (k_cell_setup), prefetched by cp.async
    __shared__ int s_next;
    __shared__ int s_tlen[8];
    __shared__ float4 s_row[kMaxRows];
    __shared__ unsigned char s_rtau[kMaxRows], s_rk[kMaxRows], s_rowlist[kMaxRows];
    __shared__ int s_rcnt[8];
    __shared__ int s_item[kMaxItems];
    __shared__ int s_nitems;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int nc = a.cg.nc;
    const double L = a.cg.L, halfL = 0.5 * a.cg.L;
    const float hw = (float)(0.5 * a.w), fw = (float)a.w;
    const unsigned lt = (1u << lane) - 1u;
    constexpr int kTL = MAXC + 64;   // per-type list capacity
    constexpr int kSetupChunks = (int)(sizeof(CellSetup) / 16);
    static_assert(kSetupChunks <= kListWarps * 32, "one 16-byte chunk per thread");
    // the cells this kernel visits: all (first pass) or the first pass's overflow list (LARGE)
    const int64_t n_visit = LARGE ? (int64_t)a.n_overflow[0] : a.ncell;
    auto cell_at = [&](int64_t k) -> int64_t { return LARGE ? (int64_t)a.overflow_cells[k] : k; };
    auto prefetch = [&](int64_t k) {   // the setup of the k-th visited cell into s_set (cp.async)
        if (k < n_visit && tid < kSetupChunks)
            cp_async16(reinterpret_cast<char*>(&s_set) + 16 * tid,
                       reinterpret_cast<const char*>(a.setups + cell_at(k)) + 16 * tid);
    };
    prefetch(blockIdx.x);
    if (tid < 8) s_rcnt[tid] = 0;   // (reset again during every cell's work items, where it is unused)
    for (int64_t kv = blockIdx.x; kv < n_visit; kv += gridDim.x) {
        const int64_t c = cell_at(kv);
        const int64_t cs = a.start[c];
        const int ccnt = (int)(a.start[c + 1] - cs);
        cp_async_wait_all();   // this cell's setup (issued during the previous cell's work items)
        __syncthreads();   // smem of the previous cell no longer in use; this cell's setup visible
        if (tid == 0) s_next = 0;   // (after the barrier: the previous cell's items are all taken)
#define s_start s_set.start
#define s_off s_set.off
#define s_dc s_set.dc
#define s_first s_set.first
#define s_last s_set.last
#define s_unsorted s_set.unsorted
        if (!s_set.any) {
            __syncthreads();   // everyone has read s_set before it is overwritten
            prefetch(kv + gridDim.x);
            continue;
        }
        const int M = s_off[27];
        if (M > MAXC || ccnt > kMaxRows) {
            if (!DIRECT && tid == 0) {   // first pass: to the LARGE pass; LARGE: to the fallback
                const int k = atomicAdd(&a.n_overflow[LARGE ? 2 : 0], 1);
                (LARGE ? a.overflow_cells2 : a.overflow_cells)[k] = (int)c;
            }
            __syncthreads();   // everyone has read s_set before it is overwritten
            prefetch(kv + gridDim.x);
            continue;
        }
        const int M32 = (M + 31) & ~31;
        if (!s_unsorted) {
            // staging by runs: candidate k of run t is slot s_off[t] + k
            for (int t = w; t < 27; t += kListWarps) {
                const int n = s_off[t + 1] - s_off[t];
                const float sx = s_dc[t][0] * fw, sy = s_dc[t][1] * fw, sz = s_dc[t][2] * fw;
                const float4* src = a.qr_cell + s_start[t];
                for (int k = lane; k < n; k += 32) {
                    float4 f = src[k];
                    f.x += sx;
                    f.y += sy;
                    f.z += sz;
                    const int m = s_off[t] + k;
                    CX[m] = f.x;
                    CY[m] = f.y;
                    CZ[m] = f.z;
                    CJ[m] = __float_as_int(f.w);
                    TM[m] = (unsigned char)type_mask(f, hw, fw, a.rb2);
                }
            }
        } else if (s_unsorted == 1) {
            // nearly sorted storage: every run is ascending (cells sorted by k_cell_sort_gather),
            // so an atom's slot in the ascending staging order is its position in its own run +
            // the atoms of the other runs below it -- whole runs by their [first, last] interval,
            // a binary search only for the few runs whose interval straddles it.  No sort, no
            // barrier; the staged order is the same as the sorted one.
            for (int t = w; t < 27; t += kListWarps) {
                const int n = s_off[t + 1] - s_off[t];
                const float sx = s_dc[t][0] * fw, sy = s_dc[t][1] * fw, sz = s_dc[t][2] * fw;
                const float4* src = a.qr_cell + s_start[t];
                for (int k = lane; k < n; k += 32) {
                    float4 f = src[k];
                    const int x = __float_as_int(f.w);
                    int m = k;
                    for (int u = 0; u < 27; u++) {
                        if (u == t || x < s_first[u]) continue;
                        const int nu = s_off[u + 1] - s_off[u];
                        if (x > s_last[u]) {
                            m += nu;
                        } else {   // x inside run u's interval: count its atoms below x
                            const int32_t* ru = a.atoms + s_start[u];
                            int lo = 0, hi = nu;
                            while (lo < hi) {
                                const int mid = (lo + hi) >> 1;
                                if (ru[mid] < x) lo = mid + 1; else hi = mid;
                            }
                            m += lo;
                        }
                    }
                    f.x += sx;
                    f.y += sy;
                    f.z += sz;
                    CX[m] = f.x;
                    CY[m] = f.y;
                    CZ[m] = f.z;
                    CJ[m] = x;
                    TM[m] = (unsigned char)type_mask(f, hw, fw, a.rb2);
                }
            }
        } else {
            // general storage order: sort the staged keys (atom id, staging slot) first
            for (int t = w; t < 27; t += kListWarps) {
                const int n = s_off[t + 1] - s_off[t];
                for (int k = lane; k < n; k += 32) {
                    const int m = s_off[t] + k;
                    key[m] = ((unsigned long long)(unsigned)a.atoms[s_start[t] + k] << 32) | (unsigned)m;
                }
            }
            const int P = next_pow2(M);
            for (int m = M + tid; m < P; m += blockDim.x) key[m] = ~0ull;
            __syncthreads();
            for (int k = 2; k <= P; k <<= 1) {
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
            for (int s = tid; s < M; s += blockDim.x) {
                const int m = (int)(key[s] & 0xffffffffull);
                int lo = 0, hi = 27;   // largest t with s_off[t] <= m
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_off[mid] <= m) lo = mid; else hi = mid;
                }
                float4 f = a.qr_cell[s_start[lo] + (m - s_off[lo])];
                f.x += s_dc[lo][0] * fw;
                f.y += s_dc[lo][1] * fw;
                f.z += s_dc[lo][2] * fw;
                CX[s] = f.x;
                CY[s] = f.y;
                CZ[s] = f.z;
                CJ[s] = __float_as_int(f.w);
                TM[s] = (unsigned char)type_mask(f, hw, fw, a.rb2);
            }
        }
        for (int s = M + tid; s < M32; s += blockDim.x) TM[s] = 0;
        if (tid == 0) {   // sentinel
            CX[MAXC] = CY[MAXC] = CZ[MAXC] = 1e30f;
            CJ[MAXC] = -1;
        }
        // rows of this cell and their half-cell types
        for (int t = tid; t < ccnt; t += blockDim.x) {
            const float4 f = a.qr_cell[cs + t];
            const int i = __float_as_int(f.w);
            unsigned char tau = 255;
            if (i >= a.row_begin && i < a.row_end) {
                s_row[t] = f;
                tau = (unsigned char)(((f.x >= hw) << 2) | ((f.y >= hw) << 1) | (f.z >= hw));
                s_rk[t] = (unsigned char)atomicAdd(&s_rcnt[tau], 1);
            }
            s_rtau[t] = tau;
        }
        __syncthreads();
        {   // warp w: the ordered slot list of type w, the rows of type w and its work items
            const int tau = w;
            unsigned short* lst = tl + tau * kTL;
            int n = 0;
            for (int ch = 0; ch < M32; ch += 32) {
                const bool mem = (TM[ch + lane] >> tau) & 1u;
                const unsigned m = __ballot_sync(0xffffffffu, mem);
                if (mem) lst[n + __popc(m & lt)] = (unsigned short)(ch + lane);
                n += __popc(m);
            }
            const int padded = (n + 63) & ~63;
            for (int k = n + lane; k < padded; k += 32) lst[k] = (unsigned short)MAXC;
            if (lane == 0) s_tlen[tau] = padded;
            int rbase = 0, ibase = 0;
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int cu = s_rcnt[u];
                if (u < tau) {
                    rbase += cu;
                    ibase += (cu + kItemRows - 1) / kItemRows;
                }
            }
            for (int t = lane; t < ccnt; t += 32)
                if (s_rtau[t] == tau) s_rowlist[rbase + s_rk[t]] = (unsigned char)t;
            const int nr = s_rcnt[tau];
            const int k = (nr + kItemRows - 1) / kItemRows;   // items of this type, sizes as equal as possible
            if (lane < k) {
                const int len = nr / k + (lane < nr % k ? 1 : 0);
                const int u0 = lane * (nr / k) + min(lane, nr % k);
                s_item[ibase + lane] = tau | ((rbase + u0) << 8) | (len << 16);
            }
            if (tau == 7 && lane == 0) s_nitems = ibase + k;
        }
        __syncthreads();
        // s_set and s_rcnt are no longer read in this cell: fetch the next cell's setup behind the
        // work items and clear the row counts for the next cell's rows phase
        if (tid < 8) s_rcnt[tid] = 0;
        prefetch(kv + gridDim.x);
        // work items: rows of one type (in registers) against the type's candidate list
        for (;;) {
            int it = 0;
            if (lane == 0) it = atomicAdd(&s_next, 1);
            it = __shfl_sync(0xffffffffu, it, 0);
            if (it >= s_nitems) break;
            const int code = s_item[it];
            const int tau = code & 0xff, u0 = (code >> 8) & 0xff, nr = code >> 16;
            LJ_CHECK_THAT(tau < 8 && nr <= kItemRows && u0 + nr <= ccnt);
            float4 ri[kItemRows];
            int32_t* dst[kItemRows];
            int cur[kItemRows];
#pragma unroll
            for (int r = 0; r < kItemRows; r++) {
                cur[r] = 0;
                ri[r] = make_float4(3e30f, 3e30f, 3e30f, __int_as_float(-2));
                dst[r] = a.out;
                if (r < nr) {
                    ri[r] = s_row[s_rowlist[u0 + r]];
                    const int64_t rr = __float_as_int(ri[r].w) - a.row_begin;
                    dst[r] = DIRECT ? a.out + a.ptr[rr] : padded_row(a.out, rr, a.il_skip);
                }
            }
            const unsigned short* lst = tl + tau * kTL;
            const int len = s_tlen[tau];
            for (int k0 = 0; k0 < len; k0 += 64) {
                const int s0 = lst[k0 + lane], s1 = lst[k0 + 32 + lane];
                LJ_CHECK_THAT(s0 <= MAXC && s1 <= MAXC);
                const int j0 = CJ[s0], j1 = CJ[s1];
                // the two candidates side by side in packed fp32x2 registers (FADD2/FFMA2,
                // row coordinate broadcast): same IEEE operations as the scalar form
                const unsigned long long cx = pack_f32x2(CX[s0], CX[s1]), cy = pack_f32x2(CY[s0], CY[s1]),
                                         cz = pack_f32x2(CZ[s0], CZ[s1]);
#pragma unroll
                for (int r = 0; r < kItemRows; r++) {
                    if (r >= nr) break;
                    const int i = __float_as_int(ri[r].w);
                    float r2a, r2b;
                    dist2_f32x2(cx, cy, cz, ri[r], r2a, r2b);
                    bool acc0 = r2a < a.lo2, acc1 = r2b < a.lo2;
                    const bool band0 = !acc0 && r2a < a.hi2, band1 = !acc1 && r2b < a.hi2;
                    if (__any_sync(0xffffffffu, band0 | band1)) {   // rare: the oracle's exact test
                        if (band0) acc0 = dist2_exact(a.q[i], a.q[j0], L, halfL) < a.rs2;
                        if (band1) acc1 = dist2_exact(a.q[i], a.q[j1], L, halfL) < a.rs2;
                    }
                    acc0 = acc0 && (HALF ? (j0 > i) : (j0 != i));
                    acc1 = acc1 && (HALF ? (j1 > i) : (j1 != i));
                    const unsigned m0 = __ballot_sync(0xffffffffu, acc0);
                    const unsigned m1 = __ballot_sync(0xffffffffu, acc1);
                    const int p0 = cur[r] + __popc(m0 & lt);
                    const int p1 = cur[r] + __popc(m0) + __popc(m1 & lt);
                    if (acc0 && (DIRECT || p0 < kRowCap)) dst[r][DIRECT ? p0 : il_off(p0, a.il_skip)] = j0;
                    if (acc1 && (DIRECT || p1 < kRowCap)) dst[r][DIRECT ? p1 : il_off(p1, a.il_skip)] = j1;
                    cur[r] += __popc(m0) + __popc(m1);
                }
            }
#ifdef LJ_CHECK
            if (DIRECT) {   // the fill pass accepts exactly the count pass's entries
#pragma unroll
                for (int r = 0; r < kItemRows; r++)
                    if (r < nr && lane == r) LJ_CHECK_THAT(cur[r] == a.npart[__float_as_int(ri[r].w) - a.row_begin]);
            }
#endif
            if (!DIRECT) {
#pragma unroll
                for (int r = 0; r < kItemRows; r++) {
                    if (r < nr && lane == r) {
                        a.npart[__float_as_int(ri[r].w) - a.row_begin] =
                            (a.clamp && cur[r] > kRowCap) ? kRowCap : cur[r];
                        if (cur[r] > kRowCap) atomicOr(&a.n_overflow[1], 1);
                    }
                }
            }
        }
    }
}

#undef s_start
#undef s_off
#undef s_dc
#undef s_first
#undef s_last
#undef s_unsorted

// Fallback for cells with more than kMaxCand candidates (dense or tiny boxes):
// one warp per row straight from global memory, per-row bitonic sort.
template <int DIRECT>
__global__ void __launch_bounds__(kListWarps * 32) k_list_fallback(ListArgs a) {
    __shared__ int rowbuf[kListWarps][kRowBuf];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double L = a.cg.L, halfL = 0.5 * a.cg.L;
    const int nover = a.n_overflow[2];
    for (int oc = blockIdx.x; oc < nover; oc += gridDim.x) {
        const int c = a.overflow_cells2[oc];
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
                        LJ_CHECK_THAT(!DIRECT || pos < a.npart[r]);
                        if (DIRECT) gdst[pos] = j;
                    }
                    cursor += __popc(m);
                }
            }
            __syncwarp();
            if (cursor <= kRowBuf || !DIRECT) {
                // (not DIRECT and cursor > kRowBuf: the row overflows the stride anyway; the
                // first kRowBuf entries, sorted, keep the stored prefix valid atom indices)
                const int m = min(cursor, kRowBuf);
                const int P = next_pow2(m > 0 ? m : 1);
                for (int k = m + lane; k < P; k += 32) buf[k] = INT_MAX;
                __syncwarp();
                warp_bitonic_sort(buf, P, lane);
                int32_t* dst = DIRECT ? gdst : padded_row(a.out, r, a.il_skip);
                const int lim = DIRECT ? cursor : min(m, kRowCap);
                const int skip = DIRECT ? 0 : a.il_skip;
                for (int k = lane; k < lim; k += 32) dst[il_off(k, skip)] = buf[k];
            } else if (lane == 0) {   // DIRECT, very long row: insertion sort in place
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
                a.npart[r] = (a.clamp && cursor > kRowCap) ? kRowCap : cursor;
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
    W.off_qr = o;
    o = align256(o + sizeof(float4) * (size_t)n);
    W.off_scan = o;
    o = align256(o + sizeof(int64_t) * (size_t)(W.scan_blocks + 1));
    W.off_over = o;    // [0] / [2] overflow cell counts, [1] row overflow flag, [3] pad, then 2 x ncell cell ids
    o = align256(o + sizeof(int32_t) * (size_t)(2 * ncell + 4));
    W.off_flags = o;   // [0] some raw coordinate outside [0, L) (set by k_cell_assign)
    o = align256(o + sizeof(int32_t) * 4);
    W.off_ptrtmp = o;  // rows + 1 int64 (padded layout: scan of the counts)
    o = align256(o + sizeof(int64_t) * (size_t)(rows + 1));
    W.off_scratch = o; // rows * kRowCap int32
    o = align256(o + sizeof(int32_t) * (size_t)rows * kRowCap);
    W.off_setup = o;   // ncell CellSetup records (k_cell_setup -> k_list_v4)
    o = align256(o + sizeof(CellSetup) * (size_t)ncell);
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
    float4* qr_cell = (float4*)(ws + W.off_qr);
    int64_t* scan = (int64_t*)(ws + W.off_scan);
    cudaError_t e;
    if ((e = cudaMemsetAsync(count, 0, sizeof(int32_t) * (size_t)cg.ncell, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (size_t)cg.ncell, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(ws + W.off_flags, 0, sizeof(int32_t) * 4, s)) != cudaSuccess) return e;
    if (n > 0) {
        k_cell_assign<<<grid_for(n, 256), 256, 0, s>>>((const rec4*)q, n, cg, cell_of, count,
                                                       (int32_t*)(ws + W.off_flags));
        g_launches++;
    }
    if ((e = launch_scan_i32_to_i64(count, start, cg.ncell, scan, W.scan_blocks, s)) != cudaSuccess) return e;
    if (n > 0) {
        k_cell_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, cell_of, start, cursor, atoms);
        k_cell_sort_gather<<<grid_for(cg.ncell, kListWarps), kListWarps * 32, 0, s>>>((const rec4*)q, cg, start,
                                                                                     atoms, q_cell, qf_cell, qr_cell,
                                                                                     cg.L / cg.nc);
        g_launches += 2;
    }
    return cudaGetLastError();
}

cudaError_t launch_rebuild_cells(double* q, const double* p, double* q_out, double* p_out, double* q_ref,
                                 int64_t* perm, int64_t n, const CellGrid& cg, char* ws, const BuildWorkspace& W,
                                 cudaStream_t s, const PeerMomenta& pm) {
    int32_t* cell_of = (int32_t*)(ws + W.off_cell_of);
    int32_t* count = (int32_t*)(ws + W.off_count);
    int64_t* start = (int64_t*)(ws + W.off_start);
    int32_t* cursor = (int32_t*)(ws + W.off_cursor);
    int32_t* atoms = (int32_t*)(ws + W.off_atoms);
    cudaError_t e;
    if ((e = cudaMemsetAsync(count, 0, sizeof(int32_t) * (size_t)cg.ncell, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (size_t)cg.ncell, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(ws + W.off_flags, 0, sizeof(int32_t) * 4, s)) != cudaSuccess) return e;   // wrapped input
    if (n > 0) {
        k_wrap_assign<<<grid_for(n, 256), 256, 0, s>>>((rec4*)q, n, cg, cell_of, count);
        g_launches++;
    }
    if ((e = launch_scan_i32_to_i64(count, start, cg.ncell, (int64_t*)(ws + W.off_scan), W.scan_blocks, s)) !=
        cudaSuccess)
        return e;
    if (n > 0) {
        k_cell_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, cell_of, start, cursor, atoms);
        k_cell_sort_permute<<<grid_for(cg.ncell, kListWarps), kListWarps * 32, 0, s>>>(
            (const rec4*)q, (const rec4*)p, cg, start, atoms, perm, (rec4*)q_out, (rec4*)p_out, (rec4*)q_ref,
            (rec4*)(ws + W.off_qcell), (float4*)(ws + W.off_qr), cg.L / cg.nc, pm);
        g_launches += 2;
    }
    return cudaGetLastError();
}

static int64_t ncell_of(const CellGrid& cg) { return cg.ncell; }

static ListArgs list_args(const double* q, const CellGrid& cg, double rs, int half, int64_t row_begin,
                          int64_t row_end, int32_t* npart, const int64_t* ptr, int32_t* out, char* ws,
                          const BuildWorkspace& W) {
    ListArgs a;
    a.q = (const rec4*)q;
    a.flags = (const int32_t*)(ws + W.off_flags);
    a.w = cg.L / cg.nc;
    {
        // v4 fp32 decision band.  A staged coordinate is u = fl32(x - o_own) + k fl32(w)
        // (k in {-1,0,1}: the neighbour cell's offset), |u| <= X = 2w + rs, carrying at most
        // 2^-24 (w + w + 2w) of rounding; a row coordinate carries <= 2^-24 w.  So each
        // fp32 displacement differs from the oracle's fp64 minimum-image displacement by
        //   eps_d <= 2^-22 X + 2^-24 rs (the fp32 subtraction near |d| ~ rs)
        //            + 2^-49 L (fp64 roundings of x - o and of the oracle's d, both sides).
        // Near r2 ~ rs2 the fp32 r2 (3 roundings) then differs from the oracle's r2 by
        // at most 2 sqrt(3) rs eps_d + 4 * 2^-24 rs2 (+ the oracle's own 2^-52 rs2);
        // the band takes 4x that.
        const double X = 2.0 * a.w + rs;
        const double eps_d = std::ldexp(X, -22) + std::ldexp(rs, -24) + std::ldexp(cg.L, -49);
        const double rs2 = rs * rs;
        const double delta = 4.0 * (2.0 * std::sqrt(3.0) * rs * eps_d + std::ldexp(4.0 * rs2, -24)) + 1e-9 * rs2;
        a.lo2 = std::nextafter((float)(rs2 - delta), 0.0f);
        a.hi2 = std::nextafter((float)(rs2 + delta), INFINITY);
        const double rb = rs * (1.0 + 1e-4) + 1e-4;   // covers fp32 coordinate errors and edge rows
        a.rb2 = std::nextafter((float)(rb * rb), INFINITY);
    }
    a.q_cell = (const rec4*)(ws + W.off_qcell);
    a.qf_cell = (const float4*)(ws + W.off_qf);
    a.qr_cell = (const float4*)(ws + W.off_qr);
    a.atoms = (const int32_t*)(ws + W.off_atoms);
    a.start = (const int64_t*)(ws + W.off_start);
    a.ncell = cg.ncell;
    a.cg = cg;
    a.rs2 = rs * rs;
    // fp32 screen: positions (|x| <= L) carry <= ~2 ulp(L) = 2.4e-7 L error per axis;
    // widen the radius by 8e-7 L + 1e-5 so every exact pair passes the screen.
    double rsc = rs + 8e-7 * cg.L + 1e-5;
    a.r_screen = (float)(rsc * (1.0 + 1e-5));
    a.half = half;
    a.row_begin = row_begin;
    a.row_end = row_end;
    a.npart = npart;
    a.ptr = ptr;
    a.out = out;
    a.n_overflow = (int32_t*)(ws + W.off_over);
    a.overflow_cells = a.n_overflow + 4;
    a.overflow_cells2 = a.overflow_cells + ncell_of(cg);
    a.setups = (const CellSetup*)(ws + W.off_setup);
    a.clamp = 0;
    a.il_skip = 0;
    return a;
}

static int list_grid(const CellGrid& cg, int per_sm) {
    int64_t g = 148 * per_sm;
    return (int)(cg.ncell < g ? cg.ncell : g);
}

constexpr size_t kListSmem = (size_t)kMaxCand * 8 + (size_t)(kMaxCand + 32) * (3 * 8 + 4 + 1);
constexpr size_t list_smem_v4(int maxc) { return (size_t)8 * (maxc + 64) * 2 + (size_t)(maxc + 32) * (16 + 1); }
constexpr int kMaxCandLarge = 2560;   // the LARGE pass: 2 CTAs per SM (86 KB of shared memory)
constexpr size_t kListSmemV4 = list_smem_v4(kMaxCand);
constexpr size_t kListSmemV4L = list_smem_v4(kMaxCandLarge);

static cudaError_t set_list_attrs() {
    // cudaFuncSetAttribute is per device: one flag per device ordinal (set once, thread-safe)
    constexpr int kMaxDevices = 64;
    static std::atomic<bool> done[kMaxDevices];
    int dev = 0;
    cudaError_t ed = cudaGetDevice(&dev);
    if (ed != cudaSuccess) return ed;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    if (!done[dev].load(std::memory_order_acquire)) {
        void (*fns[4])(ListArgs) = {k_list_v2<0, 0>, k_list_v2<0, 1>, k_list_v2<1, 0>, k_list_v2<1, 1>};
        for (auto f : fns) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kListSmem);
            if (e != cudaSuccess) return e;
        }
        void (*fns4[4])(ListArgs) = {k_list_v4<0, 0, kMaxCand, false>, k_list_v4<0, 1, kMaxCand, false>,
                                     k_list_v4<1, 0, kMaxCand, false>, k_list_v4<1, 1, kMaxCand, false>};
        for (auto f : fns4) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kListSmemV4);
            if (e != cudaSuccess) return e;
        }
        void (*fns4l[4])(ListArgs) = {k_list_v4<0, 0, kMaxCandLarge, true>, k_list_v4<0, 1, kMaxCandLarge, true>,
                                      k_list_v4<1, 0, kMaxCandLarge, true>, k_list_v4<1, 1, kMaxCandLarge, true>};
        for (auto f : fns4l) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kListSmemV4L);
            if (e != cudaSuccess) return e;
        }
        done[dev].store(true, std::memory_order_release);   // idempotent: a race sets the same attributes twice
    }
    return cudaSuccess;
}

// The exact kernel (v2/v3) and the fast kernel (v4) are both launched; each
// returns at once unless the input-range flag of k_cell_assign selects it.
template <int DIRECT>
static void launch_list_kernels(const ListArgs& a, const CellGrid& cg, int half, cudaStream_t s) {
    k_cell_setup<<<grid_for(cg.ncell * 32, 256, 148 * 16), 256, 0, s>>>(a, const_cast<CellSetup*>(a.setups));
    g_launches++;
    if (half) {
        k_list_v4<DIRECT, 1, kMaxCand, false><<<list_grid(cg, 4), kListWarps * 32, kListSmemV4, s>>>(a);
        k_list_v4<DIRECT, 1, kMaxCandLarge, true><<<list_grid(cg, 2), kListWarps * 32, kListSmemV4L, s>>>(a);
        k_list_v2<DIRECT, 1><<<list_grid(cg, 4), kListWarps * 32, kListSmem, s>>>(a);
    } else {
        k_list_v4<DIRECT, 0, kMaxCand, false><<<list_grid(cg, 4), kListWarps * 32, kListSmemV4, s>>>(a);
        k_list_v4<DIRECT, 0, kMaxCandLarge, true><<<list_grid(cg, 2), kListWarps * 32, kListSmemV4L, s>>>(a);
        k_list_v2<DIRECT, 0><<<list_grid(cg, 4), kListWarps * 32, kListSmem, s>>>(a);
    }
    k_list_fallback<DIRECT><<<148, kListWarps * 32, 0, s>>>(a);
    g_launches += 4;
}

cudaError_t launch_list_pass1(const double* q, const CellGrid& cg, double rs, int half, int64_t row_begin,
                              int64_t row_end, int32_t* npart, int32_t* out, char* ws, const BuildWorkspace& W,
                              cudaStream_t s, bool interleaved) {
    cudaError_t e = set_list_attrs();
    if (e != cudaSuccess) return e;
    ListArgs a = list_args(q, cg, rs, half, row_begin, row_end, npart, nullptr,
                           out ? out : (int32_t*)(ws + W.off_scratch), ws, W);
    a.clamp = out != nullptr;   // the caller's padded list: counts clamped to the stride
    a.il_skip = (out != nullptr && interleaved) ? kIlSkip : 0;
    e = cudaMemsetAsync(a.n_overflow, 0, 4 * sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    launch_list_kernels<0>(a, cg, half, s);
    return cudaGetLastError();
}

const int32_t* list_row_overflow_flag(char* ws, const BuildWorkspace& W) { return (const int32_t*)(ws + W.off_over) + 1; }

cudaError_t launch_list_pass2(const double* q, const CellGrid& cg, double rs, int half, int64_t row_begin,
                              int64_t row_end, int32_t* npart, const int64_t* ptr, int32_t* list, bool row_overflow,
                              char* ws, const BuildWorkspace& W, cudaStream_t s) {
    const int64_t rows = row_end - row_begin;
    if (!row_overflow) {
        k_compact<<<grid_for(rows * 32, 256, 148 * 32), 256, 0, s>>>((const int32_t*)(ws + W.off_scratch), npart, ptr,
                                                                     rows, list);
        g_launches++;
        return cudaGetLastError();
    }
    cudaError_t e = set_list_attrs();
    if (e != cudaSuccess) return e;
    ListArgs a = list_args(q, cg, rs, half, row_begin, row_end, npart, ptr, list, ws, W);
    launch_list_kernels<1>(a, cg, half, s);
    return cudaGetLastError();
}

__global__ void k_padded_pointer(int64_t* ptr, int64_t rows, int il) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= rows; r += (int64_t)gridDim.x * blockDim.x)
        if (!il)
            ptr[r] = r * (int64_t)kRowCap;
        else if (r < rows)   // entry 0 of the row, flagged (row_decode)
            ptr[r] = kIlBit | ((r >> 3) * (int64_t)(kIlRows * kRowCap) + (r & (kIlRows - 1)) * kIlGran);
        else   // the padded extent
            ptr[r] = ((rows + kIlRows - 1) / kIlRows) * (int64_t)(kIlRows * kRowCap);
}

cudaError_t launch_padded_pointer(int64_t* ptr, int64_t rows, cudaStream_t s, bool interleaved) {
    k_padded_pointer<<<grid_for(rows + 1, 256), 256, 0, s>>>(ptr, rows, interleaved ? 1 : 0);
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
