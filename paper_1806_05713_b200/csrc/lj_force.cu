// LJ force step over the sorted (CSR) Verlet list -- SURVEY §8(a) a5/a6.
//
// The method (PAPER.md Alg. lj_force, inside Alg.
// calcforce_sortedlist): for each i-atom, for each j in
// SortedList[i]: r = q_j - q_i; if r^2 < r_c^2: df = (48 - 24 r^6) dt / r^14,
// p_i -= df r (and p_j += df r for the half list; Newton-3 sign, reading C-1).
//
// B200 mapping (the paper's SIMD tricks are prior art):
//  * "i-data in registers": G lanes cooperate on one row; q_i and
//    the three accumulators stay in registers; the G partial sums are reduced
//    with warp shuffles and p_i is committed once (no atomics, full list).
//  * "AoS with padding": every partner gather is ONE 256-bit load
//    (LDG.E.ENL2.256) of a 32-byte record = one L2 sector.
//  * cutoff masking and remainder-loop elimination:
//    out-of-range pairs get df = 0 by a predicate (integer compare of the
//    IEEE bits of r^2 and r_c^2, exact for positive doubles); tail lanes
//    k >= n_i are simply inactive in the last group iteration.
//  * software pipelining: two independent partner gathers are in
//    flight per lane (memory-level parallelism instead of IPC tricks).
//  * fp64 division: 1/r^2 by MUFU.RCP64H (rcp.approx.ftz.f64) + one cubic
//    Newton correction y(1 + e + e^2), e = 1 - r^2 y, then the 1/r^2 form
//    df = dt (48 r^-6 - 24) r^-6 r^-2, algebraically the paper's expression.
//  * minimum image: raw differences are checked with integer ops on the high
//    words; the three image DADDs run only when some lane of the warp needs an
//    image (warp-uniform branch), i.e. only for rows near a box face.
#include <algorithm>
#include <climits>

#include "lj_internal.cuh"
#include "lj_force_core.cuh"

namespace lj {

namespace {

constexpr int kForceThreads = 256;

// G lanes per row, U independent partner gathers in flight per lane.
// Full list: no atomics, p_i committed once by lane 0 of the group.
// Half list: p_j += df r by fp64 REDs, p_i committed by REDs as well.
// The chunk loop runs while ANY row of the warp has entries left (warp-uniform
// trip count), so the minimum-image test can be one vote per chunk: r^2 of the
// raw differences below (L/2)^2 (integer test on the high words) proves that no
// component needs an image; otherwise (rows near a box face) the differences
// are corrected per component and r^2 recomputed.  The list layout (plain or
// interleaved; every row of a list has the same) is taken per warp by a vote.
// U = 2: at most 48 registers -> 5 CTAs (40 warps) per SM; measured 0.79 vs 0.83 ms
// (54 registers, 4 CTAs) on config 4 -- the kernel is latency/L1-bound, warps help.
template <int G, int U, bool HALF>
__global__ void __launch_bounds__(kForceThreads, U == 2 ? 5 : (U == 3 ? 4 : 3))
    k_force(const rec4* __restrict__ q, rec4* __restrict__ p, int64_t row_begin, int64_t rows,
            const int32_t* __restrict__ npart, const int64_t* __restrict__ ptr, const int32_t* __restrict__ list,
            PairConsts c, unsigned long long* n_inter) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = t / G;
    const int g = threadIdx.x % G;
    const bool active = r < rows;
    double ax = 0.0, ay = 0.0, az = 0.0;
    unsigned cnt = 0;
    const int64_t i = row_begin + (active ? r : 0);
    const rec4 qi = load_rec(q, active ? i : 0);
    const int64_t p0 = active ? ptr[r] : 0;
    const int32_t* __restrict__ lst = list + (p0 & (kIlBit - 1));
    const int n = active ? npart[r] : 0;
    const bool il = __any_sync(0xffffffffu, (p0 & kIlBit) != 0);
    LJ_CHECK_THAT(!active || il == ((p0 & kIlBit) != 0));
    if (il)
        force_row_loop<G, U, HALF, true>(q, p, i, qi, lst, n, g, c, ax, ay, az, cnt);
    else
        force_row_loop<G, U, HALF, false>(q, p, i, qi, lst, n, g, c, ax, ay, az, cnt);
    unsigned cnt_row = cnt;
    group_reduce<G>(ax, ay, az, cnt_row);
    if (active && g == 0) {
        if (HALF) {
            // p_i is concurrently a RED target of earlier rows (i in row(i'), i' < i):
            // commit with REDs too (SURVEY §8(a) a6 race hazard).
            atomicAdd(&p[i].x, ax);
            atomicAdd(&p[i].y, ay);
            atomicAdd(&p[i].z, az);
        } else {
            rec4 pi = p[i];
            pi.x += ax;
            pi.y += ay;
            pi.z += az;
            p[i] = pi;   // pad preserved (read back unchanged)
        }
    }
    count_interactions(cnt, n_inter);
}

// ---- vectorised index stream (lanes_per_row | LJ_LANES_IDXV) ---------------
// As k_force, but every lane loads V consecutive list entries with ONE vector
// load (V = 2: 64-bit, V = 4: 128-bit) and keeps their V gathers in flight.  In
// k_force a warp's index load covers 32 entries of 32/G rows (one 32-bit load
// per lane, ~10 L1 tag lookups per instruction); here it covers 32 V entries,
// cutting the index stream's share of the L1 data-pipe wavefronts -- the
// resource that binds the kernel (profiles/r01_ncu_force_v12.txt) -- by ~V.
// The row is read through the V-aligned window that contains it: window slot s
// holds list[base + s], base = pointer[r] rounded down to a multiple of V, and
// the row's entries are slots [off, off + n), off = pointer[r] - base.  A lane's
// vector load stays inside one V*4-byte aligned segment that holds at least one
// entry of the row, so it never leaves the list's allocation.  Padded lists
// (pointer = r * 196) have off = 0.
template <int V>
struct IdxVec;
template <>
struct IdxVec<2> {
    __device__ static void load(const int32_t* a, int (&j)[2]) {
        const int2 v = __ldg(reinterpret_cast<const int2*>(a));
        j[0] = v.x, j[1] = v.y;
    }
};
template <>
struct IdxVec<4> {
    __device__ static void load(const int32_t* a, int (&j)[4]) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(a));
        j[0] = v.x, j[1] = v.y, j[2] = v.z, j[3] = v.w;
    }
};

template <int G, int V, bool HALF>
__global__ void __launch_bounds__(kForceThreads, V == 2 ? 5 : 3)
    k_force_idxv(const rec4* __restrict__ q, rec4* __restrict__ p, int64_t row_begin, int64_t rows,
                 const int32_t* __restrict__ npart, const int64_t* __restrict__ ptr, const int32_t* __restrict__ list,
                 PairConsts c, unsigned long long* n_inter) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = t / G;
    const int g = threadIdx.x % G;
    const bool active = r < rows;
    double ax = 0.0, ay = 0.0, az = 0.0;
    unsigned cnt = 0;
    const int64_t i = row_begin + (active ? r : 0);
    const rec4 qi = load_rec(q, i);
    int64_t base = 0;
    int off = 0, end = 0, skip = 0;
    if (active) {
        const int64_t p0 = row_decode(list, ptr[r], skip) - list;   // (interleaved rows: 4-aligned, off = 0)
        base = p0 & ~(int64_t)(V - 1);
        off = (int)(p0 - base);
        end = off + npart[r];
    }
    const int32_t* __restrict__ win = list + base;
    // software pipeline: the next chunk's index vector is loaded before this chunk's records are used
    int jn[V];
    if (V * g < end) {
        IdxVec<V>::load(win + il_off(V * g, skip), jn);
    } else {
#pragma unroll
        for (int u = 0; u < V; u++) jn[u] = -1;
    }
    for (int s0 = V * g; __any_sync(0xffffffffu, s0 < end); s0 += V * G) {
        int j[V];
        rec4 qj[V];
#pragma unroll
        for (int u = 0; u < V; u++) {
            j[u] = (s0 + u >= off && s0 + u < end) ? jn[u] : -1;
            LJ_CHECK_THAT(j[u] < c.n_atoms);
            qj[u] = load_rec(q, j[u] >= 0 ? (int64_t)j[u] : i);   // no entry: r = 0, masked below
        }
        const int sn = s0 + V * G;
        if (sn < end) {
            IdxVec<V>::load(win + il_off(sn, skip), jn);
        } else {
#pragma unroll
            for (int u = 0; u < V; u++) jn[u] = -1;
        }
        double dx[V], dy[V], dz[V], r2[V];
        int hmax = 0;
#pragma unroll
        for (int u = 0; u < V; u++) {
            dx[u] = qj[u].x - qi.x;
            dy[u] = qj[u].y - qi.y;
            dz[u] = qj[u].z - qi.z;
            r2[u] = fma(dz[u], dz[u], fma(dy[u], dy[u], dx[u] * dx[u]));
            hmax = max(hmax, __double2hiint(r2[u]));
        }
        auto accumulate = [&]() {
            bool inr[V];
            inside_cutoff_u<V>(inr, j, r2, dx, dy, dz, c);
#pragma unroll
            for (int u = 0; u < V; u++) {
                const double inv2 = fast_rcp(r2[u]);
                const double inv6 = inv2 * inv2 * inv2;
                const bool in = inr[u];
                const double df = in ? fma(c.c48, inv6, -c.c24) * (inv6 * inv2) : 0.0;
                ax = fma(-df, dx[u], ax);
                ay = fma(-df, dy[u], ay);
                az = fma(-df, dz[u], az);
                cnt += in;
                if (HALF && in) {
                    atomicAdd(&p[j[u]].x, df * dx[u]);
                    atomicAdd(&p[j[u]].y, df * dy[u]);
                    atomicAdd(&p[j[u]].z, df * dz[u]);
                }
            }
        };
        if (__any_sync(0xffffffffu, hmax >= c.hi_L2q)) {   // some pair may need a periodic image
#pragma unroll
            for (int u = 0; u < V; u++) {
                dx[u] -= image_shift(dx[u], c.L, c.hi_halfL);
                dy[u] -= image_shift(dy[u], c.L, c.hi_halfL);
                dz[u] -= image_shift(dz[u], c.L, c.hi_halfL);
                r2[u] = fma(dz[u], dz[u], fma(dy[u], dy[u], dx[u] * dx[u]));
            }
            accumulate();
        } else {
            accumulate();
        }
    }
    unsigned cnt_row = cnt;
    group_reduce<G>(ax, ay, az, cnt_row);
    if (active && g == 0) {
        if (HALF) {
            atomicAdd(&p[i].x, ax);
            atomicAdd(&p[i].y, ay);
            atomicAdd(&p[i].z, az);
        } else {
            rec4 pi = p[i];
            pi.x += ax;
            pi.y += ay;
            pi.z += az;
            p[i] = pi;
        }
    }
    count_interactions(cnt, n_inter);
}

// ---- half list without per-entry global atomics -------
// One CTA per cell of the build's cell grid; rows = the cell's index range
// [cstart[c], cstart[c+1]) (in cell-ordered storage: exactly the cell's atoms).
// Every partner j of these rows lies in one of the 27 neighbour cells, i.e. in
// one of 27 index runs; the CTA accumulates the p_j contributions (and its own
// rows' sums) in a shared-memory window indexed by (run, offset) and flushes
// it once with one RED per component and atom -- coalesced, instead of three
// random REDs per list entry.  A partner outside the window (storage not in
// cell order, or a window larger than kWin) falls back to a global RED, so the
// result does not depend on the storage order, only the speed does.
constexpr int kWin = 1024;   // window slots (3 doubles each: 24 KB of shared memory)
#ifndef LJ_HC_THREADS
#define LJ_HC_THREADS 128    // CTA size: 8 CTAs (32 warps) per SM, so barrier waits overlap other CTAs
#endif

// Slot of partner j in the window: the window is a short ascending list of
// contiguous index segments (adjacent neighbour runs merged: ~5 for an interior
// cell), ss = segment starts padded with INT_MAX, fin = (segment end, slot - index).
template <int STEPS>
__device__ __forceinline__ int win_slot(int j, const int* ss, const int2* fin) {
    int r = 0;   // largest r with ss[r] <= j
#pragma unroll
    for (int st = 1 << (STEPS - 1); st > 0; st >>= 1) r = ss[r + st] <= j ? r + st : r;
    const int2 f = fin[r];
    return (j >= ss[r] && j < f.x) ? j + f.y : -1;
}

__device__ __forceinline__ void win_add(double* w, int slot, double v, double* gp) {
    if (slot >= 0) atomicAdd(w + slot, v);   // shared memory
    else atomicAdd(gp, v);                   // outside the window: global RED
}

__device__ __forceinline__ int axis_rank3(int v, int d, int nc) {   // as k_list_v4's axis_rank
    if (v == 0) return d == 0 ? 0 : (d == 1 ? 1 : 2);
    if (v == nc - 1) return d == 1 ? 0 : (d == -1 ? 1 : 2);
    return d + 1;
}

template <int G, int U, int kHalfCellThreads>
__global__ void __launch_bounds__(kHalfCellThreads, 1024 / kHalfCellThreads)
    k_force_half_cells(const rec4* __restrict__ q, rec4* __restrict__ p, const int32_t* __restrict__ npart,
                       const int64_t* __restrict__ ptr, const int32_t* __restrict__ list,
                       const int64_t* __restrict__ cstart, int nc, int64_t ncell, PairConsts c,
                       unsigned long long* n_inter) {
    extern __shared__ double s_acc[];                 // [3][kWin]
    __shared__ int s_rs[32], s_rn[32];                // neighbour runs in ascending cell id (rank order)
    __shared__ int s_ss[64], s_soff[64];              // window segments: start index, first slot (INT_MAX pad)
    __shared__ int2 s_fin[32];                        // window segments: (end index, slot - index)
    __shared__ int s_m, s_nseg;
    double* wx = s_acc;
    double* wy = s_acc + kWin;
    double* wz = s_acc + 2 * kWin;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int grp = tid / G, g = tid % G;
    constexpr int NG = kHalfCellThreads / G;
    unsigned cnt = 0;
    for (int64_t cell = blockIdx.x; cell < ncell; cell += gridDim.x) {
        const int64_t cs = cstart[cell];
        const int ccnt = (int)(cstart[cell + 1] - cs);
        __syncthreads();   // the previous cell's window has been flushed
        if (w == 0) {
            const int cz = (int)(cell % nc), cy = (int)((cell / nc) % nc), cx = (int)(cell / ((int64_t)nc * nc));
            int st = INT_MAX, len = 0, rank = lane;
            if (lane < 27) {
                const int dx = lane / 9 - 1, dy = (lane / 3) % 3 - 1, dz = lane % 3 - 1;
                int x = cx + dx, y = cy + dy, z = cz + dz;
                x += x < 0 ? nc : (x >= nc ? -nc : 0);
                y += y < 0 ? nc : (y >= nc ? -nc : 0);
                z += z < 0 ? nc : (z >= nc ? -nc : 0);
                const int64_t cc = ((int64_t)x * nc + y) * nc + z;
                st = (int)cstart[cc];
                // a half-list partner j > i >= cs lies at or after cs: runs before this
                // cell (lower cell ids, in cell order) get no window slots
                len = st >= cs ? (int)(cstart[cc + 1] - cstart[cc]) : 0;
                rank = axis_rank3(cx, dx, nc) * 9 + axis_rank3(cy, dy, nc) * 3 + axis_rank3(cz, dz, nc);
            }
            s_rs[rank] = st;
            s_rn[rank] = len;
            __syncwarp();
            // merge the non-empty runs (ascending) into contiguous segments
            const int st_r = s_rs[lane], len_r = s_rn[lane], end_r = st_r + len_r;
            const unsigned km = __ballot_sync(0xffffffffu, len_r > 0);
            const unsigned before = km & lt;
            const int prev = before ? 31 - __clz(before) : 0;
            const int prev_end = __shfl_sync(0xffffffffu, end_r, prev);
            const bool seg = len_r > 0 && (before == 0 || prev_end != st_r);
            const unsigned sm = __ballot_sync(0xffffffffu, seg);
            const unsigned above = lane == 31 ? 0u : sm & ~((2u << lane) - 1u);
            const int nxt = above ? __ffs(above) - 1 : 32;
            const unsigned kb = km & (nxt >= 32 ? 0xffffffffu : ((1u << nxt) - 1u));
            const int last = kb ? 31 - __clz(kb) : 0;
            const int seg_end = __shfl_sync(0xffffffffu, end_r, last);
            const int seglen = seg ? seg_end - st_r : 0;
            int incl = seglen;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int nseg = __popc(sm);
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            if (seg) {
                const int k = __popc(sm & lt);
                const int off = incl - seglen;
                s_ss[k] = st_r;
                s_soff[k] = off;
                s_fin[k] = make_int2(seg_end, off - st_r);
            }
            __syncwarp();
            if (lane >= nseg) {
                s_ss[lane] = INT_MAX;
                s_soff[lane] = INT_MAX;
            }
            s_ss[32 + lane] = INT_MAX;
            s_soff[32 + lane] = INT_MAX;
            if (lane == 0) {
                s_m = total;
                s_nseg = nseg;
            }
        }
        __syncthreads();
        const int M = s_m;
        const bool win = M <= kWin;   // (CTA-uniform)
        const bool small = s_nseg <= 8;
        if (win)
            for (int k = tid; k < M; k += kHalfCellThreads) wx[k] = wy[k] = wz[k] = 0.0;
        __syncthreads();
        for (int base = 0; base < ccnt; base += NG) {
            const bool active = base + grp < ccnt;
            const int64_t i = cs + (active ? base + grp : 0);
            const rec4 qi = load_rec(q, i);
            int skip;
            const int32_t* __restrict__ lst = row_decode(list, active ? ptr[i] : 0, skip);
            const int n = active ? npart[i] : 0;
            double ax = 0.0, ay = 0.0, az = 0.0;
            int jn[U];
#pragma unroll
            for (int u = 0; u < U; u++) jn[u] = (g + u * G < n) ? __ldg(lst + il_off(g + u * G, skip)) : -1;
            for (int k0 = g; __any_sync(0xffffffffu, k0 < n); k0 += U * G) {
                int j[U];
                rec4 qj[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    j[u] = jn[u];
                    LJ_CHECK_THAT(j[u] < c.n_atoms);
                    qj[u] = load_rec(q, j[u] >= 0 ? (int64_t)j[u] : i);
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int kn = k0 + U * G + u * G;
                    jn[u] = kn < n ? __ldg(lst + il_off(kn, skip)) : -1;
                }
                double dx[U], dy[U], dz[U], r2[U];
                int hmax = 0;
#pragma unroll
                for (int u = 0; u < U; u++) {
                    dx[u] = qj[u].x - qi.x;
                    dy[u] = qj[u].y - qi.y;
                    dz[u] = qj[u].z - qi.z;
                    r2[u] = fma(dz[u], dz[u], fma(dy[u], dy[u], dx[u] * dx[u]));
                    hmax = max(hmax, __double2hiint(r2[u]));
                }
                if (__any_sync(0xffffffffu, hmax >= c.hi_L2q)) {   // rows near a box face: periodic images
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        dx[u] -= image_shift(dx[u], c.L, c.hi_halfL);
                        dy[u] -= image_shift(dy[u], c.L, c.hi_halfL);
                        dz[u] -= image_shift(dz[u], c.L, c.hi_halfL);
                        r2[u] = fma(dz[u], dz[u], fma(dy[u], dy[u], dx[u] * dx[u]));
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const double dx_ = dx[u], dy_ = dy[u], dz_ = dz[u];
                    const bool in = j[u] >= 0 && inside_cutoff(r2[u], dx[u], dy[u], dz[u], c);
                    if (in) {
                        const double inv2 = fast_rcp(r2[u]);
                        const double inv6 = inv2 * inv2 * inv2;
                        const double df = fma(c.c48, inv6, -c.c24) * (inv6 * inv2);
                        ax = fma(-df, dx_, ax);
                        ay = fma(-df, dy_, ay);
                        az = fma(-df, dz_, az);
                        cnt++;
                        const int sl = !win ? -1 : (small ? win_slot<3>(j[u], s_ss, s_fin)
                                                          : win_slot<5>(j[u], s_ss, s_fin));
                        win_add(wx, sl, df * dx_, &p[j[u]].x);
                        win_add(wy, sl, df * dy_, &p[j[u]].y);
                        win_add(wz, sl, df * dz_, &p[j[u]].z);
                    }
                }
            }
            unsigned dummy = 0;
            group_reduce<G>(ax, ay, az, dummy);
            if (active && g == 0) {
                const int sl = !win ? -1 : (small ? win_slot<3>((int)i, s_ss, s_fin)
                                                  : win_slot<5>((int)i, s_ss, s_fin));
                win_add(wx, sl, ax, &p[i].x);
                win_add(wy, sl, ay, &p[i].y);
                win_add(wz, sl, az, &p[i].z);
            }
        }
        __syncthreads();
        if (win) {   // flush: one RED per component and touched atom, consecutive atoms per warp
            for (int k = tid; k < M; k += kHalfCellThreads) {
                const double vx = wx[k], vy = wy[k], vz = wz[k];
                if (vx != 0.0 || vy != 0.0 || vz != 0.0) {
                    int r = 0;   // the segment holding slot k: largest r with s_soff[r] <= k
#pragma unroll
                    for (int st = 16; st > 0; st >>= 1) r = s_soff[r + st] <= k ? r + st : r;
                    const int64_t a = (int64_t)s_ss[r] + (k - s_soff[r]);
                    atomicAdd(&p[a].x, vx);
                    atomicAdd(&p[a].y, vy);
                    atomicAdd(&p[a].z, vz);
                }
            }
        }
    }
    count_interactions(cnt, n_inter);
}

// ---- paper-variant ablations -------------------------
// The paper's layout axis (SoA vs AoS with padding, AoS8
// P:551-573) and its reciprocal "future issue" on the GPU: the
// full-list kernel of k_force (same lanes, same chunk loop and arithmetic)
// with the position gather / momentum commit of another layout, and the 1/r^2
// evaluated four ways.  Not on the hot path; lj_force_step_variant.
template <int LAYOUT>
struct Layout;
template <>
struct Layout<LJ_LAYOUT_AOS4> {   // x, y, z, pad: one 256-bit load
    __device__ static void pos(const double* q, int64_t, int64_t j, double& x, double& y, double& z) {
        const rec4 r = load_rec((const rec4*)q, j);
        x = r.x, y = r.y, z = r.z;
    }
    __device__ static double* mom(double* p, int64_t, int64_t i, int c) { return p + 4 * i + c; }
};
template <>
struct Layout<LJ_LAYOUT_SOA> {    // x[n], y[n], z[n]: three 8-byte gathers (three sectors)
    __device__ static void pos(const double* q, int64_t n, int64_t j, double& x, double& y, double& z) {
        x = __ldg(q + j), y = __ldg(q + n + j), z = __ldg(q + 2 * n + j);
    }
    __device__ static double* mom(double* p, int64_t n, int64_t i, int c) { return p + c * n + i; }
};
template <>
struct Layout<LJ_LAYOUT_AOS3> {   // x, y, z without padding: 24-B records, three 8-byte loads
    __device__ static void pos(const double* q, int64_t, int64_t j, double& x, double& y, double& z) {
        x = __ldg(q + 3 * j), y = __ldg(q + 3 * j + 1), z = __ldg(q + 3 * j + 2);
    }
    __device__ static double* mom(double* p, int64_t, int64_t i, int c) { return p + 3 * i + c; }
};
template <>
struct Layout<LJ_LAYOUT_AOS8> {   // one 64-B record per atom: q (x, y, z, pad) then p (x, y, z, pad)
    __device__ static void pos(const double* q, int64_t, int64_t j, double& x, double& y, double& z) {
        const rec4 r = load_rec((const rec4*)q, 2 * j);
        x = r.x, y = r.y, z = r.z;
    }
    __device__ static double* mom(double* p, int64_t, int64_t i, int c) { return p + 8 * i + 4 + c; }
};

template <int RCP>
__device__ __forceinline__ double inv_r2(double x) {
    if (RCP == LJ_RCP_NEWTON3) return fast_rcp(x);
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    if (RCP == LJ_RCP_NEWTON2) return fma(y, fma(-x, y, 1.0), y);   // one quadratic Newton step
    if (RCP == LJ_RCP_APPROX) return y;                              // MUFU.RCP64H alone
    return __drcp_rn(x);                                             // IEEE reciprocal
}

// 48 registers (5 CTAs/SM, as k_force) where it does not spill; the 8-byte-gather
// layouts need 64 (4 CTAs/SM).
template <int G, int LAYOUT, int RCP>
__global__ void __launch_bounds__(kForceThreads, (LAYOUT == LJ_LAYOUT_SOA || LAYOUT == LJ_LAYOUT_AOS3) ? 4 : 5)
    k_force_variant(const double* __restrict__ q, double* __restrict__ p, int64_t n_atoms, int64_t row_begin,
                    int64_t rows, const int32_t* __restrict__ npart, const int64_t* __restrict__ ptr,
                    const int32_t* __restrict__ list, PairConsts c, unsigned long long* n_inter) {
    constexpr int U = 2;
    using Lay = Layout<LAYOUT>;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = t / G;
    const int g = threadIdx.x % G;
    const bool active = r < rows;
    double ax = 0.0, ay = 0.0, az = 0.0;
    unsigned cnt = 0;
    const int64_t i = row_begin + (active ? r : 0);
    double qix, qiy, qiz;
    Lay::pos(q, n_atoms, active ? i : 0, qix, qiy, qiz);
    int skip;
    const int32_t* __restrict__ lst = row_decode(list, active ? ptr[r] : 0, skip);
    const int n = active ? npart[r] : 0;
    int jn[U];
#pragma unroll
    for (int u = 0; u < U; u++) jn[u] = (g + u * G < n) ? __ldg(lst + il_off(g + u * G, skip)) : -1;
    for (int k0 = g; __any_sync(0xffffffffu, k0 < n); k0 += U * G) {
        int j[U];
        double dx[U], dy[U], dz[U], r2[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            j[u] = jn[u];
            LJ_CHECK_THAT(j[u] < n_atoms);
            Lay::pos(q, n_atoms, j[u] >= 0 ? (int64_t)j[u] : i, dx[u], dy[u], dz[u]);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int kn = k0 + U * G + u * G;
            jn[u] = kn < n ? __ldg(lst + il_off(kn, skip)) : -1;
        }
        int hmax = 0;
#pragma unroll
        for (int u = 0; u < U; u++) {
            dx[u] -= qix;
            dy[u] -= qiy;
            dz[u] -= qiz;
            r2[u] = fma(dz[u], dz[u], fma(dy[u], dy[u], dx[u] * dx[u]));
            hmax = max(hmax, __double2hiint(r2[u]));
        }
        if (__any_sync(0xffffffffu, hmax >= c.hi_L2q)) {
#pragma unroll
            for (int u = 0; u < U; u++) {
                dx[u] -= image_shift(dx[u], c.L, c.hi_halfL);
                dy[u] -= image_shift(dy[u], c.L, c.hi_halfL);
                dz[u] -= image_shift(dz[u], c.L, c.hi_halfL);
                r2[u] = fma(dz[u], dz[u], fma(dy[u], dy[u], dx[u] * dx[u]));
            }
        }
        bool inr[U];
        inside_cutoff_u<U>(inr, j, r2, dx, dy, dz, c);
#pragma unroll
        for (int u = 0; u < U; u++) {
            const double inv2 = inv_r2<RCP>(r2[u]);
            const double inv6 = inv2 * inv2 * inv2;
            const bool in = inr[u];
            const double df = in ? fma(c.c48, inv6, -c.c24) * (inv6 * inv2) : 0.0;
            ax = fma(-df, dx[u], ax);
            ay = fma(-df, dy[u], ay);
            az = fma(-df, dz[u], az);
            cnt += in;
        }
    }
    unsigned cnt_row = cnt;
    group_reduce<G>(ax, ay, az, cnt_row);
    if (active && g == 0) {
        *Lay::mom(p, n_atoms, i, 0) += ax;
        *Lay::mom(p, n_atoms, i, 1) += ay;
        *Lay::mom(p, n_atoms, i, 2) += az;
    }
    count_interactions(cnt, n_inter);
}

// Roofline probe: the force kernel's access pattern (G lanes per row, U gathers
// in flight per lane, next indices prefetched, the same warp-uniform chunk loop)
// without the arithmetic.
template <int G, int U, bool IL>
__device__ __forceinline__ double probe_row_loop(const rec4* __restrict__ q, int64_t i,
                                                 const int32_t* __restrict__ lst, int n, int g) {
    constexpr bool LIN = !IL || (G % kIlGran == 0);
    constexpr int F = IL ? kIlRows : 1;
    double s = 0.0;
    int jn[U];
    int ko = eoff<IL>(g);
#pragma unroll
    for (int u = 0; u < U; u++)
        jn[u] = (g + u * G < n) ? __ldg(lst + (LIN ? ko + F * u * G : eoff<IL>(g + u * G))) : -1;
    for (int k0 = g; __any_sync(0xffffffffu, k0 < n); k0 += U * G, ko += F * U * G) {
        rec4 qj[U];
        int j[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            j[u] = jn[u];
            qj[u] = load_rec(q, j[u] >= 0 ? (int64_t)j[u] : i);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int kn = k0 + U * G + u * G;
            jn[u] = kn < n ? __ldg(lst + (LIN ? ko + F * (U * G + u * G) : eoff<IL>(kn))) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; u++) s += j[u] >= 0 ? qj[u].x + qj[u].y + qj[u].z : 0.0;
    }
    return s;
}

template <int G, int U>
__global__ void __launch_bounds__(kForceThreads, U == 2 ? 5 : (U == 3 ? 4 : 3))
    k_gather_probe(const rec4* __restrict__ q, int64_t rows, const int32_t* __restrict__ npart,
                   const int64_t* __restrict__ ptr, const int32_t* __restrict__ list, double* sink) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = t / G;
    const int g = threadIdx.x % G;
    const bool active = r < rows;
    const int64_t i = active ? r : 0;
    const int64_t p0 = active ? ptr[r] : 0;
    const int32_t* __restrict__ lst = list + (p0 & (kIlBit - 1));
    const int n = active ? npart[r] : 0;
    const double s = __any_sync(0xffffffffu, (p0 & kIlBit) != 0) ? probe_row_loop<G, U, true>(q, i, lst, n, g)
                                                                  : probe_row_loop<G, U, false>(q, i, lst, n, g);
    if (s == 1.2345678e300) sink[0] = s;   // never true: keeps the loads alive
}

// The same probe for the vectorised index stream of k_force_idxv (V entries per index load).
template <int G, int V>
__global__ void __launch_bounds__(kForceThreads, V == 2 ? 5 : 3)
    k_gather_probe_idxv(const rec4* __restrict__ q, int64_t rows, const int32_t* __restrict__ npart,
                        const int64_t* __restrict__ ptr, const int32_t* __restrict__ list, double* sink) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = t / G;
    const int g = threadIdx.x % G;
    const bool active = r < rows;
    const int64_t i = active ? r : 0;
    int64_t base = 0;
    int off = 0, end = 0, skip = 0;
    if (active) {
        const int64_t p0 = row_decode(list, ptr[r], skip) - list;   // (interleaved rows: 4-aligned, off = 0)
        base = p0 & ~(int64_t)(V - 1);
        off = (int)(p0 - base);
        end = off + npart[r];
    }
    const int32_t* __restrict__ win = list + base;
    double s = 0.0;
    int jn[V];
    if (V * g < end) {
        IdxVec<V>::load(win + il_off(V * g, skip), jn);
    } else {
#pragma unroll
        for (int u = 0; u < V; u++) jn[u] = -1;
    }
    for (int s0 = V * g; __any_sync(0xffffffffu, s0 < end); s0 += V * G) {
        int j[V];
        rec4 qj[V];
#pragma unroll
        for (int u = 0; u < V; u++) {
            j[u] = (s0 + u >= off && s0 + u < end) ? jn[u] : -1;
            qj[u] = load_rec(q, j[u] >= 0 ? (int64_t)j[u] : i);
        }
        const int sn = s0 + V * G;
        if (sn < end) {
            IdxVec<V>::load(win + il_off(sn, skip), jn);
        } else {
#pragma unroll
            for (int u = 0; u < V; u++) jn[u] = -1;
        }
#pragma unroll
        for (int u = 0; u < V; u++) s += j[u] >= 0 ? qj[u].x + qj[u].y + qj[u].z : 0.0;
    }
    if (s == 1.2345678e300) sink[0] = s;   // never true: keeps the loads alive
}

// Bit-exact "ordered" full-list kernel (DESIGN.md Pin-11): one thread per row,
// ascending j, Alg. 3 accumulating into the loaded p_i, the oracle's expression
// order and IEEE operations (explicit _rn intrinsics: no FMA contraction).
__device__ __forceinline__ double min_image_exact(double d, double L) {
    if (L > 0.0) {
        if (d > 0.5 * L)
            d = __dsub_rn(d, L);
        else if (d < -0.5 * L)
            d = __dadd_rn(d, L);
    }
    return d;
}

__global__ void __launch_bounds__(kForceThreads)
    k_force_ordered(const rec4* __restrict__ q, rec4* __restrict__ p, int64_t row_begin, int64_t rows,
                    const int32_t* __restrict__ npart, const int64_t* __restrict__ ptr,
                    const int32_t* __restrict__ list, double L, double rc2, double dt, unsigned long long* n_inter,
                    int64_t n_atoms) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned cnt = 0;
    if (r < rows) {
        const int64_t i = row_begin + r;
        const rec4 qi = load_rec(q, i);
        rec4 pi = p[i];
        int skip;
        const int32_t* row = row_decode(list, ptr[r], skip);
        const int n = npart[r];
        for (int k = 0; k < n; k++) {
            const int j = row[il_off(k, skip)];
            LJ_CHECK_THAT(j >= 0 && j < n_atoms);
            const rec4 qj = load_rec(q, j);
            double dx = min_image_exact(__dsub_rn(qj.x, qi.x), L);
            double dy = min_image_exact(__dsub_rn(qj.y, qi.y), L);
            double dz = min_image_exact(__dsub_rn(qj.z, qi.z), L);
            double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            if (r2 < rc2) {
                double r6 = __dmul_rn(__dmul_rn(r2, r2), r2);
                double r14 = __dmul_rn(__dmul_rn(r6, r6), r2);
                double df = __ddiv_rn(__dmul_rn(__dsub_rn(48.0, __dmul_rn(24.0, r6)), dt), r14);
                pi.x = __dsub_rn(pi.x, __dmul_rn(df, dx));
                pi.y = __dsub_rn(pi.y, __dmul_rn(df, dy));
                pi.z = __dsub_rn(pi.z, __dmul_rn(df, dz));
                cnt++;
            }
        }
        p[i] = pi;
    }
    count_interactions(cnt, n_inter);
}


template <bool HALF, int U>
cudaError_t launch_g(const ForceArgs& a, int lanes, cudaStream_t s) {
    if (a.rows <= 0) return cudaSuccess;
    PairConsts c = make_consts(a);
    int64_t threads = a.rows * (int64_t)lanes;
    unsigned grid = (unsigned)((threads + kForceThreads - 1) / kForceThreads);
    const rec4* q = (const rec4*)a.q;
    rec4* p = (rec4*)a.p;
#define LJ_LAUNCH(G)                                                                                        \
    k_force<G, U, HALF><<<grid, kForceThreads, 0, s>>>(q, p, a.row_begin, a.rows, a.npart, a.ptr, a.list, c, \
                                                     a.n_inter)
    switch (lanes) {
        case 1: LJ_LAUNCH(1); break;
        case 2: LJ_LAUNCH(2); break;
        case 4: LJ_LAUNCH(4); break;
        case 8: LJ_LAUNCH(8); break;
        case 16: LJ_LAUNCH(16); break;
        case 32: LJ_LAUNCH(32); break;
        default: return cudaErrorInvalidValue;
    }
#undef LJ_LAUNCH
    g_launches++;
    return cudaGetLastError();
}

template <bool HALF, int V>
cudaError_t launch_idxv(const ForceArgs& a, int G, cudaStream_t s) {
    if (a.rows <= 0) return cudaSuccess;
    PairConsts c = make_consts(a);
    const int64_t threads = a.rows * (int64_t)G;
    const unsigned grid = (unsigned)((threads + kForceThreads - 1) / kForceThreads);
    const rec4* q = (const rec4*)a.q;
    rec4* p = (rec4*)a.p;
#define LJ_LAUNCH(GG)                                                                                         \
    k_force_idxv<GG, V, HALF><<<grid, kForceThreads, 0, s>>>(q, p, a.row_begin, a.rows, a.npart, a.ptr, a.list, c, \
                                                           a.n_inter)
    switch (G) {
        case 1: LJ_LAUNCH(1); break;
        case 2: LJ_LAUNCH(2); break;
        case 4: LJ_LAUNCH(4); break;
        case 8: LJ_LAUNCH(8); break;
        case 16: LJ_LAUNCH(16); break;
        default: return cudaErrorInvalidValue;
    }
#undef LJ_LAUNCH
    g_launches++;
    return cudaGetLastError();
}

}  // namespace

// lanes encodes G (1..32) and, in its upper bits, the unroll U (lanes = G | (U << 8); U in {2, 3, 4},
// default 2); with LJ_LANES_IDXV set, U in {2, 4} is the index vector width of k_force_idxv.
template <bool HALF>
cudaError_t launch_gu(const ForceArgs& a, int lanes, cudaStream_t s) {
    const int U = (lanes >> 8) & 0xff;
    const int G = lanes & 0xff;
    if (lanes & LJ_LANES_IDXV) {
        if (U == 4) return launch_idxv<HALF, 4>(a, G, s);
        if (U == 2) return launch_idxv<HALF, 2>(a, G, s);
        return cudaErrorInvalidValue;
    }
    if (U == 4) return launch_g<HALF, 4>(a, G, s);
    if (U == 3) return launch_g<HALF, 3>(a, G, s);
    if (U == 0 || U == 2) return launch_g<HALF, 2>(a, G, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_force_full(const ForceArgs& a, int lanes, cudaStream_t s) { return launch_gu<false>(a, lanes, s); }
cudaError_t launch_force_half(const ForceArgs& a, int lanes, cudaStream_t s) { return launch_gu<true>(a, lanes, s); }

cudaError_t launch_force_half_cells(const ForceArgs& a, const int64_t* cstart, int nc, int lanes, cudaStream_t s) {
    if (a.rows <= 0) return cudaSuccess;
    const int64_t ncell = (int64_t)nc * nc * nc;
    PairConsts c = make_consts(a);
    const size_t smem = sizeof(double) * 3 * kWin;
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<int64_t>(ncell, (int64_t)sms * (1024 / LJ_HC_THREADS) * 8);
    const rec4* q = (const rec4*)a.q;
    rec4* p = (rec4*)a.p;
#define LJ_HC(G, U) k_force_half_cells<G, U, LJ_HC_THREADS><<<grid, LJ_HC_THREADS, smem, s>>>( \
        q, p, a.npart, a.ptr, a.list, cstart, nc, ncell, c, a.n_inter)
    switch (lanes) {
        case 4 | (2 << 8): LJ_HC(4, 2); break;
        case 0:
        case 8 | (2 << 8): LJ_HC(8, 2); break;
        case 4 | (3 << 8): LJ_HC(4, 3); break;
        case 2 | (2 << 8): LJ_HC(2, 2); break;
        default: return cudaErrorInvalidValue;
    }
#undef LJ_HC
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_gather_probe(const ForceArgs& a, int lanes, double* sink, cudaStream_t s) {
    if (a.rows <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((a.rows * (int64_t)(lanes & 0xff) + kForceThreads - 1) / kForceThreads);
    const rec4* q = (const rec4*)a.q;
#define LJ_PROBE(G, U) k_gather_probe<G, U><<<grid, kForceThreads, 0, s>>>(q, a.rows, a.npart, a.ptr, a.list, sink)
#define LJ_PROBEV(G, V) \
    k_gather_probe_idxv<G, V><<<grid, kForceThreads, 0, s>>>(q, a.rows, a.npart, a.ptr, a.list, sink)
    switch (lanes) {
        case 2 | (2 << 8) | LJ_LANES_IDXV: LJ_PROBEV(2, 2); break;
        case 4 | (2 << 8) | LJ_LANES_IDXV: LJ_PROBEV(4, 2); break;
        case 8 | (2 << 8) | LJ_LANES_IDXV: LJ_PROBEV(8, 2); break;
        case 2 | (4 << 8) | LJ_LANES_IDXV: LJ_PROBEV(2, 4); break;
        case 4 | (4 << 8) | LJ_LANES_IDXV: LJ_PROBEV(4, 4); break;
        case 8 | (4 << 8) | LJ_LANES_IDXV: LJ_PROBEV(8, 4); break;
        case 16 | (4 << 8) | LJ_LANES_IDXV: LJ_PROBEV(16, 4); break;
        case 2 | (2 << 8): LJ_PROBE(2, 2); break;
        case 2 | (3 << 8): LJ_PROBE(2, 3); break;
        case 8 | (4 << 8): LJ_PROBE(8, 4); break;
        case 4 | (4 << 8): LJ_PROBE(4, 4); break;
        case 16 | (3 << 8): LJ_PROBE(16, 3); break;
        case 4 | (2 << 8): LJ_PROBE(4, 2); break;
        case 4 | (3 << 8): LJ_PROBE(4, 3); break;
        case 8 | (2 << 8): LJ_PROBE(8, 2); break;
        case 8 | (3 << 8): LJ_PROBE(8, 3); break;
        case 16 | (2 << 8): LJ_PROBE(16, 2); break;
        default: return cudaErrorInvalidValue;
    }
#undef LJ_PROBE
#undef LJ_PROBEV
    g_launches++;
    return cudaGetLastError();
}

template <int G, int LAYOUT>
static cudaError_t launch_variant_rcp(const ForceArgs& a, int64_t n, int rcp, unsigned grid, PairConsts c,
                                      cudaStream_t s) {
#define LJ_V(R)                                                                                                 \
    k_force_variant<G, LAYOUT, R><<<grid, kForceThreads, 0, s>>>(a.q, a.p, n, a.row_begin, a.rows, a.npart, a.ptr, \
                                                                 a.list, c, a.n_inter)
    switch (rcp) {
        case LJ_RCP_NEWTON3: LJ_V(LJ_RCP_NEWTON3); break;
        case LJ_RCP_NEWTON2: LJ_V(LJ_RCP_NEWTON2); break;
        case LJ_RCP_APPROX: LJ_V(LJ_RCP_APPROX); break;
        case LJ_RCP_IEEE: LJ_V(LJ_RCP_IEEE); break;
        default: return cudaErrorInvalidValue;
    }
#undef LJ_V
    return cudaGetLastError();
}

template <int G>
static cudaError_t launch_variant_g(const ForceArgs& a, int64_t n, int layout, int rcp, unsigned grid, PairConsts c,
                                    cudaStream_t s) {
    switch (layout) {
        case LJ_LAYOUT_AOS4: return launch_variant_rcp<G, LJ_LAYOUT_AOS4>(a, n, rcp, grid, c, s);
        case LJ_LAYOUT_SOA: return launch_variant_rcp<G, LJ_LAYOUT_SOA>(a, n, rcp, grid, c, s);
        case LJ_LAYOUT_AOS3: return launch_variant_rcp<G, LJ_LAYOUT_AOS3>(a, n, rcp, grid, c, s);
        case LJ_LAYOUT_AOS8: return launch_variant_rcp<G, LJ_LAYOUT_AOS8>(a, n, rcp, grid, c, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_force_variant(const ForceArgs& a, int64_t n, int layout, int rcp, int lanes, cudaStream_t s) {
    if (a.rows <= 0) return cudaSuccess;
    PairConsts c = make_consts(a);
    const unsigned grid = (unsigned)((a.rows * (int64_t)lanes + kForceThreads - 1) / kForceThreads);
    cudaError_t e = lanes == 4 ? launch_variant_g<4>(a, n, layout, rcp, grid, c, s)
                  : lanes == 8 ? launch_variant_g<8>(a, n, layout, rcp, grid, c, s)
                               : cudaErrorInvalidValue;
    g_launches++;
    return e;
}

cudaError_t launch_force_ordered(const ForceArgs& a, cudaStream_t s) {
    if (a.rows <= 0) return cudaSuccess;
    unsigned grid = (unsigned)((a.rows + kForceThreads - 1) / kForceThreads);
    k_force_ordered<<<grid, kForceThreads, 0, s>>>((const rec4*)a.q, (rec4*)a.p, a.row_begin, a.rows, a.npart, a.ptr,
                                                   a.list, a.L, a.rc2, a.dt, a.n_inter, a.n);
    g_launches++;
    return cudaGetLastError();
}

}  // namespace lj
