// The force step's per-pair and per-row device code, shared by the force kernels
// (lj_force.cu) and the list builder's fused force (lj_list.cu, k_list_v4 with
// ListArgs::ff: the kick of the step after a rebuild, computed per cell right
// after the cell's rows are built).  (Product code only -- nothing here is shared
// with oracle/.)
#pragma once

#include <climits>

#include "lj_internal.cuh"

namespace lj {

struct PairConsts {
    double L;        // box side (0 = open)
    double c48, c24; // 48 dt, 24 dt
    double rc2;      // r_c^2 = rc*rc (the oracle's constant)
    int64_t n_atoms; // (bounds checks of the LJ_CHECK build)
    long long rc2_bits;
    int rc2_hi;      // high word of rc2's IEEE bits
    int hi_halfL;    // high word of L/2 (INT_MAX for open boundaries)
    int hi_L2q;      // high word of (L/2)^2: r^2 below it needs no image (INT_MAX for open boundaries)
};

__device__ __forceinline__ double fast_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    return fma(y, fma(e, e, e), y);
}

// The cutoff test on the oracle's r^2 (readings O3/C-4: r2 = (dx*dx + dy*dy) + dz*dz
// without FMA, interact iff r2 < rc2).  The kernels evaluate r^2 with FMAs
// (fma(dz, dz, fma(dy, dy, dx*dx))), which differs from the oracle's rounding by
// at most a few ulp.  The decision is taken on the HIGH words of the IEEE bits
// (r^2 > 0, so bit order = value order): hi(r2) < hi(rc2) - 1 is inside and
// hi(r2) > hi(rc2) + 1 outside for either rounding (they are >= 2^32 ulp from
// rc2); the ~3e-6-relative window in between -- ~5e-6 of the entries of the
// workloads -- is re-evaluated on the oracle's expression with explicit _rn
// operations, so the set of interacting pairs is the oracle's bit for bit.
__device__ __forceinline__ bool inside_cutoff(double r2, double dx, double dy, double dz, const PairConsts& c) {
    const int dh = __double2hiint(r2) - c.rc2_hi;
    if ((unsigned)(dh + 1) > 2u) return dh < 0;
    const double r2e = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return r2e < c.rc2;
}
// The same for U entries at once: the common decision on the high words, the
// exact re-evaluation in one rarely taken block (keeps the hot loop's registers).
template <int U>
__device__ __forceinline__ void inside_cutoff_u(bool (&in)[U], const int (&j)[U], const double (&r2)[U],
                                                const double (&dx)[U], const double (&dy)[U], const double (&dz)[U],
                                                const PairConsts& c) {
    bool near = false;
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int dh = __double2hiint(r2[u]) - c.rc2_hi;
        in[u] = j[u] >= 0 && dh < 0;
        near |= (unsigned)(dh + 1) <= 2u;
    }
    if (__builtin_expect(near, 0)) {
#pragma unroll
        for (int u = 0; u < U; u++) in[u] = j[u] >= 0 && inside_cutoff(r2[u], dx[u], dy[u], dz[u], c);
    }
}

// Periodic image shift of a raw difference: +-L when |d| > L/2 (decided on the
// high words, up to the low word -- pairs that close to L/2 are never within r_c).
__device__ __forceinline__ double image_shift(double d, double L, int hi_halfL) {
    int hi = __double2hiint(d);
    double s = ((hi & 0x7fffffff) > hi_halfL) ? L : 0.0;
    return hi < 0 ? -s : s;
}

template <int G>
__device__ __forceinline__ void group_reduce(double& ax, double& ay, double& az, unsigned& cnt) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        ax += __shfl_xor_sync(0xffffffffu, ax, o);
        ay += __shfl_xor_sync(0xffffffffu, ay, o);
        az += __shfl_xor_sync(0xffffffffu, az, o);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
}

__device__ __forceinline__ void count_interactions(unsigned cnt, unsigned long long* n_inter) {
    if (n_inter == nullptr) return;
    unsigned long long v = cnt;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(n_inter, v);
}

// Offset of a row's entry e from the row base: e (compact and padded lists) or, in
// the interleaved layout (LJ_LIST_INTERLEAVED), e + 28 (e / 4).  For G % 4 == 0 the
// entries a lane reads are e and e + d with d a multiple of 4, whose interleaved
// offsets differ by 8 d: the chunk loop then keeps compile-time load offsets in
// both layouts (LIN below) and the interleaved list costs no extra instructions.
template <bool IL>
__device__ __forceinline__ int eoff(int e) {
    return IL ? e + kIlSkip * (e >> 2) : e;
}

// One row's chunk loop of k_force (a G-lane group; accumulates into ax..cnt).
// NC: the index stream through the read-only (non-coherent) path, as in k_force; false for
// list entries written earlier in the same kernel (the builder's fused force).
template <bool NC>
__device__ __forceinline__ int load_index(const int32_t* a) {
    if (NC) return __ldg(a);
    int v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(a));
    return v;
}

template <int G, int U, bool HALF, bool IL, bool NC = true>
__device__ __forceinline__ void force_row_loop(const rec4* __restrict__ q, rec4* __restrict__ p, int64_t i,
                                               const rec4& qi, const int32_t* __restrict__ lst, int n, int g,
                                               const PairConsts& c, double& ax, double& ay, double& az,
                                               unsigned& cnt) {
    constexpr bool LIN = !IL || (G % kIlGran == 0);   // offsets linear in the entry index
    constexpr int F = IL ? kIlRows : 1;               // (LIN) offset step per entry
    // software pipeline (the GPU analogue of the paper's SWP): the
    // indices of chunk k+1 are loaded before the records of chunk k are used
    int jn[U];
    int ko = eoff<IL>(g);   // offset of entry k0 (LIN)
#pragma unroll
    for (int u = 0; u < U; u++)
        jn[u] = (g + u * G < n) ? load_index<NC>(lst + (LIN ? ko + F * u * G : eoff<IL>(g + u * G))) : -1;
    for (int k0 = g; __any_sync(0xffffffffu, k0 < n); k0 += U * G, ko += F * U * G) {
        int j[U];
        rec4 qj[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            j[u] = jn[u];
            LJ_CHECK_THAT(j[u] < c.n_atoms);
            qj[u] = load_rec(q, j[u] >= 0 ? (int64_t)j[u] : i);   // no entry: r = 0, masked below
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int kn = k0 + U * G + u * G;
            jn[u] = kn < n ? load_index<NC>(lst + (LIN ? ko + F * (U * G + u * G) : eoff<IL>(kn))) : -1;
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
        auto accumulate = [&]() {
            bool inr[U];
            inside_cutoff_u<U>(inr, j, r2, dx, dy, dz, c);
#pragma unroll
            for (int u = 0; u < U; u++) {
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
        // (the tail is duplicated in both branches so that the common path keeps r^2)
        if (__any_sync(0xffffffffu, hmax >= c.hi_L2q)) {   // some pair may need a periodic image
#pragma unroll
            for (int u = 0; u < U; u++) {
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
}


inline PairConsts make_consts(const ForceArgs& a) {
    PairConsts c;
    c.L = a.L;
    c.c48 = 48.0 * a.dt;
    c.c24 = 24.0 * a.dt;
    union {
        double d;
        long long b;
    } u;
    u.d = a.rc2;
    c.rc2_bits = u.b;
    c.rc2_hi = (int)(u.b >> 32);
    c.rc2 = a.rc2;
    c.n_atoms = a.n;
    if (a.L > 0.0) {
        u.d = 0.5 * a.L;
        c.hi_halfL = (int)(u.b >> 32);
        u.d = 0.25 * a.L * a.L;
        c.hi_L2q = (int)(u.b >> 32);
    } else {
        c.hi_halfL = INT_MAX;
        c.hi_L2q = INT_MAX;
    }
    return c;
}


}  // namespace lj
