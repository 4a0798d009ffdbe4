// Streaming kernels around the force step:
// AoS4 pack/unpack, drift, wrap + bookkeeping snapshot, max displacement, energy.
// All are HBM-streaming (one pass over 32-B records); integrate, wrap and the
// displacement are bit-identical to the oracle (explicit _rn intrinsics).
#include <climits>

#include "lj_internal.cuh"

namespace lj {

namespace {

constexpr int kThreads = 256;

__global__ void k_pack(const double* __restrict__ xyz, rec4* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        rec4 r;
        r.x = xyz[3 * i];
        r.y = xyz[3 * i + 1];
        r.z = xyz[3 * i + 2];
        r.w = 0.0;
        out[i] = r;
    }
}

__global__ void k_unpack(const rec4* __restrict__ in, double* __restrict__ xyz, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        rec4 r = in[i];
        xyz[3 * i] = r.x;
        xyz[3 * i + 1] = r.y;
        xyz[3 * i + 2] = r.z;
    }
}

// q_i += p_i dt (mass 1), same rounding as the oracle: q + (p*dt), no FMA.
__global__ void k_integrate(rec4* __restrict__ q, const rec4* __restrict__ p, int64_t begin, int64_t end,
                            double dt) {
    for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        rec4 a = q[i];
        const rec4 b = p[i];
        a.x = __dadd_rn(a.x, __dmul_rn(b.x, dt));
        a.y = __dadd_rn(a.y, __dmul_rn(b.y, dt));
        a.z = __dadd_rn(a.z, __dmul_rn(b.z, dt));
        q[i] = a;
    }
}

// Drift fused with the bookkeeping displacement (one pass over the own rows):
// q_i += p_i dt exactly as k_integrate, then |q_i - q_ref_i| exactly as k_max_disp.
__global__ void k_integrate_disp(rec4* __restrict__ q, const rec4* __restrict__ p, const rec4* __restrict__ q_ref,
                                 int64_t begin, int64_t end, double dt, unsigned long long* out);

__device__ __forceinline__ double wrap1(double x, double L) {
    double w = __dsub_rn(x, __dmul_rn(L, floor(__ddiv_rn(x, L))));
    if (w >= L) w = __dsub_rn(w, L);
    return w;
}

__global__ void k_wrap(rec4* __restrict__ q, rec4* __restrict__ q_ref, int64_t n, double L) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        rec4 a = q[i];
        a.x = wrap1(a.x, L);
        a.y = wrap1(a.y, L);
        a.z = wrap1(a.z, L);
        q[i] = a;
        if (q_ref) q_ref[i] = a;
    }
}

__device__ __forceinline__ double block_max(double v) {
    __shared__ double s[32];
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) s[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < (int)(blockDim.x >> 5) ? s[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    return v;
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double s[32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) s[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < (int)(blockDim.x >> 5) ? s[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}

// max_i |q_i - q_ref_i| (Euclidean, sqrt((dx*dx + dy*dy) + dz*dz) as the oracle).
// Non-negative doubles order like their bit patterns -> atomicMax on uint64.
__global__ void k_max_disp(const rec4* __restrict__ q, const rec4* __restrict__ q_ref, int64_t begin, int64_t end,
                           unsigned long long* out) {
    double m = 0.0;
    for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        const rec4 a = q[i], b = q_ref[i];
        double dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y), dz = __dsub_rn(a.z, b.z);
        double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
        m = fmax(m, d);
    }
    m = block_max(m);
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_integrate_disp(rec4* __restrict__ q, const rec4* __restrict__ p, const rec4* __restrict__ q_ref,
                                 int64_t begin, int64_t end, double dt, unsigned long long* out) {
    double m = 0.0;
    for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        rec4 a = q[i];
        const rec4 b = p[i];
        a.x = __dadd_rn(a.x, __dmul_rn(b.x, dt));
        a.y = __dadd_rn(a.y, __dmul_rn(b.y, dt));
        a.z = __dadd_rn(a.z, __dmul_rn(b.z, dt));
        q[i] = a;
        const rec4 r = q_ref[i];
        double dx = __dsub_rn(a.x, r.x), dy = __dsub_rn(a.y, r.y), dz = __dsub_rn(a.z, r.z);
        m = fmax(m, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz))));
    }
    m = block_max(m);
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// k_integrate_disp with the position exchange fused in:
// the thread that computes q_out_i also stores it into every push target whose
// row range holds i (a q replica of another rank, peer-mapped over NVLink), so
// the transfer is spread over the whole drift instead of following it.  The
// targets ride in the kernel's parameter space (__grid_constant__).
struct PushTargets {
    int n;
    lj_push_target t[LJ_MAX_PUSH_TARGETS];
};

__global__ void k_integrate_push(const rec4* q_in, rec4* q_out, const rec4* __restrict__ p,   // q_in may be q_out
                                 const rec4* __restrict__ q_ref, int64_t begin, int64_t end, double dt,
                                 unsigned long long* out, const __grid_constant__ PushTargets T) {
    double m = 0.0;
    for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end;
         i += (int64_t)gridDim.x * blockDim.x) {
        rec4 a = q_in[i];
        const rec4 b = p[i];
        a.x = __dadd_rn(a.x, __dmul_rn(b.x, dt));
        a.y = __dadd_rn(a.y, __dmul_rn(b.y, dt));
        a.z = __dadd_rn(a.z, __dmul_rn(b.z, dt));
        q_out[i] = a;
        for (int k = 0; k < T.n; k++)
            if (i >= T.t[k].lo && i < T.t[k].hi) reinterpret_cast<rec4*>(T.t[k].dst)[i] = a;
        const rec4 r = q_ref[i];
        double dx = __dsub_rn(a.x, r.x), dy = __dsub_rn(a.y, r.y), dz = __dsub_rn(a.z, r.z);
        m = fmax(m, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz))));
    }
    __threadfence_system();   // the peer stores are visible system-wide once the kernel has completed
    m = block_max(m);
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// ---- device-side step control (CUDA graph with a conditional rebuild) ------
// The bookkeeping decision of the MD step (reading C-16: rebuild when
// 2 max|q - q_ref| >= r_s - r_c) taken on the device: sets the graph's IF
// condition and counts rebuilds in status[0].
__global__ void k_md_decide(const double* __restrict__ disp, int count, int64_t stride, double margin,
                            cudaGraphConditionalHandle h, int64_t* status) {
    double m = disp[0];
    for (int k = 1; k < count; k++) m = fmax(m, disp[k * stride]);
    const bool r = 2.0 * m >= margin;
    cudaGraphSetConditional(h, r ? 1u : 0u);
    if (r) status[0] += 1;
}

// A build inside a graph: its entry count to status[2], a row over the padded
// stride to status[1] (sticky).
__global__ void k_build_status(const int64_t* __restrict__ total, const int32_t* __restrict__ row_overflow,
                               int64_t* status) {
    status[2] = *total;
    if (row_overflow && *row_overflow) status[1] = 1;
}

// KE over own rows and shifted PE (reading O7) over the list entries inside r_c.
// G = 8 lanes per row (as the force kernel: one 256-bit record gather per
// entry, coalesced index loads), the cutoff on the oracle's r^2 (no FMA), the
// minimum image as the oracle's branches; per-lane sums reduced per block.
constexpr int kEnergyLanes = 8;
__global__ void __launch_bounds__(kThreads)
    k_energy(const rec4* __restrict__ q, const rec4* __restrict__ p, int64_t n_atoms, int64_t row_begin, int64_t rows,
             const int32_t* __restrict__ npart, const int64_t* __restrict__ ptr, const int32_t* __restrict__ list,
             double L, double rc2, double vc, int half, double* out) {
    constexpr int G = kEnergyLanes;
    double ke = 0.0, pe = 0.0;
    const double halfL = 0.5 * L;
    const double w = half ? 1.0 : 0.5;
    const int g = threadIdx.x % G;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) / G) {
        const int64_t i = row_begin + r;
        const rec4 qi = load_rec(q, i);
        if (g == 0) {
            const rec4 pi = p[i];
            ke += 0.5 * __dadd_rn(__dadd_rn(__dmul_rn(pi.x, pi.x), __dmul_rn(pi.y, pi.y)), __dmul_rn(pi.z, pi.z));
        }
        int skip;
        const int32_t* __restrict__ l = row_decode(list, ptr[r], skip);
        const int n = npart[r];
        for (int k = g; k < n; k += G) {
            const int j = __ldg(l + il_off(k, skip));
            LJ_CHECK_THAT(j >= 0 && j < n_atoms);
            const rec4 qj = load_rec(q, j);
            double dx = qj.x - qi.x, dy = qj.y - qi.y, dz = qj.z - qi.z;
            if (L > 0.0) {
                dx = dx > halfL ? dx - L : (dx < -halfL ? dx + L : dx);
                dy = dy > halfL ? dy - L : (dy < -halfL ? dy + L : dy);
                dz = dz > halfL ? dz - L : (dz < -halfL ? dz + L : dz);
            }
            // the oracle's r^2 (reading O3, no FMA): the same pairs inside r_c
            const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            if (r2 < rc2) {
                const double inv6 = 1.0 / (r2 * r2 * r2);
                pe += w * (4.0 * (inv6 * inv6 - inv6) - vc);
            }
        }
    }
    ke = block_sum(ke);
    pe = block_sum(pe);
    if (threadIdx.x == 0) {
        atomicAdd(&out[0], ke);
        atomicAdd(&out[1], pe);
    }
}

// Interior rows for comm/compute overlap: row r is
// "boundary" if some partner lies outside [row_begin, row_end).  out[0] =
// max{i < mid : boundary} (init row_begin - 1), out[1] = min{i >= mid :
// boundary} (init row_end); [out[0] + 1, out[1]) is then the contiguous run of
// interior rows around mid = (row_begin + row_end) / 2.  One warp per row.
__global__ void k_list_interior(int64_t row_begin, int64_t row_end, const int32_t* __restrict__ npart,
                                const int64_t* __restrict__ ptr, const int32_t* __restrict__ list,
                                unsigned long long* out) {
    const int lane = threadIdx.x & 31;
    const int64_t mid = (row_begin + row_end) / 2;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < row_end - row_begin;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int n = npart[r];
        int skip;
        const int32_t* l = row_decode(list, ptr[r], skip);
        bool out_of_slab = false;
        for (int k = lane; k < n; k += 32) {
            const int j = l[il_off(k, skip)];
            out_of_slab |= j < row_begin || j >= row_end;
        }
        if (__any_sync(0xffffffffu, out_of_slab) && lane == 0) {
            const int64_t i = row_begin + r;
            if (i < mid)
                atomicMax(&out[0], (unsigned long long)(i + 1));   // stored +1 so that "none" = row_begin
            else
                atomicMin(&out[1], (unsigned long long)i);
        }
    }
}

// Halo requests: for every owner slab s (rows
// [bounds[s], bounds[s+1])), the smallest and largest partner index of the own
// rows that falls in it.  Partners of a row ascend, so each owner's entries in a
// row are one contiguous run: a warp scans its row, lanes reduce per owner in
// shared memory, one global atomic per block and owner.
constexpr int kMaxRanks = 64;

__global__ void k_partner_ranges(int64_t row_begin, int64_t row_end, const int32_t* __restrict__ npart,
                                 const int64_t* __restrict__ ptr, const int32_t* __restrict__ list,
                                 const int64_t* __restrict__ bounds, int P, long long* out) {
    __shared__ long long s_lo[kMaxRanks], s_hi[kMaxRanks];
    __shared__ long long s_b[kMaxRanks + 1];
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
        s_lo[k] = LLONG_MAX;
        s_hi[k] = -1;
    }
    for (int k = threadIdx.x; k <= P; k += blockDim.x) s_b[k] = bounds[k];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < row_end - row_begin;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int n = npart[r];
        int skip;
        const int32_t* l = row_decode(list, ptr[r], skip);
        int prev_owner = -1;   // owner of the entry before this chunk (warp-uniform)
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            const long long j = k < n ? l[il_off(k, skip)] : -1;
            int own = -1;
            if (k < n) {
                int lo = 0, hi = P;   // owner: largest s with s_b[s] <= j
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_b[mid] <= j) lo = mid; else hi = mid;
                }
                own = lo;
            }
            // ascending entries: one owner's entries are a contiguous run -- only run
            // starts and ends touch the shared minima and maxima
            int before = __shfl_up_sync(0xffffffffu, own, 1);
            if (lane == 0) before = prev_owner;
            int after = __shfl_down_sync(0xffffffffu, own, 1);
            if (lane == 31 || k + 1 >= n) after = -2;
            if (own >= 0 && own != before) atomicMin(&s_lo[own], j);
            if (own >= 0 && own != after) atomicMax(&s_hi[own], j);
            prev_owner = __shfl_sync(0xffffffffu, own, 31);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
        if (s_hi[k] >= 0) {
            atomicMin(&out[2 * k], s_lo[k]);
            atomicMax(&out[2 * k + 1], s_hi[k]);
        }
    }
}

__global__ void k_init_ranges(long long* out, int P) {
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
        out[2 * k] = LLONG_MAX;
        out[2 * k + 1] = -1;
    }
}

__global__ void k_init_interior(unsigned long long* out, int64_t row_begin, int64_t row_end) {
    out[0] = (unsigned long long)row_begin;
    out[1] = (unsigned long long)row_end;
}

}  // namespace

cudaError_t launch_list_interior(int64_t row_begin, int64_t row_end, const int32_t* npart, const int64_t* ptr,
                                 const int32_t* list, int64_t* out, cudaStream_t s) {
    k_init_interior<<<1, 1, 0, s>>>((unsigned long long*)out, row_begin, row_end);
    g_launches++;
    if (row_end > row_begin) {
        k_list_interior<<<grid_for((row_end - row_begin) * 32, kThreads, 148 * 16), kThreads, 0, s>>>(
            row_begin, row_end, npart, ptr, list, (unsigned long long*)out);
        g_launches++;
    }
    return cudaGetLastError();
}

cudaError_t launch_partner_ranges(int64_t row_begin, int64_t row_end, const int32_t* npart, const int64_t* ptr,
                                  const int32_t* list, const int64_t* bounds, int P, int64_t* out, cudaStream_t s) {
    if (P < 1 || P > kMaxRanks) return cudaErrorInvalidValue;
    k_init_ranges<<<1, 64, 0, s>>>((long long*)out, P);
    g_launches++;
    if (row_end > row_begin) {
        k_partner_ranges<<<grid_for((row_end - row_begin) * 32, kThreads, 148 * 8), kThreads, 0, s>>>(
            row_begin, row_end, npart, ptr, list, bounds, P, (long long*)out);
        g_launches++;
    }
    return cudaGetLastError();
}

cudaError_t launch_pack(const double* xyz, double* out, int64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_pack<<<grid_for(n, kThreads), kThreads, 0, s>>>(xyz, (rec4*)out, n);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_unpack(const double* in, double* xyz, int64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_unpack<<<grid_for(n, kThreads), kThreads, 0, s>>>((const rec4*)in, xyz, n);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_integrate(double* q, const double* p, int64_t begin, int64_t end, double dt, cudaStream_t s) {
    if (end <= begin) return cudaSuccess;
    k_integrate<<<grid_for(end - begin, kThreads), kThreads, 0, s>>>((rec4*)q, (const rec4*)p, begin, end, dt);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_integrate_disp(double* q, const double* p, const double* q_ref, int64_t begin, int64_t end,
                                  double dt, double* out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
    if (e != cudaSuccess || end <= begin) return e;
    k_integrate_disp<<<grid_for(end - begin, kThreads, 148 * 8), kThreads, 0, s>>>(
        (rec4*)q, (const rec4*)p, (const rec4*)q_ref, begin, end, dt, (unsigned long long*)out);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_integrate_push(const double* q_in, double* q_out, const double* p, const double* q_ref,
                                  int64_t begin, int64_t end, double dt, double* out, const lj_push_target* t,
                                  int n_targets, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
    if (e != cudaSuccess || end <= begin) return e;
    PushTargets T;
    T.n = n_targets;
    for (int k = 0; k < n_targets; k++) T.t[k] = t[k];
    k_integrate_push<<<grid_for(end - begin, kThreads, 148 * 8), kThreads, 0, s>>>(
        (const rec4*)q_in, (rec4*)q_out, (const rec4*)p, (const rec4*)q_ref, begin, end, dt,
        (unsigned long long*)out, T);
    g_launches++;
    return cudaGetLastError();
}

__global__ void k_copy_scalar(const double* __restrict__ src, double* dst) { dst[0] = src[0]; }

cudaError_t launch_copy_scalar(const double* src, double* dst, cudaStream_t s) {
    k_copy_scalar<<<1, 1, 0, s>>>(src, dst);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_md_decide(const double* disp, int count, int64_t stride, double margin,
                             cudaGraphConditionalHandle h, int64_t* status, cudaStream_t s) {
    k_md_decide<<<1, 1, 0, s>>>(disp, count, stride, margin, h, status);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_build_status(const int64_t* total, const int32_t* row_overflow, int64_t* status, cudaStream_t s) {
    k_build_status<<<1, 1, 0, s>>>(total, row_overflow, status);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_wrap(double* q, double* q_ref, int64_t n, double L, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_wrap<<<grid_for(n, kThreads), kThreads, 0, s>>>((rec4*)q, (rec4*)q_ref, n, L);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_max_disp(const double* q, const double* q_ref, int64_t begin, int64_t end, double* out,
                            cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), s);
    if (e != cudaSuccess || end <= begin) return e;
    k_max_disp<<<grid_for(end - begin, kThreads, 148 * 8), kThreads, 0, s>>>(
        (const rec4*)q, (const rec4*)q_ref, begin, end, (unsigned long long*)out);
    g_launches++;
    return cudaGetLastError();
}

cudaError_t launch_energy(const double* q, const double* p, int64_t n, int64_t row_begin, int64_t rows,
                          const int32_t* npart,
                          const int64_t* ptr, const int32_t* list, double L, double rc2, double rc, int half,
                          double* out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(double), s);
    if (e != cudaSuccess || rows <= 0) return e;
    double rc6 = rc2 * rc2 * rc2;
    double vc = 4.0 * (1.0 / (rc6 * rc6) - 1.0 / rc6);
    k_energy<<<grid_for(rows * kEnergyLanes, kThreads, 148 * 8), kThreads, 0, s>>>(
        (const rec4*)q, (const rec4*)p, n, row_begin, rows, npart, ptr, list, L, rc2, vc, half, out);
    g_launches++;
    return cudaGetLastError();
}

}  // namespace lj
