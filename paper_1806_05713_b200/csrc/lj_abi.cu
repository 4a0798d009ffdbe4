// extern "C" boundary of liblj.so (include/liblj.h): argument validation,
// error mapping, workspace carving, launch bookkeeping.  No allocation here.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "lj_internal.cuh"

namespace lj {
std::atomic<long long> g_launches{0};
}

using namespace lj;

namespace {

thread_local std::string t_last_error;

lj_status fail(lj_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
lj_status fail(lj_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    t_last_error = buf;
    return s;
}

lj_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return LJ_OK;
    return fail(LJ_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

bool aligned32(const void* p) { return ((uintptr_t)p & 31u) == 0; }

lj_status check_geom(const lj_geom& g, bool need_box) {
    if (!(g.rc > 0.0) || !(g.rs > g.rc) || !std::isfinite(g.rs))
        return fail(LJ_ERR_ARG, "geometry: need 0 < rc < rs (rc=%g rs=%g)", g.rc, g.rs);
    if (!(g.L >= 0.0) || !std::isfinite(g.L)) return fail(LJ_ERR_ARG, "geometry: L must be >= 0 (L=%g)", g.L);
    if (g.L > 0.0 && std::floor(g.L / g.rs) < 3.0)
        return fail(LJ_ERR_ARG, "geometry: floor(L/rs) must be >= 3 (L=%g rs=%g)", g.L, g.rs);
    if (need_box && !(g.L > 0.0))
        return fail(LJ_ERR_UNSUPPORTED, "list construction needs a periodic box (L > 0)");
    return LJ_OK;
}

lj_status check_n(int64_t n) {
    if (n < 0 || n > (int64_t)INT32_MAX) return fail(LJ_ERR_ARG, "n=%lld out of range [0, 2^31)", (long long)n);
    return LJ_OK;
}

lj_status check_rows(int64_t n, int64_t b, int64_t e) {
    if (b < 0 || b > e || e > n)
        return fail(LJ_ERR_ARG, "row range [%lld,%lld) not within [0,%lld]", (long long)b, (long long)e, (long long)n);
    return LJ_OK;
}

CellGrid make_grid(const lj_geom& g) {
    CellGrid cg;
    cg.L = g.L;
    cg.nc = (int)std::floor(g.L / g.rs);
    cg.inv_w = (double)cg.nc / g.L;
    cg.ncell = (int64_t)cg.nc * cg.nc * cg.nc;
    return cg;
}

#define LJ_TRY(x)                      \
    do {                               \
        lj_status _s = (x);            \
        if (_s != LJ_OK) return _s;    \
    } while (0)

#define LJ_CUDA(x, where)                                 \
    do {                                                  \
        cudaError_t _e = (x);                             \
        if (_e != cudaSuccess) return cuda_status(_e, where); \
    } while (0)

}  // namespace

extern "C" {

const char* lj_version(void) { return "liblj 0.1 (sm_100a, fp64)"; }

long long lj_launch_count(void) { return g_launches.load(); }

const char* lj_last_error(void) { return t_last_error.c_str(); }

const char* lj_status_string(lj_status s) {
    switch (s) {
        case LJ_OK: return "LJ_OK";
        case LJ_ERR_ARG: return "LJ_ERR_ARG";
        case LJ_ERR_CAPACITY: return "LJ_ERR_CAPACITY";
        case LJ_ERR_CUDA: return "LJ_ERR_CUDA";
        case LJ_ERR_UNSUPPORTED: return "LJ_ERR_UNSUPPORTED";
    }
    return "LJ_UNKNOWN";
}

lj_status lj_pack_aos4(const double* xyz, double* out, int64_t n, void* stream) {
    LJ_TRY(check_n(n));
    if (n > 0 && (!xyz || !out)) return fail(LJ_ERR_ARG, "pack: null pointer");
    if (!aligned32(out)) return fail(LJ_ERR_ARG, "pack: output not 32-byte aligned");
    LJ_CUDA(launch_pack(xyz, out, n, (cudaStream_t)stream), "lj_pack_aos4");
    return LJ_OK;
}

lj_status lj_unpack_aos4(const double* in, double* xyz, int64_t n, void* stream) {
    LJ_TRY(check_n(n));
    if (n > 0 && (!xyz || !in)) return fail(LJ_ERR_ARG, "unpack: null pointer");
    if (!aligned32(in)) return fail(LJ_ERR_ARG, "unpack: input not 32-byte aligned");
    LJ_CUDA(launch_unpack(in, xyz, n, (cudaStream_t)stream), "lj_unpack_aos4");
    return LJ_OK;
}

lj_status lj_build_list_workspace(int64_t n, lj_geom g, size_t* bytes) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(g, true));
    if (!bytes) return fail(LJ_ERR_ARG, "workspace: null output");
    CellGrid cg = make_grid(g);
    *bytes = build_workspace_layout(n, cg.ncell, n).total;   // sized for all rows
    return LJ_OK;
}

namespace {
// What precedes the list passes: the plain cell pass over q (lj_build_list) or
// the fused wrap + cells + permutation of lj_rebuild (the list is then built
// over q_out, the permuted system).
struct RebuildIO {
    double* q;   // wrapped in place
    const double* p;
    double *q_out, *p_out, *q_ref;
    int64_t* perm;
    PeerMomenta pm;   // momenta from every rank's copy of its own rows (multi-rank re-sort), else p
};

lj_status build_list_impl(const double* q, int64_t n, lj_geom g, int half, int64_t row_begin, int64_t row_end,
                          int flags, int32_t* number_of_partners, int64_t* pointer, int32_t* sorted_list,
                          int64_t capacity, int64_t* n_entries, void* workspace, size_t workspace_bytes,
                          void* stream, const RebuildIO* rb, int64_t* dev_status = nullptr) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(g, true));
    LJ_TRY(check_rows(n, row_begin, row_end));
    if (flags & ~(LJ_LIST_PADDED | LJ_LIST_DEFERRED | LJ_LIST_INTERLEAVED))
        return fail(LJ_ERR_ARG, "build_list: unknown flags 0x%x", flags);
    if ((flags & (LJ_LIST_DEFERRED | LJ_LIST_INTERLEAVED)) && !(flags & LJ_LIST_PADDED))
        return fail(LJ_ERR_ARG, "build_list: LJ_LIST_DEFERRED / LJ_LIST_INTERLEAVED need LJ_LIST_PADDED");
    if (half && (row_begin != 0 || row_end != n))
        return fail(LJ_ERR_UNSUPPORTED, "half list must cover all rows [0,n) (SURVEY §8(e))");
    if (!n_entries || !pointer || (row_end > row_begin && !number_of_partners) || (n > 0 && !q))
        return fail(LJ_ERR_ARG, "build_list: null pointer");
    if (capacity < 0) return fail(LJ_ERR_ARG, "build_list: negative capacity");
    if (capacity > 0 && !sorted_list) return fail(LJ_ERR_ARG, "build_list: null sorted_list with capacity > 0");
    if (!aligned32(q)) return fail(LJ_ERR_ARG, "build_list: q not 32-byte aligned");
    CellGrid cg = make_grid(g);
    BuildWorkspace W = build_workspace_layout(n, cg.ncell, n);
    if (!workspace || workspace_bytes < W.total)
        return fail(LJ_ERR_ARG, "build_list: workspace too small (%zu < %zu)", workspace_bytes, W.total);
    cudaStream_t s = (cudaStream_t)stream;
    char* ws = (char*)workspace;
    const int64_t rows = row_end - row_begin;
    const bool padded = (flags & LJ_LIST_PADDED) != 0;
    const bool il = (flags & LJ_LIST_INTERLEAVED) != 0;
    const int64_t padded_size = (il ? (rows + 7) / 8 * 8 : rows) * (int64_t)LJ_PADDED_ROW_STRIDE;
    if (padded && capacity < padded_size) {
        *n_entries = padded_size;
        return fail(LJ_ERR_CAPACITY, "build_list: padded layout needs capacity %lld", (long long)*n_entries);
    }
    int64_t* counts_scan = padded ? (int64_t*)(ws + W.off_ptrtmp) : pointer;
    if (rb)
        LJ_CUDA(launch_rebuild_cells(rb->q, rb->p, rb->q_out, rb->p_out, rb->q_ref, rb->perm, n, cg, ws, W, s, rb->pm),
                "lj_rebuild/cells");
    else
        LJ_CUDA(launch_cells(q, n, cg, ws, W, s), "lj_build_list/cells");
    if (rows > 0)
        LJ_CUDA(launch_list_pass1(q, cg, g.rs, half, row_begin, row_end, number_of_partners,
                                  padded ? sorted_list : nullptr, ws, W, s, il),
                "lj_build_list/pass1");
    LJ_CUDA(launch_scan_i32_to_i64(number_of_partners, counts_scan, rows, (int64_t*)(ws + W.off_scan),
                                   W.scan_blocks, s),
            "lj_build_list/scan");
    if (dev_status) {   // inside a CUDA graph (lj_md_graph): status to device memory, no synchronisation
        LJ_CUDA(launch_build_status(counts_scan + rows, rows > 0 ? list_row_overflow_flag(ws, W) : nullptr,
                                    dev_status, s),
                "lj_md_graph/status");
        LJ_CUDA(launch_padded_pointer(pointer, rows, s, il), "lj_md_graph/pointer");
        return LJ_OK;
    }
    if (flags & LJ_LIST_DEFERRED) {   // status to the caller's pinned memory, no synchronisation
        LJ_CUDA(cudaMemcpyAsync(n_entries, counts_scan + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s),
                "lj_build_list/status");
        if (rows > 0)
            LJ_CUDA(cudaMemcpyAsync(n_entries + 1, list_row_overflow_flag(ws, W), sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, s),
                    "lj_build_list/status");
        LJ_CUDA(launch_padded_pointer(pointer, rows, s, il), "lj_build_list/pointer");
        return LJ_OK;
    }
    int64_t total = 0;
    int32_t row_overflow = 0;
    LJ_CUDA(cudaMemcpyAsync(&total, counts_scan + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s),
            "lj_build_list/readback");
    if (rows > 0)
        LJ_CUDA(cudaMemcpyAsync(&row_overflow, list_row_overflow_flag(ws, W), sizeof(int32_t), cudaMemcpyDeviceToHost,
                                s),
                "lj_build_list/readback");
    LJ_CUDA(cudaStreamSynchronize(s), "lj_build_list/sync");
    *n_entries = total;
    if (padded) {
        if (row_overflow)
            return fail(LJ_ERR_UNSUPPORTED, "build_list: a row has more than %d partners; use the compact layout",
                        LJ_PADDED_ROW_STRIDE);
        LJ_CUDA(launch_padded_pointer(pointer, rows, s, il), "lj_build_list/pointer");
        return LJ_OK;
    }
    if (total > capacity)
        return fail(LJ_ERR_CAPACITY, "build_list: capacity %lld < required %lld", (long long)capacity,
                    (long long)total);
    if (rows > 0 && total > 0)
        LJ_CUDA(launch_list_pass2(q, cg, g.rs, half, row_begin, row_end, number_of_partners, pointer, sorted_list,
                                  row_overflow != 0, ws, W, s),
                "lj_build_list/pass2");
    return LJ_OK;
}

}  // namespace

lj_status lj_build_list_ex(const double* q, int64_t n, lj_geom g, int half, int64_t row_begin, int64_t row_end,
                           int flags, int32_t* number_of_partners, int64_t* pointer, int32_t* sorted_list,
                           int64_t capacity, int64_t* n_entries, void* workspace, size_t workspace_bytes,
                           void* stream) {
    return build_list_impl(q, n, g, half, row_begin, row_end, flags, number_of_partners, pointer, sorted_list,
                           capacity, n_entries, workspace, workspace_bytes, stream, nullptr);
}

lj_status lj_rebuild(double* q, const double* p, double* q_out, double* p_out, double* q_ref, int64_t* perm,
                     int64_t n, lj_geom g, int half, int64_t row_begin, int64_t row_end, int flags,
                     int32_t* number_of_partners, int64_t* pointer, int32_t* sorted_list, int64_t capacity,
                     int64_t* n_entries, void* workspace, size_t workspace_bytes, void* stream) {
    if (n > 0 && (!q || !q_out || !perm || (p && !p_out))) return fail(LJ_ERR_ARG, "rebuild: null pointer");
    if (n > 0 && (q_out == q || (p && (p_out == p || p_out == q_out)) || q_ref == q || q_ref == q_out))
        return fail(LJ_ERR_ARG, "rebuild: output buffers must be distinct from the inputs and each other");
    if (!aligned32(q) || !aligned32(q_out) || !aligned32(p) || !aligned32(p_out) || !aligned32(q_ref))
        return fail(LJ_ERR_ARG, "rebuild: records not 32-byte aligned");
    RebuildIO io{q, p, q_out, p_out, q_ref, perm, PeerMomenta()};
    return build_list_impl(q_out, n, g, half, row_begin, row_end, flags, number_of_partners, pointer, sorted_list,
                           capacity, n_entries, workspace, workspace_bytes, stream, &io);
}

lj_status lj_build_list(const double* q, int64_t n, lj_geom g, int half, int64_t row_begin, int64_t row_end,
                        int32_t* number_of_partners, int64_t* pointer, int32_t* sorted_list, int64_t capacity,
                        int64_t* n_entries, void* workspace, size_t workspace_bytes, void* stream) {
    return lj_build_list_ex(q, n, g, half, row_begin, row_end, 0, number_of_partners, pointer, sorted_list, capacity,
                            n_entries, workspace, workspace_bytes, stream);
}

lj_status lj_cell_order(const double* q, int64_t n, lj_geom g, int64_t* perm, void* workspace,
                        size_t workspace_bytes, void* stream) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(g, true));
    if (n > 0 && (!q || !perm)) return fail(LJ_ERR_ARG, "cell_order: null pointer");
    if (!aligned32(q)) return fail(LJ_ERR_ARG, "cell_order: q not 32-byte aligned");
    CellGrid cg = make_grid(g);
    BuildWorkspace W = build_workspace_layout(n, cg.ncell, n);
    if (!workspace || workspace_bytes < W.total)
        return fail(LJ_ERR_ARG, "cell_order: workspace too small (%zu < %zu)", workspace_bytes, W.total);
    cudaStream_t s = (cudaStream_t)stream;
    LJ_CUDA(launch_cells(q, n, cg, (char*)workspace, W, s), "lj_cell_order/cells");
    LJ_CUDA(launch_perm_from_cells(perm, n, (char*)workspace, W, s), "lj_cell_order/perm");
    return LJ_OK;
}

lj_status lj_permute_rows(const double* in, double* out, const int64_t* perm, int64_t n, void* stream) {
    LJ_TRY(check_n(n));
    if (n > 0 && (!in || !out || !perm)) return fail(LJ_ERR_ARG, "permute: null pointer");
    if (in == out && n > 0) return fail(LJ_ERR_ARG, "permute: in and out must differ");
    if (!aligned32(in) || !aligned32(out)) return fail(LJ_ERR_ARG, "permute: records not 32-byte aligned");
    LJ_CUDA(launch_permute(in, out, perm, n, (cudaStream_t)stream), "lj_permute_rows");
    return LJ_OK;
}

int lj_default_lanes(int64_t rows, int half) {
    // round-1 sweeps (profiles/r01_sweep_*.jsonl, tools/gu_sweep.py): config 4 G4/U3 0.766 ms, G4/U2 0.783 ms
    const bool big = !half && rows >= 500000;
    return big ? (4 | (3 << 8)) : (8 | (2 << 8));
}

lj_status lj_force_step_ex(const double* q, double* p, int64_t n, lj_geom g, double dt, int half, int64_t row_begin,
                           int64_t row_end, const int32_t* number_of_partners, const int64_t* pointer,
                           const int32_t* sorted_list, int lanes_per_row, int ordered,
                           unsigned long long* n_interactions, void* stream) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(g, false));
    LJ_TRY(check_rows(n, row_begin, row_end));
    if (!std::isfinite(dt)) return fail(LJ_ERR_ARG, "force: dt not finite");
    if (half && (row_begin != 0 || row_end != n))
        return fail(LJ_ERR_UNSUPPORTED, "half list must cover all rows [0,n) (its atomics write p of any atom)");
    if (half && ordered) return fail(LJ_ERR_UNSUPPORTED, "ordered (bit-exact) mode exists for the full list only");
    const int64_t rows = row_end - row_begin;
    if (rows > 0 && (!q || !p || !number_of_partners || !pointer))
        return fail(LJ_ERR_ARG, "force: null pointer");
    if (!aligned32(q) || !aligned32(p)) return fail(LJ_ERR_ARG, "force: q/p not 32-byte aligned");
    if (lanes_per_row & ~(0xffff | LJ_LANES_IDXV))
        return fail(LJ_ERR_ARG, "force: unknown lanes_per_row bits 0x%x", lanes_per_row);
    if ((lanes_per_row & 0xff) == 0) lanes_per_row = lj_default_lanes(row_end - row_begin, half);
    int lanes = lanes_per_row & 0xff, unroll = (lanes_per_row >> 8) & 0xff;
    const int idxv = lanes_per_row & LJ_LANES_IDXV;
    if (lanes != 1 && lanes != 2 && lanes != 4 && lanes != 8 && lanes != 16 && (lanes != 32 || idxv))
        return fail(LJ_ERR_ARG, "force: lanes_per_row G must be 1,2,4,8,16 or 32 (not 32 with LJ_LANES_IDXV) (got %d)",
                    lanes_per_row);
    if (idxv ? (unroll != 2 && unroll != 4) : (unroll != 0 && unroll != 2 && unroll != 3 && unroll != 4))
        return fail(LJ_ERR_ARG, "force: unroll (lanes_per_row >> 8) must be 0, 2, 3 or 4 (2 or 4 with "
                    "LJ_LANES_IDXV) (got %d)", unroll);
    lanes |= unroll << 8 | idxv;
    ForceArgs a;
    a.q = q;
    a.n = n;
    a.p = p;
    a.row_begin = row_begin;
    a.rows = rows;
    a.npart = number_of_partners;
    a.ptr = pointer;
    a.list = sorted_list;
    a.L = g.L;
    a.rc2 = g.rc * g.rc;
    a.dt = dt;
    a.n_inter = n_interactions;
    cudaStream_t s = (cudaStream_t)stream;
    if (ordered)
        LJ_CUDA(launch_force_ordered(a, s), "lj_force_step/ordered");
    else if (half)
        LJ_CUDA(launch_force_half(a, lanes, s), "lj_force_step/half");
    else
        LJ_CUDA(launch_force_full(a, lanes, s), "lj_force_step/full");
    return LJ_OK;
}

lj_status lj_force_step(const double* q, double* p, int64_t n, lj_geom g, double dt, int half, int64_t row_begin,
                        int64_t row_end, const int32_t* number_of_partners, const int64_t* pointer,
                        const int32_t* sorted_list, void* stream) {
    return lj_force_step_ex(q, p, n, g, dt, half, row_begin, row_end, number_of_partners, pointer, sorted_list, 0, 0,
                            nullptr, stream);
}

lj_status lj_list_cell_starts(const void* workspace, size_t workspace_bytes, int64_t n, lj_geom g,
                              int64_t* cell_start, void* stream) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(g, true));
    if (!workspace || !cell_start) return fail(LJ_ERR_ARG, "list_cell_starts: null pointer");
    const CellGrid cg = make_grid(g);
    const BuildWorkspace W = build_workspace_layout(n, cg.ncell, 0);
    if (workspace_bytes < W.off_atoms) return fail(LJ_ERR_ARG, "list_cell_starts: workspace too small");
    LJ_CUDA(cudaMemcpyAsync(cell_start, (const char*)workspace + W.off_start, sizeof(int64_t) * (cg.ncell + 1),
                            cudaMemcpyDeviceToDevice, (cudaStream_t)stream),
            "lj_list_cell_starts");
    return LJ_OK;
}

lj_status lj_force_step_half_cells(const double* q, double* p, int64_t n, lj_geom g, double dt,
                                   const int32_t* number_of_partners, const int64_t* pointer,
                                   const int32_t* sorted_list, const int64_t* cell_start, int lanes_per_row,
                                   unsigned long long* n_interactions, void* stream) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(g, true));
    if (!std::isfinite(dt)) return fail(LJ_ERR_ARG, "force_half_cells: dt not finite");
    if (n > 0 && (!q || !p || !number_of_partners || !pointer || !cell_start))
        return fail(LJ_ERR_ARG, "force_half_cells: null pointer");
    if (!aligned32(q) || !aligned32(p)) return fail(LJ_ERR_ARG, "force_half_cells: q/p not 32-byte aligned");
    if (lanes_per_row != 0 && lanes_per_row != (4 | (2 << 8)) && lanes_per_row != (8 | (2 << 8)) &&
        lanes_per_row != (4 | (3 << 8)) && lanes_per_row != (2 | (2 << 8)))
        return fail(LJ_ERR_ARG, "force_half_cells: lanes_per_row must be 0, 2|2<<8, 4|2<<8, 8|2<<8 or 4|3<<8");
    ForceArgs a;
    a.q = q;
    a.n = n;
    a.p = p;
    a.row_begin = 0;
    a.rows = n;
    a.npart = number_of_partners;
    a.ptr = pointer;
    a.list = sorted_list;
    a.L = g.L;
    a.rc2 = g.rc * g.rc;
    a.dt = dt;
    a.n_inter = n_interactions;
    LJ_CUDA(launch_force_half_cells(a, cell_start, make_grid(g).nc, lanes_per_row, (cudaStream_t)stream),
            "lj_force_step_half_cells");
    return LJ_OK;
}

lj_status lj_force_step_variant(int layout, int rcp, const double* q, double* p, int64_t n, lj_geom g, double dt,
                                int64_t row_begin, int64_t row_end, const int32_t* number_of_partners,
                                const int64_t* pointer, const int32_t* sorted_list, int lanes_per_row,
                                unsigned long long* n_interactions, void* stream) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(g, false));
    LJ_TRY(check_rows(n, row_begin, row_end));
    if (layout < LJ_LAYOUT_AOS4 || layout > LJ_LAYOUT_AOS8) return fail(LJ_ERR_ARG, "variant: unknown layout %d", layout);
    if (rcp < LJ_RCP_NEWTON3 || rcp > LJ_RCP_IEEE) return fail(LJ_ERR_ARG, "variant: unknown reciprocal %d", rcp);
    if (lanes_per_row != 4 && lanes_per_row != 8) return fail(LJ_ERR_ARG, "variant: lanes_per_row must be 4 or 8");
    if (!std::isfinite(dt)) return fail(LJ_ERR_ARG, "variant: dt not finite");
    const int64_t rows = row_end - row_begin;
    if (layout == LJ_LAYOUT_AOS8) p = const_cast<double*>(q);
    if (rows > 0 && (!q || !p || !number_of_partners || !pointer)) return fail(LJ_ERR_ARG, "variant: null pointer");
    const bool wide = layout == LJ_LAYOUT_AOS4 || layout == LJ_LAYOUT_AOS8;
    if (wide ? (!aligned32(q) || !aligned32(p)) : (((uintptr_t)q | (uintptr_t)p) & 7u))
        return fail(LJ_ERR_ARG, "variant: q/p misaligned for the layout");
    ForceArgs a;
    a.q = q;
    a.n = n;
    a.p = p;
    a.row_begin = row_begin;
    a.rows = rows;
    a.npart = number_of_partners;
    a.ptr = pointer;
    a.list = sorted_list;
    a.L = g.L;
    a.rc2 = g.rc * g.rc;
    a.dt = dt;
    a.n_inter = n_interactions;
    LJ_CUDA(launch_force_variant(a, n, layout, rcp, lanes_per_row, (cudaStream_t)stream), "lj_force_step_variant");
    return LJ_OK;
}

lj_status lj_gather_probe(const double* q, int64_t n, int64_t row_begin, int64_t row_end,
                          const int32_t* number_of_partners, const int64_t* pointer, const int32_t* sorted_list,
                          int lanes_per_row, double* sink, void* stream) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_rows(n, row_begin, row_end));
    if (!sink || (row_end > row_begin && (!q || !number_of_partners || !pointer)))
        return fail(LJ_ERR_ARG, "gather_probe: null pointer");
    if (!aligned32(q)) return fail(LJ_ERR_ARG, "gather_probe: q not 32-byte aligned");
    // same encoding and defaults as lj_force_step_ex on a full list: G | (U << 8) [| LJ_LANES_IDXV]
    if ((lanes_per_row & 0xff) == 0) lanes_per_row = lj_default_lanes(row_end - row_begin, 0);
    int lanes = lanes_per_row;
    if (((lanes >> 8) & 0xff) == 0) lanes |= 2 << 8;
    ForceArgs a;
    a.q = q;
    a.n = n;
    a.p = nullptr;
    a.row_begin = row_begin;
    a.rows = row_end - row_begin;
    a.npart = number_of_partners;
    a.ptr = pointer;
    a.list = sorted_list;
    a.L = 0;
    a.rc2 = 0;
    a.dt = 0;
    a.n_inter = nullptr;
    const cudaError_t e = launch_gather_probe(a, lanes, sink, (cudaStream_t)stream);
    if (e == cudaErrorInvalidValue) return fail(LJ_ERR_ARG, "gather_probe: unsupported lanes_per_row 0x%x", lanes_per_row);
    LJ_CUDA(e, "lj_gather_probe");
    return LJ_OK;
}

lj_status lj_list_interior(int64_t row_begin, int64_t row_end, const int32_t* number_of_partners,
                           const int64_t* pointer, const int32_t* sorted_list, int64_t* out, void* stream) {
    if (row_begin < 0 || row_end < row_begin) return fail(LJ_ERR_ARG, "list_interior: bad row range");
    if (!out || (row_end > row_begin && (!number_of_partners || !pointer || !sorted_list)))
        return fail(LJ_ERR_ARG, "list_interior: null pointer");
    LJ_CUDA(launch_list_interior(row_begin, row_end, number_of_partners, pointer, sorted_list, out,
                                 (cudaStream_t)stream),
            "lj_list_interior");
    return LJ_OK;
}

lj_status lj_list_partner_ranges(int64_t row_begin, int64_t row_end, const int32_t* number_of_partners,
                                 const int64_t* pointer, const int32_t* sorted_list, const int64_t* bounds, int P,
                                 int64_t* out, void* stream) {
    if (row_begin < 0 || row_end < row_begin) return fail(LJ_ERR_ARG, "partner_ranges: bad row range");
    if (P < 1 || P > 64) return fail(LJ_ERR_ARG, "partner_ranges: need 1 <= P <= 64 (got %d)", P);
    if (!out || !bounds || (row_end > row_begin && (!number_of_partners || !pointer || !sorted_list)))
        return fail(LJ_ERR_ARG, "partner_ranges: null pointer");
    LJ_CUDA(launch_partner_ranges(row_begin, row_end, number_of_partners, pointer, sorted_list, bounds, P, out,
                                  (cudaStream_t)stream),
            "lj_list_partner_ranges");
    return LJ_OK;
}

lj_status lj_integrate(double* q, const double* p, int64_t begin, int64_t end, double dt, void* stream) {
    if (begin < 0 || end < begin || end > (int64_t)INT32_MAX)
        return fail(LJ_ERR_ARG, "integrate: bad range [%lld,%lld)", (long long)begin, (long long)end);
    if (end > begin && (!q || !p)) return fail(LJ_ERR_ARG, "integrate: null pointer");
    if (!aligned32(q) || !aligned32(p)) return fail(LJ_ERR_ARG, "integrate: q/p not 32-byte aligned");
    if (!std::isfinite(dt)) return fail(LJ_ERR_ARG, "integrate: dt not finite");
    LJ_CUDA(launch_integrate(q, p, begin, end, dt, (cudaStream_t)stream), "lj_integrate");
    return LJ_OK;
}

lj_status lj_integrate_displacement(double* q, const double* p, const double* q_ref, int64_t begin, int64_t end,
                                   double dt, double* max_disp, void* stream) {
    if (begin < 0 || end < begin || end > (int64_t)INT32_MAX)
        return fail(LJ_ERR_ARG, "integrate_displacement: bad range [%lld,%lld)", (long long)begin, (long long)end);
    if (!max_disp || (end > begin && (!q || !p || !q_ref))) return fail(LJ_ERR_ARG, "integrate_displacement: null pointer");
    if (!aligned32(q) || !aligned32(p) || !aligned32(q_ref))
        return fail(LJ_ERR_ARG, "integrate_displacement: not 32-byte aligned");
    if (!std::isfinite(dt)) return fail(LJ_ERR_ARG, "integrate_displacement: dt not finite");
    LJ_CUDA(launch_integrate_disp(q, p, q_ref, begin, end, dt, max_disp, (cudaStream_t)stream),
            "lj_integrate_displacement");
    return LJ_OK;
}

lj_status lj_integrate_push(const double* q_in, double* q_out, const double* p, const double* q_ref, int64_t begin,
                            int64_t end, double dt, double* max_disp, const lj_push_target* targets, int n_targets,
                            void* stream) {
    if (begin < 0 || end < begin || end > (int64_t)INT32_MAX)
        return fail(LJ_ERR_ARG, "integrate_push: bad range [%lld,%lld)", (long long)begin, (long long)end);
    if (n_targets < 0 || n_targets > LJ_MAX_PUSH_TARGETS || (n_targets > 0 && !targets))
        return fail(LJ_ERR_ARG, "integrate_push: need 0 <= n_targets <= %d and a target array", LJ_MAX_PUSH_TARGETS);
    if (!max_disp || (end > begin && (!q_in || !q_out || !p || !q_ref)))
        return fail(LJ_ERR_ARG, "integrate_push: null pointer");
    if (!aligned32(q_in) || !aligned32(q_out) || !aligned32(p) || !aligned32(q_ref))
        return fail(LJ_ERR_ARG, "integrate_push: not 32-byte aligned");
    for (int k = 0; k < n_targets; k++) {
        if (!targets[k].dst || !aligned32(targets[k].dst))
            return fail(LJ_ERR_ARG, "integrate_push: target %d: null or misaligned dst", k);
        if (targets[k].lo < 0 || targets[k].hi < targets[k].lo)
            return fail(LJ_ERR_ARG, "integrate_push: target %d: bad rows [%lld,%lld)", k, (long long)targets[k].lo,
                        (long long)targets[k].hi);
    }
    if (!std::isfinite(dt)) return fail(LJ_ERR_ARG, "integrate_push: dt not finite");
    LJ_CUDA(launch_integrate_push(q_in, q_out, p, q_ref, begin, end, dt, max_disp, targets, n_targets,
                                  (cudaStream_t)stream),
            "lj_integrate_push");
    return LJ_OK;
}

// cuMemGetAddressRange through the runtime's driver entry point (liblj.so does not
// link libcuda, so that it loads on machines without a driver).
typedef int (*pfn_get_range)(unsigned long long*, size_t*, unsigned long long);

lj_status lj_ipc_get_handle(const void* ptr, void* handle, int64_t* offset) {
    if (!ptr || !handle || !offset) return fail(LJ_ERR_ARG, "ipc_get_handle: null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess)
        return fail(LJ_ERR_CUDA, "ipc_get_handle: cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    if (((pfn_get_range)fn)(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0)
        return fail(LJ_ERR_ARG, "ipc_get_handle: not a device allocation");
    cudaIpcMemHandle_t h;
    LJ_CUDA(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base), "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
    return LJ_OK;
}

lj_status lj_ipc_open(const void* handle, int64_t offset, void** ptr) {
    if (!handle || !ptr || offset < 0) return fail(LJ_ERR_ARG, "ipc_open: bad argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    LJ_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    *ptr = (char*)base + offset;
    return LJ_OK;
}

lj_status lj_ipc_close(void* ptr) {
    if (!ptr) return fail(LJ_ERR_ARG, "ipc_close: null pointer");
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess)
        return fail(LJ_ERR_CUDA, "ipc_close: cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    if (((pfn_get_range)fn)(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0)
        return fail(LJ_ERR_ARG, "ipc_close: not a mapped allocation");
    LJ_CUDA(cudaIpcCloseMemHandle((void*)(uintptr_t)base), "cudaIpcCloseMemHandle");
    return LJ_OK;
}

// ---- the MD step as a CUDA graph with a device-side rebuild decision --------
struct lj_md_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    long long kernels_steps = 0, kernels_rebuild = 0;   // all unrolled steps (no rebuild) / one rebuild
    std::vector<cudaEvent_t> ev;   // per step: force begin, force end
    std::vector<char> timed;       // the step's force kernel sits between its two events
};

lj_status lj_md_graph_create(const lj_md_graph_desc* d, lj_md_graph** out) {
    if (!d || !out) return fail(LJ_ERR_ARG, "md_graph: null pointer");
    *out = nullptr;
    const int64_t n = d->n;
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(d->g, true));
    if (n < 1) return fail(LJ_ERR_ARG, "md_graph: n must be >= 1");
    if (d->steps < 1 || d->steps > 100000) return fail(LJ_ERR_ARG, "md_graph: steps must be in [1, 100000]");
    if (!std::isfinite(d->dt)) return fail(LJ_ERR_ARG, "md_graph: dt not finite");
    if (d->energy_every < 0 || (d->energy_every > 0 && !d->energies))
        return fail(LJ_ERR_ARG, "md_graph: energy_every needs an energies buffer");
    if (!d->q || !d->p || !d->q_ref || !d->perm || !d->disp || !d->status || !d->number_of_partners || !d->pointer ||
        !d->sorted_list || !d->workspace || (d->reorder && (!d->q_alt || !d->p_alt)))
        return fail(LJ_ERR_ARG, "md_graph: null pointer");
    if (!aligned32(d->q) || !aligned32(d->p) || !aligned32(d->q_ref) || !aligned32(d->q_alt) || !aligned32(d->p_alt))
        return fail(LJ_ERR_ARG, "md_graph: records not 32-byte aligned");
    const int64_t need = (d->interleaved ? (n + 7) / 8 * 8 : n) * (int64_t)LJ_PADDED_ROW_STRIDE;
    if (d->capacity < need) return fail(LJ_ERR_CAPACITY, "md_graph: the padded list needs capacity %lld", (long long)need);
    const CellGrid cg = make_grid(d->g);
    const BuildWorkspace W = build_workspace_layout(n, cg.ncell, n);
    if (d->workspace_bytes < W.total) return fail(LJ_ERR_ARG, "md_graph: workspace too small");
    lj_md_graph* gr = new lj_md_graph();
    cudaStream_t cs = nullptr;
    auto done = [&](lj_status r) {
        if (cs) cudaStreamDestroy(cs);
        if (r != LJ_OK) {
            lj_md_graph_destroy(gr);
        } else {
            *out = gr;
        }
        return r;
    };
#define LJ_G(x, where)                                              \
    do {                                                            \
        cudaError_t _e = (x);                                       \
        if (_e != cudaSuccess) return done(cuda_status(_e, where)); \
    } while (0)
    LJ_G(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "md_graph/stream");
    LJ_G(cudaGraphCreate(&gr->graph, 0), "md_graph/create");
    ForceArgs fa;
    fa.q = d->q;
    fa.n = n;
    fa.p = d->p;
    fa.row_begin = 0;
    fa.rows = n;
    fa.npart = d->number_of_partners;
    fa.ptr = d->pointer;
    fa.list = d->sorted_list;
    fa.L = d->g.L;
    fa.rc2 = d->g.rc * d->g.rc;
    fa.dt = d->dt;
    fa.n_inter = d->n_interactions;
    const int lanes = lj_default_lanes(n, 0);   // lj_force_step_ex's defaults
    const size_t rec = sizeof(double) * 4 * (size_t)n;
    gr->ev.resize(2 * (size_t)d->steps, nullptr);
    gr->timed.assign((size_t)d->steps, 0);
    for (auto& ev : gr->ev) LJ_G(cudaEventCreate(&ev), "md_graph/event");
    cudaGraphNode_t prev = nullptr;
    for (int k = 0; k < d->steps; k++) {
        // kick (between two event records: the force kernel's duration per step) + drift +
        // displacement + the decision, captured straight into the graph after the previous step
        LJ_G(cudaStreamBeginCaptureToGraph(cs, gr->graph, prev ? &prev : nullptr, nullptr, prev ? 1 : 0,
                                           cudaStreamCaptureModeRelaxed),
             "md_graph/capture");
        long long l0 = g_launches;
        cudaGraphConditionalHandle h = 0;
        cudaError_t e = cudaSuccess;
        if (d->energy_every > 0 && k % d->energy_every == 0) {
            // sample step: p_n = p_{n-1/2} + F dt/2, (KE, PE) at the synchronised p, the second half kick
            ForceArgs half_kick = fa;
            half_kick.dt = 0.5 * d->dt;
            e = launch_force_full(half_kick, lanes, cs);
            if (e == cudaSuccess)
                e = launch_energy(d->q, d->p, n, 0, n, d->number_of_partners, d->pointer, d->sorted_list, d->g.L,
                                  d->g.rc * d->g.rc, d->g.rc, 0, d->energies + 2 * (k / d->energy_every), cs);
            half_kick.n_inter = nullptr;
            if (e == cudaSuccess) e = launch_force_full(half_kick, lanes, cs);
        } else {   // the force kernel between two event nodes: its duration per step
            e = cudaEventRecordWithFlags(gr->ev[2 * k], cs, cudaEventRecordExternal);
            if (e == cudaSuccess) e = launch_force_full(fa, lanes, cs);
            if (e == cudaSuccess) e = cudaEventRecordWithFlags(gr->ev[2 * k + 1], cs, cudaEventRecordExternal);
            gr->timed[k] = 1;
        }
        if (e == cudaSuccess) e = launch_integrate_disp(d->q, d->p, d->q_ref, 0, n, d->dt, d->disp, cs);
        if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, gr->graph, 0, cudaGraphCondAssignDefault);
        if (e == cudaSuccess) e = launch_md_decide(d->disp, 1, 0, d->g.rs - d->g.rc, h, d->status, cs);
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        cudaStreamCaptureStatus cst;
        if (e == cudaSuccess) e = cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps);
        std::vector<cudaGraphNode_t> leaf;
        if (e == cudaSuccess) leaf.assign(deps, deps + ndeps);
        cudaGraph_t tmp;
        cudaError_t e2 = cudaStreamEndCapture(cs, &tmp);
        LJ_G(e, "md_graph/step");
        LJ_G(e2, "md_graph/capture-end");
        gr->kernels_steps += g_launches - l0;
        // IF (rebuild): the body is the bookkeeping rebuild, captured into the conditional's graph
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        LJ_G(cudaGraphAddNode(&prev, gr->graph, leaf.data(), leaf.size(), &cp), "md_graph/conditional");
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        LJ_G(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
             "md_graph/capture-body");
        l0 = g_launches;
        lj_status st = LJ_OK;
        const int lflags = LJ_LIST_PADDED | (d->interleaved ? LJ_LIST_INTERLEAVED : 0);
        if (d->reorder) {   // as lj_rebuild, then the permuted state back into q / p
            RebuildIO io{d->q, d->p, d->q_alt, d->p_alt, d->q_ref, d->perm, PeerMomenta()};
            st = build_list_impl(d->q_alt, n, d->g, 0, 0, n, lflags, d->number_of_partners, d->pointer,
                                 d->sorted_list, d->capacity, d->status + 2, d->workspace, d->workspace_bytes, cs,
                                 &io, d->status);
            if (st == LJ_OK) e = cudaMemcpyAsync(d->q, d->q_alt, rec, cudaMemcpyDeviceToDevice, cs);
            if (st == LJ_OK && e == cudaSuccess)
                e = cudaMemcpyAsync(d->p, d->p_alt, rec, cudaMemcpyDeviceToDevice, cs);
        } else {            // wrap + snapshot, then the list (as lj_wrap + lj_build_list_ex)
            e = launch_wrap(d->q, d->q_ref, n, d->g.L, cs);
            if (e == cudaSuccess)
                st = build_list_impl(d->q, n, d->g, 0, 0, n, lflags, d->number_of_partners, d->pointer,
                                     d->sorted_list, d->capacity, d->status + 2, d->workspace, d->workspace_bytes,
                                     cs, nullptr, d->status);
        }
        e2 = cudaStreamEndCapture(cs, &tmp);
        if (st != LJ_OK) return done(st);
        LJ_G(e, "md_graph/rebuild");
        LJ_G(e2, "md_graph/capture-body-end");
        if (k == 0) gr->kernels_rebuild = g_launches - l0;
    }
    LJ_G(cudaGraphInstantiate(&gr->exec, gr->graph, 0), "md_graph/instantiate");
    LJ_G(cudaGraphUpload(gr->exec, cs), "md_graph/upload");   // the first launch pays no upload
    LJ_G(cudaStreamSynchronize(cs), "md_graph/upload");
#undef LJ_G
    return done(LJ_OK);
}

lj_status lj_md_capture_rebuild(const lj_md_rebuild_desc* d, void* stream, long long* kernels_per_rebuild) {
    if (!d) return fail(LJ_ERR_ARG, "md_capture_rebuild: null descriptor");
    const int64_t n = d->n;
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(d->g, true));
    LJ_TRY(check_rows(n, d->row_begin, d->row_end));
    if (n < 1) return fail(LJ_ERR_ARG, "md_capture_rebuild: n must be >= 1");
    if (!d->q || !d->q_ref || !d->number_of_partners || !d->pointer || !d->sorted_list || !d->workspace ||
        !d->disp || !d->status)
        return fail(LJ_ERR_ARG, "md_capture_rebuild: null pointer");
    if (!aligned32(d->q) || !aligned32(d->q_ref)) return fail(LJ_ERR_ARG, "md_capture_rebuild: records not 32-byte aligned");
    if (d->disp_count < 1 || d->disp_count > 4096 || d->disp_stride < 0)
        return fail(LJ_ERR_ARG, "md_capture_rebuild: need 1 <= disp_count <= 4096, disp_stride >= 0");
    if (d->reorder) {
        if (!d->q_alt || !d->p || !d->p_alt || !d->perm || !d->p_peers)
            return fail(LJ_ERR_ARG, "md_capture_rebuild: reorder needs q_alt, p, p_alt, perm and p_peers");
        if (!aligned32(d->q_alt) || !aligned32(d->p) || !aligned32(d->p_alt))
            return fail(LJ_ERR_ARG, "md_capture_rebuild: records not 32-byte aligned");
        if (d->n_own < 1 || n % d->n_own != 0 || d->row_begin % d->n_own != 0 || d->row_end - d->row_begin != d->n_own)
            return fail(LJ_ERR_ARG, "md_capture_rebuild: reorder needs equal slabs (n_own divides n, own rows = "
                        "one slab)");
        if (d->q_alt == d->q || d->p_alt == d->p) return fail(LJ_ERR_ARG, "md_capture_rebuild: alt buffers must differ");
    }
    const int64_t rows = d->row_end - d->row_begin;
    const int64_t need = (d->interleaved ? (rows + 7) / 8 * 8 : rows) * (int64_t)LJ_PADDED_ROW_STRIDE;
    if (d->capacity < need)
        return fail(LJ_ERR_CAPACITY, "md_capture_rebuild: the padded list needs capacity %lld", (long long)need);
    const CellGrid cg = make_grid(d->g);
    const BuildWorkspace W = build_workspace_layout(n, cg.ncell, n);
    if (d->workspace_bytes < W.total) return fail(LJ_ERR_ARG, "md_capture_rebuild: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    cudaStreamCaptureStatus cst;
    cudaGraph_t graph = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    LJ_CUDA(cudaStreamGetCaptureInfo(s, &cst, nullptr, &graph, &deps, &ndeps), "md_capture_rebuild/info");
    if (cst != cudaStreamCaptureStatusActive || !graph)
        return fail(LJ_ERR_ARG, "md_capture_rebuild: the stream is not being captured");
    cudaGraphConditionalHandle h;
    LJ_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault), "md_capture_rebuild/handle");
    LJ_CUDA(launch_md_decide(d->disp, d->disp_count, d->disp_stride, d->g.rs - d->g.rc, h, d->status, s),
            "md_capture_rebuild/decide");
    LJ_CUDA(cudaStreamGetCaptureInfo(s, &cst, nullptr, &graph, &deps, &ndeps), "md_capture_rebuild/info");
    std::vector<cudaGraphNode_t> leaf(deps, deps + ndeps);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    LJ_CUDA(cudaGraphAddNode(&node, graph, leaf.data(), leaf.size(), &cp), "md_capture_rebuild/conditional");
    // the body: captured on a private stream into the conditional's graph
    cudaStream_t bs = nullptr;
    LJ_CUDA(cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking), "md_capture_rebuild/stream");
    cudaError_t e = cudaStreamBeginCaptureToGraph(bs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeRelaxed);
    const long long l0 = g_launches;
    lj_status st = LJ_OK;
    const int lflags = LJ_LIST_PADDED | (d->interleaved ? LJ_LIST_INTERLEAVED : 0);
    if (e == cudaSuccess) {
        if (d->reorder) {
            // as lj_rebuild -- wrap, cells, the cell-order permutation of q (replicated) and q_ref --
            // with the own new rows' momenta read from the rank that owned each atom (d->p_peers,
            // NVLink loads of the peers' copies), then the permuted state back into q / own p rows
            RebuildIO io{d->q, nullptr, d->q_alt, d->p_alt, d->q_ref, d->perm, PeerMomenta()};
            io.pm.table = d->p_peers;
            io.pm.n_own = d->n_own;
            io.pm.own_lo = d->row_begin;
            io.pm.own_hi = d->row_end;
            st = build_list_impl(d->q_alt, n, d->g, 0, d->row_begin, d->row_end, lflags,
                                 d->number_of_partners, d->pointer, d->sorted_list, d->capacity, d->status + 2,
                                 d->workspace, d->workspace_bytes, bs, &io, d->status);
            const size_t rec = sizeof(double) * 4;
            if (st == LJ_OK) e = cudaMemcpyAsync(d->q, d->q_alt, rec * (size_t)n, cudaMemcpyDeviceToDevice, bs);
            if (st == LJ_OK && e == cudaSuccess)
                e = cudaMemcpyAsync(d->p + 4 * d->row_begin, d->p_alt + 4 * d->row_begin,
                                    rec * (size_t)(d->row_end - d->row_begin), cudaMemcpyDeviceToDevice, bs);
        } else {
            e = launch_wrap(d->q, d->q_ref, n, d->g.L, bs);
            if (e == cudaSuccess)
                st = build_list_impl(d->q, n, d->g, 0, d->row_begin, d->row_end, lflags,
                                     d->number_of_partners, d->pointer, d->sorted_list, d->capacity, d->status + 2,
                                     d->workspace, d->workspace_bytes, bs, nullptr, d->status);
        }
        cudaGraph_t tmp;
        const cudaError_t e2 = cudaStreamEndCapture(bs, &tmp);
        if (e == cudaSuccess) e = e2;
    }
    cudaStreamDestroy(bs);
    if (st != LJ_OK) return st;
    LJ_CUDA(e, "md_capture_rebuild/body");
    if (kernels_per_rebuild) *kernels_per_rebuild = g_launches - l0;
    // later captured work on `stream` follows the IF node
    LJ_CUDA(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies),
            "md_capture_rebuild/deps");
    return LJ_OK;
}

lj_status lj_copy_records(const double* src, double* dst, int64_t n, void* stream) {
    if (n < 0 || (n > 0 && (!src || !dst))) return fail(LJ_ERR_ARG, "copy_records: bad argument");
    if (!aligned32(src) || !aligned32(dst)) return fail(LJ_ERR_ARG, "copy_records: not 32-byte aligned");
    if (n == 0 || src == dst) return LJ_OK;
    LJ_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * 4 * (size_t)n, cudaMemcpyDeviceToDevice, (cudaStream_t)stream),
            "lj_copy_records");
    return LJ_OK;
}

lj_status lj_copy_bytes(void* dst, const void* src, size_t bytes, void* stream) {
    if (bytes > 0 && (!src || !dst)) return fail(LJ_ERR_ARG, "copy_bytes: null pointer");
    if (bytes == 0 || src == dst) return LJ_OK;
    LJ_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream), "lj_copy_bytes");
    return LJ_OK;
}

lj_status lj_permute_rows_peers(double* q, double* q_out, double* q_ref, double* p_out,
                                const double* const* p_peers, int64_t n_own, int64_t own_lo, int64_t own_hi,
                                int64_t* perm, int64_t n, lj_geom g, void* workspace, size_t workspace_bytes,
                                void* stream) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(g, true));
    if (n > 0 && (!q || !q_out || !p_out || !p_peers || !perm)) return fail(LJ_ERR_ARG, "permute_rows_peers: null pointer");
    if (!aligned32(q) || !aligned32(q_out) || !aligned32(q_ref) || !aligned32(p_out))
        return fail(LJ_ERR_ARG, "permute_rows_peers: records not 32-byte aligned");
    if (n_own < 1 || n % n_own != 0 || own_lo < 0 || own_lo > own_hi || own_hi > n)
        return fail(LJ_ERR_ARG, "permute_rows_peers: need n_own dividing n and 0 <= own_lo <= own_hi <= n");
    if (q_out == q) return fail(LJ_ERR_ARG, "permute_rows_peers: q_out must differ from q");
    const CellGrid cg = make_grid(g);
    const BuildWorkspace W = build_workspace_layout(n, cg.ncell, n);
    if (!workspace || workspace_bytes < W.total) return fail(LJ_ERR_ARG, "permute_rows_peers: workspace too small");
    PeerMomenta pm;
    pm.table = p_peers;
    pm.n_own = n_own;
    pm.own_lo = own_lo;
    pm.own_hi = own_hi;
    LJ_CUDA(launch_rebuild_cells(q, nullptr, q_out, p_out, q_ref, perm, n, cg, (char*)workspace, W,
                                 (cudaStream_t)stream, pm),
            "lj_permute_rows_peers");
    return LJ_OK;
}

lj_status lj_publish_scalar(const double* src, double* dst, void* stream) {
    if (!src || !dst) return fail(LJ_ERR_ARG, "publish_scalar: null pointer");
    LJ_CUDA(launch_copy_scalar(src, dst, (cudaStream_t)stream), "lj_publish_scalar");
    return LJ_OK;
}

lj_status lj_md_graph_force_ms(const lj_md_graph* gr, float* ms, int n) {
    if (!gr || !ms || n < 0 || 2 * (size_t)n > gr->ev.size()) return fail(LJ_ERR_ARG, "md_graph_force_ms: bad argument");
    for (int k = 0; k < n; k++) {   // sample steps (split kick, no events) report 0
        ms[k] = 0.0f;
        if (gr->timed[k]) LJ_CUDA(cudaEventElapsedTime(ms + k, gr->ev[2 * k], gr->ev[2 * k + 1]), "event");
    }
    return LJ_OK;
}

lj_status lj_md_graph_launch(lj_md_graph* gr, void* stream) {
    if (!gr || !gr->exec) return fail(LJ_ERR_ARG, "md_graph_launch: bad argument");
    LJ_CUDA(cudaGraphLaunch(gr->exec, (cudaStream_t)stream), "cudaGraphLaunch");
    return LJ_OK;
}

lj_status lj_md_graph_kernels(const lj_md_graph* gr, long long* per_step, long long* per_rebuild) {
    if (!gr || !per_step || !per_rebuild) return fail(LJ_ERR_ARG, "md_graph_kernels: null pointer");
    *per_step = gr->kernels_steps;
    *per_rebuild = gr->kernels_rebuild;
    return LJ_OK;
}

lj_status lj_md_graph_destroy(lj_md_graph* gr) {
    if (!gr) return LJ_OK;
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    if (gr->graph) cudaGraphDestroy(gr->graph);
    for (auto ev : gr->ev)
        if (ev) cudaEventDestroy(ev);
    delete gr;
    return LJ_OK;
}

lj_status lj_wrap(double* q, double* q_ref, int64_t n, double L, void* stream) {
    LJ_TRY(check_n(n));
    if (!(L > 0.0) || !std::isfinite(L)) return fail(LJ_ERR_ARG, "wrap: L must be > 0");
    if (n > 0 && !q) return fail(LJ_ERR_ARG, "wrap: null q");
    if (!aligned32(q) || !aligned32(q_ref)) return fail(LJ_ERR_ARG, "wrap: records not 32-byte aligned");
    LJ_CUDA(launch_wrap(q, q_ref, n, L, (cudaStream_t)stream), "lj_wrap");
    return LJ_OK;
}

lj_status lj_max_displacement(const double* q, const double* q_ref, int64_t begin, int64_t end, double* out,
                              void* stream) {
    if (begin < 0 || end < begin || end > (int64_t)INT32_MAX)
        return fail(LJ_ERR_ARG, "max_displacement: bad range");
    if (!out || (end > begin && (!q || !q_ref))) return fail(LJ_ERR_ARG, "max_displacement: null pointer");
    if (!aligned32(q) || !aligned32(q_ref)) return fail(LJ_ERR_ARG, "max_displacement: not 32-byte aligned");
    LJ_CUDA(launch_max_disp(q, q_ref, begin, end, out, (cudaStream_t)stream), "lj_max_displacement");
    return LJ_OK;
}

lj_status lj_energy(const double* q, const double* p, int64_t n, lj_geom g, int64_t row_begin, int64_t row_end,
                    const int32_t* number_of_partners, const int64_t* pointer, const int32_t* sorted_list, int half,
                    double* out, void* stream) {
    LJ_TRY(check_n(n));
    LJ_TRY(check_geom(g, false));
    LJ_TRY(check_rows(n, row_begin, row_end));
    if (!out) return fail(LJ_ERR_ARG, "energy: null out");
    if (row_end > row_begin && (!q || !p || !number_of_partners || !pointer))
        return fail(LJ_ERR_ARG, "energy: null pointer");
    if (!aligned32(q) || !aligned32(p)) return fail(LJ_ERR_ARG, "energy: not 32-byte aligned");
    LJ_CUDA(launch_energy(q, p, n, row_begin, row_end - row_begin, number_of_partners, pointer, sorted_list, g.L,
                          g.rc * g.rc, g.rc, half, out, (cudaStream_t)stream),
            "lj_energy");
    return LJ_OK;
}

}  // extern "C"
