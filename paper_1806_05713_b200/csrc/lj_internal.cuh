// Internal declarations shared by the liblj CUDA translation units.
// (Product code only -- nothing here is shared with oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>

#include "../../include/liblj.h"

namespace lj {

// The paper's "AoS with padding" record: x, y, z, pad.
// 32-byte alignment makes one record exactly one 256-bit load (LDG.E.ENL2.256
// on sm_100a) and exactly one 32-byte L2 sector.
struct __align__(32) rec4 {
    double x, y, z, w;
};

extern std::atomic<long long> g_launches;

// Bounds checks of the memory-safety build (liblj_check.so, -DLJ_CHECK; tests/test_gpu_checked.py):
// a violated condition prints where and traps, which surfaces as a CUDA error at the next
// synchronising call.  Compiled out of liblj.so.
#ifdef LJ_CHECK
#define LJ_CHECK_THAT(cond)                                                                            \
    do {                                                                                               \
        if (!(cond)) {                                                                                 \
            printf("liblj check failed: %s (%s:%d, block %d thread %d)\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                                 \
            __trap();                                                                                  \
        }                                                                                              \
    } while (0)
#else
#define LJ_CHECK_THAT(cond) \
    do {                    \
    } while (0)
#endif

// 256-bit read-only load of one record (compiles to LDG.E.ENL2.256.CONSTANT).
__device__ __forceinline__ rec4 load_rec(const rec4* __restrict__ a, int64_t i) {
    rec4 r;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
                 : "l"(a + i));
    return r;
}

// Interleaved padded list (LJ_LIST_INTERLEAVED): the rows of a
// padded list in blocks of kIlRows, their entries interleaved in granules of
// kIlGran -- granule k of the block holds entries [4k, 4k+4) of row 0, then of
// row 1, ..., row 7 -- so that the index loads of a warp whose 8 rows x 4 lanes
// read entries 4k..4k+3 of 8 consecutive rows are ONE 128-B line instead of 8
// (tools/layout_probe.py: the gather replay 14 % faster).  pointer[r] holds the
// address of the row's entry 0 with bit 62 set; entry e of the row is at
// pointer + e + kIlSkip * (e / kIlGran).  Every list consumer decodes the row
// with row_decode, so compact, padded and interleaved lists all read correctly.
constexpr int kIlRows = 8, kIlGran = 4;
constexpr int kIlSkip = (kIlRows - 1) * kIlGran;   // 28
constexpr int64_t kIlBit = 1LL << 62;
__device__ __forceinline__ const int32_t* row_decode(const int32_t* list, int64_t p0, int& skip) {
    skip = (p0 & kIlBit) ? kIlSkip : 0;
    return list + (p0 & (kIlBit - 1));
}
// offset of entry e from the row base (skip from row_decode)
__device__ __forceinline__ int il_off(int e, int skip) { return e + skip * (e >> 2); }

// Cell geometry shared by the list builder and the cell-order pass.
struct CellGrid {
    double L, inv_w;   // inv_w = nc / L
    int nc;
    int64_t ncell;
};

// Workspace carve-out (offsets in bytes, 256-B aligned).
struct BuildWorkspace {
    size_t off_cell_of, off_count, off_start, off_cursor, off_atoms, off_qcell, off_qf, off_qr, off_scan, off_over,
        off_flags, off_ptrtmp, off_scratch, off_setup, total;
    int64_t scan_blocks;
};

BuildWorkspace build_workspace_layout(int64_t n, int64_t ncell, int64_t rows);

// Launchers (return cudaGetLastError()).
cudaError_t launch_cells(const double* q, int64_t n, const CellGrid& cg, char* ws, const BuildWorkspace& W,
                         cudaStream_t s);
// lj_rebuild: wrap q in place, cells, and the cell-order permutation applied to q/p (q_out, p_out, q_ref), with
// the builder's staging arrays prepared for the permuted system
// Momenta source of the re-sort: either p (all n records valid), or -- the multi-rank step,
// a device table of P pointers to every rank's copy of its own rows
// (peer-mapped over NVLink), rank = atom / n_own; only p_out rows [own_lo, own_hi) are written.
struct PeerMomenta {
    const double* const* table = nullptr;
    int64_t n_own = 0, own_lo = 0, own_hi = 0;
};
cudaError_t launch_rebuild_cells(double* q, const double* p, double* q_out, double* p_out, double* q_ref,
                                 int64_t* perm, int64_t n, const CellGrid& cg, char* ws, const BuildWorkspace& W,
                                 cudaStream_t s, const PeerMomenta& pm = PeerMomenta());
// pass 1: every row into the per-row scratch (stride kRowCap), counts into npart
// (out == nullptr: the workspace scratch; else the caller's padded list)
cudaError_t launch_list_pass1(const double* q, const CellGrid& cg, double rs, int half, int64_t row_begin,
                              int64_t row_end, int32_t* npart, int32_t* out, char* ws, const BuildWorkspace& W,
                              cudaStream_t s, bool interleaved = false);
cudaError_t launch_padded_pointer(int64_t* ptr, int64_t rows, cudaStream_t s, bool interleaved = false);
// pass 2: scratch -> CSR, or (if some row overflowed the scratch) a direct fill at pointer[r]
cudaError_t launch_list_pass2(const double* q, const CellGrid& cg, double rs, int half, int64_t row_begin,
                              int64_t row_end, int32_t* npart, const int64_t* ptr, int32_t* list, bool row_overflow,
                              char* ws, const BuildWorkspace& W, cudaStream_t s);
const int32_t* list_row_overflow_flag(char* ws, const BuildWorkspace& W);
// exclusive scan of int32 counts -> int64 offsets (out has n+1 entries)
cudaError_t launch_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, int64_t* block_sums,
                                   int64_t nblocks, cudaStream_t s);
cudaError_t launch_perm_from_cells(int64_t* perm, int64_t n, char* ws, const BuildWorkspace& W, cudaStream_t s);
cudaError_t launch_permute(const double* in, double* out, const int64_t* perm, int64_t n, cudaStream_t s);

struct ForceArgs {
    const double* q;
    double* p;
    int64_t n;   // atoms (the range every list index must lie in)
    int64_t row_begin, rows;
    const int32_t* npart;
    const int64_t* ptr;
    const int32_t* list;
    double L, rc2, dt;
    unsigned long long* n_inter;
};
cudaError_t launch_force_full(const ForceArgs& a, int lanes, cudaStream_t s);
cudaError_t launch_force_half(const ForceArgs& a, int lanes, cudaStream_t s);
cudaError_t launch_force_half_cells(const ForceArgs& a, const int64_t* cstart, int nc, int lanes, cudaStream_t s);
cudaError_t launch_force_ordered(const ForceArgs& a, cudaStream_t s);
cudaError_t launch_force_variant(const ForceArgs& a, int64_t n, int layout, int rcp, int lanes, cudaStream_t s);
cudaError_t launch_gather_probe(const ForceArgs& a, int lanes, double* sink, cudaStream_t s);

cudaError_t launch_pack(const double* xyz, double* out, int64_t n, cudaStream_t s);
cudaError_t launch_unpack(const double* in, double* xyz, int64_t n, cudaStream_t s);
cudaError_t launch_integrate(double* q, const double* p, int64_t begin, int64_t end, double dt, cudaStream_t s);
cudaError_t launch_integrate_disp(double* q, const double* p, const double* q_ref, int64_t begin, int64_t end,
                                  double dt, double* out, cudaStream_t s);
cudaError_t launch_integrate_push(const double* q_in, double* q_out, const double* p, const double* q_ref,
                                  int64_t begin, int64_t end, double dt, double* out, const lj_push_target* t,
                                  int n_targets, cudaStream_t s);
cudaError_t launch_wrap(double* q, double* q_ref, int64_t n, double L, cudaStream_t s);
cudaError_t launch_md_decide(const double* disp, int count, int64_t stride, double margin,
                             cudaGraphConditionalHandle h, int64_t* status, cudaStream_t s);
cudaError_t launch_copy_scalar(const double* src, double* dst, cudaStream_t s);
cudaError_t launch_build_status(const int64_t* total, const int32_t* row_overflow, int64_t* status, cudaStream_t s);
cudaError_t launch_max_disp(const double* q, const double* q_ref, int64_t begin, int64_t end, double* out,
                            cudaStream_t s);
cudaError_t launch_partner_ranges(int64_t row_begin, int64_t row_end, const int32_t* npart, const int64_t* ptr,
                                  const int32_t* list, const int64_t* bounds, int P, int64_t* out, cudaStream_t s);
cudaError_t launch_list_interior(int64_t row_begin, int64_t row_end, const int32_t* npart, const int64_t* ptr,
                                 const int32_t* list, int64_t* out, cudaStream_t s);
cudaError_t launch_energy(const double* q, const double* p, int64_t n, int64_t row_begin, int64_t rows,
                          const int32_t* npart,
                          const int64_t* ptr, const int32_t* list, double L, double rc2, double rc, int half,
                          double* out, cudaStream_t s);

inline int grid_for(int64_t work, int block, int max_blocks = 148 * 64) {
    int64_t g = (work + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}

}  // namespace lj
