/*
 * liblj.h -- C ABI of the B200 (sm_100a) Lennard-Jones force hot path of
 * Watanabe & Nakagawa, arXiv 1806.05713.  Implemented by
 * paper_1806_05713_b200/liblj.so (hand-written CUDA, fp64, no tensor cores).
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers owned by the caller unless stated; the
 *    library allocates nothing on the device (workspaces are caller-provided)
 *    and keeps no global device state.
 *  - q, p: n records of 4 doubles (x, y, z, pad) -- the paper's "AoS with
 *    padding" layout (Fig. aos4).  Base address 32-byte
 *    aligned (checked: one 256-bit load per record).  The pad is never read
 *    into arithmetic and is preserved by every call.
 *  - Lists are the paper's sorted list (Fig. sorted_list) in
 *    CSR form, local to a row range [row_begin, row_end): row r <-> atom
 *    row_begin + r; number_of_partners[rows] (int32), pointer[rows+1] (int64;
 *    the builder writes pointer[0] = 0, consumers only read row r's entries at
 *    sorted_list + pointer[r], so a contiguous sub-range of rows is addressed by
 *    offsetting number_of_partners and pointer), sorted_list (int32 global atom
 *    indices, ascending within a row).  n < 2^31 is checked.
 *  - Full list (half = 0): row i holds every j != i with r_ij^2 < rs^2.
 *    Half list (half = 1): row i holds only j > i (each pair once, PAPER.md
 *    Alg. calcforce_sortedlist); a half list must cover all rows [0, n).
 *  - Geometry: L > 0 is a periodic cube of side L (minimum image, DESIGN.md
 *    reading C-3); L == 0 is open space (force/energy only).  0 < rc < rs.
 *  - Stream-ordered and asynchronous on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream), except lj_build_list, which
 *    synchronises `stream` once to read the entry count.
 *  - Errors: arguments are validated before anything is enqueued; a failure
 *    returns LJ_ERR_ARG and launches nothing.  A CUDA launch error returns
 *    LJ_ERR_CUDA; lj_last_error() gives the detail (thread-local).  Faults of
 *    already-enqueued kernels surface at the next synchronising call.  No
 *    exception or abort crosses the ABI.
 *  - Re-entrant on different streams with disjoint outputs.
 */
#ifndef LIBLJ_H
#define LIBLJ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LJ_OK = 0,
    LJ_ERR_ARG = 1,          /* invalid argument; nothing launched */
    LJ_ERR_CAPACITY = 2,     /* list capacity too small; *n_entries = required */
    LJ_ERR_CUDA = 3,         /* CUDA runtime error; see lj_last_error() */
    LJ_ERR_UNSUPPORTED = 4   /* valid but unsupported combination */
} lj_status;

/* L: periodic box side (0 = open); rc: cutoff ("simple
 * truncation", interact iff r^2 < rc^2); rs: search length of the Verlet list
 * ("register each pair within a search length r_s"). */
typedef struct {
    double L;
    double rc;
    double rs;
} lj_geom;

/* ---- layout (§8(a) a1) --------------------------------------------------- */

/* xyz: n x 3 doubles (device) -> out: n x 4 doubles, pad = 0. */
lj_status lj_pack_aos4(const double *xyz, double *out, int64_t n, void *stream);
/* in: n x 4 -> xyz: n x 3 (drops the pad). */
lj_status lj_unpack_aos4(const double *in, double *xyz, int64_t n, void *stream);

/* ---- neighbour list (§8(a) a2-a4) ---------------------- */

/* Bytes of device workspace lj_build_list / lj_cell_order need for n atoms. */
lj_status lj_build_list_workspace(int64_t n, lj_geom g, size_t *bytes);

/* Linked-cell Verlet list: cells of side L/nc, nc =
 * floor(L/rs) >= 3 (requires L > 0); cell of an atom from its position wrapped
 * into [0,L); pairs accepted iff the minimum-image r^2 = (dx*dx + dy*dy) + dz*dz,
 * evaluated without FMA, is < rs*rs (bit-identical to the oracle's test).
 * Rows [row_begin, row_end) are built; half = 1 needs the full range.
 * Outputs number_of_partners[rows], pointer[rows+1], sorted_list[capacity].
 * *n_entries (HOST) receives the required entry count.  If capacity is too
 * small the call returns LJ_ERR_CAPACITY (list contents undefined; capacity 0
 * is a size query).  Synchronises `stream` once. */
lj_status lj_build_list(const double *q, int64_t n, lj_geom g, int half,
                        int64_t row_begin, int64_t row_end,
                        int32_t *number_of_partners, int64_t *pointer,
                        int32_t *sorted_list, int64_t capacity, int64_t *n_entries,
                        void *workspace, size_t workspace_bytes, void *stream);

/* Layout flag of lj_build_list_ex: row r of the list starts at
 * pointer[r] = r * LJ_PADDED_ROW_STRIDE (rows padded to a fixed stride; entries
 * past number_of_partners[r] are undefined).  Saves the compaction pass of the
 * compact CSR; every consumer of a list (force, energy) reads only
 * [pointer[r], pointer[r] + number_of_partners[r]). */
#define LJ_LIST_PADDED 1
/* With LJ_LIST_PADDED only: do not synchronise.  n_entries must then point to
 * 2 int64 of PINNED host memory, written in stream order: [0] = the number of
 * valid entries, [1] = non-zero if a row exceeded the stride (the list is then
 * invalid -- rebuild with the compact layout); [1] must be 0 on entry.  The
 * caller reads them after a later synchronisation (the MD driver: at the next
 * displacement readback), so a rebuild costs no host round trip. */
#define LJ_LIST_DEFERRED 2
/* With LJ_LIST_PADDED only: the rows in blocks of 8 (rows row_begin + 8b ..
 * + 8b + 7), their entries interleaved in granules of 4 -- granule k of a block
 * holds entries 4k..4k+3 of its row 0, then of its row 1, ..., of its row 7
 * -- so that the force kernel's index loads (4 lanes per row, 8
 * rows per warp) are one 128-byte line each.  pointer[r] = the position of
 * row r's entry 0 with bit 62 set (LJ_LIST_IL_BIT); entry e of row r is at
 * (pointer[r] & (LJ_LIST_IL_BIT - 1)) + e + 28 * (e / 4); pointer[rows] = the
 * padded extent.  capacity must be >= ceil(rows / 8) * 8 * LJ_PADDED_ROW_STRIDE.
 * Every consumer of a list in this library (force, energy, row
 * classification) reads compact, padded and interleaved lists alike. */
#define LJ_LIST_INTERLEAVED 4
#define LJ_LIST_IL_BIT (1LL << 62)
#ifndef LJ_PADDED_ROW_STRIDE
/* 196 entries = 784 B: not a multiple of the 128-B line, so the rows a warp
 * reads do not all start on the same DRAM channel / L2 slice (strides of 640 or
 * 768 B made the force step 10 % slower, tools/stride_sweep.sh). */
#define LJ_PADDED_ROW_STRIDE 196
#endif

/* lj_build_list with layout flags (0 = compact CSR, as lj_build_list).  With
 * LJ_LIST_PADDED, capacity must be >= rows * LJ_PADDED_ROW_STRIDE (rows rounded
 * up to a multiple of 8 with LJ_LIST_INTERLEAVED; else
 * LJ_ERR_CAPACITY, *n_entries = that size); *n_entries receives the number of
 * valid entries; a row longer than the stride returns LJ_ERR_UNSUPPORTED (use
 * the compact layout).  Same synchronisation as lj_build_list. */
lj_status lj_build_list_ex(const double *q, int64_t n, lj_geom g, int half, int64_t row_begin, int64_t row_end,
                           int flags, int32_t *number_of_partners, int64_t *pointer, int32_t *sorted_list,
                           int64_t capacity, int64_t *n_entries, void *workspace, size_t workspace_bytes,
                           void *stream);

/* Fused bookkeeping rebuild (PAPER.md:190-192 with the config-3 reordering):
 * wrap q into [0,L) in place (as lj_wrap), perm = the cell order of the wrapped
 * q (as lj_cell_order), q_out = q[perm], p_out = p[perm] (skipped if p == NULL),
 * q_ref = q_out (skipped if NULL), and the list of rows [row_begin, row_end) of
 * the PERMUTED system q_out -- every output bit-identical to lj_wrap +
 * lj_cell_order + lj_permute_rows + lj_build_list_ex(q_out, ...), from a single
 * cell pass.  Outputs must not alias inputs or each other.  List arguments,
 * flags, capacity protocol and synchronisation as lj_build_list_ex (a repeated
 * call after LJ_ERR_CAPACITY with the same arguments is valid: wrapping is
 * idempotent). */
lj_status lj_rebuild(double *q, const double *p, double *q_out, double *p_out, double *q_ref, int64_t *perm,
                     int64_t n, lj_geom g, int half, int64_t row_begin, int64_t row_end, int flags,
                     int32_t *number_of_partners, int64_t *pointer, int32_t *sorted_list, int64_t capacity,
                     int64_t *n_entries, void *workspace, size_t workspace_bytes, void *stream);

/* Spatial reordering (BASELINE.json config 3): perm[new] = old, the stable
 * sort of the atoms by cell id (cx*nc + cy)*nc + cz (same cells as the list). */
lj_status lj_cell_order(const double *q, int64_t n, lj_geom g, int64_t *perm,
                        void *workspace, size_t workspace_bytes, void *stream);

/* out[k] = in[perm[k]] for n records of 4 doubles (in != out). */
lj_status lj_permute_rows(const double *in, double *out, const int64_t *perm, int64_t n, void *stream);

/* ---- force (§8(a) a5/a6; PAPER.md Alg. lj_force + Alg. calcforce_sortedlist) */

/* One force step: for every own row i and every j in its row with
 * r^2 < rc^2: df = (48 - 24 r^6) dt / r^14, p_i -= df r_vec,
 * and for a half list also p_j += df r_vec (Newton 3; PAPER.md:172 prints
 * "-", reading C-1).  r_vec = minimum-image q_j - q_i.
 * Full list: only p of own rows changes, deterministic, no atomics.
 * Half list: p of any atom changes (fp64 atomics; summation order not
 * deterministic).  p is indexed by global atom index. */
lj_status lj_force_step(const double *q, double *p, int64_t n, lj_geom g, double dt, int half,
                        int64_t row_begin, int64_t row_end,
                        const int32_t *number_of_partners, const int64_t *pointer,
                        const int32_t *sorted_list, void *stream);

/* lanes_per_row flag: the list indices are read V = U (2 or 4) at a time with
 * one 64/128-bit load per thread (fewer L1 requests for the index stream). */
#define LJ_LANES_IDXV (1 << 16)

/* Tuning / instrumentation variant of lj_force_step.
 * lanes_per_row = G | (U << 8) [| LJ_LANES_IDXV]: G (1,2,4,8,16,32) threads
 * cooperate on a row, U (2,3,4; 0 = 2) partner gathers in flight per thread;
 * with LJ_LANES_IDXV, G in (1,2,4,8,16) and U in (2,4) is the index vector
 * width.  0 = the library default (lj_default_lanes).
 * n_interactions: NULL or a device uint64 to which the
 * number of list entries inside r_c is ADDED (pair interactions; a full list
 * counts each pair twice).  ordered != 0 (full list only): one thread per row,
 * ascending j, the oracle's exact expression order (Alg. 3 accumulating into
 * the loaded p_i, IEEE division, no FMA) -- bit-identical to the oracle. */
/* The lanes_per_row lj_force_step uses for `rows` rows of a full (half = 0) or
 * half list (the round-2 sweeps). */
int lj_default_lanes(int64_t rows, int half);

lj_status lj_force_step_ex(const double *q, double *p, int64_t n, lj_geom g, double dt, int half,
                           int64_t row_begin, int64_t row_end,
                           const int32_t *number_of_partners, const int64_t *pointer,
                           const int32_t *sorted_list, int lanes_per_row, int ordered,
                           unsigned long long *n_interactions, void *stream);

/* ---- half list without per-entry global atomics ------ */

/* The cell structure of the last list build (lj_build_list[_ex] / lj_rebuild
 * with this workspace, n and g): cell_start (device, ncell + 1 int64, ncell =
 * floor(L/rs)^3) = the first position of every cell in the cell-sorted atom
 * order; for cell-ordered storage (lj_rebuild's output, or lj_cell_order +
 * lj_permute_rows before the build) cell c holds atoms [cell_start[c],
 * cell_start[c+1]).  Asynchronous (one device copy). */
lj_status lj_list_cell_starts(const void *workspace, size_t workspace_bytes, int64_t n, lj_geom g,
                              int64_t *cell_start, void *stream);

/* lj_force_step for a HALF list over all rows [0, n) (Alg. 3, PAPER.md
 * P:247-267) without per-entry global atomics: one CTA per cell takes the rows
 * [cell_start[c], cell_start[c+1]) and accumulates the p_j contributions of
 * its rows -- and the rows' own sums -- in a shared-memory window over the 27
 * neighbour cells' index ranges, then adds the window to p with one fp64 RED
 * per component and atom.  Same result as lj_force_step(half = 1) up to
 * summation order (C-12); any storage order is correct (partners outside the
 * window take a global RED), cell-ordered storage is the fast case.
 * lanes_per_row: 0 (= 8 | 2 << 8), 2 | 2 << 8, 4 | 2 << 8, 8 | 2 << 8 or 4 | 3 << 8.
 * n_interactions as lj_force_step_ex.  Asynchronous. */
lj_status lj_force_step_half_cells(const double *q, double *p, int64_t n, lj_geom g, double dt,
                                   const int32_t *number_of_partners, const int64_t *pointer,
                                   const int32_t *sorted_list, const int64_t *cell_start, int lanes_per_row,
                                   unsigned long long *n_interactions, void *stream);

/* ---- paper-variant ablations (not the hot path) ------- */

/* Position/momentum layouts of the paper's variant axis (PAPER.md:117-126,
 * 341-353, 551-573).  q and p are n atoms in the given layout (for AOS8 both
 * live in q's 64-byte records and p is ignored). */
#define LJ_LAYOUT_AOS4 0   /* x, y, z, pad: 32-B records (the library's layout) */
#define LJ_LAYOUT_SOA 1    /* x[n], y[n], z[n]: 3n doubles, x block first */
#define LJ_LAYOUT_AOS3 2   /* x, y, z without padding: 24-B records */
#define LJ_LAYOUT_AOS8 3   /* q.x, q.y, q.z, pad, p.x, p.y, p.z, pad: 64-B records */
/* 1/r^2 evaluation (the paper's reciprocal "future issue"). */
#define LJ_RCP_NEWTON3 0   /* rcp.approx + one cubic Newton step (lj_force_step) */
#define LJ_RCP_NEWTON2 1   /* rcp.approx + one quadratic Newton step */
#define LJ_RCP_APPROX 2    /* rcp.approx (MUFU.RCP64H) alone */
#define LJ_RCP_IEEE 3      /* correctly rounded reciprocal */

/* lj_force_step (full list only) in another layout / reciprocal: the same
 * lanes-per-row kernel structure and arithmetic as lj_force_step, only the
 * gathers, the momentum commit or 1/r^2 differ (so LJ_LAYOUT_* with
 * LJ_RCP_NEWTON3 give bit-identical momenta).  lanes_per_row: 4 or 8.
 * Alignment: 32 B for AOS4/AOS8, 8 B otherwise. */
lj_status lj_force_step_variant(int layout, int rcp, const double *q, double *p, int64_t n, lj_geom g, double dt,
                                int64_t row_begin, int64_t row_end, const int32_t *number_of_partners,
                                const int64_t *pointer, const int32_t *sorted_list, int lanes_per_row,
                                unsigned long long *n_interactions, void *stream);

/* Roofline probe (not part of the method): the memory traffic of lj_force_step
 * on a full list -- the same lanes-per-row mapping and gathers in flight
 * (lanes_per_row = G | (U << 8) as lj_force_step_ex, 0 = its defaults), index
 * loads and 256-bit record gathers -- with no arithmetic beyond a running sum
 * written to *sink (device double).  Its duration is the gather-bandwidth floor
 * of the force kernel (SURVEY §8(d) "gather-only replay of the actual CSR list"). */
lj_status lj_gather_probe(const double *q, int64_t n, int64_t row_begin, int64_t row_end,
                          const int32_t *number_of_partners, const int64_t *pointer,
                          const int32_t *sorted_list, int lanes_per_row, double *sink, void *stream);

/* Interior rows of a row-split full list (comm/compute
 * overlap): out (device, 2 x int64) = {A, B} such that every row in [A, B)
 * has all its partners inside [row_begin, row_end) -- the force on those rows
 * needs no position of another rank, so it can run while the all-gather of
 * the other ranks' positions is in flight.  [A, B) is the contiguous interior
 * run around the middle row (A = row_begin, B = row_end if no row looks
 * outside).  Asynchronous. */
lj_status lj_list_interior(int64_t row_begin, int64_t row_end, const int32_t *number_of_partners,
                           const int64_t *pointer, const int32_t *sorted_list, int64_t *out, void *stream);

/* Halo requests of a row-split list (halo exchange in place
 * of the all-gather): the P owner slabs are rows [bounds[s], bounds[s+1])
 * (bounds: device, P + 1 int64, ascending, bounds[P] = n); out (device, 2P
 * int64) = for every s, {min, max} of the partner indices of rows [row_begin,
 * row_end) that lie in slab s, or {INT64_MAX, -1} if none.  The force on these
 * rows reads exactly positions [min, max] of each slab it touches.  1 <= P <=
 * 64.  Asynchronous. */
lj_status lj_list_partner_ranges(int64_t row_begin, int64_t row_end, const int32_t *number_of_partners,
                                 const int64_t *pointer, const int32_t *sorted_list, const int64_t *bounds, int P,
                                 int64_t *out, void *stream);

/* ---- integration and bookkeeping (§8(a) a7, a9) --------------------------- */

/* Drift q_i += p_i dt for atoms [begin, end) (mass 1), bit-identical to the
 * oracle (no FMA).  Positions are not wrapped. */
lj_status lj_integrate(double *q, const double *p, int64_t begin, int64_t end, double dt, void *stream);

/* lj_integrate followed by lj_max_displacement(q, q_ref, begin, end, max_disp)
 * in one pass over the own rows (both results bit-identical to the two calls). */
lj_status lj_integrate_displacement(double *q, const double *p, const double *q_ref, int64_t begin, int64_t end,
                                   double dt, double *max_disp, void *stream);

/* ---- fused drift + NVLink push ------------------------ */

/* One destination of lj_integrate_push: rows [lo, hi) of the caller's own range
 * are also stored to dst (a q replica of another rank, n records, mapped into
 * this process -- by lj_ipc_open on another GPU of the node, or any device
 * pointer), at the same row index. */
typedef struct {
    double *dst;
    int64_t lo, hi;
} lj_push_target;

#ifndef LJ_MAX_PUSH_TARGETS
#define LJ_MAX_PUSH_TARGETS 63
#endif

/* lj_integrate_displacement with the position exchange fused in: for own rows
 * [begin, end), q_out_i = q_in_i + p_i dt (bit-identical to lj_integrate),
 * *max_disp = max |q_out_i - q_ref_i| (as lj_max_displacement), and every
 * updated record is also stored straight into targets[k].dst for the targets
 * whose [lo, hi) holds i -- one kernel, the peer stores issued by the threads
 * that computed the records (no separate copy or collective).  q_out may equal
 * q_in.  The kernel ends with a system-scope fence: once it has completed
 * (e.g. ordered before a collective on the same stream), the stores are
 * visible to the peers.  The CALLER orders the pushes against the peers'
 * readers (the MD driver double-buffers the replicas).
 * 0 <= n_targets <= LJ_MAX_PUSH_TARGETS; targets is a host array; every dst
 * 32-byte aligned.  Asynchronous. */
lj_status lj_integrate_push(const double *q_in, double *q_out, const double *p, const double *q_ref,
                            int64_t begin, int64_t end, double dt, double *max_disp,
                            const lj_push_target *targets, int n_targets, void *stream);

/* CUDA IPC for the push targets (one process per GPU).  lj_ipc_get_handle:
 * a 64-byte handle of the device allocation holding ptr, and ptr's byte offset
 * inside it.  lj_ipc_open (another process): map that allocation (peer access
 * enabled lazily) and return the pointer at `offset`; lj_ipc_close unmaps it
 * (pass the pointer lj_ipc_open returned).  Synchronous. */
lj_status lj_ipc_get_handle(const void *ptr, void *handle /* 64 bytes */, int64_t *offset);
lj_status lj_ipc_open(const void *handle, int64_t offset, void **ptr);
lj_status lj_ipc_close(void *ptr);

/* ---- the MD step as a CUDA graph ("capture the whole
 * step ... a conditional node can skip the rebuild"; one rank) -------------- */

/* Buffers of a single-rank leapfrog MD (BASELINE.json configs 4-5, reading O8 /
 * C-16), all device memory owned by the caller and used by every launch. */
typedef struct {
    double *q, *p;            /* n AoS4 records each: the state, updated in place (p's pad is carried) */
    double *q_alt, *p_alt;    /* n records each: scratch of the re-sorting rebuild (reorder != 0) */
    double *q_ref;            /* n records: positions at the last build (written by every rebuild) */
    int64_t *perm;            /* n: scratch (perm of the last re-sort) */
    int64_t n;
    lj_geom g;
    double dt;
    int32_t *number_of_partners; /* the current full list over rows [0, n), padded layout (LJ_LIST_PADDED) */
    int64_t *pointer;
    int32_t *sorted_list;
    int64_t capacity;         /* >= n * LJ_PADDED_ROW_STRIDE */
    void *workspace;          /* lj_build_list_workspace(n, g) bytes */
    size_t workspace_bytes;
    double *disp;             /* 1 double: scratch (max displacement) */
    unsigned long long *n_interactions; /* NULL or a counter, as lj_force_step_ex */
    int64_t *status;          /* 4 int64: [0] += rebuilds, [1] = 1 if a rebuilt row overflowed the stride
                                 (the list is then invalid), [2] = entries of the last rebuild */
    int reorder;              /* re-sort into cell order at every rebuild (as lj_rebuild) */
    int steps;                /* steps per launch, 1..100000 (unrolled in the graph) */
    int energy_every;         /* 0, or sample (KE, PE) at steps k % energy_every == 0 of every launch: the
                                 kick is split in two halves around lj_energy (reading O8, synchronised p) */
    double *energies;         /* 2 doubles per sample (ceil(steps / energy_every) samples), if energy_every */
    int interleaved;          /* the list is LJ_LIST_INTERLEAVED (rebuilds keep that layout; capacity as there) */
} lj_md_graph_desc;

typedef struct lj_md_graph lj_md_graph;

/* Instantiate one MD step as a CUDA graph: p += F(q) dt (lj_force_step, full
 * list); q += p dt with the displacement (lj_integrate_displacement); a
 * one-thread kernel takes the bookkeeping decision on the device (2 max|q -
 * q_ref| >= rs - rc) and sets the condition of an IF node whose body is the
 * rebuild -- reorder: lj_rebuild into q_alt / p_alt, then copied back into
 * q / p; else lj_wrap(q, q_ref) + the build -- with its status to `status`.
 * The d->steps steps are unrolled into one graph, so a launch is host-free: no
 * readback per step or per rebuild.
 * Bit-identical to the same calls made one by one.  The list must be current
 * before the first launch (e.g. from lj_rebuild). */
lj_status lj_md_graph_create(const lj_md_graph_desc *d, lj_md_graph **out);
/* Run the graph's `steps` steps on `stream` (asynchronous; one launch). */
lj_status lj_md_graph_launch(lj_md_graph *gr, void *stream);
/* After a launch has completed: ms[k] = duration of step k's force kernel (CUDA
 * events recorded around it inside the graph), k < min(n, steps). */
lj_status lj_md_graph_force_ms(const lj_md_graph *gr, float *ms, int n);
/* Kernels one launch runs without its rebuilds (all unrolled steps) / per rebuild. */
lj_status lj_md_graph_kernels(const lj_md_graph *gr, long long *steps_total, long long *per_rebuild);
lj_status lj_md_graph_destroy(lj_md_graph *gr);

/* ---- the multi-rank step under the caller's stream capture (P > 1; SURVEY
 * §8(f) NEXT-1 "capture the whole step, NCCL included, in a CUDA graph") ---- */

/* Buffers of one rank's bookkeeping rebuild (rows split into
 * equal slabs); device memory owned by the caller.  Without
 * reorder the atoms keep their storage slots; with reorder every rebuild
 * re-sorts them into cell order as lj_rebuild does (the fast path of the list
 * builder needs cell-ordered storage). */
typedef struct {
    double *q;                /* n records: replicated positions (complete after the position exchange) */
    double *q_ref;            /* n records: bookkeeping reference (written by every rebuild) */
    int64_t n;
    lj_geom g;
    int64_t row_begin, row_end;   /* own rows */
    int32_t *number_of_partners;  /* own rows' padded list (LJ_LIST_PADDED), current before the first launch */
    int64_t *pointer;
    int32_t *sorted_list;
    int64_t capacity;         /* >= (row_end - row_begin) * LJ_PADDED_ROW_STRIDE */
    void *workspace;          /* lj_build_list_workspace(n, g) bytes */
    size_t workspace_bytes;
    const double *disp;       /* the decision reads max_k disp[k * disp_stride], k < disp_count: e.g. the */
    int disp_count;           /* pads of every rank's first q record after the all-gather (see */
    int64_t disp_stride;      /* lj_publish_scalar), or one all-reduced double (count 1, stride 0) */
    int64_t *status;          /* 4 int64, as lj_md_graph_desc.status */
    int reorder;              /* re-sort all atoms into cell order at every rebuild (as lj_rebuild); the own
                                 rows then change owner-rank, their momenta are read from p_peers: */
    double *q_alt;            /* n records: scratch */
    double *p;                /* n records: this rank's momenta (own rows [row_begin, row_end) valid) */
    double *p_alt;            /* n records: scratch */
    int64_t *perm;            /* n: scratch */
    const double *const *p_peers; /* DEVICE array of P pointers: rank k's copy of its own rows' momenta
                                 (n records, rows [k n_own, (k+1) n_own) valid; peer-mapped, e.g. CUDA
                                 IPC), current when the rebuild runs -- see lj_copy_records */
    int64_t n_own;            /* rows per rank (equal slabs; own rows = one slab) */
    int interleaved;          /* the list is LJ_LIST_INTERLEAVED (rebuilds keep that layout; capacity as there) */
} lj_md_rebuild_desc;

/* Called while `stream` is being captured into a CUDA graph (cudaStreamBeginCapture
 * in relaxed mode, e.g. inside torch.cuda.graph holding the step's NCCL
 * collectives): appends to the capture a one-thread kernel that takes the
 * bookkeeping decision (rebuild iff 2 max_k disp[k*stride] >= rs - rc, reading
 * C-16) and an IF node whose body wraps all n records of q
 * (q_ref = the wrapped q, as lj_wrap) -- with reorder, also re-sorts every atom
 * into cell order (as lj_permute_rows_peers, the permuted q / own p copied back
 * into q / p) -- and rebuilds the own rows' padded list (as lj_build_list_ex,
 * status to d->status as lj_md_graph).  Work captured
 * afterwards on `stream` depends on the IF node.  *kernels_per_rebuild (if not
 * NULL) = kernels the body launches.  LJ_ERR_ARG if `stream` is not capturing. */
lj_status lj_md_capture_rebuild(const lj_md_rebuild_desc *d, void *stream, long long *kernels_per_rebuild);

/* dst[k] = src[k] for n records (device, stream-ordered; src == dst is a no-op): e.g. a
 * rank's own momenta into the buffer its peers read at a re-sorting rebuild. */
lj_status lj_copy_records(const double *src, double *dst, int64_t n, void *stream);

/* bytes from src to dst, stream-ordered, either side device or page-locked host
 * memory (cudaMemcpyAsync, direction from the addresses): the per-step state
 * copies of the end-to-end step graph (md.LeapfrogMD.graph_host_io), capturable
 * into a CUDA graph.  Asynchronous. */
lj_status lj_copy_bytes(void *dst, const void *src, size_t bytes, void *stream);

/* The multi-rank re-sort on its own (lj_rebuild's cell pass without the list):
 * q (n records, replicated) is wrapped in place, perm[new] = old is the stable
 * cell order, q_out = q permuted, q_ref = q_out (if not NULL), and for the own
 * new rows [own_lo, own_hi) p_out[k] = p_peers[perm[k] / n_own][perm[k]] -- the
 * momenta read from the rank that owned the atom (device table of P pointers,
 * peer-mapped).  Rows of p_out outside [own_lo, own_hi) are not written. */
lj_status lj_permute_rows_peers(double *q, double *q_out, double *q_ref, double *p_out,
                                const double *const *p_peers, int64_t n_own, int64_t own_lo, int64_t own_hi,
                                int64_t *perm, int64_t n, lj_geom g, void *workspace, size_t workspace_bytes,
                                void *stream);

/* dst[0] = src[0] (device doubles), stream-ordered: e.g. the rank's maximum
 * displacement into the pad lane of its first own q record, which the position
 * all-gather then carries to every rank -- the bookkeeping decision without a
 * separate all-reduce.  Pads are ignored by every kernel. */
lj_status lj_publish_scalar(const double *src, double *dst, void *stream);

/* Wrap q into [0,L) (x -= L floor(x/L); x -= L if x >= L) for atoms [0,n) and,
 * if q_ref != NULL, copy the wrapped records to q_ref (the bookkeeping
 * reference of PAPER.md:190-192). */
lj_status lj_wrap(double *q, double *q_ref, int64_t n, double L, void *stream);

/* *out (device double) = max_{i in [begin,end)} |q_i - q_ref_i| (Euclidean). */
lj_status lj_max_displacement(const double *q, const double *q_ref, int64_t begin, int64_t end,
                              double *out, void *stream);

/* ---- energy (§8(a) a10; PAPER.md:146 Eq. lj with V(r_c) = 0) -------------- */

/* out (device, 2 doubles) = {KE over own rows, PE over the list's entries
 * inside r_c}: PE counts each half-list entry once and each full-list entry
 * 1/2 (so row ranges partition the sum).  Overwrites out. */
lj_status lj_energy(const double *q, const double *p, int64_t n, lj_geom g,
                    int64_t row_begin, int64_t row_end,
                    const int32_t *number_of_partners, const int64_t *pointer,
                    const int32_t *sorted_list, int half, double *out, void *stream);

/* ---- diagnostics ---------------------------------------------------------- */

const char *lj_status_string(lj_status s);
const char *lj_last_error(void);
/* Number of kernels this library has launched in the process (all threads). */
long long lj_launch_count(void);
/* Library version string. */
const char *lj_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LIBLJ_H */
