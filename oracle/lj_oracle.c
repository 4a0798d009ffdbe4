/*
 * lj_oracle.c -- plain, slow, single-threaded CPU oracle for the LJ force hot
 * path of Watanabe & Nakagawa, arXiv 1806.05713 ("SIMD Vectorization for the
 * Lennard-Jones Potential with AVX2 and AVX-512 instructions").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, constant generator or helper with the CUDA path
 * (paper_1806_05713_b200/csrc); neither includes the other.
 *
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fno-fast-math -shared -fPIC
 * (no FMA contraction, no reassociation: every expression below is evaluated
 * in the order written, in IEEE binary64).
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; C-n / O-n / Pin-n =
 * the readings in DESIGN.md.
 *
 * Layout: the oracle uses its own plain layout, positions and momenta as
 * (n,3) row-major double arrays, not the product's padded AoS4.
 *
 * Pins (tests/test_oracle_*.py): every function here is pinned to something
 * other than itself -- closed forms (Pin-1..4), SPEC worked examples (Pin-8),
 * brute force (Pin-5, Pin-6), conservation laws (Pin-7, Pin-10).  The only
 * unpinned property is the summation order inside a row, which the paper
 * leaves free.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- geometry ------------------------------------------------------------ */

/* Minimum image per axis (reading O2 / C-3: periodic cube of side L;
 * L == 0 means open boundaries).  Valid while |d| < 1.5 L. */
static double minimum_image(double d, double L)
{
    if (L > 0.0) {
        if (d > 0.5 * L)
            d -= L;
        else if (d < -0.5 * L)
            d += L;
    }
    return d;
}

/* r = q_j - q_i and r^2 = r . r  (Alg. 1 lines 1-2), reading O3:
 * r2 = (dx*dx + dy*dy) + dz*dz in that association, no FMA. */
static double relative(const double *qi, const double *qj, double L, double r[3])
{
    r[0] = minimum_image(qj[0] - qi[0], L);
    r[1] = minimum_image(qj[1] - qi[1], L);
    r[2] = minimum_image(qj[2] - qi[2], L);
    return (r[0] * r[0] + r[1] * r[1]) + r[2] * r[2];
}

/* Alg. 1 lines 3-5: r6 = r2*r2*r2, r14 = r6*r6*r2,
 * df = (48 - 24 r6) dt / r14. */
static double impulse_coefficient(double r2, double dt)
{
    double r6 = (r2 * r2) * r2;
    double r14 = (r6 * r6) * r2;
    return ((48.0 - 24.0 * r6) * dt) / r14;
}

/* ---- counting sort of a pair list (Fig. sorted_list) ----------- */

/* Stable counting sort of pairs (pi[k], pj[k]) by pi into offsets[n+1] and
 * jidx[npairs]: "This list can be constructed by a counting sort".
 * pairs [(0,1),(0,3),(2,5),(0,7)], n=8 -> offsets
 * [0,3,3,4,4,4,4,4,4], j [1,3,7,5]  (Pin-8). Returns npairs. */
int64_t lj_oracle_sort_pair_list(const int32_t *pi, const int32_t *pj, int64_t npairs, int64_t n,
                                 int64_t *offsets, int32_t *jidx)
{
    int64_t i, k;
    int64_t *fill;
    for (i = 0; i <= n; i++)
        offsets[i] = 0;
    for (k = 0; k < npairs; k++)          /* histogram of i */
        offsets[pi[k] + 1] += 1;
    for (i = 0; i < n; i++)               /* exclusive prefix sum */
        offsets[i + 1] += offsets[i];
    fill = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (i = 0; i < n; i++)
        fill[i] = offsets[i];
    for (k = 0; k < npairs; k++)          /* stable placement */
        jidx[fill[pi[k]]++] = pj[k];
    free(fill);
    return npairs;
}

/* ---- neighbour list, O(N^2) brute force (definition) --------------------- */

/* Verlet list with search length rs: every pair with r2 < rs2 (strict,
 * reading C-4), j != i.  half != 0: only i < j (each pair once, as Alg. 3
 * updates both atoms); half == 0: both (i,j) and (j,i).
 * Rows [row_begin,row_end) are kept, as a row-local CSR (pointer[0] = 0).
 * Pairs are emitted in double-loop order and grouped with the counting sort
 * above, which leaves every row ascending in j (reading C-10).
 * Returns the number of entries; fills the outputs only if cap >= that. */
int64_t lj_oracle_list_brute(const double *q, int64_t n, double L, double rs, int half,
                             int64_t row_begin, int64_t row_end,
                             int32_t *number_of_partners, int64_t *pointer, int32_t *sorted_list,
                             int64_t cap)
{
    const double rs2 = rs * rs;
    int64_t i, j, np = 0, k = 0, rows = row_end - row_begin;
    int32_t *pi, *pj;
    int64_t *offsets;
    double r[3];
    for (i = 0; i < n; i++)
        for (j = i + 1; j < n; j++)
            if (relative(&q[3 * i], &q[3 * j], L, r) < rs2) {
                if (i >= row_begin && i < row_end)
                    np++;
                if (!half && j >= row_begin && j < row_end)
                    np++;
            }
    if (cap < np)
        return np;
    pi = (int32_t *)malloc((size_t)(np > 0 ? np : 1) * sizeof(int32_t));
    pj = (int32_t *)malloc((size_t)(np > 0 ? np : 1) * sizeof(int32_t));
    for (i = 0; i < n; i++)
        for (j = i + 1; j < n; j++)
            if (relative(&q[3 * i], &q[3 * j], L, r) < rs2) {
                if (i >= row_begin && i < row_end) {
                    pi[k] = (int32_t)(i - row_begin);
                    pj[k] = (int32_t)j;
                    k++;
                }
                if (!half && j >= row_begin && j < row_end) {
                    pi[k] = (int32_t)(j - row_begin);
                    pj[k] = (int32_t)i;
                    k++;
                }
            }
    offsets = (int64_t *)malloc((size_t)(rows + 1) * sizeof(int64_t));
    lj_oracle_sort_pair_list(pi, pj, np, rows, offsets, sorted_list);
    for (i = 0; i < rows; i++) {
        pointer[i] = offsets[i];
        number_of_partners[i] = (int32_t)(offsets[i + 1] - offsets[i]);
    }
    pointer[rows] = offsets[rows];
    free(offsets);
    free(pi);
    free(pj);
    return np;
}

/* ---- neighbour list, linked-cell method ----------------------- */

/* Cell grid: nc = floor(L/rs) cells per side, nc >= 3 so the 27 stencil
 * cells are distinct.  An atom's cell is computed from its position wrapped
 * into [0,L) (reading C-3): xw = x - L*floor(x/L), xw -= L if xw >= L;
 * c = floor(xw * (nc/L)), clamped to nc-1.  Cell id = (cx*nc + cy)*nc + cz. */
static int64_t cell_coord(double x, double L, double inv_w, int64_t nc)
{
    double xw = x - L * floor(x / L);
    int64_t c;
    if (xw >= L)
        xw -= L;
    c = (int64_t)floor(xw * inv_w);
    if (c > nc - 1)
        c = nc - 1;
    if (c < 0)
        c = 0;
    return c;
}

int64_t lj_oracle_cells_per_side(double L, double rs)
{
    return (int64_t)floor(L / rs);
}

int64_t lj_oracle_cell_id(double x, double y, double z, double L, double rs)
{
    int64_t nc = lj_oracle_cells_per_side(L, rs);
    double inv_w = (double)nc / L;
    return (cell_coord(x, L, inv_w, nc) * nc + cell_coord(y, L, inv_w, nc)) * nc + cell_coord(z, L, inv_w, nc);
}

static int cmp_int32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Same contract as lj_oracle_list_brute (requires L > 0 and floor(L/rs) >= 3;
 * returns -1 otherwise).  The classic linked list: head[cell], next[atom]
 * (P:188-189), then for each own row i the 27 neighbouring cells are scanned;
 * the row is grouped by construction and sorted ascending (reading C-10). */
int64_t lj_oracle_list_cells(const double *q, int64_t n, double L, double rs, int half,
                             int64_t row_begin, int64_t row_end,
                             int32_t *number_of_partners, int64_t *pointer, int32_t *sorted_list,
                             int64_t cap)
{
    const double rs2 = rs * rs;
    int64_t nc, ncell, i, rows = row_end - row_begin, total = 0, pass;
    double inv_w, r[3];
    int64_t *head, *next, *cell_of;
    if (!(L > 0.0))
        return -1;
    nc = lj_oracle_cells_per_side(L, rs);
    if (nc < 3)
        return -1;
    inv_w = (double)nc / L;
    ncell = nc * nc * nc;
    head = (int64_t *)malloc((size_t)ncell * sizeof(int64_t));
    next = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    cell_of = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * 3 * sizeof(int64_t));
    for (i = 0; i < ncell; i++)
        head[i] = -1;
    for (i = 0; i < n; i++) {
        int64_t cx = cell_coord(q[3 * i + 0], L, inv_w, nc);
        int64_t cy = cell_coord(q[3 * i + 1], L, inv_w, nc);
        int64_t cz = cell_coord(q[3 * i + 2], L, inv_w, nc);
        int64_t c = (cx * nc + cy) * nc + cz;
        cell_of[3 * i + 0] = cx;
        cell_of[3 * i + 1] = cy;
        cell_of[3 * i + 2] = cz;
        next[i] = head[c];
        head[c] = i;
    }
    /* pass 0 counts, pass 1 fills (only if the capacity suffices) */
    for (pass = 0; pass < 2; pass++) {
        int64_t pos = 0;
        if (pass == 1 && cap < total)
            break;
        for (i = row_begin; i < row_end; i++) {
            int64_t start = pos;
            int dx, dy, dz;
            for (dx = -1; dx <= 1; dx++)
                for (dy = -1; dy <= 1; dy++)
                    for (dz = -1; dz <= 1; dz++) {
                        int64_t cx = (cell_of[3 * i + 0] + dx + nc) % nc;
                        int64_t cy = (cell_of[3 * i + 1] + dy + nc) % nc;
                        int64_t cz = (cell_of[3 * i + 2] + dz + nc) % nc;
                        int64_t j = head[(cx * nc + cy) * nc + cz];
                        for (; j >= 0; j = next[j]) {
                            if (j == i || (half && j < i))
                                continue;
                            if (relative(&q[3 * i], &q[3 * j], L, r) < rs2) {
                                if (pass == 1)
                                    sorted_list[pos] = (int32_t)j;
                                pos++;
                            }
                        }
                    }
            if (pass == 1) {
                qsort(&sorted_list[start], (size_t)(pos - start), sizeof(int32_t), cmp_int32);
                pointer[i - row_begin] = start;
                number_of_partners[i - row_begin] = (int32_t)(pos - start);
            }
        }
        if (pass == 0)
            total = pos;
        else
            pointer[rows] = pos;
    }
    free(head);
    free(next);
    free(cell_of);
    return total;
}

/* Spatial (cell-order) reordering, BASELINE.json config 3: stable counting sort
 * of the atoms by cell id; perm[new] = old.  Returns -1 on a bad geometry. */
int64_t lj_oracle_cell_order(const double *q, int64_t n, double L, double rs, int64_t *perm)
{
    int64_t nc, ncell, i;
    int64_t *count, *key;
    if (!(L > 0.0))
        return -1;
    nc = lj_oracle_cells_per_side(L, rs);
    if (nc < 3)
        return -1;
    ncell = nc * nc * nc;
    count = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
    key = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (i = 0; i < n; i++) {
        key[i] = lj_oracle_cell_id(q[3 * i], q[3 * i + 1], q[3 * i + 2], L, rs);
        count[key[i] + 1]++;
    }
    for (i = 0; i < ncell; i++)
        count[i + 1] += count[i];
    for (i = 0; i < n; i++)
        perm[count[key[i]]++] = i;
    free(count);
    free(key);
    return 0;
}

/* ---- force (Alg. 3, with Alg. 1 arithmetic) --------- */

/* One force step over the sorted list, exactly in the order of Alg. 3:
 *   for i (ascending): load q_i, p_i; for j in SortedList[i] (ascending):
 *     load q_j; if |q_j - q_i| < r_c: df; p_i -= df r; [half] p_j += df r
 *   store p_i.
 * Alg. 1 line 7 prints p_j <- p_j - df r; Newton's third law requires +
 * (reading C-1).  The cutoff is strict on squares, r2 < rc2 (C-4).
 * half == 0: full list, only p of own rows changes (no p_j update).
 * p is indexed by global atom index; row r is atom row_begin + r. */
void lj_oracle_force_step(const double *q, double *p, int64_t n, double L, double rc, double dt, int half,
                          int64_t row_begin, int64_t row_end,
                          const int32_t *number_of_partners, const int64_t *pointer,
                          const int32_t *sorted_list)
{
    const double rc2 = rc * rc;
    int64_t i, k;
    double r[3];
    (void)n;
    for (i = row_begin; i < row_end; i++) {
        const double *qi = &q[3 * i];
        double pix = p[3 * i + 0], piy = p[3 * i + 1], piz = p[3 * i + 2];
        int64_t beg = pointer[i - row_begin];
        int64_t cnt = number_of_partners[i - row_begin];
        for (k = beg; k < beg + cnt; k++) {
            int64_t j = sorted_list[k];
            double r2 = relative(qi, &q[3 * j], L, r);
            if (r2 < rc2) {
                double df = impulse_coefficient(r2, dt);
                pix = pix - df * r[0];
                piy = piy - df * r[1];
                piz = piz - df * r[2];
                if (half) {
                    p[3 * j + 0] = p[3 * j + 0] + df * r[0];
                    p[3 * j + 1] = p[3 * j + 1] + df * r[1];
                    p[3 * j + 2] = p[3 * j + 2] + df * r[2];
                }
            }
        }
        p[3 * i + 0] = pix;
        p[3 * i + 1] = piy;
        p[3 * i + 2] = piz;
    }
}

/* All-core TIMING build only (SURVEY §8(d) "an optional OpenMP
 * full-list build on all cores"): lj_oracle_force_step for a FULL list with the
 * rows split over OpenMP threads.  Full-list rows are independent (no p_j
 * writes), so every row runs exactly the arithmetic, in exactly the order, of
 * lj_oracle_force_step -- the results are bit-identical (tests/test_oracle_force.py).
 * Built without -fopenmp (liblj_oracle.so) the pragma is ignored; the bench's
 * all-core leg loads liblj_oracle_omp.so (-fopenmp).  Never used for parity. */
void lj_oracle_force_step_full_rows_parallel(const double *q, double *p, int64_t n, double L, double rc, double dt,
                                             int64_t row_begin, int64_t row_end,
                                             const int32_t *number_of_partners, const int64_t *pointer,
                                             const int32_t *sorted_list)
{
    const double rc2 = rc * rc;
    int64_t i;
    (void)n;
#pragma omp parallel for schedule(static)
    for (i = row_begin; i < row_end; i++) {
        const double *qi = &q[3 * i];
        double r[3];
        double pix = p[3 * i + 0], piy = p[3 * i + 1], piz = p[3 * i + 2];
        int64_t beg = pointer[i - row_begin];
        int64_t cnt = number_of_partners[i - row_begin];
        int64_t k;
        for (k = beg; k < beg + cnt; k++) {
            int64_t j = sorted_list[k];
            double r2 = relative(qi, &q[3 * j], L, r);
            if (r2 < rc2) {
                double df = impulse_coefficient(r2, dt);
                pix = pix - df * r[0];
                piy = piy - df * r[1];
                piz = piz - df * r[2];
            }
        }
        p[3 * i + 0] = pix;
        p[3 * i + 1] = piy;
        p[3 * i + 2] = piz;
    }
}

/* The plain definition without any list: for every unordered pair i < j with
 * r2 < rc2 (canonical double loop), Alg. 1 with the sign fix. */
void lj_oracle_force_brute(const double *q, double *p, int64_t n, double L, double rc, double dt)
{
    const double rc2 = rc * rc;
    int64_t i, j;
    double r[3];
    for (i = 0; i < n; i++)
        for (j = i + 1; j < n; j++) {
            double r2 = relative(&q[3 * i], &q[3 * j], L, r);
            if (r2 < rc2) {
                double df = impulse_coefficient(r2, dt);
                p[3 * i + 0] -= df * r[0];
                p[3 * i + 1] -= df * r[1];
                p[3 * i + 2] -= df * r[2];
                p[3 * j + 0] += df * r[0];
                p[3 * j + 1] += df * r[1];
                p[3 * j + 2] += df * r[2];
            }
        }
}

/* Parity denominator (reading C-12): S_ik = |p0_ik| + sum over the pairs of i
 * inside r_c of dt (48 + 24 r^6)/r^14 |r_k|, the component's sum of absolute
 * contributions.  Rows of the given list; with half != 0 each entry also adds
 * to atom j.  S has 3n entries (global index); p0 may be NULL (treated as 0). */
void lj_oracle_abs_contrib(const double *q, const double *p0, int64_t n, double L, double rc, double dt, int half,
                           int64_t row_begin, int64_t row_end,
                           const int32_t *number_of_partners, const int64_t *pointer,
                           const int32_t *sorted_list, double *S)
{
    const double rc2 = rc * rc;
    int64_t i, k, c;
    double r[3];
    for (i = 0; i < 3 * n; i++)
        S[i] = p0 ? fabs(p0[i]) : 0.0;
    for (i = row_begin; i < row_end; i++) {
        int64_t beg = pointer[i - row_begin];
        int64_t cnt = number_of_partners[i - row_begin];
        for (k = beg; k < beg + cnt; k++) {
            int64_t j = sorted_list[k];
            double r2 = relative(&q[3 * i], &q[3 * j], L, r);
            if (r2 < rc2) {
                double r6 = (r2 * r2) * r2;
                double r14 = (r6 * r6) * r2;
                double a = ((48.0 + 24.0 * r6) * dt) / r14;
                for (c = 0; c < 3; c++) {
                    S[3 * i + c] += a * fabs(r[c]);
                    if (half)
                        S[3 * j + c] += a * fabs(r[c]);
                }
            }
        }
    }
}

/* ---- integration, bookkeeping, energy ------------------------------------ */

/* Drift q_i += p_i dt (mass 1; reading C-8), atoms [begin,end); no wrap. */
void lj_oracle_integrate(double *q, const double *p, int64_t begin, int64_t end, double dt)
{
    int64_t i;
    for (i = 3 * begin; i < 3 * end; i++)
        q[i] = q[i] + p[i] * dt;
}

/* Wrap positions into [0,L) (reading C-3). */
void lj_oracle_wrap(double *q, int64_t n, double L)
{
    int64_t i;
    for (i = 0; i < 3 * n; i++) {
        double x = q[i] - L * floor(q[i] / L);
        if (x >= L)
            x -= L;
        q[i] = x;
    }
}

/* Bookkeeping (reading C-16): max_i |q_i - q_ref_i| over
 * [begin,end), Euclidean, no minimum image (q is never wrapped between builds). */
double lj_oracle_max_displacement(const double *q, const double *q_ref, int64_t begin, int64_t end)
{
    int64_t i;
    double m = 0.0;
    for (i = begin; i < end; i++) {
        double dx = q[3 * i] - q_ref[3 * i];
        double dy = q[3 * i + 1] - q_ref[3 * i + 1];
        double dz = q[3 * i + 2] - q_ref[3 * i + 2];
        double d = sqrt((dx * dx + dy * dy) + dz * dz);
        if (d > m)
            m = d;
    }
    return m;
}

/* Shifted LJ pair energy (Eq. 1, with V(r_c) = 0; reading O7):
 * 4 (r^-12 - r^-6) - 4 (rc^-12 - rc^-6). */
static double shifted_potential(double r2, double rc)
{
    double rc2 = rc * rc;
    double rc6 = (rc2 * rc2) * rc2;
    double vc = 4.0 * (1.0 / (rc6 * rc6) - 1.0 / rc6);
    double r6 = (r2 * r2) * r2;
    double inv6 = 1.0 / r6;
    return 4.0 * (inv6 * inv6 - inv6) - vc;
}

double lj_oracle_pair_energy(double r2, double rc)
{
    if (!(r2 < rc * rc))
        return 0.0;
    return shifted_potential(r2, rc);
}

/* out[0] = KE = 1/2 sum_{own rows} |p|^2; out[1] = PE over the list's entries
 * inside r_c: each entry once for a half list, 1/2 per entry for a full list
 * (so that row ranges of a full list partition the unique-pair sum). */
void lj_oracle_energy(const double *q, const double *p, int64_t n, double L, double rc, int half,
                      int64_t row_begin, int64_t row_end,
                      const int32_t *number_of_partners, const int64_t *pointer,
                      const int32_t *sorted_list, double *out)
{
    const double rc2 = rc * rc;
    int64_t i, k;
    double ke = 0.0, pe = 0.0, r[3];
    (void)n;
    for (i = row_begin; i < row_end; i++) {
        int64_t beg = pointer[i - row_begin];
        int64_t cnt = number_of_partners[i - row_begin];
        ke += 0.5 * ((p[3 * i] * p[3 * i] + p[3 * i + 1] * p[3 * i + 1]) + p[3 * i + 2] * p[3 * i + 2]);
        for (k = beg; k < beg + cnt; k++) {
            double r2 = relative(&q[3 * i], &q[3 * sorted_list[k]], L, r);
            if (r2 < rc2)
                pe += half ? shifted_potential(r2, rc) : 0.5 * shifted_potential(r2, rc);
        }
    }
    out[0] = ke;
    out[1] = pe;
}

/* PE over all unordered pairs by definition (O(N^2)). */
double lj_oracle_energy_brute(const double *q, int64_t n, double L, double rc)
{
    int64_t i, j;
    double pe = 0.0, r[3];
    for (i = 0; i < n; i++)
        for (j = i + 1; j < n; j++)
            pe += lj_oracle_pair_energy(relative(&q[3 * i], &q[3 * j], L, r), rc);
    return pe;
}

/* ---- NVE dynamics (BASELINE.json configs 4-5; reading O8) ---------------- */

/* Velocity Verlet, kick-drift-kick, with the bookkeeping rebuild (C-16):
 *   p += F(q) dt/2;  q += p dt;
 *   if 2 max|q - q_ref| >= rs - rc: wrap q, rebuild full list, q_ref <- q;
 *   p += F(q) dt/2.
 * The half-kick impulse F(q) dt/2 of the end of step n is reused at the start
 * of step n+1 (same value, one evaluation).  energies: (steps/sample_every + 1)
 * rows of {KE, PE, E} at steps 0, s, 2s, ...  Returns the number of rebuilds
 * (excluding the initial build), or -1 on a bad geometry. */
int64_t lj_oracle_md_run(double *q, double *p, int64_t n, double L, double rc, double rs, double dt,
                         int64_t steps, int64_t sample_every, double *energies)
{
    int64_t step, i, cap, rebuilds = 0, ns = 0;
    int32_t *np_ = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int64_t *ptr = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    int32_t *lst;
    double *qref = (double *)malloc((size_t)(3 * n) * sizeof(double));
    double *kick = (double *)malloc((size_t)(3 * n) * sizeof(double));
    double e[2];

    lj_oracle_wrap(q, n, L);
    cap = lj_oracle_list_cells(q, n, L, rs, 0, 0, n, np_, ptr, NULL, 0);
    if (cap < 0)
        return -1;
    cap = cap + cap / 4 + 1024;
    lst = (int32_t *)malloc((size_t)cap * sizeof(int32_t));
    lj_oracle_list_cells(q, n, L, rs, 0, 0, n, np_, ptr, lst, cap);
    memcpy(qref, q, (size_t)(3 * n) * sizeof(double));

    /* F(q0) dt/2 */
    memset(kick, 0, (size_t)(3 * n) * sizeof(double));
    lj_oracle_force_step(q, kick, n, L, rc, 0.5 * dt, 0, 0, n, np_, ptr, lst);
    if (energies && sample_every > 0) {
        lj_oracle_energy(q, p, n, L, rc, 0, 0, n, np_, ptr, lst, e);
        energies[0] = e[0];
        energies[1] = e[1];
        energies[2] = e[0] + e[1];
        ns = 1;
    }
    for (step = 1; step <= steps; step++) {
        for (i = 0; i < 3 * n; i++)
            p[i] = p[i] + kick[i];
        lj_oracle_integrate(q, p, 0, n, dt);
        if (2.0 * lj_oracle_max_displacement(q, qref, 0, n) >= rs - rc) {
            int64_t need;
            lj_oracle_wrap(q, n, L);
            need = lj_oracle_list_cells(q, n, L, rs, 0, 0, n, np_, ptr, lst, cap);
            if (need > cap) {
                cap = need + need / 4;
                free(lst);
                lst = (int32_t *)malloc((size_t)cap * sizeof(int32_t));
                lj_oracle_list_cells(q, n, L, rs, 0, 0, n, np_, ptr, lst, cap);
            }
            memcpy(qref, q, (size_t)(3 * n) * sizeof(double));
            rebuilds++;
        }
        memset(kick, 0, (size_t)(3 * n) * sizeof(double));
        lj_oracle_force_step(q, kick, n, L, rc, 0.5 * dt, 0, 0, n, np_, ptr, lst);
        for (i = 0; i < 3 * n; i++)
            p[i] = p[i] + kick[i];
        if (energies && sample_every > 0 && step % sample_every == 0) {
            lj_oracle_energy(q, p, n, L, rc, 0, 0, n, np_, ptr, lst, e);
            energies[3 * ns + 0] = e[0];
            energies[3 * ns + 1] = e[1];
            energies[3 * ns + 2] = e[0] + e[1];
            ns++;
        }
    }
    free(np_);
    free(ptr);
    free(lst);
    free(qref);
    free(kick);
    return rebuilds;
}
