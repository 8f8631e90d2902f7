/*
 * nemd_oracle.c -- CPU fp64 ORACLE for the cell-list force path of
 * arXiv 1412.3784 ("cell lists for NEMD in a deforming periodic box").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path under paper_1412_3784_b200/ and neither includes the other.
 *
 * Plain, slow, obviously-correct fp64 loops.  Compiled with
 * -ffp-contract=off so every a*b+c below is two correctly rounded
 * operations, in the association order written (reading R16:
 * "canonical fp64 arithmetic").  Citations: P:n = /root/reference/PAPER.md
 * line n; readings Rn are listed in DESIGN.md section 3.
 *
 * Matrices are row-major double[9]; the COLUMNS of L are the box vectors
 * v1, v2, v3 (Eq. 1).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;

static double wtime(void)
{
#ifdef _OPENMP
    return omp_get_wtime();
#else
    return 0.0;
#endif
}

/* ------------------------------------------------------------------ */
/* Lattice geometry          */
/* ------------------------------------------------------------------ */

/* L^{-1} = adj(L)/det(L); cofactors as (a*b)-(c*d); det by first-row
 * expansion ((L00*C00 + L01*C01) + L02*C02).  Reading R16.
 * Returns 0 on success, 1 if det <= 0 or non-finite (P:32 needs a basis). */
int or_inv3(const double *L, double *Li, double *det_out)
{
    double C00 = L[4] * L[8] - L[5] * L[7];
    double C01 = L[5] * L[6] - L[3] * L[8];
    double C02 = L[3] * L[7] - L[4] * L[6];
    double C10 = L[2] * L[7] - L[1] * L[8];
    double C11 = L[0] * L[8] - L[2] * L[6];
    double C12 = L[1] * L[6] - L[0] * L[7];
    double C20 = L[1] * L[5] - L[2] * L[4];
    double C21 = L[2] * L[3] - L[0] * L[5];
    double C22 = L[0] * L[4] - L[1] * L[3];
    double det = (L[0] * C00 + L[1] * C01) + L[2] * C02;
    if (det_out) *det_out = det;
    if (!(det > 0.0) || !isfinite(det)) return 1;
    /* (L^{-1})_{rc} = C_{cr} / det */
    Li[0] = C00 / det; Li[1] = C10 / det; Li[2] = C20 / det;
    Li[3] = C01 / det; Li[4] = C11 / det; Li[5] = C21 / det;
    Li[6] = C02 / det; Li[7] = C12 / det; Li[8] = C22 / det;
    return 0;
}

static double norm3(double x, double y, double z) { return sqrt((x * x + y * y) + z * z); }

/* Box heights h_k = distance between the two faces not containing v_k
 * (Fig. "fig:bh"; reading R7): h_k = 1/||row_k(L^{-1})||. */
void or_heights(const double *Li, double *h)
{
    for (int k = 0; k < 3; ++k) h[k] = 1.0 / norm3(Li[3 * k], Li[3 * k + 1], Li[3 * k + 2]);
}

/* Dynamic-size cell counts c_i = floor(h_i / d_cut). */
void or_ds_dims(const double *h, double rc, int *c)
{
    for (int k = 0; k < 3; ++k) c[k] = (int)floor(h[k] / rc);
}

/* QR of L by Gram-Schmidt on the columns, r_kk > 0 (R8).
 * Q row-major with columns e1,e2,e3; R upper triangular row-major. */
void or_qr(const double *L, double *Q, double *R)
{
    double v1[3] = {L[0], L[3], L[6]}, v2[3] = {L[1], L[4], L[7]}, v3[3] = {L[2], L[5], L[8]};
    double r11 = norm3(v1[0], v1[1], v1[2]);
    double e1[3] = {v1[0] / r11, v1[1] / r11, v1[2] / r11};
    double r12 = (e1[0] * v2[0] + e1[1] * v2[1]) + e1[2] * v2[2];
    double u2[3] = {v2[0] - r12 * e1[0], v2[1] - r12 * e1[1], v2[2] - r12 * e1[2]};
    double r22 = norm3(u2[0], u2[1], u2[2]);
    double e2[3] = {u2[0] / r22, u2[1] / r22, u2[2] / r22};
    double e3[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                    e1[0] * e2[1] - e1[1] * e2[0]};
    double r13 = (e1[0] * v3[0] + e1[1] * v3[1]) + e1[2] * v3[2];
    double r23 = (e2[0] * v3[0] + e2[1] * v3[1]) + e2[2] * v3[2];
    double r33 = (e3[0] * v3[0] + e3[1] * v3[1]) + e3[2] * v3[2];
    for (int r = 0; r < 3; ++r) { Q[3 * r + 0] = e1[r]; Q[3 * r + 1] = e2[r]; Q[3 * r + 2] = e3[r]; }
    R[0] = r11; R[1] = r12; R[2] = r13;
    R[3] = 0.0; R[4] = r22; R[5] = r23;
    R[6] = 0.0; R[7] = 0.0; R[8] = r33;
}

/* Dynamic-offset cell counts l_i = floor(r_ii / d_cut) and the
 * rectangular cell widths w_i = r_ii / l_i. */
void or_do_dims(const double *R, double rc, int *l, double *w)
{
    for (int k = 0; k < 3; ++k) {
        l[k] = (int)floor(R[4 * k] / rc);
        w[k] = R[4 * k] / (double)l[k];
    }
}

/* ------------------------------------------------------------------ */
/* Fractional coordinates, wrap into Omega, cell keys                   */
/* ------------------------------------------------------------------ */

/* lambda = L^{-1} q, rows evaluated as (a*x + b*y) + c*z ("convert
 * particle positions to the underlying lattice basis"; R16). */
static inline void frac(const double *Li, const double *q, double *lam)
{
    for (int k = 0; k < 3; ++k)
        lam[k] = (Li[3 * k] * q[0] + Li[3 * k + 1] * q[1]) + Li[3 * k + 2] * q[2];
}

/* Lattice shift s = L n, (L_a0 n0 + L_a1 n1) + L_a2 n2 (R16). */
static inline void lshift(const double *L, const int *n, double *s)
{
    for (int a = 0; a < 3; ++a)
        s[a] = (L[3 * a] * (double)n[0] + L[3 * a + 1] * (double)n[1]) + L[3 * a + 2] * (double)n[2];
}

/* Wrap each particle into the unit cell Omega (Eq. 2): if any
 * lambda_k is outside [0,1), q <- round_prec(q - L floor(lambda)) once
 * (readings R14, R15).  prec: 0 = values are fp32 (round result to float),
 * 1 = fp64.  In place on q (n x 3).  Returns number of particles moved. */
i64 or_wrap(i64 n, double *q, const double *L, int prec)
{
    double Li[9], det;
    if (or_inv3(L, Li, &det)) return -1;
    i64 moved = 0;
#pragma omp parallel for reduction(+ : moved) schedule(static)
    for (i64 i = 0; i < n; ++i) {
        double lam[3];
        frac(Li, q + 3 * i, lam);
        if (lam[0] < 0.0 || lam[0] >= 1.0 || lam[1] < 0.0 || lam[1] >= 1.0 || lam[2] < 0.0 ||
            lam[2] >= 1.0) {
            int nn[3] = {(int)floor(lam[0]), (int)floor(lam[1]), (int)floor(lam[2])};
            double s[3];
            lshift(L, nn, s);
            for (int a = 0; a < 3; ++a) {
                double v = q[3 * i + a] - s[a];
                q[3 * i + a] = prec == 0 ? (double)(float)v : v;
            }
            moved++;
        }
    }
    return moved;
}

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* DS cell of one particle: a_k = clamp(floor(lambda_k c_k), 0, c_k-1)
 * (reading R14).  Cell index is x-fastest. */
static inline i64 ds_cell(const double *lam, const int *c, int *a)
{
    for (int k = 0; k < 3; ++k) a[k] = clampi((int)floor(lam[k] * (double)c[k]), 0, c[k] - 1);
    return (i64)a[0] + (i64)c[0] * ((i64)a[1] + (i64)c[1] * (i64)a[2]);
}

/* DO cell of one particle (Eqs. 11-12 with reading R1: the x
 * update is "mod r11"; R2: applied to Omega-wrapped points, z untouched).
 * (x,y,z) = R lambda; ky = floor(y/r22); y' = y - ky r22;
 * x'' = x - ky r12; kx = floor(x''/r11); x' = x'' - kx r11.
 * The rearranged copy is q + L nh with nh = (-kx, -ky, 0). */
static inline i64 do_cell(const double *lam, const double *R, const int *l, const double *w, int *a,
                          int *nh)
{
    double x = (R[0] * lam[0] + R[1] * lam[1]) + R[2] * lam[2];
    double y = R[4] * lam[1] + R[5] * lam[2];
    double z = R[8] * lam[2];
    double ky = floor(y / R[4]);
    double yp = y - ky * R[4];
    double xpp = x - ky * R[1];
    double kx = floor(xpp / R[0]);
    double xp = xpp - kx * R[0];
    a[0] = clampi((int)floor(xp / w[0]), 0, l[0] - 1);
    a[1] = clampi((int)floor(yp / w[1]), 0, l[1] - 1);
    a[2] = clampi((int)floor(z / w[2]), 0, l[2] - 1);
    nh[0] = -(int)kx;
    nh[1] = -(int)ky;
    nh[2] = 0;
    return (i64)a[0] + (i64)l[0] * ((i64)a[1] + (i64)l[1] * (i64)a[2]);
}

/* Exported: rearranged rotated coordinates (x', y', z) and home shift for
 * points given in the rotated frame (x, y, z) = R lambda (Eqs. 11-12). */
void or_do_rearrange(i64 n, const double *xyz, const double *R, double *out, int32_t *nh)
{
    for (i64 i = 0; i < n; ++i) {
        double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        double ky = floor(y / R[4]);
        double yp = y - ky * R[4];
        double xpp = x - ky * R[1];
        double kx = floor(xpp / R[0]);
        out[3 * i] = xpp - kx * R[0];
        out[3 * i + 1] = yp;
        out[3 * i + 2] = z;
        nh[3 * i] = -(int)kx; nh[3 * i + 1] = -(int)ky; nh[3 * i + 2] = 0;
    }
}

/* Geometry bundle for one box and one variant. */
typedef struct {
    double L[9], Li[9], det, h[3];
    int variant;       /* 0 = dynamic size (DS), 1 = dynamic offset (DO) */
    int dims[3];       /* c (DS) or l (DO) */
    double Q[9], R[9]; /* DO */
    double w[3];       /* DO */
    double d21, d31, d32; /* DO offsets in cell units: r12/w1, r13/w1, r23/w2 */
} geom_t;

/* Returns 0 ok, 1 bad box, 2 degenerate grid (DS c_k < 3; DO l1,l2 < 4 or l3 < 3; R9). */
static int geom_init(geom_t *g, const double *L, double rc, int variant)
{
    memcpy(g->L, L, sizeof(double) * 9);
    if (or_inv3(L, g->Li, &g->det)) return 1;
    or_heights(g->Li, g->h);
    g->variant = variant;
    if (variant == 0) {
        or_ds_dims(g->h, rc, g->dims);
        if (g->dims[0] < 3 || g->dims[1] < 3 || g->dims[2] < 3) return 2;
    } else {
        or_qr(L, g->Q, g->R);
        or_do_dims(g->R, rc, g->dims, g->w);
        if (g->dims[0] < 4 || g->dims[1] < 4 || g->dims[2] < 3) return 2;
        g->d21 = g->R[1] / g->w[0];
        g->d31 = g->R[2] / g->w[0];
        g->d32 = g->R[5] / g->w[1];
    }
    return 0;
}

/* Exported: cell keys (and DO home shifts) for n stored positions.
 * Returns 0 / 1 bad box / 2 degenerate.  dims_out[3] = grid. */
int or_cell_keys(int variant, i64 n, const double *q, const double *L, double rc, i64 *cell,
                 int32_t *nhome, int32_t *dims_out)
{
    geom_t g;
    int st = geom_init(&g, L, rc, variant);
    if (st) return st;
    for (int k = 0; k < 3; ++k) dims_out[k] = g.dims[k];
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) {
        double lam[3];
        int a[3], nh[3] = {0, 0, 0};
        frac(g.Li, q + 3 * i, lam);
        if (variant == 0)
            cell[i] = ds_cell(lam, g.dims, a);
        else
            cell[i] = do_cell(lam, g.R, g.dims, g.w, a, nh);
        if (nhome) { nhome[3 * i] = nh[0]; nhome[3 * i + 1] = nh[1]; nhome[3 * i + 2] = nh[2]; }
    }
    return 0;
}

/* Counting sort into cells; within a cell ascending particle index
 * (= gid; reading R27).  cell_start has ncell+1 entries. */
void or_cell_sort(i64 n, const i64 *cell, i64 ncell, i64 *cell_start, i64 *order)
{
    memset(cell_start, 0, sizeof(i64) * (size_t)(ncell + 1));
    for (i64 i = 0; i < n; ++i) cell_start[cell[i] + 1]++;
    for (i64 c = 0; c < ncell; ++c) cell_start[c + 1] += cell_start[c];
    i64 *fill = (i64 *)malloc(sizeof(i64) * (size_t)ncell);
    memcpy(fill, cell_start, sizeof(i64) * (size_t)ncell);
    for (i64 i = 0; i < n; ++i) order[fill[cell[i]]++] = i;
    free(fill);
}

/* ------------------------------------------------------------------ */
/* Neighborhoods (stencils)                                             */
/* ------------------------------------------------------------------ */

typedef struct { i64 cell; int n[3]; } sten_t; /* neighbor cell + lattice crossing */

static inline i64 floordiv_i(i64 a, i64 b) { i64 q = a / b; if ((a % b) && ((a < 0) != (b < 0))) q--; return q; }

/* DS: the 27-cell neighborhood: m = a + delta,
 * n_k = floor(m_k/c_k), m_k -= n_k c_k. */
static int ds_stencil(const geom_t *g, const int *a, sten_t *out)
{
    int k = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int m[3] = {a[0] + dx, a[1] + dy, a[2] + dz}, nn[3];
                for (int t = 0; t < 3; ++t) {
                    nn[t] = (int)floordiv_i(m[t], g->dims[t]);
                    m[t] -= nn[t] * g->dims[t];
                }
                out[k].cell = (i64)m[0] + (i64)g->dims[0] * ((i64)m[1] + (i64)g->dims[1] * (i64)m[2]);
                out[k].n[0] = nn[0]; out[k].n[1] = nn[1]; out[k].n[2] = nn[2];
                k++;
            }
    return k;
}

/* DO: neighborhood by exact interval overlap in cell units (P:609,
 * P:673-687; readings R3, R4, R5).  For layer kk: n3 = floor(kk/l3);
 * rows m over [j-1-n3*d32, j+2-n3*d32) rounded out; per row n2 =
 * floor(m/l2), x-offset o = n3*d31 + n2*d21; columns over [i-1-o, i+2-o)
 * rounded out; n1 = floor(col/l1).  Gives 27/30/34/36 cells for the four
 * cases of P:679-686 on generic boxes and 27 at equilibrium. */
static int do_stencil(const geom_t *g, const int *a, sten_t *out)
{
    const int l1 = g->dims[0], l2 = g->dims[1], l3 = g->dims[2];
    int k = 0;
    for (int dz = -1; dz <= 1; ++dz) {
        int kk = a[2] + dz;
        int n3 = (int)floordiv_i(kk, l3);
        int kd = kk - n3 * l3;
        double oy = (double)n3 * g->d32;
        int m0 = (int)floor((double)(a[1] - 1) - oy);
        int m1 = (int)ceil((double)(a[1] + 2) - oy); /* half-open */
        for (int m = m0; m < m1; ++m) {
            int n2 = (int)floordiv_i(m, l2);
            int jd = m - n2 * l2;
            double ox = (double)n3 * g->d31 + (double)n2 * g->d21;
            int c0 = (int)floor((double)(a[0] - 1) - ox);
            int c1 = (int)ceil((double)(a[0] + 2) - ox);
            for (int col = c0; col < c1; ++col) {
                int n1 = (int)floordiv_i(col, l1);
                int id = col - n1 * l1;
                out[k].cell = (i64)id + (i64)l1 * ((i64)jd + (i64)l2 * (i64)kd);
                out[k].n[0] = n1; out[k].n[1] = n2; out[k].n[2] = n3;
                k++;
            }
        }
    }
    return k;
}

/* Exported: stencil of one cell (for the case-count pins). */
int or_stencil(int variant, const double *L, double rc, const int32_t *cell3, i64 *cells, int32_t *ncross)
{
    geom_t g;
    if (geom_init(&g, L, rc, variant)) return -1;
    sten_t st[64];
    int a[3] = {cell3[0], cell3[1], cell3[2]};
    int k = variant == 0 ? ds_stencil(&g, a, st) : do_stencil(&g, a, st);
    for (int t = 0; t < k; ++t) {
        cells[t] = st[t].cell;
        ncross[3 * t] = st[t].n[0]; ncross[3 * t + 1] = st[t].n[1]; ncross[3 * t + 2] = st[t].n[2];
    }
    return k;
}

/* Exported: histogram of neighborhood sizes over all cells (index = size, 0..63). */
int or_stencil_histogram(int variant, const double *L, double rc, i64 *hist, int32_t *dims_out)
{
    geom_t g;
    int stt = geom_init(&g, L, rc, variant);
    if (stt) return stt;
    memset(hist, 0, sizeof(i64) * 64);
    sten_t st[64];
    for (int k = 0; k < 3; ++k) dims_out[k] = g.dims[k];
    for (int z = 0; z < g.dims[2]; ++z)
        for (int y = 0; y < g.dims[1]; ++y)
            for (int x = 0; x < g.dims[0]; ++x) {
                int a[3] = {x, y, z};
                int k = variant == 0 ? ds_stencil(&g, a, st) : do_stencil(&g, a, st);
                hist[k]++;
            }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Pair set, forces, energy, virial                                      */
/* ------------------------------------------------------------------ */

/* Canonical displacement d = (q_j + L n) - q_i and r^2 = (dx^2+dy^2)+dz^2
 * (pair-set definition; reading R16). */
static inline double pair_d(const double *qi, const double *qj, const double *L, const int *n, double *d)
{
    double s[3];
    lshift(L, n, s);
    for (int a = 0; a < 3; ++a) d[a] = (qj[a] + s[a]) - qi[a];
    return (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
}

/* splitmix64 finalizer, for order-independent per-particle pair digests. */
static inline uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

typedef struct { double rc2, eps, sig2, ushift; } pot_t;

typedef struct {
    long double F[3], U, W[6];
    uint32_t cnt;
    uint64_t hsum, hxor;
    i64 cand;
} acc_t;

/* One member (i,j,n) of the pair set (r^2 < rc^2 strictly, R10):
 * LJ 12-6, energy shifted (R11): fr = 24 eps (2 s^12 - s^6)/r^2 with
 * s^2 = sigma^2/r^2; F_i -= fr d; U_i += (phi(r) - phi(rc))/2;
 * W_i += fr d (x) d / 2 (R12).  Membership was decided by the canonical
 * fp64 test; the force uses d = (q_j + L n) - q_i evaluated in x87
 * extended precision (64-bit mantissa) so the oracle's own rounding stays
 * far below the fp64 tolerance it referees (R16).
 * Digest key = gid_j | (n+8) nibbles. */
static inline void acc_pair(acc_t *acc, const pot_t *p, const double *qi, const double *qj, const double *L,
                            i64 gj, const int *n)
{
    long double d[3];
    for (int a = 0; a < 3; ++a) {
        long double s = ((long double)L[3 * a] * n[0] + (long double)L[3 * a + 1] * n[1]) +
                        (long double)L[3 * a + 2] * n[2];
        d[a] = ((long double)qj[a] + s) - (long double)qi[a];
    }
    long double r2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
    long double s2 = (long double)p->sig2 / r2;
    long double s6 = s2 * s2 * s2;
    long double s12 = s6 * s6;
    long double fr = 24.0L * p->eps * (2.0L * s12 - s6) / r2;
    acc->F[0] -= fr * d[0];
    acc->F[1] -= fr * d[1];
    acc->F[2] -= fr * d[2];
    acc->U += 0.5L * (4.0L * p->eps * (s12 - s6) - p->ushift);
    acc->W[0] += 0.5L * fr * d[0] * d[0];
    acc->W[1] += 0.5L * fr * d[1] * d[1];
    acc->W[2] += 0.5L * fr * d[2] * d[2];
    acc->W[3] += 0.5L * fr * d[0] * d[1];
    acc->W[4] += 0.5L * fr * d[0] * d[2];
    acc->W[5] += 0.5L * fr * d[1] * d[2];
    uint64_t key = (uint64_t)gj | ((uint64_t)(n[0] + 8) << 32) | ((uint64_t)(n[1] + 8) << 36) |
                   ((uint64_t)(n[2] + 8) << 40);
    uint64_t h = mix64(key);
    acc->cnt++;
    acc->hsum += h;
    acc->hxor ^= h;
}

typedef struct {
    double *F, *U, *W; /* per evaluated particle: 3, 1, 6 */
    uint32_t *cnt;
    uint64_t *hsum, *hxor;
    int32_t *pairs; i64 pair_cap; i64 *npairs; /* optional (i, j, n0, n1, n2) list */
} out_t;

static void store(out_t *o, i64 k, const acc_t *a)
{
    if (o->F) { o->F[3 * k] = (double)a->F[0]; o->F[3 * k + 1] = (double)a->F[1]; o->F[3 * k + 2] = (double)a->F[2]; }
    if (o->U) o->U[k] = (double)a->U;
    if (o->W) for (int t = 0; t < 6; ++t) o->W[6 * k + t] = (double)a->W[t];
    if (o->cnt) o->cnt[k] = a->cnt;
    if (o->hsum) o->hsum[k] = a->hsum;
    if (o->hxor) o->hxor[k] = a->hxor;
}

static void push_pair(out_t *o, i64 i, i64 j, const int *n)
{
    if (!o->pairs) return;
    i64 slot;
#pragma omp atomic capture
    slot = (*o->npairs)++;
    if (slot < o->pair_cap) {
        int32_t *p = o->pairs + 5 * slot;
        p[0] = (int32_t)i; p[1] = (int32_t)j; p[2] = n[0]; p[3] = n[1]; p[4] = n[2];
    }
}

/*
 * Exported: evaluate the pair set and the forces / energy / virial for the
 * particles listed in idx (or all if idx == NULL), by
 *   method 0: brute force over all j and the complete image range
 *             n_k in [ceil(-rc/h_k - dlam_k), floor(rc/h_k - dlam_k)]
 *             ("loop over all pairs"), widened by 1e-9;
 *   method 1: dynamic-size cell list;
 *   method 2: dynamic-offset cell list.
 * q are the stored (already wrapped) positions in fp64.  Outputs are per
 * evaluated particle (row k for idx[k]).  stats[0] = candidates (distance
 * checks, cell methods), stats[1] = ordered interactions, stats[2..4] = grid,
 * stats[5] = cell-list build time and stats[6] = pair-loop time (ns, wall).
 * Returns 0, or 1 bad box, 2 degenerate grid.
 */
int or_evaluate(int method, i64 n, const double *q, const double *L, double rc, double eps, double sigma,
                double ushift, i64 nidx, const i64 *idx, double *F, double *U, double *W, uint32_t *cnt,
                uint64_t *hsum, uint64_t *hxor, int32_t *pairs, i64 pair_cap, i64 *npairs, i64 *stats)
{
    pot_t pot = {rc * rc, eps, sigma * sigma, ushift};
    out_t o = {F, U, W, cnt, hsum, hxor, pairs, pair_cap, npairs};
    if (npairs) *npairs = 0;
    i64 ne = idx ? nidx : n;
    i64 tot_cand = 0, tot_int = 0;
    memset(stats, 0, sizeof(i64) * 7);

    if (method == 0) {
        double Li[9], det, h[3];
        if (or_inv3(L, Li, &det)) return 1;
        or_heights(Li, h);
        double *lam = (double *)malloc(sizeof(double) * 3 * (size_t)n);
#pragma omp parallel for schedule(static)
        for (i64 i = 0; i < n; ++i) frac(Li, q + 3 * i, lam + 3 * i);
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : tot_cand, tot_int)
        for (i64 k = 0; k < ne; ++k) {
            i64 i = idx ? idx[k] : k;
            acc_t acc;
            memset(&acc, 0, sizeof acc);
            for (i64 j = 0; j < n; ++j) {
                int lo[3], hi[3];
                for (int t = 0; t < 3; ++t) {
                    double dl = lam[3 * j + t] - lam[3 * i + t];
                    lo[t] = (int)ceil(-rc / h[t] - dl - 1e-9);
                    hi[t] = (int)floor(rc / h[t] - dl + 1e-9);
                }
                int nn[3];
                for (nn[0] = lo[0]; nn[0] <= hi[0]; ++nn[0])
                    for (nn[1] = lo[1]; nn[1] <= hi[1]; ++nn[1])
                        for (nn[2] = lo[2]; nn[2] <= hi[2]; ++nn[2]) {
                            if (j == i && nn[0] == 0 && nn[1] == 0 && nn[2] == 0) continue;
                            double d[3];
                            double r2 = pair_d(q + 3 * i, q + 3 * j, L, nn, d);
                            acc.cand++;
                            if (r2 < pot.rc2) {
                                acc_pair(&acc, &pot, q + 3 * i, q + 3 * j, L, j, nn);
                                push_pair(&o, i, j, nn);
                            }
                        }
            }
            store(&o, k, &acc);
            tot_cand += acc.cand;
            tot_int += acc.cnt;
        }
        free(lam);
        stats[0] = tot_cand;
        stats[1] = tot_int;
        return 0;
    }

    geom_t g;
    int st = geom_init(&g, L, rc, method == 1 ? 0 : 1);
    if (st) return st;
    double t0 = wtime();
    i64 ncell = (i64)g.dims[0] * g.dims[1] * g.dims[2];
    i64 *cell = (i64 *)malloc(sizeof(i64) * (size_t)n);
    int32_t *nh = (int32_t *)calloc((size_t)n * 3, sizeof(int32_t));
    int32_t *a3 = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)n);
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n; ++i) {
        double lam[3];
        int a[3], hh[3] = {0, 0, 0};
        frac(g.Li, q + 3 * i, lam);
        cell[i] = g.variant == 0 ? ds_cell(lam, g.dims, a) : do_cell(lam, g.R, g.dims, g.w, a, hh);
        for (int t = 0; t < 3; ++t) { nh[3 * i + t] = hh[t]; a3[3 * i + t] = a[t]; }
    }
    i64 *cs = (i64 *)malloc(sizeof(i64) * (size_t)(ncell + 1));
    i64 *order = (i64 *)malloc(sizeof(i64) * (size_t)n);
    or_cell_sort(n, cell, ncell, cs, order);
    double t1 = wtime();

#pragma omp parallel for schedule(dynamic, 64) reduction(+ : tot_cand, tot_int)
    for (i64 k = 0; k < ne; ++k) {
        i64 i = idx ? idx[k] : k;
        acc_t acc;
        memset(&acc, 0, sizeof acc);
        sten_t stn[64];
        int a[3] = {a3[3 * i], a3[3 * i + 1], a3[3 * i + 2]};
        int ns = g.variant == 0 ? ds_stencil(&g, a, stn) : do_stencil(&g, a, stn);
        for (int e = 0; e < ns; ++e) {
            for (i64 t = cs[stn[e].cell]; t < cs[stn[e].cell + 1]; ++t) {
                i64 j = order[t];
                /* n_total = n_cross + nh_j - nh_i (DS: nh = 0) */
                int nn[3] = {stn[e].n[0] + nh[3 * j] - nh[3 * i], stn[e].n[1] + nh[3 * j + 1] - nh[3 * i + 1],
                             stn[e].n[2] + nh[3 * j + 2] - nh[3 * i + 2]};
                if (j == i && nn[0] == 0 && nn[1] == 0 && nn[2] == 0) continue;
                double d[3];
                double r2 = pair_d(q + 3 * i, q + 3 * j, L, nn, d);
                acc.cand++;
                if (r2 < pot.rc2) {
                    acc_pair(&acc, &pot, q + 3 * i, q + 3 * j, L, j, nn);
                    push_pair(&o, i, j, nn);
                }
            }
        }
        store(&o, k, &acc);
        tot_cand += acc.cand;
        tot_int += acc.cnt;
    }
    stats[0] = tot_cand;
    stats[1] = tot_int;
    stats[2] = g.dims[0]; stats[3] = g.dims[1]; stats[4] = g.dims[2];
    stats[5] = (i64)((t1 - t0) * 1e9);
    stats[6] = (i64)((wtime() - t1) * 1e9);
    free(cell); free(nh); free(a3); free(cs); free(order);
    return 0;
}

int or_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
