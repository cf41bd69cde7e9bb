/*
 * blr_oracle.c -- fp64 CPU ORACLE for the block-low-rank (BLR) prefill forward product
 * of arXiv 2512.20861 ("memory-efficient BLR kernels").
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code, header,
 * constant or helper with the CUDA path in paper_2512_20861_b200/csrc/.
 *
 * Every function is the paper's definition written out with plain loops in double precision,
 * no blocking, no fusion, no reordering beyond what the cited equation states.  Inputs are the
 * bf16-rounded values widened exactly to double by the caller.
 *
 * Notation (§2.1): n tokens, i input features, o output features, r rank.
 *   X in R^{n x i}, Y = X W, W in R^{i x o}
 *   blocks: l in [b1] (input), k in [b2] (output), p = i/b1, q = o/b2
 * All arrays are row-major, contiguous.  Indices are 0-based (the paper uses 1-based).
 *
 * Parity status: every function below is pinned by tests/test_oracle_pins.py (see the
 * pin list in DESIGN.md §3); none is "parity unpinned".
 */
#include <stdint.h>
#include <string.h>

typedef int64_t i64;

/* ------------------------------------------------------------------------------------------ */
/* Dense: Y = X W  ("the corresponding linear layer Y = XW").                     */
/* ------------------------------------------------------------------------------------------ */
void orc_dense_forward(i64 n, i64 i, i64 o, const double* X, const double* W, double* Y)
{
#pragma omp parallel for schedule(static)
    for (i64 t = 0; t < n; ++t) {
        for (i64 c = 0; c < o; ++c) {
            double acc = 0.0;
            for (i64 a = 0; a < i; ++a) acc += X[t * i + a] * W[a * o + c];
            Y[t * o + c] = acc;
        }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Low-rank: W = V U, V in R^{i x r}, U in R^{r x o}.                            */
/* ------------------------------------------------------------------------------------------ */
void orc_lowrank_weight(i64 i, i64 o, i64 r, const double* V, const double* U, double* W)
{
    for (i64 a = 0; a < i; ++a)
        for (i64 c = 0; c < o; ++c) {
            double acc = 0.0;
            for (i64 rho = 0; rho < r; ++rho) acc += V[a * r + rho] * U[rho * o + c];
            W[a * o + c] = acc;
        }
}

/* Structured low-rank forward, "the factorization is stored and used directly":
 * Z = X V (n x r), then Y = Z U.  Z is kept per row (rows are independent). */
void orc_lowrank_forward(i64 n, i64 i, i64 o, i64 r, const double* X, const double* V,
                         const double* U, double* Y, double* scratch /* n*r */)
{
#pragma omp parallel for schedule(static)
    for (i64 t = 0; t < n; ++t) {
        double* Z = scratch + t * r;
        for (i64 rho = 0; rho < r; ++rho) {
            double acc = 0.0;
            for (i64 a = 0; a < i; ++a) acc += X[t * i + a] * V[a * r + rho];
            Z[rho] = acc;
        }
        for (i64 c = 0; c < o; ++c) {
            double acc = 0.0;
            for (i64 rho = 0; rho < r; ++rho) acc += Z[rho] * U[rho * o + c];
            Y[t * o + c] = acc;
        }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Monarch.  W_{l,k} = V_{l,k} U_{l,k} in R^{p x q}, per-block rank r'.      */
/* Storage: Vst in R^{b1 x (r' b2) x p}, Ust in R^{b2 x q x (b1 r')}.            */
/* Composite-index readings (readings R2, R3):                          */
/*   Vst middle dim (r' b2):  layout 0 = "contiguous along b2 then r'"  -> m = rho*b2 + k        */
/*                            layout 1 = after re-layout (1), r' first  -> m = k*r' + rho        */
/*   Ust inner dim (b1 r'):   "contiguous along r' then b1"             -> l*r' + rho            */
/* so V_{l,k}[a, rho] = Vst[l, m(rho,k), a] and U_{l,k}[rho, c] = Ust[k, c, l*r' + rho].        */
/* ------------------------------------------------------------------------------------------ */
static i64 monarch_m(i64 rho, i64 k, i64 b2, i64 rp, int layout)
{
    return layout == 0 ? rho * b2 + k : k * rp + rho;
}

/* Dense reconstruction: W[l*p + a, k*q + c] = sum_rho V_{l,k}[a,rho] U_{l,k}[rho,c]
 * (rows l-major, columns k-major, canonical output order, PAPER.md L53 / reading R4). */
void orc_monarch_weight(i64 b1, i64 b2, i64 rp, i64 p, i64 q, const double* Vst,
                        const double* Ust, int layout, double* W)
{
    const i64 i = b1 * p, o = b2 * q, R = rp * b2, K2 = b1 * rp;
    (void)i;
    for (i64 l = 0; l < b1; ++l)
        for (i64 k = 0; k < b2; ++k)
            for (i64 a = 0; a < p; ++a)
                for (i64 c = 0; c < q; ++c) {
                    double acc = 0.0;
                    for (i64 rho = 0; rho < rp; ++rho) {
                        const double v = Vst[(l * R + monarch_m(rho, k, b2, rp, layout)) * p + a];
                        const double u = Ust[(k * q + c) * K2 + l * rp + rho];
                        acc += v * u;
                    }
                    W[(l * p + a) * o + k * q + c] = acc;
                }
}

/* Structured Monarch forward: Y_k = sum_l X_l W_{l,k} with W_{l,k} = V_{l,k}U_{l,k}
 * evaluated without forming W: z = X_l V_{l,k} (r' values per row), then Y_k += z U_{l,k}. */
void orc_monarch_forward(i64 n, i64 b1, i64 b2, i64 rp, i64 p, i64 q, const double* X,
                         const double* Vst, const double* Ust, int layout, double* Y)
{
    const i64 i = b1 * p, o = b2 * q, R = rp * b2, K2 = b1 * rp;
#pragma omp parallel for schedule(static)
    for (i64 t = 0; t < n; ++t) {
        for (i64 c = 0; c < o; ++c) Y[t * o + c] = 0.0;
        for (i64 k = 0; k < b2; ++k)
            for (i64 l = 0; l < b1; ++l)
                for (i64 rho = 0; rho < rp; ++rho) {
                    const double* vrow = Vst + (l * R + monarch_m(rho, k, b2, rp, layout)) * p;
                    double z = 0.0;
                    for (i64 a = 0; a < p; ++a) z += X[t * i + l * p + a] * vrow[a];
                    for (i64 c = 0; c < q; ++c)
                        Y[t * o + k * q + c] += z * Ust[(k * q + c) * K2 + l * rp + rho];
                }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* BLAST.  W_{l,k} = V_l S_{l,k} U_k, V_l in R^{p x r}, S_{l,k} = diag in     */
/* R^{r x r}, U_k in R^{r x q}; stored as Vst (b1,p,r), Sst (b1,b2,r), Ust (b2,r,q) (L81).       */
/* ------------------------------------------------------------------------------------------ */
void orc_blast_weight(i64 b1, i64 b2, i64 r, i64 p, i64 q, const double* Vst, const double* Sst,
                      const double* Ust, double* W)
{
    const i64 o = b2 * q;
    for (i64 l = 0; l < b1; ++l)
        for (i64 k = 0; k < b2; ++k)
            for (i64 a = 0; a < p; ++a)
                for (i64 c = 0; c < q; ++c) {
                    double acc = 0.0;
                    for (i64 rho = 0; rho < r; ++rho)
                        acc += Vst[(l * p + a) * r + rho] * Sst[(l * b2 + k) * r + rho] *
                               Ust[(k * r + rho) * q + c];
                    W[(l * p + a) * o + k * q + c] = acc;
                }
}

/* Structured BLAST forward: Y_k = ( sum_l (X_l V_l) S_{l,k} ) U_k.
 * Per row: Z_l = X_l V_l for every l; Z''_k = sum_l Z_l S_{l,k}; Y_k = Z''_k U_k. */
void orc_blast_forward(i64 n, i64 b1, i64 b2, i64 r, i64 p, i64 q, const double* X,
                       const double* Vst, const double* Sst, const double* Ust, double* Y,
                       double* scratch /* n * (b1*r + r) */)
{
    const i64 i = b1 * p, o = b2 * q;
#pragma omp parallel for schedule(static)
    for (i64 t = 0; t < n; ++t) {
        double* Z = scratch + t * (b1 * r + r);  /* Z[l*r + rho] = (X_l V_l)[t, rho] */
        double* Zpp = Z + b1 * r;                /* Z''_k[t, rho] for the current k   */
        for (i64 l = 0; l < b1; ++l)
            for (i64 rho = 0; rho < r; ++rho) {
                double acc = 0.0;
                for (i64 a = 0; a < p; ++a) acc += X[t * i + l * p + a] * Vst[(l * p + a) * r + rho];
                Z[l * r + rho] = acc;
            }
        for (i64 k = 0; k < b2; ++k) {
            for (i64 rho = 0; rho < r; ++rho) {
                double acc = 0.0;
                for (i64 l = 0; l < b1; ++l) acc += Z[l * r + rho] * Sst[(l * b2 + k) * r + rho];
                Zpp[rho] = acc;
            }
            for (i64 c = 0; c < q; ++c) {
                double acc = 0.0;
                for (i64 rho = 0; rho < r; ++rho) acc += Zpp[rho] * Ust[(k * r + rho) * q + c];
                Y[t * o + k * q + c] = acc;
            }
        }
    }
}

/* Number of OpenMP threads the oracle will use (reported as cpu_baseline.cores). */
int orc_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count for subsequent calls (timing only: the arithmetic and its order per output element
   do not depend on it).  n <= 0 restores the OpenMP default. */
void orc_set_num_threads(int n)
{
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    extern int omp_get_num_procs(void);
    omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
#else
    (void)n;
#endif
}
