/*
 * escs_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the hot path of
 * arXiv 2506.15174 ("enumerate-and-sparse-coarsen", ESC).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, table or helper
 * with the CUDA path (paper_2506_15174_b200/csrc); neither includes the other.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * DESIGN.md "Reading Rk" = the reading of a silent/garbled passage we adopted.
 *
 * Two functions:
 *
 *  oracle_spmm       C = A x B with A in CSR, fp64 accumulation in CSR order.
 *                    This is the plain definition of Listing 1:
 *                      for i, for k, for j: if (A[i][k]) C[i][j] += A[i][k]*B[k][j]
 *                    ESC reaches exactly this result up to fp32 rounding
 *                    order (the method only re-maps iterations).
 *                    Pinned by tests/test_oracle.py against numpy dense A@B,
 *                    exact dyadic cases, identity A and one-nonzero rows.
 *
 *  oracle_partition  The enumeration plan ("TA") built the way the
 *                    paper's dataTransformer does it: iterate over
 *                    the dense image of each UFi-row panel once (O(M*K)),
 *                    compute each column's UFi-bit nonzero pattern, bucket the
 *                    panel's columns by pattern (one enumerated block per
 *                    pattern), lay the values out in
 *                    kernel traversal order (Listing 7, read as
 *                    DESIGN.md Reading R1), and cut each panel's column stream
 *                    into balanced items of at most T columns (north_star
 *                    "balanced tiles"; DESIGN.md Reading R7).
 *                    Pinned by the golden plan (S:123/S:132/S:501), the
 *                    exhaustive 15-pattern matrix, brute-force
 *                    enumeration on tiny inputs and invariants I1-I7.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* oracle_spmm                                                               */
/* ------------------------------------------------------------------------- */
/*
 * rows == NULL: compute all m rows, C is m x ncols.
 * rows != NULL: compute only rows[0..nrows), C is nrows x ncols (sampled check
 *               at full sizes).
 * absum (nullable): sum_t |vals[t]| * |B[colidx[t]][j]|, same shape as C.
 * nterms (nullable): number of CSR terms in each computed row.
 * Returns 0, or -1 on a malformed CSR (caller bug; the oracle does not repair).
 */
int oracle_spmm(int64_t m, int64_t k, int32_t ncols,
                const int32_t *rowptr, const int32_t *colidx,
                const float *vals, const float *B,
                const int64_t *rows, int64_t nrows,
                double *C, double *absum, int32_t *nterms, int32_t nthreads)
{
    int64_t nout = rows ? nrows : m;
    int bad = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16) reduction(|:bad)
#endif
    for (int64_t o = 0; o < nout; o++) {
        int64_t i = rows ? rows[o] : o;
        if (i < 0 || i >= m) { bad |= 1; continue; }
        double *c = C + o * (int64_t)ncols;
        double *a = absum ? absum + o * (int64_t)ncols : NULL;
        for (int32_t j = 0; j < ncols; j++) { c[j] = 0.0; if (a) a[j] = 0.0; }
        /* CSR order: t ascending within row i (Listing 1's k loop). */
        for (int64_t t = rowptr[i]; t < rowptr[i + 1]; t++) {
            int64_t kk = colidx[t];
            if (kk < 0 || kk >= k) { bad |= 1; break; }
            double av = (double)vals[t];
            const float *b = B + kk * (int64_t)ncols;
            for (int32_t j = 0; j < ncols; j++) {
                c[j] += av * (double)b[j];          /* product exact in fp64 */
                if (a) a[j] += fabs(av) * fabs((double)b[j]);
            }
        }
        if (nterms) nterms[o] = (int32_t)(rowptr[i + 1] - rowptr[i]);
    }
    return bad ? -1 : 0;
}

/* ------------------------------------------------------------------------- */
/* oracle_partition                                                          */
/* ------------------------------------------------------------------------- */
/*
 * Output arrays are caller-allocated with capacities:
 *   grp_panel, grp_mask            : cap_groups
 *   grp_col_ptr, grp_val_ptr       : cap_groups + 1
 *   gcol, slot_src                 : max(nnz, 1)
 *   item_panel, item_group_begin   : cap_items
 *   item_gcol_ptr                  : cap_items + 1
 * header[11] = version, m, k, nnz, bCols, h, T, nP, NG, G, n_items.
 * Returns 0 on success, -1 on bad arguments, -2 on capacity overflow.
 */
#define ORACLE_PLAN_VERSION 1

int oracle_partition(int64_t m, int64_t k, int64_t nnz,
                     const int32_t *rowptr, const int32_t *colidx,
                     int32_t bCols, int32_t h, int32_t T,
                     int32_t *header,
                     int32_t *grp_panel, int32_t *grp_mask,
                     int32_t *grp_col_ptr, int32_t *grp_val_ptr,
                     int32_t *gcol, int32_t *slot_src,
                     int32_t *item_panel, int32_t *item_group_begin,
                     int32_t *item_gcol_ptr,
                     int64_t cap_groups, int64_t cap_items)
{
    if (m < 1 || k < 1 || nnz < 0 || h < 1 || h > 16 || T < 1) return -1;
    int64_t nP = (m + h - 1) / h;                 /* Reading R2: ragged last panel */
    int64_t nmask = (int64_t)1 << h;

    /* Dense image of one panel: pattern of every column, and where each
     * (row r, column c) nonzero lives in CSR ("if (A[i][k])").     */
    int32_t *mask = (int32_t *)calloc((size_t)k, sizeof(int32_t));
    int32_t *pos = (int32_t *)malloc((size_t)h * (size_t)k * sizeof(int32_t));
    int64_t *count = (int64_t *)calloc((size_t)nmask, sizeof(int64_t));
    int64_t *gfirst = (int64_t *)malloc((size_t)nmask * sizeof(int64_t));
    int64_t *fill = (int64_t *)calloc((size_t)nmask, sizeof(int64_t));
    if (!mask || !pos || !count || !gfirst || !fill) {
        free(mask); free(pos); free(count); free(gfirst); free(fill);
        return -1;
    }

    int64_t NG = 0, G = 0, NI = 0, V = 0;  /* groups, gcols, items, value slots */
    int rc = 0;
    grp_col_ptr[0] = 0;
    grp_val_ptr[0] = 0;
    item_gcol_ptr[0] = 0;

    for (int64_t P = 0; P < nP && rc == 0; P++) {
        int64_t r0 = P * h;
        int64_t rows = (m - r0 < h) ? (m - r0) : h;

        /* 1. scan the panel's rows: bit r of mask[c] <=> A(r0+r, c) != 0
         *    (the unrolled conditionals of Listing 3).          */
        for (int64_t r = 0; r < rows; r++)
            for (int64_t t = rowptr[r0 + r]; t < rowptr[r0 + r + 1]; t++) {
                mask[colidx[t]] |= (int32_t)1 << r;
                pos[r * k + colidx[t]] = (int32_t)t;
            }

        /* 2. count columns per pattern over the dense column range. */
        for (int64_t mu = 0; mu < nmask; mu++) { count[mu] = 0; fill[mu] = 0; }
        for (int64_t c = 0; c < k; c++) count[mask[c]]++;

        /* 3. one group (enumerated block x row panel) per non-empty
         *    pattern, patterns ascending (Reading R3), pattern 0 never
         *    materialised (P:286-310 enumerates the 2^UFi-1 non-zero ones). */
        int64_t pgroup0 = NG, pstream0 = G;
        for (int64_t mu = 1; mu < nmask; mu++) {
            if (count[mu] == 0) continue;
            if (NG >= cap_groups) { rc = -2; break; }
            int p = __builtin_popcountll((unsigned long long)mu);
            gfirst[mu] = NG;
            grp_panel[NG] = (int32_t)P;
            grp_mask[NG] = (int32_t)mu;
            grp_col_ptr[NG + 1] = (int32_t)(grp_col_ptr[NG] + count[mu]);   /* "RPP" */
            grp_val_ptr[NG + 1] = (int32_t)(grp_val_ptr[NG] + count[mu] * p); /* "NPP" */
            NG++;
        }
        if (rc) break;

        /* 4. place columns, ascending within each group ("Cols"), and the
         *    value slots in Listing 7's traversal order: column-major over
         *    the group's columns, pattern rows ascending (Reading R1).     */
        for (int64_t c = 0; c < k; c++) {
            int32_t mu = mask[c];
            if (mu == 0) continue;
            int64_t g = gfirst[mu];
            int64_t ci = fill[mu]++;                        /* column ordinal */
            gcol[grp_col_ptr[g] + ci] = (int32_t)c;
            int p = __builtin_popcount((unsigned)mu);
            int rank = 0;
            for (int r = 0; r < h; r++) {
                if (!((mu >> r) & 1)) continue;
                slot_src[grp_val_ptr[g] + ci * p + rank] = pos[(int64_t)r * k + c];
                rank++;
            }
            V += p;
        }
        int64_t SP = grp_col_ptr[NG] - pstream0;            /* panel stream length */
        G += SP;

        /* 5. balanced items of the panel stream (Reading R7):
         *    n_P = max(1, ceil(S_P/T)); item q = [q*S_P/n_P, (q+1)*S_P/n_P). */
        int64_t nPi = (SP + T - 1) / T;
        if (nPi < 1) nPi = 1;
        for (int64_t q = 0; q < nPi; q++) {
            if (NI >= cap_items) { rc = -2; break; }
            int64_t s0 = (q * SP) / nPi, s1 = ((q + 1) * SP) / nPi;
            /* last group of the panel whose stream start <= s0 */
            int64_t gb = pgroup0;
            for (int64_t g = pgroup0; g < NG; g++)
                if (grp_col_ptr[g] - pstream0 <= s0) gb = g;
            item_panel[NI] = (int32_t)P;
            item_group_begin[NI] = (int32_t)gb;
            item_gcol_ptr[NI] = (int32_t)(pstream0 + s0);
            item_gcol_ptr[NI + 1] = (int32_t)(pstream0 + s1);
            NI++;
        }

        /* 6. reset the dense panel image (the O(K) part of O(M*K)). */
        for (int64_t c = 0; c < k; c++) mask[c] = 0;
    }

    free(mask); free(pos); free(count); free(gfirst); free(fill);
    if (rc) return rc;
    if (V != nnz) return -1;   /* conservation; cannot fail on valid CSR */

    header[0] = ORACLE_PLAN_VERSION;
    header[1] = (int32_t)m;   header[2] = (int32_t)k;  header[3] = (int32_t)nnz;
    header[4] = bCols;        header[5] = h;           header[6] = T;
    header[7] = (int32_t)nP;  header[8] = (int32_t)NG; header[9] = (int32_t)G;
    header[10] = (int32_t)NI;
    return 0;
}
