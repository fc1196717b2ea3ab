/*
 * h2_oracle.c -- plain, slow, obviously-correct CPU oracle of the H^2 matrix-vector product
 *
 *     Y := alpha * A~ * X + beta * Y,   A~ = A_de + sum_l sum_{(t,s)} U^l_t S^l_ts V^l_s^T
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code with the
 * CUDA path (paper_2109_05451_b200/) and includes none of its headers.
 *
 * It follows the paper's algorithm step by step, by direct recursion over a pointer tree it
 * builds itself from the flat input arrays, in FP64, in a fixed per-output order.  OpenMP runs
 * independent subtrees (tasks) and independent rows (parallel loops) concurrently; every output
 * value is still computed by one thread in the same order as the sequential recursion, so the
 * result is bitwise identical for any thread count (SURVEY.md §8(c) "OpenMP is allowed over
 * independent subtrees and rows with a fixed per-output order"; pinned by a test):
 *   1. forward(s)   upsweep      PAPER.md:239-254 (sec. "Distributed Upsweep", alg:upsweep2):
 *                   leaf: xh_s = V_s^T x_s ; inner: xh_s = F_{s1}^T xh_{s1} + F_{s2}^T xh_{s2}
 *   2. couplings    PAPER.md:328-329 ("Distributed Intermediate Multiplication"):
 *                   yh_t = sum_{s in b_t} S_ts xh_s, s ascending
 *   3. backward(t)  downsweep    PAPER.md:379-399 (alg:downsweep): yh_t += E_t yh_parent,
 *                   top-down; leaf: y_t = U_t yh_t
 *   4. dense        PAPER.md:225: y_t += sum_s D_ts x_s, s ascending
 *   5. epilogue     BLAS semantics (reading R12): Y = alpha*y + beta*Y; beta == 0 -> Y not read;
 *                   alpha == 0 -> steps 1-4 skipped.
 * Storage: every small r x c matrix column-major; X, Y are
 * N x nv column-major with leading dimension N, rows in cluster-tree order.
 * Levels: global numbering, root = 0, leaves = q (reading R2).  Transfer E^l_c is k^l x k^{l-1}
 * (reading R1).  Parity: pinned by the -m "not gpu" tests (dense assembly, closed forms,
 * all-dense case, linearity); see DESIGN.md "Oracle pins".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t N;
    int32_t m, q;
    const int32_t *ranks;               /* [q+1] k^l                                   */
    const int64_t *leaf_ptr;            /* [2^q + 1] row offsets of the leaves           */
    const double *U_leaf, *V_leaf;      /* [2^q][k^q][m]  (m x k^q col-major per leaf)   */
    const double *const *E, *const *F;  /* [q+1]; E[l]: [2^l][k^{l-1}][k^l]; E[0] unused */
    const int64_t *const *S_rowptr;     /* [q+1]; [2^l + 1]                              */
    const int32_t *const *S_col;        /* [q+1]; column node index within level l       */
    const double *const *S;             /* [q+1]; [nblk_l][k^l][k^l]                     */
    const int64_t *D_rowptr;            /* [2^q + 1]                                     */
    const int32_t *D_col;               /* leaf column index                             */
    const double *D;                    /* [n_D][m][m]                                   */
} h2o_input;

typedef struct node {
    int level;
    int64_t index;                      /* position within its level                    */
    int k;                              /* k^level                                      */
    struct node *parent, *child[2];
    int64_t row_begin, row_end;         /* rows of X / Y covered by this cluster        */
    const double *E, *F;                /* transfer to the parent (k x k_parent)         */
    const double *U, *V;                /* leaves only (m x k)                          */
    int64_t ncoup; const double **S; struct node **coup_col;
    int64_t ndense; const double **D; struct node **dense_col;
    double *xh, *yh;                    /* k x nv each                                  */
    int needed;
} node;

typedef struct {
    const h2o_input *in;
    int nv;
    const double *X;
    double *y;                          /* N x nv accumulator for y = A~ X */
    node **level_nodes;                 /* [q+1] arrays of 2^l nodes       */
    int par_levels;                     /* spawn subtree tasks above this level */
} ctx;

/* ---------------------------------------------------------------- tree construction */
static node *build_tree(const h2o_input *in, int nv, node ***levels_out)
{
    int q = in->q;
    node **levels = (node **)calloc((size_t)q + 1, sizeof(node *));
    for (int l = 0; l <= q; l++) {
        int64_t n = (int64_t)1 << l;
        levels[l] = (node *)calloc((size_t)n, sizeof(node));
        for (int64_t i = 0; i < n; i++) {
            node *t = &levels[l][i];
            t->level = l; t->index = i; t->k = in->ranks[l];
            t->parent = l ? &levels[l - 1][i / 2] : NULL;
            t->xh = (double *)calloc((size_t)t->k * nv, sizeof(double));
            t->yh = (double *)calloc((size_t)t->k * nv, sizeof(double));
            if (l) {
                size_t sz = (size_t)t->k * in->ranks[l - 1];
                t->E = in->E[l] + (size_t)i * sz;
                t->F = in->F[l] + (size_t)i * sz;
            }
            /* couplings of block row t at level l */
            int64_t b0 = in->S_rowptr[l][i], b1 = in->S_rowptr[l][i + 1];
            t->ncoup = b1 - b0;
            t->S = (const double **)malloc(sizeof(double *) * (size_t)(t->ncoup + 1));
            t->coup_col = (node **)malloc(sizeof(node *) * (size_t)(t->ncoup + 1));
        }
    }
    for (int l = 0; l <= q; l++) {
        int64_t n = (int64_t)1 << l;
        size_t kk = (size_t)in->ranks[l] * in->ranks[l];
        for (int64_t i = 0; i < n; i++) {
            node *t = &levels[l][i];
            if (l < q) { t->child[0] = &levels[l + 1][2 * i]; t->child[1] = &levels[l + 1][2 * i + 1]; }
            int64_t b0 = in->S_rowptr[l][i];
            for (int64_t b = 0; b < t->ncoup; b++) {
                t->S[b] = in->S[l] + (size_t)(b0 + b) * kk;
                t->coup_col[b] = &levels[l][in->S_col[l][b0 + b]];
            }
        }
    }
    /* leaves: rows, explicit bases, dense blocks */
    int64_t nleaf = (int64_t)1 << q;
    size_t mk = (size_t)in->m * in->ranks[q], mm = (size_t)in->m * in->m;
    for (int64_t i = 0; i < nleaf; i++) {
        node *t = &levels[q][i];
        t->row_begin = in->leaf_ptr[i]; t->row_end = in->leaf_ptr[i + 1];
        t->U = in->U_leaf + (size_t)i * mk;
        t->V = in->V_leaf + (size_t)i * mk;
        int64_t b0 = in->D_rowptr[i], b1 = in->D_rowptr[i + 1];
        t->ndense = b1 - b0;
        t->D = (const double **)malloc(sizeof(double *) * (size_t)(t->ndense + 1));
        t->dense_col = (node **)malloc(sizeof(node *) * (size_t)(t->ndense + 1));
        for (int64_t b = 0; b < t->ndense; b++) {
            t->D[b] = in->D + (size_t)(b0 + b) * mm;
            t->dense_col[b] = &levels[q][in->D_col[b0 + b]];
        }
    }
    for (int l = q - 1; l >= 0; l--) {          /* inner clusters cover their children's rows */
        int64_t n = (int64_t)1 << l;
        for (int64_t i = 0; i < n; i++) {
            node *t = &levels[l][i];
            t->row_begin = t->child[0]->row_begin; t->row_end = t->child[1]->row_end;
        }
    }
    *levels_out = levels;
    return &levels[0][0];
}

static void free_tree(const h2o_input *in, node **levels)
{
    for (int l = 0; l <= in->q; l++) {
        int64_t n = (int64_t)1 << l;
        for (int64_t i = 0; i < n; i++) {
            node *t = &levels[l][i];
            free(t->xh); free(t->yh); free(t->S); free(t->coup_col);
            if (l == in->q) { free(t->D); free(t->dense_col); }
        }
        free(levels[l]);
    }
    free(levels);
}

/* ---------------------------------------------------------------- 1. upsweep (forward) */
static void forward(ctx *c, node *s)
{
    int nv = c->nv, k = s->k;
    int64_t N = c->in->N;
    memset(s->xh, 0, sizeof(double) * (size_t)k * nv);
    if (s->child[0] == NULL) {                  /* leaf: xh_s = V_s^T x_s */
        int m = c->in->m;
        int64_t rows = s->row_end - s->row_begin;
        for (int n = 0; n < nv; n++)
            for (int a = 0; a < k; a++) {
                double acc = 0.0;
                for (int64_t i = 0; i < rows; i++)
                    acc += s->V[(size_t)a * m + i] * c->X[(size_t)n * N + s->row_begin + i];
                s->xh[(size_t)n * k + a] = acc;
            }
        return;
    }
    /* the two child subtrees are independent: recurse concurrently, then accumulate in order */
    #pragma omp task if (s->level < c->par_levels)
    forward(c, s->child[0]);
    forward(c, s->child[1]);
    #pragma omp taskwait
    for (int ci = 0; ci < 2; ci++) {            /* inner: xh_s = sum_c F_c^T xh_c */
        node *ch = s->child[ci];
        int kc = ch->k;
        for (int n = 0; n < nv; n++)
            for (int b = 0; b < k; b++) {
                double acc = 0.0;
                for (int a = 0; a < kc; a++)
                    acc += ch->F[(size_t)b * kc + a] * ch->xh[(size_t)n * kc + a];
                s->xh[(size_t)n * k + b] += acc;
            }
    }
}

/* ---------------------------------------------------------------- 2. coupling multiply */
static void couple(ctx *c, node *t)
{
    int nv = c->nv, k = t->k;
    memset(t->yh, 0, sizeof(double) * (size_t)k * nv);
    for (int64_t b = 0; b < t->ncoup; b++) {    /* yh_t += S_ts xh_s, s ascending */
        const double *S = t->S[b];
        const node *s = t->coup_col[b];
        for (int n = 0; n < nv; n++)
            for (int a = 0; a < k; a++) {
                double acc = 0.0;
                for (int bb = 0; bb < k; bb++)
                    acc += S[(size_t)bb * k + a] * s->xh[(size_t)n * k + bb];
                t->yh[(size_t)n * k + a] += acc;
            }
    }
}

/* ---------------------------------------------------------------- 3. downsweep (backward) */
static void backward(ctx *c, node *t)
{
    int nv = c->nv, k = t->k;
    int64_t N = c->in->N;
    if (!t->needed) return;
    if (t->parent) {                            /* yh_t += E_t yh_parent (parent already updated) */
        const node *p = t->parent;
        int kp = p->k;
        for (int n = 0; n < nv; n++)
            for (int a = 0; a < k; a++) {
                double acc = 0.0;
                for (int b = 0; b < kp; b++)
                    acc += t->E[(size_t)b * k + a] * p->yh[(size_t)n * kp + b];
                t->yh[(size_t)n * k + a] += acc;
            }
    }
    if (t->child[0] == NULL) {                  /* leaf: y_t = U_t yh_t */
        int m = c->in->m;
        int64_t rows = t->row_end - t->row_begin;
        for (int n = 0; n < nv; n++)
            for (int64_t i = 0; i < rows; i++) {
                double acc = 0.0;
                for (int a = 0; a < k; a++)
                    acc += t->U[(size_t)a * m + i] * t->yh[(size_t)n * k + a];
                c->y[(size_t)n * N + t->row_begin + i] = acc;
            }
        return;
    }
    #pragma omp task if (t->level < c->par_levels)
    backward(c, t->child[0]);
    backward(c, t->child[1]);
    #pragma omp taskwait
}

/* ---------------------------------------------------------------- 4. dense near field */
static void dense(ctx *c, node *t)
{
    int nv = c->nv, m = c->in->m;
    int64_t N = c->in->N;
    int64_t rows = t->row_end - t->row_begin;
    for (int64_t b = 0; b < t->ndense; b++) {   /* y_t += D_ts x_s, s ascending */
        const double *D = t->D[b];
        const node *s = t->dense_col[b];
        int64_t cols = s->row_end - s->row_begin;
        for (int n = 0; n < nv; n++)
            for (int64_t i = 0; i < rows; i++) {
                double acc = 0.0;
                for (int64_t j = 0; j < cols; j++)
                    acc += D[(size_t)j * m + i] * c->X[(size_t)n * N + s->row_begin + j];
                c->y[(size_t)n * N + t->row_begin + i] += acc;
            }
    }
}

/*
 * h2o_matvec: Y := alpha A~ X + beta Y.  leaf_mask (optional, [2^q]): when non-NULL only the
 * rows of leaves with leaf_mask[i] != 0 are computed and written (sampled-row oracle of
 * SURVEY.md §8(c)); the upsweep is always complete, couplings and the downsweep are evaluated
 * only on the ancestors of the sampled leaves -- the same arithmetic restricted to the rows asked.
 * Returns 0, or -1 on bad arguments / allocation failure.
 */
int h2o_matvec(const h2o_input *in, int nv, double alpha, const double *X, double beta,
               double *Y, const unsigned char *leaf_mask)
{
    if (!in || nv < 1 || !X || !Y || in->q < 0 || in->m < 1) return -1;
    int q = in->q;
    int64_t N = in->N, nleaf = (int64_t)1 << q;
    double *y = (double *)calloc((size_t)N * nv, sizeof(double));
    if (!y) return -1;
    if (alpha != 0.0) {
        node **levels = NULL;
        node *root = build_tree(in, nv, &levels);
        ctx c = { in, nv, X, y, levels, q < 12 ? q : 12 };
        for (int64_t i = 0; i < nleaf; i++) {
            if (leaf_mask && !leaf_mask[i]) continue;
            for (node *t = &levels[q][i]; t; t = t->parent) t->needed = 1;
        }
        #pragma omp parallel
        #pragma omp single
        forward(&c, root);                                       /* 1 */
        for (int l = 0; l <= q; l++) {                           /* 2 */
            int64_t n = (int64_t)1 << l;
            #pragma omp parallel for schedule(dynamic, 16)
            for (int64_t i = 0; i < n; i++)
                if (levels[l][i].needed) couple(&c, &levels[l][i]);
        }
        #pragma omp parallel
        #pragma omp single
        backward(&c, root);                                      /* 3 */
        #pragma omp parallel for schedule(dynamic, 16)
        for (int64_t i = 0; i < nleaf; i++)                      /* 4 */
            if (levels[q][i].needed) dense(&c, &levels[q][i]);
        free_tree(in, levels);
    }
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nleaf; i++) {                        /* 5 */
        if (leaf_mask && !leaf_mask[i]) continue;
        for (int n = 0; n < nv; n++)
            for (int64_t r = in->leaf_ptr[i]; r < in->leaf_ptr[i + 1]; r++) {
                size_t o = (size_t)n * N + r;
                Y[o] = (beta == 0.0) ? alpha * y[o] : alpha * y[o] + beta * Y[o];
            }
    }
    free(y);
    return 0;
}

/* Per-phase trees for the per-phase parity tests: xh_out / yh_out (may be NULL) receive, for
 * every level l, the 2^l nodes' (k^l x nv) blocks concatenated level by level: xh after the
 * upsweep (step 1) and yh after the coupling multiply (step 2, before the downsweep). */
int h2o_trees(const h2o_input *in, int nv, const double *X, double *xh_out, double *yh_out)
{
    if (!in || nv < 1 || !X) return -1;
    int q = in->q;
    double *y = (double *)calloc((size_t)in->N * nv, sizeof(double));
    if (!y) return -1;
    node **levels = NULL;
    node *root = build_tree(in, nv, &levels);
    ctx c = { in, nv, X, y, levels, q < 12 ? q : 12 };
    #pragma omp parallel
    #pragma omp single
    forward(&c, root);
    for (int l = 0; l <= q; l++) {
        int64_t n = (int64_t)1 << l;
        #pragma omp parallel for schedule(dynamic, 16)
        for (int64_t i = 0; i < n; i++) couple(&c, &levels[l][i]);
    }
    size_t off = 0;
    for (int l = 0; l <= q; l++)
        for (int64_t i = 0; i < ((int64_t)1 << l); i++) {
            size_t sz = (size_t)levels[l][i].k * nv;
            if (xh_out) memcpy(xh_out + off, levels[l][i].xh, sz * sizeof(double));
            if (yh_out) memcpy(yh_out + off, levels[l][i].yh, sz * sizeof(double));
            off += sz;
        }
    free_tree(in, levels);
    free(y);
    return 0;
}

/* Threads used by the OpenMP regions of later calls (n < 1: the OpenMP default); returns the
 * thread count in effect (1 when built without OpenMP). */
int h2o_set_threads(int n)
{
#ifdef _OPENMP
    if (n >= 1) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}
