/*
 * oracle/cce_oracle.c -- the CPU oracle for the fused linear cross-entropy
 * (Cut Cross-Entropy) hot path of arxiv 2601.02609 ("Chronicals").
 *
 * TEST INFRASTRUCTURE ONLY.  This file is a plain, slow, obviously-correct
 * fp64 statement of what the CUDA path computes.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * leg may load it.  It shares no code, header, table or constant generator
 * with paper_2601_02609_b200/ (the product path), and the product path never
 * calls it.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line, "S:<line>" =
 * /root/reference/SPEC.md line (interface ideas only).  Readings of the paper
 * taken where it is silent or garbled are listed in DESIGN.md ("Readings").
 *
 * What is computed (reading R1-R8):
 *   z[n,v]  = sum_d H[n,d] * W[v,d]                 logits, P:555 (z_c = h W_c^T)
 *   m_n     = max_v z[n,v]                          stable form
 *   lse_n   = m_n + log sum_v exp(z[n,v] - m_n)
 *   l_n     = lse_n - z[n, y_n]                      P:243-248 (Def. Cross-Entropy Loss)
 *   loss    = (1/n_valid) sum_{valid n} l_n          mean over non-ignored rows
 *   G[n,v]  = (dloss/n_valid) (exp(z[n,v]-lse_n) - 1[v == y_n])
 *                                                    P:254-258 (Prop. CE Gradient)
 *   dH[n,:] = sum_v G[n,v] W[v,:]                    P:666 (grad_h += probs @ W[chunk])
 *   dW[v,:] = sum_n G[n,v] H[n,:]                    P:667 (grad_W[chunk] += probs^T @ h)
 * Regularised variant (oracle_cce_reg), the paper's definitions
 * with label smoothing eps and z-loss weight lam (both 0 gives the above exactly):
 *   l_n     = (1-eps) (lse_n - z[n,y_n])                     (1-eps) L(z, c)
 *           + eps (lse_n - (1/V) sum_v z[n,v])               eps L_uniform(z)
 *           + lam lse_n^2                                    Z-loss, added
 *   G[n,v]  = s [ (1-eps)(p - 1[v==y]) + eps (p - 1/V) + 2 lam lse_n p ],  p = exp(z - lse_n)
 *             (the three terms' gradients: P:254-258; d/dz of -mean z = -1/V)
 * Rows whose label equals ignore_index are skipped:
 * they get lse = 0, dH row = 0 and contribute nothing to dW or to the mean.
 *
 * Inputs are fp64 arrays (the Python wrapper converts bf16 bit patterns to
 * fp64 exactly: a bf16 is the top half of an IEEE fp32); labels are int32.  Every output element is summed by one thread in a fixed order, so
 * results are reproducible run to run.  Parallelism is OpenMP over rows
 * (forward / dH) and over vocabulary rows (dW); there is no blocking, fusion
 * or reordering of the arithmetic beyond the definitions above.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_LABEL_RANGE 1   /* S:242-244 "target out of range" */
#define ORACLE_ERR_INVALID 2
#define ORACLE_ERR_NOMEM 3


int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Label validation (reading R3): a label is either ignore_index or in
 * [0, V).  Returns ORACLE_ERR_LABEL_RANGE on the first offending label. */
int oracle_validate(const int32_t *labels, int64_t N, int64_t V,
                    int32_t ignore_index, int64_t *n_valid) {
    int64_t c = 0;
    for (int64_t n = 0; n < N; ++n) {
        int32_t y = labels[n];
        if (y == ignore_index) continue;
        if (y < 0 || (int64_t)y >= V) return ORACLE_ERR_LABEL_RANGE;
        ++c;
    }
    *n_valid = c;
    return ORACLE_OK;
}

/* One materialised logit row z[v] = sum_d h[d] W[v,d]. */
static void logit_row(const double *h, const double *W, int64_t D, int64_t V,
                      double *z) {
    for (int64_t v = 0; v < V; ++v) {
        const double *w = W + v * D;
        double acc = 0.0;
        for (int64_t d = 0; d < D; ++d) acc += h[d] * w[d];
        z[v] = acc;
    }
}

/* Two-pass stable log-sum-exp: m = max z, lse = m + log sum exp(z-m). */
static double lse_two_pass(const double *z, int64_t V) {
    double m = -INFINITY;
    for (int64_t v = 0; v < V; ++v) if (z[v] > m) m = z[v];
    double s = 0.0;
    for (int64_t v = 0; v < V; ++v) s += exp(z[v] - m);
    return m + log(s);
}

/*
 * Full forward + backward on the whole problem (the plain definition).
 *   H[N,D], W[V,D] fp64; labels[N]; dloss = upstream gradient of the mean loss.
 *   Outputs: *loss, lse[N] (0 for ignored rows), *n_valid, and (if non-NULL)
 *   dH[N,D], dW[V,D], all fp64.  With n_valid == 0: loss = 0 and zero grads
 *   (reading R2).
 */
/* dL/dz[v] of one valid row's loss (before the mean scale), R11/R12. */
static double row_grad(double zv, double lse, int is_target, double eps, double lam, int64_t V) {
    double p = exp(zv - lse);
    double ce = p - (is_target ? 1.0 : 0.0);
    double uni = p - 1.0 / (double)V;                 /* d/dz of lse - mean z */
    double zl = 2.0 * lam * lse * p;
    return (1.0 - eps) * ce + eps * uni + zl;
}

/*
 * reduction: 0 = mean over valid rows, 1 = sum, 2 = none.
 * The upstream gradient of row n's loss is dloss / n_valid (mean), dloss (sum) or
 * dloss_rows[n] (none); with "none" *loss receives the [N] per-row losses (0 for
 * ignored rows).
 */
int oracle_cce_full(const double *H, const double *W, const int32_t *labels,
                    int64_t N, int64_t D, int64_t V, int32_t ignore_index,
                    double eps, double lam, int reduction,
                    double dloss, const double *dloss_rows,
                    double *loss, double *lse, int64_t *n_valid,
                    double *dH, double *dW) {
    if (N < 0 || D <= 0 || V <= 0 || reduction < 0 || reduction > 2) return ORACLE_ERR_INVALID;
    if (reduction == 2 && !dloss_rows && (dH || dW)) return ORACLE_ERR_INVALID;
    int64_t nv = 0;
    int rc = oracle_validate(labels, N, V, ignore_index, &nv);
    if (rc) return rc;
    *n_valid = nv;
    double *row_loss = (double *)calloc((size_t)(N > 0 ? N : 1), sizeof(double));
    double *rscale = (double *)calloc((size_t)(N > 0 ? N : 1), sizeof(double));
    if (!row_loss || !rscale) { free(row_loss); free(rscale); return ORACLE_ERR_NOMEM; }
    for (int64_t n = 0; n < N; ++n) {                   /* reading R6 */
        if (labels[n] == ignore_index) continue;
        rscale[n] = reduction == 0 ? dloss / (double)nv : (reduction == 1 ? dloss : (dloss_rows ? dloss_rows[n] : 0.0));
    }
    int nomem = 0;

    /* Pass 1, parallel over rows: materialise z, lse, l_n, G row, dH row. */
#pragma omp parallel
    {
        double *h = (double *)malloc((size_t)D * sizeof(double));
        double *z = (double *)malloc((size_t)V * sizeof(double));
        if (!h || !z) {
#pragma omp atomic write
            nomem = 1;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t n = 0; n < N; ++n) {
            if (!h || !z) continue;
            int32_t y = labels[n];
            if (y == ignore_index) {
                lse[n] = 0.0;
                if (dH) for (int64_t d = 0; d < D; ++d) dH[n * D + d] = 0.0;
                continue;
            }
            for (int64_t d = 0; d < D; ++d) h[d] = H[n * D + d];
            logit_row(h, W, D, V, z);
            double l = lse_two_pass(z, V);
            lse[n] = l;
            double zsum = 0.0;
            for (int64_t v = 0; v < V; ++v) zsum += z[v];
            row_loss[n] = (1.0 - eps) * (l - z[y]) + eps * (l - zsum / (double)V) + lam * l * l;
            if (dH) {
                double *out = dH + n * D;
                for (int64_t d = 0; d < D; ++d) out[d] = 0.0;
                for (int64_t v = 0; v < V; ++v) {
                    double g = rscale[n] * row_grad(z[v], l, v == y, eps, lam, V);
                    const double *w = W + v * D;
                    for (int64_t d = 0; d < D; ++d) out[d] += g * w[d];
                }
            }
        }
        free(h);
        free(z);
    }
    if (nomem) { free(row_loss); free(rscale); return ORACLE_ERR_NOMEM; }

    /* Mean / sum over valid rows, summed in row order; or the rows themselves. */
    if (reduction == 2) {
        for (int64_t n = 0; n < N; ++n) loss[n] = labels[n] != ignore_index ? row_loss[n] : 0.0;
    } else {
        double acc = 0.0;
        for (int64_t n = 0; n < N; ++n) if (labels[n] != ignore_index) acc += row_loss[n];
        *loss = reduction == 1 ? acc : (nv > 0 ? acc / (double)nv : 0.0);
    }
    free(row_loss);

    /* Pass 2, parallel over vocabulary rows: recompute z[n,v], G[n,v], dW[v,:]. */
    if (dW) {
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t v = 0; v < V; ++v) {
            double *out = dW + v * D;
            const double *w = W + v * D;
            for (int64_t d = 0; d < D; ++d) out[d] = 0.0;
            for (int64_t n = 0; n < N; ++n) {
                int32_t y = labels[n];
                if (y == ignore_index) continue;
                const double *hr = H + n * D;
                double zv = 0.0;
                for (int64_t d = 0; d < D; ++d) zv += hr[d] * w[d];
                double g = rscale[n] * row_grad(zv, lse[n], v == y, eps, lam, V);
                for (int64_t d = 0; d < D; ++d) out[d] += g * hr[d];
            }
        }
    }
    free(rscale);
    return ORACLE_OK;
}

int oracle_cce_reg(const double *H, const double *W, const int32_t *labels,
                   int64_t N, int64_t D, int64_t V, int32_t ignore_index,
                   double eps, double lam,
                   double dloss, double *loss, double *lse, int64_t *n_valid,
                   double *dH, double *dW) {
    return oracle_cce_full(H, W, labels, N, D, V, ignore_index, eps, lam, 0, dloss, NULL, loss, lse, n_valid,
                           dH, dW);
}

/* The unregularised loss (eps = lam = 0). */
int oracle_cce(const double *H, const double *W, const int32_t *labels,
               int64_t N, int64_t D, int64_t V, int32_t ignore_index,
               double dloss, double *loss, double *lse, int64_t *n_valid,
               double *dH, double *dW) {
    return oracle_cce_reg(H, W, labels, N, D, V, ignore_index, 0.0, 0.0, dloss, loss, lse, n_valid, dH, dW);
}

/*
 * The dlogits matrix itself, G[N,V] (fp64), for tiny problems only: the
 * quantity the paper's backward forms chunk by chunk.  Ignored
 * rows are all-zero.
 */
int oracle_dlogits_reg(const double *H, const double *W, const int32_t *labels,
                       int64_t N, int64_t D, int64_t V, int32_t ignore_index,
                       double eps, double lam, double dloss, double *G) {
    int64_t nv = 0;
    int rc = oracle_validate(labels, N, V, ignore_index, &nv);
    if (rc) return rc;
    double scale = nv > 0 ? dloss / (double)nv : 0.0;
    double *h = (double *)malloc((size_t)D * sizeof(double));
    double *z = (double *)malloc((size_t)V * sizeof(double));
    if (!h || !z) { free(h); free(z); return ORACLE_ERR_NOMEM; }
    for (int64_t n = 0; n < N; ++n) {
        int32_t y = labels[n];
        if (y == ignore_index) {
            for (int64_t v = 0; v < V; ++v) G[n * V + v] = 0.0;
            continue;
        }
        for (int64_t d = 0; d < D; ++d) h[d] = H[n * D + d];
        logit_row(h, W, D, V, z);
        double l = lse_two_pass(z, V);
        for (int64_t v = 0; v < V; ++v)
            G[n * V + v] = scale * row_grad(z[v], l, v == y, eps, lam, V);
    }
    free(h);
    free(z);
    return ORACLE_OK;
}

int oracle_dlogits(const double *H, const double *W, const int32_t *labels,
                   int64_t N, int64_t D, int64_t V, int32_t ignore_index,
                   double dloss, double *G) {
    return oracle_dlogits_reg(H, W, labels, N, D, V, ignore_index, 0.0, 0.0, dloss, G);
}

/*
 * Sampled rows (for parity at full size): for each listed row index r (which
 * must be a valid row), lse[r], z_y[r] and -- if dH_rows != NULL -- the dH row
 * scale * sum_v (exp(z-lse) - 1[v==y]) W[v,:], with scale = dloss / n_valid
 * passed in by the caller (n_valid is a count over the whole batch).
 * Outputs are indexed by position in `rows`.
 */
int oracle_cce_rows(const double *H, const double *W, const int32_t *labels,
                    int64_t D, int64_t V, double scale,
                    const int64_t *rows, int64_t nrows,
                    double *lse_out, double *zy_out, double *dH_rows) {
    int nomem = 0, bad = 0;
#pragma omp parallel
    {
        double *h = (double *)malloc((size_t)D * sizeof(double));
        double *z = (double *)malloc((size_t)V * sizeof(double));
        if (!h || !z) {
#pragma omp atomic write
            nomem = 1;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < nrows; ++i) {
            if (!h || !z) continue;
            int64_t n = rows[i];
            int32_t y = labels[n];
            if (y < 0 || (int64_t)y >= V) {
#pragma omp atomic write
                bad = 1;
                continue;
            }
            for (int64_t d = 0; d < D; ++d) h[d] = H[n * D + d];
            logit_row(h, W, D, V, z);
            double l = lse_two_pass(z, V);
            lse_out[i] = l;
            zy_out[i] = z[y];
            if (dH_rows) {
                double *out = dH_rows + i * D;
                for (int64_t d = 0; d < D; ++d) out[d] = 0.0;
                for (int64_t v = 0; v < V; ++v) {
                    double g = scale * (exp(z[v] - l) - (v == y ? 1.0 : 0.0));
                    const double *w = W + v * D;
                    for (int64_t d = 0; d < D; ++d) out[d] += g * w[d];
                }
            }
        }
        free(h);
        free(z);
    }
    if (nomem) return ORACLE_ERR_NOMEM;
    return bad ? ORACLE_ERR_LABEL_RANGE : ORACLE_OK;
}

/*
 * Sampled vocabulary rows of dW (for parity at full size).  Needs lse[n] of
 * every valid row (computed by this oracle, e.g. via oracle_cce_rows over all
 * valid rows).  dW[v,:] = scale * sum_{valid n} (exp(z[n,v]-lse_n) - 1[v==y_n]) H[n,:].
 */
int oracle_dW_rows(const double *H, const double *W, const int32_t *labels,
                   int64_t N, int64_t D, int32_t ignore_index, const double *lse,
                   double scale, const int64_t *vrows, int64_t nv_rows,
                   double *dW_rows) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < nv_rows; ++i) {
        int64_t v = vrows[i];
        const double *w = W + v * D;
        double *out = dW_rows + i * D;
        for (int64_t d = 0; d < D; ++d) out[d] = 0.0;
        for (int64_t n = 0; n < N; ++n) {
            int32_t y = labels[n];
            if (y == ignore_index) continue;
            const double *hr = H + n * D;
            double zv = 0.0;
            for (int64_t d = 0; d < D; ++d) zv += hr[d] * w[d];
            double g = scale * (exp(zv - lse[n]) - (v == y ? 1.0 : 0.0));
            for (int64_t d = 0; d < D; ++d) out[d] += g * hr[d];
        }
    }
    return ORACLE_OK;
}

/*
 * Online softmax over a sequence, exactly as Def. "Online Softmax"
 * (P:511-519): m_i = max(m_{i-1}, x_i); d_i = d_{i-1} e^{m_{i-1}-m_i} + e^{x_i-m_i},
 * with the empty state m_0 = -inf, d_0 = 0 and e^{-inf} = 0 (S:37 ledger).
 * Returns log d_n + m_n (Theorem).
 */
double oracle_online_lse(const double *x, int64_t n) {
    double m = -INFINITY, d = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double mn = x[i] > m ? x[i] : m;
        double scale_old = (m == -INFINITY) ? 0.0 : exp(m - mn);
        d = d * scale_old + exp(x[i] - mn);
        m = mn;
    }
    return log(d) + m;
}

/*
 * Per-shard partial statistics for vocabulary-sharded parity:
 * for valid row n, over the local vocabulary slice W_local = W[off : off+V_local]
 * (global ids), m = max_v z, d = sum_v exp(z - m), z_y = z[y - off] if this shard
 * owns y_n else 0.  Empty shards give (m=-inf, d=0, z_y=0).  Ignored rows give
 * (-inf, 0, 0).  This is the per-shard instance of the two-pass definition;
 * combining shards is done by the caller (tests) following P:521-541.
 */
int oracle_partial_stats(const double *H, const double *W_local,
                         const int32_t *labels, int64_t N, int64_t D,
                         int64_t V_local, int64_t vocab_offset, int32_t ignore_index,
                         double *m_out, double *d_out, double *zy_out) {
    int nomem = 0;
#pragma omp parallel
    {
        double *h = (double *)malloc((size_t)D * sizeof(double));
        double *z = (double *)malloc((size_t)(V_local > 0 ? V_local : 1) * sizeof(double));
        if (!h || !z) {
#pragma omp atomic write
            nomem = 1;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t n = 0; n < N; ++n) {
            if (!h || !z) continue;
            int32_t y = labels[n];
            m_out[n] = -INFINITY; d_out[n] = 0.0; zy_out[n] = 0.0;
            if (y == ignore_index || V_local == 0) continue;
            for (int64_t d = 0; d < D; ++d) h[d] = H[n * D + d];
            logit_row(h, W_local, D, V_local, z);
            double m = -INFINITY;
            for (int64_t v = 0; v < V_local; ++v) if (z[v] > m) m = z[v];
            double s = 0.0;
            for (int64_t v = 0; v < V_local; ++v) s += exp(z[v] - m);
            m_out[n] = m; d_out[n] = s;
            int64_t yl = (int64_t)y - vocab_offset;
            if (yl >= 0 && yl < V_local) zy_out[n] = z[yl];
        }
        free(h);
        free(z);
    }
    return nomem ? ORACLE_ERR_NOMEM : ORACLE_OK;
}

/*
 * One AdamW step in the order of the paper's fused kernel,
 * Alg. "Fused AdamW Triton Kernel (Complete)", which is Def. AdamW
 * with a pre-supplied clipping coefficient:
 *   g  = g * clip_coef
 *   th = th * (1 - lr * wd)                       decoupled weight decay
 *   m  = b1 m + (1 - b1) g ;  v = b2 v + (1 - b2) g^2
 *   th = th - lr * (m / bc1) / (sqrt(v / bc2) + eps),   bc_i = 1 - b_i^t (host)
 * In place over n elements, fp64.
 */
void oracle_adamw_step(double *theta, const double *grad, double *m, double *v, int64_t n,
                       double lr, double b1, double b2, double eps, double wd, double clip_coef,
                       double bc1, double bc2) {
    for (int64_t i = 0; i < n; ++i) {
        double g = grad[i] * clip_coef;
        double th = theta[i] * (1.0 - lr * wd);
        m[i] = b1 * m[i] + (1.0 - b1) * g;
        v[i] = b2 * v[i] + (1.0 - b2) * g * g;
        double mh = m[i] / bc1;
        double vh = v[i] / bc2;
        theta[i] = th - lr * (mh / (sqrt(vh) + eps));
    }
}

/*
 * RMSNorm prologue ("the final-RMSNorm prologue, the step before
 * the path: norm H on load, with rstd cached").  Def. Root Mean Square Layer
 * Normalization:
 *   r_n    = sqrt((1/D) sum_i x[n,i]^2 + eps),   rstd_n = 1 / r_n   (Alg. P:722-724)
 *   y[n,i] = x[n,i] * rstd_n * gamma_i                                   (Alg. P:725)
 * In place of nothing: y, rstd out; fp64.
 */
void oracle_rmsnorm_fwd(const double *x, const double *gamma, int64_t N, int64_t D, double eps, double *y,
                        double *rstd) {
    for (int64_t n = 0; n < N; ++n) {
        const double *xr = x + n * D;
        double ss = 0.0;
        for (int64_t i = 0; i < D; ++i) ss += xr[i] * xr[i];
        const double r = sqrt(ss / (double)D + eps);
        rstd[n] = 1.0 / r;
        for (int64_t i = 0; i < D; ++i) y[n * D + i] = xr[i] * rstd[n] * gamma[i];
    }
}

/*
 * RMSNorm backward: the exact gradient of Def. RMSNorm.  With
 * xbar = x rstd and dy the upstream gradient of y:
 *   dx[n,k]  = rstd_n (gamma_k dy[n,k] - xbar[n,k] (1/D) sum_i dy[n,i] gamma_i xbar[n,i])
 *   dgamma_k = sum_n dy[n,k] xbar[n,k]                        (Alg. P:745, summed over rows)
 * This is Prop. "RMSNorm Backward Pass" and the Alg. with two
 * garbles corrected (reading R18): the Prop. drops the 1/D of the mean and
 * both apply gamma_k to the second term as well.  Differentiating y_i = x_i gamma_i / r,
 * r = sqrt(mean x^2 + eps): dy_i/dx_k = gamma_i delta_ik / r - x_i gamma_i x_k / (D r^3),
 * which gives the line above.  Rows with skip[n] != 0 (ignored rows, never read by the
 * CE path) get dx = 0 and add nothing to dgamma.  fp64, fixed order.
 */
void oracle_rmsnorm_bwd(const double *dy, const double *x, const double *gamma, const double *rstd,
                        const int32_t *skip, int64_t N, int64_t D, double *dx, double *dgamma) {
    for (int64_t i = 0; i < D; ++i) dgamma[i] = 0.0;
    for (int64_t n = 0; n < N; ++n) {
        double *dxr = dx + n * D;
        if (skip && skip[n]) {
            for (int64_t i = 0; i < D; ++i) dxr[i] = 0.0;
            continue;
        }
        const double *xr = x + n * D, *dyr = dy + n * D;
        const double rs = rstd[n];
        double c1 = 0.0;
        for (int64_t i = 0; i < D; ++i) c1 += dyr[i] * gamma[i] * (xr[i] * rs);
        c1 /= (double)D;
        for (int64_t k = 0; k < D; ++k) dxr[k] = rs * (gamma[k] * dyr[k] - (xr[k] * rs) * c1);
        for (int64_t k = 0; k < D; ++k) dgamma[k] += dyr[k] * (xr[k] * rs);
    }
}

/* fp64 -> bf16 bit pattern: fp64 -> fp32 (RNE), then fp32 -> bf16 (RNE, ties to the even
 * bf16 pattern; overflow rounds to inf, NaN stays a quiet NaN of the same sign).  The CE
 * path consumes bf16 H formed in fp32 arithmetic (reading R18), hence the two
 * steps.  Pinned by tests/test_oracle_pins.py::test_to_bf16_* (exact rational rounding
 * and torch's float32 -> bfloat16 cast on ties, +-1 ulp, subnormals, the max, NaN). */
void oracle_to_bf16(const double *a, int64_t n, uint16_t *out) {
    for (int64_t i = 0; i < n; ++i) {
        const float f = (float)a[i];
        uint32_t u;
        memcpy(&u, &f, 4);
        if ((u & 0x7FFFFFFFu) > 0x7F800000u) {   /* NaN: keep the sign, quiet */
            out[i] = (uint16_t)((u >> 16) | 0x0040u);
            continue;
        }
        u += 0x7FFFu + ((u >> 16) & 1u);
        out[i] = (uint16_t)(u >> 16);
    }
}
