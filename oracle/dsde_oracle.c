/*
 * dsde_oracle.c — plain, slow, obviously-correct CPU oracle for the DSDE
 * speculative-verification hot path (arXiv 2509.01083, "DSDE").
 *
 * ======================================================================
 * TEST INFRASTRUCTURE. This file is NOT part of the product. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load liboracle.so. It shares no code, header, table or helper
 * with the CUDA path under paper_2509_01083_b200/csrc/, and neither side
 * includes or links the other.
 * ======================================================================
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n (the reference
 * texts), SURVEY §8(c) = the reading of the paper this oracle follows
 * (decisions D1..D17, listed again in DESIGN.md).
 *
 * Arithmetic: IEEE fp64 throughout. bf16/fp32 logits are converted to
 * double exactly (a bf16 pattern b is the fp32 pattern b<<16). Every
 * reduction is a sequential left-to-right loop in ascending token order;
 * there is no blocking, fusion, online softmax or reordering.
 *
 * Parts:
 *   C0  Philox4x32-10 (Salmon et al., SC'11; the Random123 reference
 *       algorithm) and the 53-bit uniform map res53.         [D6]
 *   C1  verify: softmax, KL(p||q), accept test min(1, p/q), first
 *       rejection, residual max(0,p-q) / bonus inverse-CDF sample.
 *       P:163; S:125-127 (standard speculative sampling);
 *       D1 (KL direction), D3, D5, D7.
 *   C2  signal: KLD history ring (Fig.5), calibration Eq.1
 *       (P:181), SF Eq.3, weights Eq.5, weighted mean
 *       Eq.6, weighted variance Eq.7, WVIR Eq.4,
 *       conditional prediction Eq.8 / Eq.2.
 *   C3  cap: Eq.9-11: cap = arithmetic mean of predictions,
 *       integerised by exact round-half-even (D14); next = min(SL^, cap,
 *       budget).
 *
 * Parity pins: see tests/test_oracle_*.py. Every function here has at
 * least one pin that does not re-type its formula (closed forms,
 * brute-force distribution tests, library routines, KAT vectors).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ */
/* C0. Philox4x32-10 and res53                                          */
/* ------------------------------------------------------------------ */

/* One Philox round (Salmon et al. 2011, Random123 philox4x32round). */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n[4];
    n[0] = hi1 ^ c[1] ^ k[0];
    n[1] = lo1;
    n[2] = hi0 ^ c[3] ^ k[1];
    n[3] = lo0;
    memcpy(c, n, sizeof(n));
}

/* Philox4x32 with 10 rounds; the key is bumped by the Weyl constants
 * between rounds (9 bumps for 10 rounds). */
OR_EXPORT void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                                    uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k[0] += 0x9E3779B9u;
            k[1] += 0xBB67AE85u;
        }
        philox_round(c, k);
    }
    memcpy(out, c, sizeof(c));
}

/* res53(a, b) = ((a >> 5) * 2^26 + (b >> 6)) * 2^-53, a double in [0,1). */
OR_EXPORT double oracle_res53(uint32_t a, uint32_t b) {
    return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

/* D6: the two uniforms of one (sequence, position): Philox keyed by the
 * 64-bit seed (key = (lo32, hi32)), counter 0; words 0-1 -> u_acc,
 * words 2-3 -> u_smp. */
OR_EXPORT void oracle_uniforms(uint64_t seed, double* u_acc, double* u_smp) {
    const uint32_t ctr[4] = {0u, 0u, 0u, 0u};
    const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t w[4];
    oracle_philox4x32_10(ctr, key, w);
    *u_acc = oracle_res53(w[0], w[1]);
    *u_smp = oracle_res53(w[2], w[3]);
}

/* D23: the uniforms of proposal j >= 1 of a recovery draw: Philox keyed by the
 * slot's seed, counter (j, 0, 0, 0); words 0-1 -> u_prop (the proposal's
 * inverse CDF over p), words 2-3 -> u_keep (its accept test). Counter 0 is
 * D6's (u_acc, u_smp). */
OR_EXPORT void oracle_proposal_uniforms(uint64_t seed, uint32_t j, double* u_prop, double* u_keep) {
    const uint32_t ctr[4] = {j, 0u, 0u, 0u};
    const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t w[4];
    oracle_philox4x32_10(ctr, key, w);
    *u_prop = oracle_res53(w[0], w[1]);
    *u_keep = oracle_res53(w[2], w[3]);
}

/* ------------------------------------------------------------------ */
/* C1. Verify                                                           */
/* ------------------------------------------------------------------ */

/* dtype codes of the oracle's own API: 0 = fp32 logits, 1 = bf16 logits. */
static double logit_at(const void* base, int dtype, int64_t row, int64_t ld, int64_t v) {
    if (dtype == 0) {
        const float* p = (const float*)base;
        return (double)p[row * ld + v];
    }
    const uint16_t* p = (const uint16_t*)base;
    const uint32_t bits = (uint32_t)p[row * ld + v] << 16;
    float f;
    memcpy(&f, &bits, sizeof(f));
    return (double)f;
}

static void load_row(double* dst, const void* base, int dtype, int64_t row, int64_t ld, int V) {
    for (int v = 0; v < V; ++v) dst[v] = logit_at(base, dtype, row, ld, v);
}

/* log-sum-exp of a row by the plain two-pass definition:
 * m = max_v x_v ; lse = m + log(sum_v exp(x_v - m)). */
static double row_lse(const double* x, int V) {
    double m = x[0];
    for (int v = 1; v < V; ++v)
        if (x[v] > m) m = x[v];
    double s = 0.0;
    for (int v = 0; v < V; ++v) s += exp(x[v] - m);
    return m + log(s);
}

/* KL(p||q) = sum_v p_v (log p_v - log q_v), p = softmax(t), q = softmax(d);
 * terms with p_v == 0 contribute 0 (D1: target relative to draft). */
OR_EXPORT double oracle_row_kld(int V, const double* t, const double* d) {
    const double lt = row_lse(t, V), ld = row_lse(d, V);
    double kl = 0.0;
    for (int v = 0; v < V; ++v) {
        const double logp = t[v] - lt;
        const double p = exp(logp);
        if (p == 0.0) continue;
        kl += p * (logp - (d[v] - ld));
    }
    return kl;
}

/* Draft entropy H(q) = -sum_v q_v log q_v, q = softmax(d) (SURVEY §8(f) f2:
 * the paper's optional entropy signal next to the KLD); terms
 * with q_v == 0 contribute 0. */
OR_EXPORT double oracle_row_entropy(int V, const double* d) {
    const double ld = row_lse(d, V);
    double h = 0.0;
    for (int v = 0; v < V; ++v) {
        const double logq = d[v] - ld;
        const double q = exp(logq);
        if (q == 0.0) continue;
        h -= q * logq;
    }
    return h;
}

/* H(q) of every draft row of a batch (rows in the layout of oracle_verify). */
OR_EXPORT void oracle_draft_entropy(int n_rows, int V, int dtype, const void* draft, int64_t ld_d,
                                    double* out) {
    double* d = (double*)malloc(sizeof(double) * (size_t)V);
    for (int r = 0; r < n_rows; ++r) {
        load_row(d, draft, dtype, r, ld_d, V);
        out[r] = oracle_row_entropy(V, d);
    }
    free(d);
}

/* log r = log p(x) - log q(x) (S:125 acceptance ratio p(x)/q(x)). */
OR_EXPORT double oracle_row_log_ratio(int V, const double* t, const double* d, int x) {
    return (t[x] - row_lse(t, V)) - (d[x] - row_lse(d, V));
}

/* Inverse-CDF draw over non-negative weights w[0..V) (D7): the smallest v
 * with C_v = sum_{u<=v} w_u  >  u * R, R = sum_u w_u, summed sequentially
 * in ascending token order. Returns -1 if R == 0. lo/hi receive
 * C_{v-1}/R and C_v/R of the chosen token (for the tie bands of D16). */
static int inverse_cdf(const double* w, int V, double u, double* R_out, double* lo, double* hi) {
    double R = 0.0;
    for (int v = 0; v < V; ++v) R += w[v];
    *R_out = R;
    if (!(R > 0.0)) return -1;
    const double target = u * R;
    double c = 0.0;
    int last_pos = -1;
    for (int v = 0; v < V; ++v) {
        const double prev = c;
        c += w[v];
        if (w[v] > 0.0) last_pos = v;
        if (c > target) {
            *lo = prev / R;
            *hi = c / R;
            return v;
        }
    }
    /* Unreachable in exact arithmetic (u < 1 => u*R < R = C_{V-1}); kept so a
     * rounding corner can never emit a zero-mass token. */
    *lo = 1.0;
    *hi = 1.0;
    return last_pos;
}

/* Flags written per slot (oracle's own codes). */
#define OR_FLAG_ACCEPT_TIE 1   /* |u_acc - min(1,r)| < 1e-6 at this position */
#define OR_FLAG_SAMPLE_TIE 2   /* |u_smp - boundary| < 1e-6 for the drawn token */
#define OR_FLAG_FALLBACK 4     /* residual mass R == 0: sampled from p instead */
#define OR_FLAG_PROPOSAL_FALLBACK 8  /* D23: none of the OR_PROPOSALS proposals kept: D7 draw */

/* D23: proposals of a recovery draw before the D7 inverse CDF takes over. */
#define OR_PROPOSALS 256

typedef struct {
    int V, dtype;
    const int32_t* cu_sl;
    const int32_t* draft_tokens;
    const void* tl;
    int64_t ld_t;
    const void* dl;
    int64_t ld_d;
    const uint64_t* seeds;
    int32_t* accepted_len;   /* [B] */
    int32_t* emitted;        /* [sum k + B] */
    double* kld;             /* [sum k] */
    double* log_ratio;       /* [sum k]  log p(x_j) - log q(x_j)   */
    double* u_acc;           /* [sum k + B] */
    double* u_smp;           /* [sum k + B] */
    double* samp_diag;       /* [B][3] : R, lo, hi of the final draw */
    int32_t* flags;          /* [sum k + B] */
    int greedy;              /* 1: T = 0 verification (f1) */
    const double* temps;     /* [B] per-sequence temperature (f1) or NULL = 1; T_i == 0: greedy */
    int resample;            /* recovery draw: 0 = D23 proposals from p, 1 = D7 inverse CDF (default) */
    int b0, b1;              /* sequence range for this worker */
    int status;
} verify_job;

/* argmax of a row, smallest index among equal maxima (D18) */
static int row_argmax(const double* x, int V) {
    int best = 0;
    for (int v = 1; v < V; ++v)
        if (x[v] > x[best]) best = v;
    return best;
}

/* Verification of one sequence i (S:125-127 / P:260):
 *   for j in [0,k): KL_j (all positions, D3), r_j = p(x_j)/q(x_j),
 *   acc_j = u_acc(i,j) < min(1, r_j) (D5);
 *   a = first j with !acc_j, else k (prefix shape S:111);
 *   a <  k: recovery token ~ normalize(max(0, p - q)) on row a;
 *   a == k: bonus token ~ p on target row k;
 *   emitted = x_0..x_{a-1}, token, then DSDE pad (-1) up to slot k. */
/* Logit row (sequence i) as the method sees it: the stored value divided by
 * the sequence's temperature T_i > 0 (p = softmax(t / T), q = softmax(d / T):
 * sampling at temperature T; D20). T_i == 0 (greedy) and no
 * temperatures use the stored values (T = 1 semantics for the KLD, D18).
 * Masked tokens (-inf logits, top-k / top-p, D21) stay -inf. */
static void load_row_t(double* dst, const verify_job* J, const void* base, int64_t row, int64_t ld, int i) {
    load_row(dst, base, J->dtype, row, ld, J->V);
    if (J->temps && J->temps[i] > 0.0)
        for (int v = 0; v < J->V; ++v) dst[v] = dst[v] / J->temps[i];
}

/* a row with no finite logit (everything masked) or a +inf / NaN logit is not
 * a distribution */
static int row_ok(const double* x, int V) {
    int fin = 0;
    for (int v = 0; v < V; ++v) {
        if (isnan(x[v]) || x[v] == INFINITY) return 0;
        if (x[v] > -INFINITY) fin = 1;
    }
    return fin;
}

static int verify_one(verify_job* J, int i, double* t, double* d, double* w) {
    const int V = J->V;
    const int32_t base = J->cu_sl[i];
    const int k = J->cu_sl[i + 1] - base;
    if (k < 1) return -1;
    const int greedy = J->greedy || (J->temps && J->temps[i] == 0.0);
    const int64_t trow0 = (int64_t)base + i; /* target row of (i, j) = cu_sl[i] + i + j */
    const int64_t slot0 = (int64_t)base + i; /* output slot of (i, j), j in [0, k]     */
    int a = k;
    for (int j = 0; j < k; ++j) {
        const int x = J->draft_tokens[base + j];
        if (x < 0 || x >= V) return -1;
        load_row_t(t, J, J->tl, trow0 + j, J->ld_t, i);
        load_row_t(d, J, J->dl, (int64_t)base + j, J->ld_d, i);
        if (!row_ok(t, V) || !row_ok(d, V)) return -1;
        if (d[x] == -INFINITY) return -1; /* x ~ q: a token the draft masked cannot be drafted (D21) */
        const double kl = oracle_row_kld(V, t, d);
        const double lr = oracle_row_log_ratio(V, t, d, x);
        double ua, us;
        oracle_uniforms(J->seeds[slot0 + j], &ua, &us);
        J->kld[base + j] = kl;
        J->log_ratio[base + j] = lr;
        J->u_acc[slot0 + j] = ua;
        J->u_smp[slot0 + j] = us;
        J->flags[slot0 + j] = 0;
        if (greedy) {
            /* T = 0: accept iff x_j is the target argmax */
            if (a == k && x != row_argmax(t, V)) a = j;
            continue;
        }
        const double r = exp(lr);
        const double pacc = r < 1.0 ? r : 1.0;
        if (fabs(ua - pacc) < 1e-6) J->flags[slot0 + j] |= OR_FLAG_ACCEPT_TIE;
        if (a == k && !(ua < pacc)) a = j;
    }
    {
        double ua, us;
        oracle_uniforms(J->seeds[slot0 + k], &ua, &us);
        J->u_acc[slot0 + k] = ua;
        J->u_smp[slot0 + k] = us;
        J->flags[slot0 + k] = 0;
    }
    /* The draw of the final token uses u_smp of slot a (recovery at the
     * first rejected position, or the bonus position a == k) (D6). */
    const double u = J->u_smp[slot0 + a];
    int tok, stie = 0;
    double R = 0.0, lo = 0.0, hi = 0.0;
    if (greedy) {
        /* the target argmax of row a (recovery, a < k) or of the bonus row k */
        load_row_t(t, J, J->tl, trow0 + a, J->ld_t, i);
        if (!row_ok(t, V)) return -1;
        tok = row_argmax(t, V);
    } else if (a < k) {
        load_row_t(t, J, J->tl, trow0 + a, J->ld_t, i);
        load_row_t(d, J, J->dl, (int64_t)base + a, J->ld_d, i);
        const double lt = row_lse(t, V), ld = row_lse(d, V);
        int kept = 0;
        tok = -1;
        if (J->resample == 0) {
            /* D23: propose v ~ p by the inverse CDF (D7) with u_prop of
             * proposal j, keep it with probability max(0, p_v - q_v) / p_v
             * (u_keep < that); the first kept proposal is the recovery token.
             * A kept proposal is distributed as normalize(max(0, p - q))
             * (P(v kept) = p_v max(0, p_v - q_v) / p_v). */
            for (int v = 0; v < V; ++v) w[v] = exp(t[v] - lt);   /* p_v */
            for (uint32_t j = 1; j <= OR_PROPOSALS && !kept; ++j) {
                double up, uk;
                oracle_proposal_uniforms(J->seeds[slot0 + a], j, &up, &uk);
                const int v = inverse_cdf(w, V, up, &R, &lo, &hi);
                if (v < 0) break;
                if (fabs(up - lo) < 1e-6 || fabs(up - hi) < 1e-6) stie = 1;
                const double pv = w[v], qv = exp(d[v] - ld);
                const double keep = pv > qv ? (pv - qv) / pv : 0.0;
                if (fabs(uk - keep) < 1e-6) stie = 1;
                if (uk < keep) {
                    tok = v;
                    kept = 1;
                }
            }
            if (!kept) J->flags[slot0 + a] |= OR_FLAG_PROPOSAL_FALLBACK;
        }
        if (!kept) {
            /* D7: inverse CDF over rho_v = max(0, p_v - q_v) with u_smp */
            for (int v = 0; v < V; ++v) {
                const double pv = exp(t[v] - lt), qv = exp(d[v] - ld);
                w[v] = pv - qv > 0.0 ? pv - qv : 0.0;
            }
            tok = inverse_cdf(w, V, u, &R, &lo, &hi);
            if (tok < 0) { /* R == 0: fall back to p (D7) */
                for (int v = 0; v < V; ++v) w[v] = exp(t[v] - lt);
                tok = inverse_cdf(w, V, u, &R, &lo, &hi);
                J->flags[slot0 + a] |= OR_FLAG_FALLBACK;
            }
            if (fabs(u - lo) < 1e-6 || fabs(u - hi) < 1e-6) stie = 1;
        }
    } else {
        load_row_t(t, J, J->tl, trow0 + k, J->ld_t, i);
        if (!row_ok(t, V)) return -1;
        const double lt = row_lse(t, V);
        for (int v = 0; v < V; ++v) w[v] = exp(t[v] - lt);  /* p_v */
        tok = inverse_cdf(w, V, u, &R, &lo, &hi);
        if (fabs(u - lo) < 1e-6 || fabs(u - hi) < 1e-6) stie = 1;
    }
    if (stie) J->flags[slot0 + a] |= OR_FLAG_SAMPLE_TIE;
    J->samp_diag[3 * i + 0] = R;
    J->samp_diag[3 * i + 1] = lo;
    J->samp_diag[3 * i + 2] = hi;
    J->accepted_len[i] = a;
    for (int j = 0; j < a; ++j) J->emitted[slot0 + j] = J->draft_tokens[base + j];
    J->emitted[slot0 + a] = tok;
    for (int j = a + 1; j <= k; ++j) J->emitted[slot0 + j] = -1; /* reserved pad id */
    return 0;
}

static void* verify_worker(void* arg) {
    verify_job* J = (verify_job*)arg;
    double* t = (double*)malloc(sizeof(double) * (size_t)J->V);
    double* d = (double*)malloc(sizeof(double) * (size_t)J->V);
    double* w = (double*)malloc(sizeof(double) * (size_t)J->V);
    J->status = 0;
    if (!t || !d || !w) J->status = -2;
    for (int i = J->b0; i < J->b1 && J->status == 0; ++i)
        if (verify_one(J, i, t, d, w) != 0) J->status = -1;
    free(t);
    free(d);
    free(w);
    return NULL;
}

/* Batched verify over B sequences with ragged k_i (Ragged Q).
 * resample selects the recovery draw's reading: 0 = D23 (proposals from p),
 * 1 = D7 (inverse CDF over max(0, p - q), the default).
 * Layout: draft row of (i,j) = cu_sl[i]+j; target row of (i,j) =
 * cu_sl[i]+i+j for j in [0,k_i]; per-slot outputs (emitted, u_acc, u_smp,
 * flags) use the target-row index. nthreads <= 1 runs serially.
 * Returns 0, or -1 on invalid data (k < 1, token out of range). */
OR_EXPORT int oracle_verify_temp(int B, int V, int dtype, const int32_t* cu_sl,
                                 const int32_t* draft_tokens, const void* target_logits, int64_t ld_t,
                                 const void* draft_logits, int64_t ld_d, const uint64_t* seeds,
                                 int32_t* accepted_len, int32_t* emitted, double* kld,
                                 double* log_ratio, double* u_acc, double* u_smp, double* samp_diag,
                                 int32_t* flags, int nthreads, int greedy, const double* temps,
                                 int resample) {
    if (B < 1 || V < 2 || (dtype != 0 && dtype != 1) || (resample != 0 && resample != 1)) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > B) nthreads = B;
    verify_job* jobs = (verify_job*)calloc((size_t)nthreads, sizeof(verify_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) {
        free(jobs);
        free(th);
        return -2;
    }
    for (int n = 0; n < nthreads; ++n) {
        verify_job* J = &jobs[n];
        J->V = V;
        J->dtype = dtype;
        J->cu_sl = cu_sl;
        J->draft_tokens = draft_tokens;
        J->tl = target_logits;
        J->ld_t = ld_t;
        J->dl = draft_logits;
        J->ld_d = ld_d;
        J->seeds = seeds;
        J->accepted_len = accepted_len;
        J->emitted = emitted;
        J->kld = kld;
        J->log_ratio = log_ratio;
        J->u_acc = u_acc;
        J->u_smp = u_smp;
        J->samp_diag = samp_diag;
        J->flags = flags;
        J->greedy = greedy;
        J->temps = temps;
        J->resample = resample;
        J->b0 = (int)((int64_t)B * n / nthreads);
        J->b1 = (int)((int64_t)B * (n + 1) / nthreads);
    }
    int rc = 0;
    if (nthreads == 1) {
        verify_worker(&jobs[0]);
    } else {
        for (int n = 0; n < nthreads; ++n) pthread_create(&th[n], NULL, verify_worker, &jobs[n]);
        for (int n = 0; n < nthreads; ++n) pthread_join(th[n], NULL);
    }
    for (int n = 0; n < nthreads; ++n)
        if (jobs[n].status != 0) rc = jobs[n].status;
    free(jobs);
    free(th);
    return rc;
}

/* Global T = 0 (greedy = 1) or T = 1 (greedy = 0) verification. */
OR_EXPORT int oracle_verify_mode(int B, int V, int dtype, const int32_t* cu_sl,
                                 const int32_t* draft_tokens, const void* target_logits, int64_t ld_t,
                                 const void* draft_logits, int64_t ld_d, const uint64_t* seeds,
                                 int32_t* accepted_len, int32_t* emitted, double* kld,
                                 double* log_ratio, double* u_acc, double* u_smp, double* samp_diag,
                                 int32_t* flags, int nthreads, int greedy) {
    return oracle_verify_temp(B, V, dtype, cu_sl, draft_tokens, target_logits, ld_t, draft_logits, ld_d,
                              seeds, accepted_len, emitted, kld, log_ratio, u_acc, u_smp, samp_diag, flags,
                              nthreads, greedy, NULL, 1);
}

/* The rejection-sampling verification (the default, C1). */
OR_EXPORT int oracle_verify(int B, int V, int dtype, const int32_t* cu_sl, const int32_t* draft_tokens,
                            const void* target_logits, int64_t ld_t, const void* draft_logits,
                            int64_t ld_d, const uint64_t* seeds, int32_t* accepted_len,
                            int32_t* emitted, double* kld, double* log_ratio, double* u_acc,
                            double* u_smp, double* samp_diag, int32_t* flags, int nthreads) {
    return oracle_verify_mode(B, V, dtype, cu_sl, draft_tokens, target_logits, ld_t, draft_logits,
                              ld_d, seeds, accepted_len, emitted, kld, log_ratio, u_acc, u_smp,
                              samp_diag, flags, nthreads, 0);
}

/* ------------------------------------------------------------------ */
/* C2. Signal: calibration, SF, weighted variance, WVIR, SL prediction  */
/* ------------------------------------------------------------------ */

#define OR_MAX_WIN 256

typedef struct {
    double delta;       /* decay factor, Eq.5 (default 0.85)       */
    int n_short;        /* short window N = 10                    */
    int n_long;         /* long window  N = 30                    */
    int sl_min;         /* SL_min = 2                             */
    int sl_ceiling;     /* hard bound on SL_max (D17)                     */
    double epsilon;     /* 1e-6                                   */
    int calib_steps;    /* preliminary steps (D12 default 5)       */
    int calib_sl;       /* SL used while calibrating (D12 default 4)      */
    int window_unit;    /* 0 = per-token observations, 1 = per-step means (D8) */
    int cap_mode;       /* 0 = none (cap = max), 1 = mean / MSE (Eq.11)   */
    int entropy_mode;   /* 0 = KLD signal only; 1 = also the draft-entropy predictor (D22) */
    double entropy_gamma; /* gamma of the entropy bound alpha_H = 1 - sqrt(gamma H) (D22) */
} oracle_cfg;

typedef struct {
    double hist[OR_MAX_WIN]; /* most recent LAST; at most n_long kept          */
    int n_hist;
    int steps;               /* verification steps observed                     */
    int sl_a_max;            /* Eq.1 SL_A,max (accepted draft tokens, D12)      */
    double kld_sum;          /* for mu_KLD,pre                                  */
    long kld_cnt;
    double kld_max;          /* KLD_pre,max                                     */
    int sl_max;              /* calibrated SL_max (0 while calibrating)         */
} oracle_seq;

typedef struct {
    oracle_cfg cfg;
    int n;
    oracle_seq* seq;
} oracle_state;

/* Eq.5-7 literally, two-pass: values[0] is the most recent (i = 1),
 * alpha_i = delta^(i-1); mu_w = sum a_i x_i / sum a_i;
 * Var_w = sum a_i (x_i - mu_w)^2 / sum a_i. */
OR_EXPORT double oracle_weighted_variance(const double* values_recent_first, int N, double delta) {
    if (N < 1) return NAN;
    double sa = 0.0, sax = 0.0;
    for (int i = 1; i <= N; ++i) {
        const double a = pow(delta, (double)(i - 1));
        sa += a;
        sax += a * values_recent_first[i - 1];
    }
    const double mu = sax / sa;
    double sv = 0.0;
    for (int i = 1; i <= N; ++i) {
        const double a = pow(delta, (double)(i - 1));
        const double e = values_recent_first[i - 1] - mu;
        sv += a * e * e;
    }
    return sv / sa;
}

/* Eq.3: SF = exp(2 mu_last) - 1. */
OR_EXPORT double oracle_scale_factor(double mu_last) { return exp(2.0 * mu_last) - 1.0; }

/* Eq.1 with D11: raw = SL_A,max (1 + mu/(max + eps)); SL_max =
 * clamp(rint(raw), sl_min+1, sl_ceiling); SL_A,max == 0 -> sl_min+1.
 * rint() rounds half to even under the default rounding mode. */
OR_EXPORT int oracle_calibrate(int sl_a_max, double mu_pre, double kld_pre_max, int sl_min,
                               int sl_ceiling, double epsilon, double* raw_out) {
    const double raw = (double)sl_a_max * (1.0 + mu_pre / (kld_pre_max + epsilon));
    if (raw_out) *raw_out = raw;
    if (sl_a_max == 0) return sl_min + 1;
    double r = rint(raw);
    if (r < sl_min + 1) r = sl_min + 1;
    if (r > sl_ceiling) r = sl_ceiling;
    return (int)r;
}

/* Eq.8 (with Eq.2 in its first branch) + D11 rounding and clamp.
 * x_out receives the pre-round value (or sl_min for the second branch). */
OR_EXPORT int oracle_predict_sl(double penalty, int sl_max, int sl_min, double* x_out) {
    double x;
    if (penalty <= 1.0)
        x = (1.0 - penalty) * (double)(sl_max - sl_min) + (double)sl_min;
    else
        x = (double)sl_min;
    if (x_out) *x_out = x;
    double r = rint(x);
    if (r < sl_min) r = sl_min;
    if (r > sl_max) r = sl_max;
    return (int)r;
}

OR_EXPORT oracle_state* oracle_state_new(const oracle_cfg* cfg, int n) {
    if (!cfg || n < 1 || cfg->n_long > OR_MAX_WIN || cfg->n_short >= cfg->n_long) return NULL;
    oracle_state* s = (oracle_state*)calloc(1, sizeof(oracle_state));
    if (!s) return NULL;
    s->cfg = *cfg;
    s->n = n;
    s->seq = (oracle_seq*)calloc((size_t)n, sizeof(oracle_seq));
    if (!s->seq) {
        free(s);
        return NULL;
    }
    return s;
}

OR_EXPORT void oracle_state_free(oracle_state* s) {
    if (!s) return;
    free(s->seq);
    free(s);
}

OR_EXPORT void oracle_state_reset(oracle_state* s, const int32_t* slots, int n) {
    for (int i = 0; i < n; ++i) memset(&s->seq[slots[i]], 0, sizeof(oracle_seq));
}

static void hist_append(oracle_seq* q, int n_long, double x) {
    if (q->n_hist == n_long) { /* evict the oldest (ring semantics) */
        memmove(q->hist, q->hist + 1, sizeof(double) * (size_t)(n_long - 1));
        q->n_hist--;
    }
    q->hist[q->n_hist++] = x;
}

/* Observe one verification step of B sequences and predict SL^ for each.
 * diag (optional) [B][8]: mu_last, sf, var_short, var_long, wvir, penalty,
 * x (pre-round SL^), sl_max. Calibrating sequences (D12) return calib_sl
 * and report their flag in calibrating[i] (1) — they are not capped and
 * do not enter the cap mean. */
/* The draft-entropy predictor ("KLD variance (optionally
 * combined with entropy)"; the entropy early-stopping bound of AdaEDL,
 * P:135), reading D22: with H the mean draft entropy of the step's positions,
 * alpha_H = max(0, 1 - sqrt(gamma H)) bounds the per-token acceptance from
 * below, and SL_H maps it to [SL_min, SL_max] as Eq.8 maps 1 - penalty:
 * SL_H = clamp(rint(alpha_H (SL_max - SL_min) + SL_min)). x_out: pre-round value. */
OR_EXPORT int oracle_entropy_sl(double h_mean, double gamma, int sl_max, int sl_min, double* x_out) {
    double a = 1.0 - sqrt(gamma * h_mean);
    if (a < 0.0) a = 0.0;
    const double x = a * (double)(sl_max - sl_min) + (double)sl_min;
    if (x_out) *x_out = x;
    double r = rint(x);
    if (r < sl_min) r = sl_min;
    if (r > sl_max) r = sl_max;
    return (int)r;
}

/* entropy (optional, [sum k]): the draft entropy of every draft position;
 * with cfg.entropy_mode = 1 the post-calibration prediction is
 * min(SL^ of Eq.8, SL_H) (D22). */
OR_EXPORT int oracle_update_signal_ent(oracle_state* s, int B, const int32_t* slots,
                                       const int32_t* cu_sl, const double* kld,
                                       const int32_t* accepted_len, const double* entropy,
                                       int32_t* sl_hat, int32_t* calibrating, double* diag) {
    const oracle_cfg* c = &s->cfg;
    for (int i = 0; i < B; ++i) {
        oracle_seq* q = &s->seq[slots[i]];
        const int k = cu_sl[i + 1] - cu_sl[i];
        if (k < 1) return -1;
        const double* kl = kld + cu_sl[i];
        /* mu_KLD,last: mean of the KLDs of the most recent step. */
        double sum = 0.0;
        for (int j = 0; j < k; ++j) sum += kl[j];
        const double mu_last = sum / (double)k;
        /* Fig.5: append this step's KLDs to the history window (D8). */
        if (c->window_unit == 0)
            for (int j = 0; j < k; ++j) hist_append(q, c->n_long, kl[j]);
        else
            hist_append(q, c->n_long, mu_last);
        q->steps++;
        /* No calibration configured: SL_max is the hard ceiling (D17). */
        if (c->calib_steps < 1 && q->sl_max == 0) q->sl_max = c->sl_ceiling;
        /* Calibration phase, Eq.1. */
        if (q->steps <= c->calib_steps) {
            if (accepted_len[i] > q->sl_a_max) q->sl_a_max = accepted_len[i];
            for (int j = 0; j < k; ++j) {
                q->kld_sum += kl[j];
                q->kld_cnt++;
                if (kl[j] > q->kld_max) q->kld_max = kl[j];
            }
            if (q->steps == c->calib_steps) {
                const double mu_pre = q->kld_sum / (double)q->kld_cnt;
                q->sl_max = oracle_calibrate(q->sl_a_max, mu_pre, q->kld_max, c->sl_min,
                                             c->sl_ceiling, c->epsilon, NULL);
            }
        }
        /* Windows: last min(n, n_short) and min(n, n_long) observations,
         * most recent first (i = 1 is the most recent). */
        double recent[OR_MAX_WIN];
        for (int m = 0; m < q->n_hist; ++m) recent[m] = q->hist[q->n_hist - 1 - m];
        double var_s = NAN, var_l = NAN, wvir;
        if (q->n_hist < c->n_short) {
            wvir = 1.0; /* warm-up (D9) */
        } else {
            var_s = oracle_weighted_variance(recent, c->n_short, c->delta);
            var_l = oracle_weighted_variance(recent, q->n_hist, c->delta);
            wvir = (var_l < 1e-12) ? 1.0 : var_s / var_l; /* Eq.4; flat-history guard D10 */
        }
        const double sf = oracle_scale_factor(mu_last);
        const double penalty = sf * wvir;
        double x = NAN;
        int calib = q->steps < c->calib_steps;
        int out;
        if (calib) {
            out = c->calib_sl;
        } else {
            out = oracle_predict_sl(penalty, q->sl_max, c->sl_min, &x);
            if (c->entropy_mode == 1 && entropy) {
                double hs = 0.0;
                for (int j = 0; j < k; ++j) hs += entropy[cu_sl[i] + j];
                const int sl_h = oracle_entropy_sl(hs / (double)k, c->entropy_gamma, q->sl_max, c->sl_min, NULL);
                if (sl_h < out) out = sl_h;
            }
        }
        sl_hat[i] = out;
        if (calibrating) calibrating[i] = calib;
        if (diag) {
            double* g = diag + 8 * (size_t)i;
            g[0] = mu_last;
            g[1] = sf;
            g[2] = var_s;
            g[3] = var_l;
            g[4] = wvir;
            g[5] = penalty;
            g[6] = x;
            g[7] = (double)q->sl_max;
        }
    }
    return 0;
}

OR_EXPORT int oracle_update_signal(oracle_state* s, int B, const int32_t* slots,
                                   const int32_t* cu_sl, const double* kld,
                                   const int32_t* accepted_len, int32_t* sl_hat,
                                   int32_t* calibrating, double* diag) {
    return oracle_update_signal_ent(s, B, slots, cu_sl, kld, accepted_len, NULL, sl_hat, calibrating, diag);
}

/* ------------------------------------------------------------------ */
/* C3. Cap                                                              */
/* ------------------------------------------------------------------ */

/* Eq.11: cap = (1/N) sum SL^_i over the N non-calibrating sequences,
 * integerised by exact round-half-even on the rational sum/N (D14).
 * cap_mode 0 (no cap): cap = max SL^_i. With N == 0 the cap is sl_ceiling.
 * next_sl_i = calibrating ? calib_sl : min(SL^_i, cap); then min(., budget_i)
 * when a budget is given. */
OR_EXPORT int oracle_next_sl(const oracle_cfg* c, int B, const int32_t* sl_hat,
                             const int32_t* calibrating, const int32_t* budget,
                             int32_t* next_sl, int32_t* cap_out) {
    long long sum = 0, n = 0;
    int mx = 0;
    for (int i = 0; i < B; ++i) {
        if (calibrating[i]) continue;
        sum += sl_hat[i];
        n += 1;
        if (sl_hat[i] > mx) mx = sl_hat[i];
    }
    int cap;
    if (n == 0) {
        cap = c->sl_ceiling;
    } else if (c->cap_mode == 0) {
        cap = mx;
    } else {
        long long q = sum / n, r = sum % n; /* sum >= 0 */
        if (2 * r > n || (2 * r == n && (q & 1))) q += 1;
        cap = (int)q;
    }
    *cap_out = cap;
    for (int i = 0; i < B; ++i) {
        int v = calibrating[i] ? c->calib_sl : (sl_hat[i] < cap ? sl_hat[i] : cap);
        if (budget && budget[i] < v) v = budget[i];
        next_sl[i] = v;
    }
    return 0;
}

/* Convenience for multi-rank partition tests: the exact (sum, n) partial. */
OR_EXPORT void oracle_cap_partial(int B, const int32_t* sl_hat, const int32_t* calibrating,
                                  long long* sum, long long* n) {
    *sum = 0;
    *n = 0;
    for (int i = 0; i < B; ++i) {
        if (calibrating[i]) continue;
        *sum += sl_hat[i];
        *n += 1;
    }
}
