/*
 * oracle.c — plain, slow, obviously-correct fp64 CPU oracle for the fixed fan-in
 * (uniform sparsity) output layer of arXiv 2306.03725.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2306_03725_b200/ + its CUDA library) never links, imports or calls it,
 * and shares no code, header, helper, table or constant generator with it.
 *
 * Citations: P:n = reference PAPER.md line n (LaTeX source of the paper),
 *            S:n = reference SPEC.md line n, SURVEY §x = /root/repo/SURVEY.md.
 * Notation: L labels (this shard: L rows, first global id row_begin),
 * k connections per label (the paper's s), m = width of the layer the sparse layer
 * reads (the paper's features dimension), B = mini-batch size.
 * Layouts: W[L][k], idx[L][k] label-major (the paper's s x L, transposed; SURVEY §0
 * reading #2); h[B][m]; y, g[B][L]; dh[B][m].
 *
 * Every floating-point computation is fp64 except the init-W word map, which our
 * RNG reading (reading R17) defines in fp32 and which is emulated here.
 * Loops follow the paper's algorithms in the paper's order; no blocking, fusion
 * or reordering.
 *
 * Parity pins (tests/test_oracle_pins.py): Fig. 1c worked example, dense-with-mask
 * equivalence, central finite differences, BCE/Adam closed forms, Random123 Philox
 * known-answer vectors, redistribution invariants and a hand-derived Fig. 1c
 * redistribution, top-k / P@k worked examples.  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* Timing mode: with oracle_set_threads(n > 1) the loops over labels (and
 * over Adam's elements) are shared by n OpenMP threads.  Every output element is still
 * computed by one thread in the loop order written below, so y, g, dW, db and Adam are
 * bit-identical to the 1-thread run; Alg. 2's dh is accumulated in per-thread private
 * arrays over contiguous label ranges and summed in thread order (a different, fixed fp64
 * summation order), and the loss total is an OpenMP sum.  The default is 1 thread: the
 * parity tests run the plain sequential loops.                                          */
static int g_threads = 1;
void oracle_set_threads(int32_t n) { g_threads = n > 1 ? n : 1; }
int32_t oracle_get_threads(void) { return g_threads; }

/* ------------------------------------------------------------------------- */
/* Alg. 1: score of label `label` for instance `instance`:
 *   value = 0; for weight_idx in range(s): source = indices[weight_idx, label];
 *   feature = features[instance, source]; value += feature * weights[weight_idx, label]
 * plus the per-label bias of the north-star formula y[b,j] = sum_i W[j,i] h[b,idx[j,i]] + b_j
 * (reading R3).  Ay is the companion sum of |terms| used for tolerances
 * (reading R19).                                                      */
void oracle_forward(int64_t L, int32_t m, int32_t k, int32_t B,
                    const double* W, const int32_t* idx, const double* bias,
                    const double* h, double* y, double* Ay)
{
    for (int32_t instance = 0; instance < B; ++instance) {
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t label = 0; label < L; ++label) {
            double value = bias[label];
            double avalue = fabs(bias[label]);
            for (int32_t weight_idx = 0; weight_idx < k; ++weight_idx) {
                int32_t source = idx[label * k + weight_idx];
                double feature = h[(int64_t)instance * m + source];
                value += feature * W[label * k + weight_idx];
                avalue += fabs(feature * W[label * k + weight_idx]);
            }
            y[(int64_t)instance * L + label] = value;
            if (Ay) Ay[(int64_t)instance * L + label] = avalue;
        }
    }
}

/* Shortlist scoring ("a trivial matrix slicing operation"): Alg. 1 restricted
 * to the (instance, label) pairs of a CSR candidate list: for cand_ptr[b] <= p < cand_ptr[b+1],
 *   y[p] = bias[j] + sum_i W[j,i] h[b, idx[j,i]],  j = cand_ids[p] - row_begin,
 * and y[p] = 0 when j is outside this shard's rows [0, L) (reading R24).  Ay as above.  */
void oracle_score_shortlist(int64_t L, int64_t row_begin, int32_t m, int32_t k, int32_t B,
                            const double* W, const int32_t* idx, const double* bias, const double* h,
                            const int32_t* cand_ptr, const int32_t* cand_ids, double* y, double* Ay)
{
    for (int32_t instance = 0; instance < B; ++instance) {
        for (int32_t p = cand_ptr[instance]; p < cand_ptr[instance + 1]; ++p) {
            int64_t label = (int64_t)cand_ids[p] - row_begin;
            double value = 0.0, avalue = 0.0;
            if (label >= 0 && label < L) {
                value = bias[label];
                avalue = fabs(bias[label]);
                for (int32_t weight_idx = 0; weight_idx < k; ++weight_idx) {
                    int32_t source = idx[label * k + weight_idx];
                    double feature = h[(int64_t)instance * m + source];
                    value += feature * W[label * k + weight_idx];
                    avalue += fabs(feature * W[label * k + weight_idx]);
                }
            }
            y[p] = value;
            Ay[p] = avalue;
        }
    }
}

/* Is global label `gid` a positive of instance b?  y in {0,1}^L stored sparse
 * (P:92-97): positives of b are lbl_ids[lbl_ptr[b] .. lbl_ptr[b+1]).            */
static int is_positive(const int32_t* lbl_ptr, const int32_t* lbl_ids, int32_t b, int64_t gid)
{
    for (int32_t q = lbl_ptr[b]; q < lbl_ptr[b + 1]; ++q)
        if ((int64_t)lbl_ids[q] == gid) return 1;
    return 0;
}

/* Logistic sigma, evaluated in the form that does not overflow. */
static double sigmoid(double x)
{
    if (x >= 0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

/* Binary cross-entropy with logits, one-vs-all over all labels (
 * S:264-272).  loss = s_g * sum_{b,j} [ softplus(y) - t*y ]
 *                   = s_g * sum_{b,j} [ max(y,0) - t*y + log1p(exp(-|y|)) ]
 * dloss/dy = s_g * (sigma(y) - t), written as s_g*sigma(y) for t=0 and
 * -s_g*sigma(-y) for t=1 (same value; no cancellation; reading R5).
 * s_g = grad_scale (default 1/B; reading R4).                                 */
void oracle_bce_grad(int64_t L, int64_t row_begin, int32_t B, const double* y,
                     const int32_t* lbl_ptr, const int32_t* lbl_ids, double s_g,
                     double* g, double* loss)
{
    double total = 0.0;
    for (int32_t b = 0; b < B; ++b) {
        #pragma omp parallel for schedule(static) reduction(+ : total) if (g_threads > 1) num_threads(g_threads)
        for (int64_t j = 0; j < L; ++j) {
            double yy = y[(int64_t)b * L + j];
            int t = is_positive(lbl_ptr, lbl_ids, b, row_begin + j);
            g[(int64_t)b * L + j] = t ? -s_g * sigmoid(-yy) : s_g * sigmoid(yy);
            total += (yy > 0 ? yy : 0.0) - (t ? yy : 0.0) + log1p(exp(-fabs(yy)));
        }
    }
    if (loss) *loss = s_g * total;
}

/* Squared hinge, the paper's main loss: l(y, yhat) = max(0, 1 - y yhat)^2 with
 * y = +1 for positives and -1 for negatives; dl/dyhat = -2 y max(0, 1 - y yhat),
 * "exactly zero whenever y yhat >= 1" — the implicit negative mining of §3.3.
 * g = s_g * dl/dyhat, loss = s_g * sum_{b,j} l.                                            */
void oracle_sqh_grad(int64_t L, int64_t row_begin, int32_t B, const double* y,
                     const int32_t* lbl_ptr, const int32_t* lbl_ids, double s_g,
                     double* g, double* loss)
{
    double total = 0.0;
    for (int32_t b = 0; b < B; ++b) {
        #pragma omp parallel for schedule(static) reduction(+ : total) if (g_threads > 1) num_threads(g_threads)
        for (int64_t j = 0; j < L; ++j) {
            double yy = y[(int64_t)b * L + j];
            double t = is_positive(lbl_ptr, lbl_ids, b, row_begin + j) ? 1.0 : -1.0;
            double margin = 1.0 - t * yy;
            double hinge = margin > 0.0 ? margin : 0.0;
            g[(int64_t)b * L + j] = s_g * (-2.0 * t * hinge);
            total += hinge * hinge;
        }
    }
    if (loss) *loss = s_g * total;
}

/* Alg. 3: gradient of one structural non-zero weight:
 *   source = indices[weight_idx, label]; result = 0
 *   for instance in range(batch_size): out = backward[instance, label];
 *       feature = features[instance, source]; result += feature * out
 * (the paper's `if out == 0: continue` skip changes nothing arithmetically for
 * BCE, whose gradient has no exact zeros).
 * db[j] = sum_b g[b,j] (bias gradient, north star).  A* = sums of |terms|.      */
void oracle_weight_grad(int64_t L, int32_t m, int32_t k, int32_t B,
                        const int32_t* idx, const double* h, const double* g,
                        double* dW, double* AdW, double* db, double* Adb)
{
    #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
    for (int64_t label = 0; label < L; ++label) {
        for (int32_t weight_idx = 0; weight_idx < k; ++weight_idx) {
            int32_t source = idx[label * k + weight_idx];
            double result = 0.0, aresult = 0.0;
            for (int32_t instance = 0; instance < B; ++instance) {
                double out = g[(int64_t)instance * L + label];
                double feature = h[(int64_t)instance * m + source];
                result += feature * out;
                aresult += fabs(feature * out);
            }
            dW[label * k + weight_idx] = result;
            if (AdW) AdW[label * k + weight_idx] = aresult;
        }
        double s = 0.0, as = 0.0;
        for (int32_t instance = 0; instance < B; ++instance) {
            s += g[(int64_t)instance * L + label];
            as += fabs(g[(int64_t)instance * L + label]);
        }
        db[label] = s;
        if (Adb) Adb[label] = as;
    }
}

/* Alg. 2: contribution of (instance, label) to the feature gradient:
 *   out = backward[instance, label]
 *   for weight_idx in range(s): source = indices[weight_idx, label]
 *       gradient[instance, source] += weights[weight_idx, label] * out
 * (the paper's atomicAdd becomes a plain += in this sequential loop; labels and
 * slots visited in ascending order).  dh is overwritten (zeroed first).         */
void oracle_input_grad(int64_t L, int32_t m, int32_t k, int32_t B,
                       const double* W, const int32_t* idx, const double* g,
                       double* dh, double* Adh)
{
    memset(dh, 0, sizeof(double) * (size_t)B * (size_t)m);
    if (Adh) memset(Adh, 0, sizeof(double) * (size_t)B * (size_t)m);
#ifdef _OPENMP
    if (g_threads > 1) {
        /* timing mode: thread r owns labels [r L / n, (r+1) L / n) and a private dh (and Adh);
         * the partials are summed in thread order.                                        */
        const int n = g_threads;
        const size_t Bm = (size_t)B * (size_t)m;
        double* part = (double*)calloc((size_t)n * Bm * (Adh ? 2 : 1), sizeof(double));
        if (part) {
            #pragma omp parallel num_threads(n)
            {
                const int r = omp_get_thread_num();
                double* pd = part + (size_t)r * Bm;
                double* pa = Adh ? part + (size_t)(n + r) * Bm : NULL;
                for (int32_t instance = 0; instance < B; ++instance) {
                    for (int64_t label = L * r / n; label < L * (r + 1) / n; ++label) {
                        double out = g[(int64_t)instance * L + label];
                        for (int32_t weight_idx = 0; weight_idx < k; ++weight_idx) {
                            int32_t source = idx[label * k + weight_idx];
                            double weight = W[label * k + weight_idx];
                            pd[(int64_t)instance * m + source] += weight * out;
                            if (pa) pa[(int64_t)instance * m + source] += fabs(weight * out);
                        }
                    }
                }
                #pragma omp barrier
                #pragma omp for schedule(static)
                for (int64_t e = 0; e < (int64_t)Bm; ++e) {
                    for (int q = 0; q < n; ++q) {
                        dh[e] += part[(size_t)q * Bm + e];
                        if (Adh) Adh[e] += part[(size_t)(n + q) * Bm + e];
                    }
                }
            }
            free(part);
            return;
        }
    }
#endif
    for (int32_t instance = 0; instance < B; ++instance) {
        for (int64_t label = 0; label < L; ++label) {
            double out = g[(int64_t)instance * L + label];
            for (int32_t weight_idx = 0; weight_idx < k; ++weight_idx) {
                int32_t source = idx[label * k + weight_idx];
                double weight = W[label * k + weight_idx];
                dh[(int64_t)instance * m + source] += weight * out;
                if (Adh) Adh[(int64_t)instance * m + source] += fabs(weight * out);
            }
        }
    }
}

/* Adam (Kingma & Ba, the optimizer of P:677-678) with bias correction, epsilon
 * outside the square root (reading R6), one global step counter t that
 * the caller has already incremented (t >= 1, reading R7):
 *   m = b1 m + (1-b1) q;  v = b2 v + (1-b2) q^2;
 *   p -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)                  */
void oracle_adam(int64_t n, double* p, const double* q, double* mo, double* ve,
                 int64_t t, double lr, double beta1, double beta2, double eps)
{
    double bc1 = 1.0 - pow(beta1, (double)t);
    double bc2 = 1.0 - pow(beta2, (double)t);
    #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
    for (int64_t e = 0; e < n; ++e) {
        mo[e] = beta1 * mo[e] + (1.0 - beta1) * q[e];
        ve[e] = beta2 * ve[e] + (1.0 - beta2) * q[e] * q[e];
        double mhat = mo[e] / bc1;
        double vhat = ve[e] / bc2;
        p[e] -= lr * mhat / (sqrt(vhat) + eps);
    }
}

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al., SC'11, "Parallel random numbers: as easy as
 * 1, 2, 3"; Random123).  Round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2;
 * c' = (hi1^c1^k0, lo1, hi0^c3^k1, lo0); key bump by the Weyl constants
 * between rounds.  Pinned by the Random123 known-answer vectors.               */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The w-th 32-bit word of the stream keyed (seed) with counter (n, row, step, domain),
 * n = w / 4, consumed in order (reading R13).                        */
static uint32_t stream_word(uint64_t seed, uint32_t row, uint32_t step, uint32_t domain, uint64_t w)
{
    uint32_t ctr[4] = { (uint32_t)(w / 4), row, step, domain };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t out[4];
    oracle_philox4x32_10(ctr, key, out);
    return out[w % 4];
}

/* Uniform integer in [0, m) from one 32-bit word by Lemire's multiply-shift with
 * exact rejection: x = u*m; reject if (x mod 2^32) < (2^32 mod m); else x >> 32.
 * Returns -1 on rejection.                                                      */
static int64_t lemire(uint32_t u, uint32_t m)
{
    uint64_t x = (uint64_t)u * (uint64_t)m;
    uint32_t low = (uint32_t)x;
    uint32_t threshold = (uint32_t)((((uint64_t)1) << 32) % (uint64_t)m);
    if (low < threshold) return -1;
    return (int64_t)(x >> 32);
}

/* Initialization ("we initialize the connections uniformly randomly,
 * potentially subject to the constraint that each label gets the same amount of
 * connections"; S:333 for the value range):
 *  idx row j: the first k distinct accepted candidates of domain 0, in draw order;
 *  W[j][i] = a * (2 * ((u >> 8) * 2^-24) - 1) evaluated in fp32, u = word i of
 *  domain 1 (reading R17); a = fp32(init_scale).                      */
void oracle_init(int64_t L, int64_t row_begin, int32_t m, int32_t k, uint64_t seed,
                 float a, int32_t* idx, float* W)
{
    for (int64_t j = 0; j < L; ++j) {
        uint32_t row = (uint32_t)(row_begin + j);
        int32_t count = 0;
        for (uint64_t w = 0; count < k; ++w) {
            int64_t c = lemire(stream_word(seed, row, 0, 0, w), (uint32_t)m);
            if (c < 0) continue;
            int dup = 0;
            for (int32_t q = 0; q < count; ++q) if (idx[j * k + q] == (int32_t)c) dup = 1;
            if (dup) continue;
            idx[j * k + count] = (int32_t)c;
            ++count;
        }
        for (int32_t i = 0; i < k; ++i) {
            uint32_t u = stream_word(seed, row, 0, 1, (uint64_t)i);
            float unit = (float)(u >> 8) * (1.0f / 16777216.0f);   /* exact in fp32 */
            float centered = 2.0f * unit - 1.0f;                    /* exact in fp32 */
            volatile float value = a * centered;                    /* one fp32 rounding */
            W[j * k + i] = value;
        }
    }
}

/* SET prune / redistribute / regrow ("the 10% lowest-magnitude
 * weights are randomly redistributed"), per label row (reading R8):
 *  p = floor(alpha * k) slots with the smallest key (|W|, slot) are pruned (R9);
 *  p new indices are drawn uniformly from [0, m) minus the row's pre-call index
 *  set (R10) from the regrow stream (domain 2, step = the caller's step, R13/R14),
 *  rejecting candidates already accepted;  the i-th accepted index goes to the
 *  i-th pruned slot in ascending slot order (R12); W = mW = vW = 0 there (R11).
 * W, mW, vW are fp64 here; |W| is compared numerically (so -0 == +0).          */
void oracle_redistribute(int64_t L, int64_t row_begin, int32_t m, int32_t k, int32_t p,
                         uint64_t seed, uint64_t step,
                         double* W, int32_t* idx, double* mW, double* vW)
{
    int32_t* pruned = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
    int32_t* accepted = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
    for (int64_t j = 0; j < L; ++j) {
        /* prune: rank of slot i = #slots with strictly smaller key */
        int32_t np = 0;
        for (int32_t i = 0; i < k; ++i) {
            double ai = fabs(W[j * k + i]);
            int32_t rank = 0;
            for (int32_t q = 0; q < k; ++q) {
                double aq = fabs(W[j * k + q]);
                if (aq < ai || (aq == ai && q < i)) ++rank;
            }
            if (rank < p) pruned[np++] = i;          /* ascending slot order */
        }
        /* regrow */
        uint32_t row = (uint32_t)(row_begin + j);
        int32_t na = 0;
        for (uint64_t w = 0; na < p; ++w) {
            int64_t c = lemire(stream_word(seed, row, (uint32_t)step, 2, w), (uint32_t)m);
            if (c < 0) continue;
            int taken = 0;
            for (int32_t q = 0; q < k; ++q) if (idx[j * k + q] == (int32_t)c) taken = 1;
            for (int32_t q = 0; q < na; ++q) if (accepted[q] == (int32_t)c) taken = 1;
            if (taken) continue;
            accepted[na++] = (int32_t)c;
        }
        for (int32_t q = 0; q < p; ++q) {
            int32_t slot = pruned[q];
            idx[j * k + slot] = accepted[q];
            W[j * k + slot] = 0.0;
            mW[j * k + slot] = 0.0;
            vW[j * k + slot] = 0.0;
        }
    }
    free(pruned);
    free(accepted);
}

/* ------------------------------------------------------------------------- */
/* top-k prediction ("selecting the k highest scoring labels"):
 * order labels by (score descending, global id ascending) and keep K.  */
typedef struct { double score; int64_t id; } scored_label;

static int by_score_then_id(const void* a, const void* b)
{
    const scored_label* x = (const scored_label*)a;
    const scored_label* z = (const scored_label*)b;
    if (x->score > z->score) return -1;
    if (x->score < z->score) return 1;
    if (x->id < z->id) return -1;
    if (x->id > z->id) return 1;
    return 0;
}

void oracle_topk(int64_t L, int64_t row_begin, int32_t B, const double* y, int32_t K,
                 double* scores, int64_t* ids)
{
    scored_label* row = (scored_label*)malloc(sizeof(scored_label) * (size_t)L);
    for (int32_t b = 0; b < B; ++b) {
        for (int64_t j = 0; j < L; ++j) {
            row[j].score = y[(int64_t)b * L + j];
            row[j].id = row_begin + j;
        }
        qsort(row, (size_t)L, sizeof(scored_label), by_score_then_id);
        for (int32_t q = 0; q < K; ++q) {
            scores[(int64_t)b * K + q] = row[q].score;
            ids[(int64_t)b * K + q] = row[q].id;
        }
    }
    free(row);
}

/* Precision at k, Eq. (1): P@k = k^-1 sum_j y_j yhat_j, i.e. the
 * number of predicted labels that are positives divided by k (even if the
 * instance has fewer than k positives, reading R16); averaged over instances. */
double oracle_precision_at_k(int32_t B, int32_t K, const int64_t* ids,
                             const int32_t* lbl_ptr, const int32_t* lbl_ids)
{
    double total = 0.0;
    for (int32_t b = 0; b < B; ++b) {
        int32_t hits = 0;
        for (int32_t q = 0; q < K; ++q)
            if (is_positive(lbl_ptr, lbl_ids, b, ids[(int64_t)b * K + q])) ++hits;
        total += (double)hits / (double)K;
    }
    return total / (double)B;
}

/* ========================================================================= */
/* NEXT-2: the intermediate layer of the proposed architecture,
 * features -> input dropout -> dense W_d -> uniform-sparse W (Fig. 2, P:1013-1022;
 * "adding an intermediate layer between the embedding layer and the final
 * classification layer"; "we apply dropout to the input features",
 * P:686-689).  Layouts: x, xt [B][d] (d = feature dimension), Wd [d][m] (input
 * feature major), bd [m], z, h, dh [B][m].  Readings R25-R28.       */

/* Input dropout (inverted dropout as TF's tf.nn.dropout, reading R25):
 *   u = word f of the stream keyed (seed) with counter (f/4, b, step, domain 3);
 *   kept iff (u >> 8) * 2^-24 >= p;  xt[b][f] = x[b][f] * s if kept, else 0,
 * with s = fp32(1 / (1 - p)) supplied by the caller.  keep[b][f] = 0/1.         */
void oracle_dropout(int32_t B, int32_t d, double p, double s, uint64_t seed, uint32_t step,
                    const double* x, double* xt, uint8_t* keep)
{
    for (int32_t b = 0; b < B; ++b) {
        for (int32_t f = 0; f < d; ++f) {
            uint32_t u = stream_word(seed, (uint32_t)b, step, 3, (uint64_t)f);
            double unit = (double)(u >> 8) / 16777216.0;
            int kept = unit >= p;
            keep[(int64_t)b * d + f] = (uint8_t)kept;
            xt[(int64_t)b * d + f] = kept ? x[(int64_t)b * d + f] * s : 0.0;
        }
    }
}

/* Dense intermediate layer, forward: z[b][c] = bd[c] + sum_f xt[b][f] Wd[f][c]
 * (f ascending), h = max(z, 0) (ReLU; the activation is unnamed in the paper, reading
 * R18).  Az = |bd[c]| + sum_f |xt[b][f] Wd[f][c]| (R19 companion).               */
void oracle_dense_forward(int32_t B, int32_t d, int32_t m, const double* Wd, const double* bd,
                          const double* xt, double* z, double* Az, double* h)
{
    for (int32_t b = 0; b < B; ++b) {
        for (int32_t c = 0; c < m; ++c) {
            double value = bd[c], avalue = fabs(bd[c]);
            for (int32_t f = 0; f < d; ++f) {
                double term = xt[(int64_t)b * d + f] * Wd[(int64_t)f * m + c];
                value += term;
                avalue += fabs(term);
            }
            z[(int64_t)b * m + c] = value;
            Az[(int64_t)b * m + c] = avalue;
            h[(int64_t)b * m + c] = value > 0.0 ? value : 0.0;
        }
    }
}

/* Dense intermediate layer, backward: dz = dh * [z > 0] (ReLU'(0) = 0, reading R26);
 *   dWd[f][c] = sum_b xt[b][f] dz[b][c] (b ascending),  dbd[c] = sum_b dz[b][c],
 * with the |term| companions AdWd, Adbd.  The input gradient (w.r.t. the fixed
 * features) is not needed: the embeddings are not trained.           */
void oracle_dense_backward(int32_t B, int32_t d, int32_t m, const double* xt, const double* z,
                           const double* dh, double* dWd, double* AdWd, double* dbd, double* Adbd)
{
    for (int32_t f = 0; f < d; ++f) {
        for (int32_t c = 0; c < m; ++c) {
            double value = 0.0, avalue = 0.0;
            for (int32_t b = 0; b < B; ++b) {
                double dz = z[(int64_t)b * m + c] > 0.0 ? dh[(int64_t)b * m + c] : 0.0;
                double term = xt[(int64_t)b * d + f] * dz;
                value += term;
                avalue += fabs(term);
            }
            dWd[(int64_t)f * m + c] = value;
            AdWd[(int64_t)f * m + c] = avalue;
        }
    }
    for (int32_t c = 0; c < m; ++c) {
        double value = 0.0, avalue = 0.0;
        for (int32_t b = 0; b < B; ++b) {
            double dz = z[(int64_t)b * m + c] > 0.0 ? dh[(int64_t)b * m + c] : 0.0;
            value += dz;
            avalue += fabs(dz);
        }
        dbd[c] = value;
        Adbd[c] = avalue;
    }
}

/* Dense init (reading R27; TF's Dense default is Glorot-uniform): Wd[f][c] =
 * a * (2 * ((u >> 8) * 2^-24) - 1) in fp32 with u = word c of the stream keyed (seed)
 * with counter (c/4, f, 0, domain 4) (the R17 word map on a new domain);
 * a = fp32(init_scale), default sqrt(6 / (d + m)); bd = 0.                       */
void oracle_dense_init(int32_t d, int32_t m, uint64_t seed, float a, float* Wd)
{
    for (int32_t f = 0; f < d; ++f) {
        for (int32_t c = 0; c < m; ++c) {
            uint32_t u = stream_word(seed, (uint32_t)f, 0, 4, (uint64_t)c);
            float unit = (float)(u >> 8) * (1.0f / 16777216.0f);
            float centered = 2.0f * unit - 1.0f;
            volatile float value = a * centered;
            Wd[(int64_t)f * m + c] = value;
        }
    }
}
