/*
 * aps_oracle.c -- plain, slow, obviously-correct CPU oracle for the APS
 * (Auto-Precision Scaling, arXiv 1911.08907) gradient synchronisation.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1911_08907_b200/, libaps.so) never links, calls
 * or executes anything under oracle/.  This file shares no code, header,
 * table or constant generator with the CUDA path.
 *
 * Citations: "P:n" is a line of the paper's LaTeX source, with
 * the algorithm / equation / table it falls in.  "A<k>" is a reading of the
 * paper listed in DESIGN.md (section "Readings").  "O<k>" is an oracle step
 * of SURVEY.md section 8(c).
 *
 * Arithmetic: every value is carried in IEEE binary64 where the paper gives
 * no precision; the operations the paper performs in fp32 (Alg. 1's scale
 * g*2^f, the low-precision accumulator's fp32 add that CPD re-quantises, the
 * cast back and the unscale) are done in binary32 exactly as written.
 * Requires FLT_EVAL_METHOD == 0 (x86-64 SSE) and no -ffast-math /
 * -ffp-contract.
 *
 * Pins (tests/test_oracle_*.py): Table 2 ranges, torch dtype equivalence
 * (float8_e5m2, float16, bfloat16, float8_e4m3fn below 248), brute-force
 * argmin enumeration, the paper's worked shifts (Fig. aps_comparing), the
 * no-overflow invariant, (8,23) transparency, exact-rounding of the ring add
 * and numpy.packbits for the layout.  Parity of the ring-chunk layout (O7)
 * is a design rule with no paper pin: "parity unpinned (layout)" -- see
 * DESIGN.md.
 */
#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if !defined(FLT_EVAL_METHOD) || FLT_EVAL_METHOD != 0
#error "oracle needs FLT_EVAL_METHOD == 0 so float arithmetic is IEEE binary32"
#endif

/* status codes, same numeric values as the product's, written here independently */
enum { OR_OK = 0, OR_ERR_ARG = 1, OR_ERR_FORMAT = 2, OR_ERR_NONFINITE = 6 };

#define OR_TILE 128 /* O7: elements per tile (design rule, not in the paper) */
#define OR_EMPTY INT32_MIN  /* FindMaxExp of an all-zero tensor: "-INF" (Alg. 1) */
#define OR_NONFINITE INT32_MAX

/* ------------------------------------------------------------------ */
/* O1  Format.  Table `precision_range` P:184-198; Alg. 1 P:237-242.   */
/* ------------------------------------------------------------------ */

/* Validity (A-readings in DESIGN.md): 2 <= e <= 8 (e = 1 has bias 0 and no
 * normal numbers), 0 <= m <= 23, 1 + e + m <= 32.  CPD: "exp bits <= 8 and
 * man bits <= 23". */
int oracle_format_valid(int e, int m)
{
    if (e < 2 || e > 8 || m < 0 || m > 23 || 1 + e + m > 32) return OR_ERR_FORMAT;
    return OR_OK;
}

/* upper_bound_exp <- 2^(exp_bits-1) - 1   (Alg. 1 line 1) */
int oracle_bias(int e) { return (1 << (e - 1)) - 1; }

/* ------------------------------------------------------------------ */
/* O1  decode: code -> value.  IEEE-style layout s | E | M, sign MSB.  */
/* normal (1 + M/2^m) * 2^(E-bias); subnormal M * 2^(1-bias-m);        */
/* all-ones exponent reserved (M = 0: Inf, else NaN).                  */
/* ------------------------------------------------------------------ */
float oracle_decode1(uint32_t code, int e, int m)
{
    const int bias = oracle_bias(e);
    const uint32_t sign = (code >> (e + m)) & 1u;
    const uint32_t E = (code >> m) & ((1u << e) - 1u);
    const uint32_t M = code & ((m == 0) ? 0u : ((1u << m) - 1u));
    double v;
    if (E == (1u << e) - 1u) {
        v = (M == 0) ? INFINITY : NAN;
    } else if (E == 0) {
        v = ldexp((double)M, 1 - bias - m);
    } else {
        v = ldexp(1.0 + ldexp((double)M, -m), (int)E - bias);
    }
    if (sign) v = -v;
    return (float)v; /* every finite value of a format with e<=8, m<=23 is exact in binary32 */
}

/* encode a non-negative value v that is EXACTLY representable in (e,m),
 * or equal to 2^(bias+1) (the stand-in for +Inf in O6). */
static uint32_t encode_magnitude(double v, int e, int m)
{
    const int bias = oracle_bias(e);
    if (v == 0.0) return 0u;
    if (v >= ldexp(1.0, bias + 1)) return ((1u << e) - 1u) << m; /* Inf */
    if (v < ldexp(1.0, 1 - bias)) {                              /* subnormal: E = 0 */
        double M = v / ldexp(1.0, 1 - bias - m);
        return (uint32_t)M;
    }
    int k;
    double f = frexp(v, &k); /* v = f * 2^k, f in [0.5, 1) */
    (void)f;
    k -= 1;                  /* v in [2^k, 2^(k+1)) */
    double M = (v / ldexp(1.0, k) - 1.0) * ldexp(1.0, m);
    return ((uint32_t)(k + bias) << m) | (uint32_t)M;
}

/* ------------------------------------------------------------------ */
/* O6  Cast(x, exp_bit, man_bit): round-to-nearest-even into   */
/* (e,m) with gradual underflow ("smaller than 2^-16 ... cast to 0",   */
/* P:278, A10) and IEEE overflow ("greater than 2^15 will overflow and */
/* cast to INF", A11).  Ties go to the candidate whose          */
/* magnitude code is even (A9; equals IEEE ties-to-even for m >= 1).   */
/* Method: the two representable neighbours lo <= |x| < hi are found   */
/* from the quantum of |x|'s binade; 2|x| is compared with lo + hi.    */
/* All of it is exact in binary64.                                     */
/* ------------------------------------------------------------------ */
uint32_t oracle_cast1(float x, int e, int m)
{
    const int bias = oracle_bias(e);
    const uint32_t sbit = (signbit(x) ? 1u : 0u) << (e + m);
    const uint32_t inf_code = sbit | (((1u << e) - 1u) << m);
    if (isnan(x)) /* canonical NaN: mantissa MSB set; m = 0 has no NaN code (A12) */
        return (m > 0) ? (inf_code | (1u << (m - 1))) : inf_code;
    if (isinf(x)) return inf_code;

    const double a = fabs((double)x);
    if (a == 0.0) return sbit;                       /* signed zero (A15) */
    if (a >= ldexp(1.0, bias + 1)) return inf_code;  /* past every candidate */

    int k;
    (void)frexp(a, &k);
    k -= 1;                                          /* a in [2^k, 2^(k+1)) */
    const int qexp = ((k > 1 - bias) ? k : (1 - bias)) - m;
    const double quantum = ldexp(1.0, qexp);         /* spacing of (e,m) values around a */
    const double lo = floor(a / quantum) * quantum;  /* largest value <= a */
    const double hi = lo + quantum;                  /* smallest value >  a (2^(bias+1) = Inf) */
    const uint32_t clo = encode_magnitude(lo, e, m);
    const uint32_t chi = encode_magnitude(hi, e, m);
    uint32_t mag;
    if (2.0 * a < lo + hi) mag = clo;
    else if (2.0 * a > lo + hi) mag = chi;
    else mag = (clo % 2u == 0u) ? clo : chi;        /* tie: even code */
    return sbit | mag;
}

int oracle_cast(const float *x, uint32_t *codes, int64_t n, int e, int m)
{
    if (oracle_format_valid(e, m)) return OR_ERR_FORMAT;
    if (n < 0 || (n > 0 && (!x || !codes))) return OR_ERR_ARG;
    for (int64_t i = 0; i < n; ++i) codes[i] = oracle_cast1(x[i], e, m);
    return OR_OK;
}

int oracle_decode(const uint32_t *codes, float *x, int64_t n, int e, int m)
{
    if (oracle_format_valid(e, m)) return OR_ERR_FORMAT;
    if (n < 0 || (n > 0 && (!x || !codes))) return OR_ERR_ARG;
    for (int64_t i = 0; i < n; ++i) x[i] = oracle_decode1(codes[i], e, m);
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* O2/O3  FindMaxExp(g * N)   (Alg. 1 line 3; function P:260-271)*/
/*   max over i != 0 of ceil(log2(abs(i)))  ->  -INF for an all-zero   */
/*   tensor.  Reading A2: the product N*|g_i| is taken exactly (Eq. 4, */
/*   P:375, writes ceil(log2|N*g^|)).  Reading A5: exact ceil(log2)    */
/*   also for fp32 subnormals.  ceil(log2(.)) is monotone, so the max  */
/*   over elements equals ceil(log2(N * max|g_i|)).                    */
/*   Returns OR_EMPTY (A3), or OR_NONFINITE when any element is Inf/NaN*/
/*   (A4).                                                             */
/* ------------------------------------------------------------------ */
static int32_t ceil_log2_exact(double v) /* v > 0, exact */
{
    int k;
    double f = frexp(v, &k); /* v = f * 2^k with f in [0.5, 1) */
    return (f == 0.5) ? (k - 1) : k;
}

int32_t oracle_find_max_exp(const float *g, int64_t n, int N)
{
    int32_t max_exp = OR_EMPTY; /* "max_exp <- -INF" */
    for (int64_t i = 0; i < n; ++i) {
        if (!isfinite(g[i])) return OR_NONFINITE;
        if (g[i] != 0.0f) {                                     /* "if i != 0" */
            int32_t t = ceil_log2_exact((double)N * fabs((double)g[i])); /* ceil(log2(abs(N*i))) */
            if (t > max_exp) max_exp = t;
        }
    }
    return max_exp;
}

/* O4  f~ <- upper_bound_exp - AllReduce(max_grad_exp, MAX)   (Alg. 1 line 4,
 * P:246; Eq. (4) P:375 with p^ = 2^upper_bound_exp, reading A1).
 * All-zero layer: f~ = 0 (A3). */
int32_t oracle_scale_exp(int e, int32_t E)
{
    if (E == OR_EMPTY) return 0;
    return oracle_bias(e) - E;
}

/* O5  g <- g * 2^f~  (Alg. 1 line 5): one binary32 result, RNE,
 * gradual underflow (A8: ldexpf semantics).  (double)g * 2^f is exact in
 * binary64 for every f~ that can arise, so the only rounding is the cast to
 * float. */
float oracle_scale(float g, int32_t ft) { return (float)ldexp((double)g, ft); }

/* O8 helper: one low-precision accumulation step as CPD simulates it
 * (reading A13): the addends are cast back to fp32, added in
 * fp32, and the sum is re-quantised. */
uint32_t oracle_ring_add(uint32_t acc, uint32_t addend, int e, int m)
{
    float s = oracle_decode1(acc, e, m) + oracle_decode1(addend, e, m); /* fl32 add */
    return oracle_cast1(s, e, m);
}

/* O10  g <- Cast(low_g, 8, 23); g <- g / 2^f~   (Alg. 1 lines 7-8,
 * P:254-256), then the average over N ranks (north_star; reading A16):
 * out = fl32( fl32(dec(s) * 2^-f~) / N ). */
float oracle_unscale1(uint32_t s, int32_t ft, int N, int average, int e, int m)
{
    float g = oracle_decode1(s, e, m);               /* Cast(low_g, 8, 23): exact */
    float t = (float)ldexp((double)g, -ft);          /* g / 2^f~, one binary32 rounding */
    if (average) t = t / (float)N;                   /* IEEE binary32 division */
    return t;
}

/* ------------------------------------------------------------------ */
/* O7  Layout (design rule; parity unpinned by the paper).            */
/*   Layer l occupies T_l = ceil(n_l / 128) tiles from tile offset    */
/*   o_l = sum_{k<l} T_k (caller's layer order); T = sum T_l;         */
/*   T' = p * ceil(T / p); chunk c = tiles [c T'/p, (c+1) T'/p).      */
/* O11 Pack: code i of the whole buffer occupies bits [i b, (i+1) b), */
/*   LSB-first, in a little-endian byte stream (tile t = bytes        */
/*   [16 b t, 16 b (t+1)) ).  Padding codes are +0.                    */
/* ------------------------------------------------------------------ */
int64_t oracle_total_tiles(int p, int n_layers, const int64_t *numels)
{
    int64_t T = 0;
    for (int l = 0; l < n_layers; ++l) T += (numels[l] + OR_TILE - 1) / OR_TILE;
    return ((T + p - 1) / p) * p; /* T' */
}

int64_t oracle_packed_bytes(int p, int e, int m, int n_layers, const int64_t *numels)
{
    if (oracle_format_valid(e, m) || p < 1 || n_layers < 1 || !numels) return -1;
    const int b = 1 + e + m;
    return 16 * (int64_t)b * oracle_total_tiles(p, n_layers, numels);
}

void oracle_put_code(uint8_t *buf, int64_t i, int b, uint32_t code)
{
    for (int j = 0; j < b; ++j) {
        int64_t bit = i * b + j;
        uint8_t mask = (uint8_t)(1u << (bit % 8));
        if ((code >> j) & 1u) buf[bit / 8] |= mask;
        else buf[bit / 8] &= (uint8_t)~mask;
    }
}

uint32_t oracle_get_code(const uint8_t *buf, int64_t i, int b)
{
    uint32_t code = 0;
    for (int j = 0; j < b; ++j) {
        int64_t bit = i * b + j;
        if ((buf[bit / 8] >> (bit % 8)) & 1u) code |= (1u << j);
    }
    return code;
}

int oracle_pack(const uint32_t *codes, int64_t n, int b, uint8_t *out)
{
    if (b < 1 || b > 32 || n < 0) return OR_ERR_ARG;
    for (int64_t i = 0; i < n; ++i) oracle_put_code(out, i, b, codes[i]);
    return OR_OK;
}

int oracle_unpack(const uint8_t *buf, int64_t n, int b, uint32_t *codes)
{
    if (b < 1 || b > 32 || n < 0) return OR_ERR_ARG;
    for (int64_t i = 0; i < n; ++i) codes[i] = oracle_get_code(buf, i, b);
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Whole APS synchronisation for p simulated ranks, Alg. 1 */
/* in the paper's order: FindMaxExp -> AllReduce(MAX) -> f~ -> scale   */
/* -> Cast -> AllReduce(SUM) as a ring with a re-       */
/* quantise after every add -> Cast back -> unscale (and   */
/* average, A16).                                                      */
/*                                                                     */
/* grads: p * n_layers host pointers, rank-major (grads[r*n_layers+l]).*/
/* ftilde_out[n_layers]; packed_out: p * packed_bytes or NULL (each    */
/* rank's codes after Cast, O11); reduced_out: packed_bytes or NULL    */
/* (the codes every rank holds after the all-reduce, O8/O9); out:      */
/* n_layers host pointers (fp32), or NULL.                             */
/* n_threads >= 1: the element loops of each step are split into       */
/* contiguous ranges run by that many threads (every element's         */
/* arithmetic is independent of the split, and a maximum is            */
/* order-independent, so the results are bit-identical for any         */
/* n_threads -- pinned by tests/test_oracle_aps.py).                   */
/* Returns OR_OK, OR_ERR_ARG, OR_ERR_FORMAT or OR_ERR_NONFINITE.       */
/* ------------------------------------------------------------------ */

/* a contiguous element range [i0, i1) of layer l of rank r */
typedef struct { int r, l; int64_t i0, i1; } or_range;

typedef struct {
    int p, e, m, n_layers, average, n_threads, tid;
    const int64_t *numels;
    const float *const *grads;
    const int64_t *tile_off;   /* first tile of each layer (O7) */
    const int32_t *ft;
    const or_range *rng;       /* the step's ranges */
    int64_t n_rng;
    int32_t *rng_E;            /* step 1: FindMaxExp of each range */
    uint32_t *q;               /* [p][ncodes] Cast codes */
    uint32_t *s;               /* [ncodes] reduced codes */
    int64_t ncodes, chunk_codes;
    float *const *out;
    int step;
} or_job;

#define OR_RANGE 262144 /* elements per range of the threaded steps */

static void *or_worker(void *arg)
{
    const or_job *J = (const or_job *)arg;
    if (J->step == 1) {        /* Alg. 1 line 3: FindMaxExp(g * N) of each range */
        for (int64_t k = J->tid; k < J->n_rng; k += J->n_threads) {
            const or_range R = J->rng[k];
            J->rng_E[k] = oracle_find_max_exp(J->grads[(size_t)R.r * J->n_layers + R.l] + R.i0, R.i1 - R.i0, J->p);
        }
    } else if (J->step == 2) { /* Alg. 1 lines 5-6: Cast(g * 2^f~) into the O7 layout */
        for (int64_t k = J->tid; k < J->n_rng; k += J->n_threads) {
            const or_range R = J->rng[k];
            const float *g = J->grads[(size_t)R.r * J->n_layers + R.l];
            uint32_t *dst = J->q + (size_t)R.r * J->ncodes + J->tile_off[R.l] * OR_TILE;
            for (int64_t i = R.i0; i < R.i1; ++i) dst[i] = oracle_cast1(oracle_scale(g[i], J->ft[R.l]), J->e, J->m);
        }
    } else if (J->step == 3) { /* Alg. 1 line 7: the ring sum, element by element */
        const int64_t lo = J->ncodes * J->tid / J->n_threads, hi = J->ncodes * (J->tid + 1) / J->n_threads;
        for (int64_t i = lo; i < hi; ++i) {
            const int c = (int)(i / J->chunk_codes); /* the chunk (and owner) of code i */
            uint32_t acc = J->q[(size_t)((c + 1) % J->p) * J->ncodes + i];
            for (int j = 2; j <= J->p; ++j)
                acc = oracle_ring_add(acc, J->q[(size_t)((c + j) % J->p) * J->ncodes + i], J->e, J->m);
            J->s[i] = acc;
        }
    } else {                   /* Alg. 1 lines 8-9: Cast back, unscale, average */
        for (int64_t k = J->tid; k < J->n_rng; k += J->n_threads) {
            const or_range R = J->rng[k];
            const uint32_t *src = J->s + J->tile_off[R.l] * OR_TILE;
            for (int64_t i = R.i0; i < R.i1; ++i)
                J->out[R.l][i] = oracle_unscale1(src[i], J->ft[R.l], J->p, J->average, J->e, J->m);
        }
    }
    return NULL;
}

/* run step `step` of job J on J->n_threads threads (the calling thread is one of them) */
static void or_run(or_job *J, int step)
{
    const int nt = J->n_threads;
    or_job *jobs = (or_job *)malloc(sizeof(or_job) * (size_t)nt);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nt);
    for (int t = 0; t < nt; ++t) {
        jobs[t] = *J;
        jobs[t].tid = t;
        jobs[t].step = step;
    }
    for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, or_worker, &jobs[t]);
    or_worker(&jobs[0]);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
}

/* ranges of <= OR_RANGE elements covering every (rank < pr, layer) */
static or_range *or_ranges(int pr, int n_layers, const int64_t *numels, int64_t *n_out)
{
    int64_t n = 0;
    for (int l = 0; l < n_layers; ++l) n += (int64_t)pr * ((numels[l] + OR_RANGE - 1) / OR_RANGE);
    or_range *R = (or_range *)malloc(sizeof(or_range) * (size_t)n);
    int64_t k = 0;
    for (int r = 0; r < pr; ++r)
        for (int l = 0; l < n_layers; ++l)
            for (int64_t i0 = 0; i0 < numels[l]; i0 += OR_RANGE) {
                R[k].r = r;
                R[k].l = l;
                R[k].i0 = i0;
                R[k].i1 = i0 + OR_RANGE < numels[l] ? i0 + OR_RANGE : numels[l];
                ++k;
            }
    *n_out = n;
    return R;
}

int oracle_aps_sync(int p, int e, int m, int n_layers, const int64_t *numels,
                    const float *const *grads, int average, int32_t *ftilde_out,
                    uint8_t *packed_out, uint8_t *reduced_out, float *const *out, int n_threads)
{
    if (oracle_format_valid(e, m)) return OR_ERR_FORMAT;
    if (p < 1 || n_layers < 1 || !numels || !grads || n_threads < 1) return OR_ERR_ARG;
    for (int l = 0; l < n_layers; ++l)
        if (numels[l] < 1) return OR_ERR_ARG;

    const int b = 1 + e + m;
    const int64_t Tp = oracle_total_tiles(p, n_layers, numels); /* T' */
    const int64_t ncodes = Tp * OR_TILE;
    const int64_t nbytes = 16 * (int64_t)b * Tp;
    int64_t *tile_off = (int64_t *)malloc(sizeof(int64_t) * (size_t)n_layers);
    for (int l = 0, t = 0; l < n_layers; ++l) {
        tile_off[l] = t;
        t += (int)((numels[l] + OR_TILE - 1) / OR_TILE);
    }
    or_job J;
    memset(&J, 0, sizeof J);
    J.p = p; J.e = e; J.m = m; J.n_layers = n_layers; J.average = average; J.n_threads = n_threads;
    J.numels = numels; J.grads = grads; J.tile_off = tile_off;
    J.ncodes = ncodes; J.chunk_codes = (Tp / p) * OR_TILE; J.out = out;

    /* Alg. 1 line 3: max_grad_exp <- FindMaxExp(g * N), on every rank;
     * line 4: AllReduce(max_grad_exp, MAX).  (The max over ranges equals
     * FindMaxExp of the whole layer: ceil(log2(N x)) is monotone in x.) */
    int32_t *E = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_layers);
    int32_t *ft = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_layers);
    int64_t n_rng;
    or_range *rng = or_ranges(p, n_layers, numels, &n_rng);
    int32_t *rng_E = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_rng);
    J.rng = rng; J.n_rng = n_rng; J.rng_E = rng_E;
    or_run(&J, 1);
    int nonfinite = 0;
    for (int l = 0; l < n_layers; ++l) E[l] = OR_EMPTY;
    for (int64_t k = 0; k < n_rng; ++k) {
        if (rng_E[k] == OR_NONFINITE) nonfinite = 1;
        if (rng_E[k] > E[rng[k].l]) E[rng[k].l] = rng_E[k];
    }
    for (int l = 0; l < n_layers; ++l) {
        ft[l] = oracle_scale_exp(e, E[l]); /* f~ <- upper_bound_exp - E */
        if (ftilde_out) ftilde_out[l] = ft[l];
    }
    free(rng_E);
    if (nonfinite) { /* A4: outputs unspecified, the error is reported */
        free(E); free(ft); free(rng); free(tile_off);
        return OR_ERR_NONFINITE;
    }
    J.ft = ft;

    /* Alg. 1 lines 5-6: g <- g * 2^f~ ; low_g <- Cast(g, exp_bit, man_bit),
     * placed in the O7 layout (padding codes are +0). */
    uint32_t *q = (uint32_t *)calloc((size_t)p * (size_t)ncodes, sizeof(uint32_t));
    J.q = q;
    or_run(&J, 2);
    if (packed_out)
        for (int r = 0; r < p; ++r) {
            uint8_t *pk = packed_out + (size_t)r * (size_t)nbytes;
            memset(pk, 0, (size_t)nbytes);
            oracle_pack(q + (size_t)r * ncodes, ncodes, b, pk);
        }

    /* Alg. 1 line 7: low_g <- AllReduce(low_g, SUM), as a ring with
     * the low-precision accumulator re-quantising after each add.
     * O8: chunk c is accumulated in rank order c+1, c+2, ..., c (the owner
     * adds last, "add a local gradient with the summation of all other
     * nodes' local gradients in the last step").  O9: every rank then holds
     * the same codes. */
    uint32_t *s = (uint32_t *)calloc((size_t)ncodes, sizeof(uint32_t));
    J.s = s;
    or_run(&J, 3);
    if (reduced_out) {
        memset(reduced_out, 0, (size_t)nbytes);
        oracle_pack(s, ncodes, b, reduced_out);
    }

    /* Alg. 1 lines 8-9: g <- Cast(low_g, 8, 23); g <- g / 2^f~; average. */
    if (out) {
        free(rng);
        rng = or_ranges(1, n_layers, numels, &n_rng);
        J.rng = rng; J.n_rng = n_rng;
        or_run(&J, 4);
    }
    free(q); free(s); free(E); free(ft); free(rng); free(tile_off);
    return OR_OK;
}

/* Element-wise O8 step over arrays (loop over oracle_ring_add; test helper). */
int oracle_ring_add_n(const uint32_t *acc, const uint32_t *addend, uint32_t *out, int64_t n, int e, int m)
{
    if (oracle_format_valid(e, m)) return OR_ERR_FORMAT;
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_ring_add(acc[i], addend[i], e, m);
    return OR_OK;
}

/* Element-wise O10 over arrays (loop over oracle_unscale1; test helper). */
int oracle_unscale_n(const uint32_t *s, float *out, int64_t n, int32_t ft, int N, int average, int e, int m)
{
    if (oracle_format_valid(e, m)) return OR_ERR_FORMAT;
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_unscale1(s[i], ft, N, average, e, m);
    return OR_OK;
}

/* Element-wise O5+O6 over arrays: codes[i] = Cast(g[i] * 2^f~) (test helper). */
int oracle_scale_cast_n(const float *g, uint32_t *codes, int64_t n, int32_t ft, int e, int m)
{
    if (oracle_format_valid(e, m)) return OR_ERR_FORMAT;
    for (int64_t i = 0; i < n; ++i) codes[i] = oracle_cast1(oracle_scale(g[i], ft), e, m);
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Per-layer formats (hybrid precision, Table      */
/* `last_layer_precision` P:571-584 and P:545: "IEEE FP32 for the       */
/* gradient of the last layer ... low precision for all other layers"). */
/* Layer l has format (e[l], m[l]) and code width b_l; its tiles are     */
/* 16*b_l bytes.  Padding tiles (T..T') continue the last layer's        */
/* format.  Tile t starts at byte sum_{u<t} 16*b(u); chunk c = tiles     */
/* [c T'/p, (c+1) T'/p) as before; every element is cast, re-quantised   */
/* and decoded in its own layer's format.                                */
/* ------------------------------------------------------------------ */
int64_t oracle_packed_bytes_mixed(int p, int n_layers, const int64_t *numels, const int *e, const int *m)
{
    if (p < 1 || n_layers < 1 || !numels || !e || !m) return -1;
    int64_t bytes = 0, T = 0;
    for (int l = 0; l < n_layers; ++l) {
        if (oracle_format_valid(e[l], m[l])) return -1;
        const int64_t Tl = (numels[l] + OR_TILE - 1) / OR_TILE;
        bytes += 16 * (int64_t)(1 + e[l] + m[l]) * Tl;
        T += Tl;
    }
    const int64_t Tp = ((T + p - 1) / p) * p;
    return bytes + 16 * (int64_t)(1 + e[n_layers - 1] + m[n_layers - 1]) * (Tp - T);
}

int oracle_aps_sync_mixed(int p, const int *e, const int *m, int n_layers, const int64_t *numels,
                          const float *const *grads, int average, int32_t *ftilde_out,
                          uint8_t *packed_out, uint8_t *reduced_out, float *const *out)
{
    if (p < 1 || n_layers < 1 || !numels || !grads || !e || !m) return OR_ERR_ARG;
    for (int l = 0; l < n_layers; ++l) {
        if (oracle_format_valid(e[l], m[l])) return OR_ERR_FORMAT;
        if (numels[l] < 1) return OR_ERR_ARG;
    }
    const int64_t Tp = oracle_total_tiles(p, n_layers, numels);
    const int64_t ncodes = Tp * OR_TILE;
    const int64_t chunk_codes = (Tp / p) * OR_TILE;
    const int64_t nbytes = oracle_packed_bytes_mixed(p, n_layers, numels, e, m);
    /* per-code layer (padding codes belong to the last layer) and tile byte offsets */
    int *lay = (int *)malloc(sizeof(int) * (size_t)ncodes);
    int64_t *tile_byte = (int64_t *)malloc(sizeof(int64_t) * (size_t)(Tp + 1));
    {
        int64_t i = 0, t = 0, byte = 0;
        for (int l = 0; l < n_layers; ++l) {
            const int64_t Tl = (numels[l] + OR_TILE - 1) / OR_TILE;
            for (int64_t k = 0; k < Tl * OR_TILE; ++k) lay[i++] = l;
            for (int64_t k = 0; k < Tl; ++k, ++t) { tile_byte[t] = byte; byte += 16 * (1 + e[l] + m[l]); }
        }
        for (; i < ncodes; ++i) lay[i] = n_layers - 1;
        for (; t < Tp; ++t) { tile_byte[t] = byte; byte += 16 * (1 + e[n_layers - 1] + m[n_layers - 1]); }
        tile_byte[Tp] = byte;
    }
    /* Alg. 1 lines 3-4 per layer, in the layer's format */
    int32_t *ft = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_layers);
    int nonfinite = 0;
    for (int l = 0; l < n_layers; ++l) {
        int32_t Emax = OR_EMPTY;
        for (int r = 0; r < p; ++r) {
            int32_t Er = oracle_find_max_exp(grads[(size_t)r * n_layers + l], numels[l], p);
            if (Er == OR_NONFINITE) nonfinite = 1;
            if (Er > Emax) Emax = Er;
        }
        ft[l] = oracle_scale_exp(e[l], Emax);
        if (ftilde_out) ftilde_out[l] = ft[l];
    }
    if (nonfinite) { free(lay); free(tile_byte); free(ft); return OR_ERR_NONFINITE; }
    /* lines 5-6: scale and Cast in the layer's format */
    uint32_t *q = (uint32_t *)calloc((size_t)p * (size_t)ncodes, sizeof(uint32_t));
    for (int r = 0; r < p; ++r) {
        int64_t off = 0;
        for (int l = 0; l < n_layers; ++l) {
            const float *g = grads[(size_t)r * n_layers + l];
            for (int64_t i = 0; i < numels[l]; ++i)
                q[(size_t)r * ncodes + off + i] = oracle_cast1(oracle_scale(g[i], ft[l]), e[l], m[l]);
            off += OR_TILE * ((numels[l] + OR_TILE - 1) / OR_TILE);
        }
    }
    /* line 7: the ring with a re-quantise after every add, element in its own format */
    uint32_t *s = (uint32_t *)calloc((size_t)ncodes, sizeof(uint32_t));
    for (int c = 0; c < p; ++c)
        for (int64_t i = c * chunk_codes; i < (c + 1) * chunk_codes; ++i) {
            const int l = lay[i];
            uint32_t acc = q[(size_t)((c + 1) % p) * ncodes + i];
            for (int j = 2; j <= p; ++j) acc = oracle_ring_add(acc, q[(size_t)((c + j) % p) * ncodes + i], e[l], m[l]);
            s[i] = acc;
        }
    /* O11 per tile: code k of tile t at bit k*b inside the tile's bytes */
    for (int which = 0; which <= p; ++which) {
        uint8_t *dst = which < p ? (packed_out ? packed_out + (size_t)which * (size_t)nbytes : NULL) : reduced_out;
        const uint32_t *src = which < p ? q + (size_t)which * ncodes : s;
        if (!dst) continue;
        memset(dst, 0, (size_t)nbytes);
        for (int64_t t = 0; t < Tp; ++t) {
            const int l = lay[t * OR_TILE];
            const int b = 1 + e[l] + m[l];
            oracle_pack(src + t * OR_TILE, OR_TILE, b, dst + tile_byte[t]);
        }
    }
    /* lines 8-9 */
    if (out) {
        int64_t off = 0;
        for (int l = 0; l < n_layers; ++l) {
            for (int64_t i = 0; i < numels[l]; ++i) out[l][i] = oracle_unscale1(s[off + i], ft[l], p, average, e[l], m[l]);
            off += OR_TILE * ((numels[l] + OR_TILE - 1) / OR_TILE);
        }
    }
    free(q); free(s); free(lay); free(tile_byte); free(ft);
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Stochastic rounding ("some          */
/* researchers prefer stochastic rounding ... which can get an         */
/* unbiased estimate for high precision values").  Reading A26: x     */
/* between its representable neighbours lo <= |x| < hi rounds to hi   */
/* with probability (|x| - lo) / (hi - lo), decided by a 32-bit       */
/* random number r: up iff r < (|x| - lo) / (hi - lo) * 2^32 (exact   */
/* comparison in binary64).  r comes from the counter-based generator */
/* SplitMix64 (Steele, Lea, Flood 2014): output = mix(seed + (ctr+1) * */
/* 0x9E3779B97F4A7C15), r = output >> 32, keyed by ctr = phase << 40 | */
/* i (i = the element's code index in the packed layout; phase r for  */
/* rank r's Cast, p - 1 + a for the a-th add of the element's fold),  */
/* so results do not depend on thread order.                          */
/* ------------------------------------------------------------------ */
uint64_t oracle_splitmix64(uint64_t seed, uint64_t ctr)
{
    uint64_t z = seed + (ctr + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint32_t sr_rand(uint64_t seed, uint64_t phase, int64_t i)
{
    return (uint32_t)(oracle_splitmix64(seed, (phase << 40) | (uint64_t)i) >> 32);
}

uint32_t oracle_cast_sr1(float x, int e, int m, uint32_t r)
{
    const int bias = oracle_bias(e);
    const uint32_t sbit = (signbit(x) ? 1u : 0u) << (e + m);
    const uint32_t inf_code = sbit | (((1u << e) - 1u) << m);
    if (isnan(x) || isinf(x)) return oracle_cast1(x, e, m);
    const double a = fabs((double)x);
    if (a == 0.0) return sbit;
    if (a >= ldexp(1.0, bias + 1)) return inf_code;
    int k;
    (void)frexp(a, &k);
    k -= 1;
    const int qexp = ((k > 1 - bias) ? k : (1 - bias)) - m;
    const double quantum = ldexp(1.0, qexp);
    const double lo = floor(a / quantum) * quantum;
    const double hi = lo + quantum;                   /* 2^(bias+1) stands for Inf */
    if (a == lo) return sbit | encode_magnitude(lo, e, m);
    const double frac = (a - lo) / quantum;           /* exact: quantum is a power of two */
    const int up = (double)r < frac * 4294967296.0;
    return sbit | encode_magnitude(up ? hi : lo, e, m);
}

int oracle_cast_sr(const float *x, uint32_t *codes, int64_t n, int e, int m, uint64_t seed, uint64_t phase)
{
    if (oracle_format_valid(e, m)) return OR_ERR_FORMAT;
    for (int64_t i = 0; i < n; ++i) codes[i] = oracle_cast_sr1(x[i], e, m, sr_rand(seed, phase, i));
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Reduction order and accumulator.    */
/*                                                                     */
/* NEXT-3, hierarchical all-reduce: "partition the nodes   */
/* into groups ... (1) within each group, all worker nodes send their  */
/* local gradients to the master node; (2) ring all-reduce across all  */
/* the master nodes; (3) within each group, the master node broadcasts */
/* the global gradients".  Reading A23: p ranks form G =   */
/* p/k groups of k consecutive ranks; step (1) is the ring reduce of   */
/* the group (its step count 2(k-1) of the paper's 4(k-1)+2(p/k-1),    */
/* P:528), i.e. O7/O8 applied inside the group: tile t lies in group   */
/* chunk c1 = t / (T'/k) and is accumulated over group members in      */
/* local order c1+1, ..., c1; step (2) is O8 over the G group sums:    */
/* tile t lies in master chunk c2 = t / (T'/G), accumulated over groups*/
/* c2+1, ..., c2; step (3) moves codes only.  k = 1 and k = p are the  */
/* flat ring of O8.                                                    */
/*                                                                     */
/* NEXT-4, CPD accumulator: "use a higher precision to     */
/* store the accumulator", "arbitrary low precision (<= 32 bits) for   */
/* the accumulator", "the Kahan summation algorithm".  Reading A24:    */
/* the running sum is held in the accumulator format (ae, am); every   */
/* arithmetic result is an fp32 operation re-quantised to (ae, am)     */
/* (CPD's emulation, as in O8); the first addend is cast into the      */
/* accumulator; the final sum is cast to the wire format once.  Kahan  */
/* (Higham's compensated summation): y = x - c; t = s + y;             */
/* c = (t - s) - y; s = t, each result re-quantised; c starts at 0 in  */
/* every fold (a group's compensation is not sent to its master).      */
/* ------------------------------------------------------------------ */
static float acc_q(float x, int ae, int am) { return oracle_decode1(oracle_cast1(x, ae, am), ae, am); }

/* Sum x[0..n-1] in the given order in accumulator format (ae, am). */
static float oracle_fold(const float *x, int n, int ae, int am, int kahan)
{
    float s = acc_q(x[0], ae, am);
    float c = 0.0f;
    for (int j = 1; j < n; ++j) {
        if (!kahan) {
            s = acc_q(s + x[j], ae, am);                 /* fl32 add, re-quantise */
        } else {
            const float y = acc_q(x[j] - c, ae, am);
            const float t = acc_q(s + y, ae, am);
            c = acc_q(acc_q(t - s, ae, am) - y, ae, am);
            s = t;
        }
    }
    return s;
}

/* One element's all-reduce: q[r] = rank r's wire code of the element
 * (r = 0..p-1), t = its tile, Tp = T'.  Returns the reduced wire code. */
/* The same element's all-reduce with stochastic rounding after every add
 * (wire-format accumulator, no compensation; reading A26): the a-th add of
 * the fold (a = 1..p-1, in fold order across groups) draws phase p - 1 + a. */
static uint32_t reduce1_sr(const uint32_t *q, int p, int64_t i, int64_t Tp, int group_k, int e, int m, uint64_t seed)
{
    const int k = group_k, G = p / group_k;
    const int64_t t = i / OR_TILE, c1 = t / (Tp / k), c2 = t / (Tp / G);
    int a = 0;
    float S = 0.0f;
    for (int gi = 0; gi < G; ++gi) {
        const int g = (int)((c2 + 1 + gi) % G);
        float s = oracle_decode1(q[g * k + (int)((c1 + 1) % k)], e, m);
        for (int j = 1; j < k; ++j) {
            const float x = oracle_decode1(q[g * k + (int)((c1 + 1 + j) % k)], e, m);
            ++a;
            s = oracle_decode1(oracle_cast_sr1(s + x, e, m, sr_rand(seed, (uint64_t)(p - 1 + a), i)), e, m);
        }
        if (gi == 0) {
            S = s;
        } else {
            ++a;
            S = oracle_decode1(oracle_cast_sr1(S + s, e, m, sr_rand(seed, (uint64_t)(p - 1 + a), i)), e, m);
        }
    }
    return oracle_cast1(S, e, m); /* S is a wire value: exact */
}

uint32_t oracle_reduce1(const uint32_t *q, int p, int64_t t, int64_t Tp, int group_k, int e, int m,
                        int ae, int am, int kahan)
{
    const int k = group_k, G = p / group_k;
    const int64_t c1 = t / (Tp / k), c2 = t / (Tp / G);
    float gs[256], xs[256];
    for (int gi = 0; gi < G; ++gi) {
        const int g = (int)((c2 + 1 + gi) % G);          /* masters in ring order c2+1, ..., c2 */
        for (int j = 0; j < k; ++j)                      /* members in ring order c1+1, ..., c1 */
            xs[j] = oracle_decode1(q[g * k + (int)((c1 + 1 + j) % k)], e, m);
        gs[gi] = oracle_fold(xs, k, ae, am, kahan);
    }
    return oracle_cast1(oracle_fold(gs, G, ae, am, kahan), e, m);
}

/* oracle_aps_sync with a reduction order (group_k: 1 <= k <= p, k | p,
 * p <= 256) and an accumulator format (ae, am) with optional Kahan
 * compensation.  group_k = 1 (or p), (ae, am) = (e, m), kahan = 0 is
 * oracle_aps_sync. */
int oracle_aps_sync_ex(int p, int e, int m, int n_layers, const int64_t *numels, const float *const *grads,
                       int average, int group_k, int ae, int am, int kahan, int sr, uint64_t seed,
                       int32_t *ftilde_out, uint8_t *packed_out, uint8_t *reduced_out, float *const *out)
{
    if (oracle_format_valid(e, m) || oracle_format_valid(ae, am)) return OR_ERR_FORMAT;
    if (p < 1 || p > 256 || n_layers < 1 || !numels || !grads) return OR_ERR_ARG;
    if (group_k < 1 || group_k > p || p % group_k) return OR_ERR_ARG;
    if (sr && (kahan || ae != e || am != m)) return OR_ERR_ARG; /* A26: SR with the wire accumulator only */
    for (int l = 0; l < n_layers; ++l)
        if (numels[l] < 1) return OR_ERR_ARG;
    const int b = 1 + e + m;
    const int64_t Tp = oracle_total_tiles(p, n_layers, numels);
    const int64_t ncodes = Tp * OR_TILE;
    const int64_t nbytes = 16 * (int64_t)b * Tp;

    /* Alg. 1 lines 3-4 */
    int32_t *ft = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_layers);
    int nonfinite = 0;
    for (int l = 0; l < n_layers; ++l) {
        int32_t Emax = OR_EMPTY;
        for (int r = 0; r < p; ++r) {
            int32_t Er = oracle_find_max_exp(grads[(size_t)r * n_layers + l], numels[l], p);
            if (Er == OR_NONFINITE) nonfinite = 1;
            if (Er > Emax) Emax = Er;
        }
        ft[l] = oracle_scale_exp(e, Emax);
        if (ftilde_out) ftilde_out[l] = ft[l];
    }
    if (nonfinite) { free(ft); return OR_ERR_NONFINITE; }
    /* lines 5-6 */
    uint32_t *q = (uint32_t *)calloc((size_t)p * (size_t)ncodes, sizeof(uint32_t));
    for (int r = 0; r < p; ++r) {
        int64_t off = 0;
        for (int l = 0; l < n_layers; ++l) {
            const float *g = grads[(size_t)r * n_layers + l];
            for (int64_t i = 0; i < numels[l]; ++i) {
                const float y = oracle_scale(g[i], ft[l]);
                q[(size_t)r * ncodes + off + i] =
                    sr ? oracle_cast_sr1(y, e, m, sr_rand(seed, (uint64_t)r, off + i)) : oracle_cast1(y, e, m);
            }
            off += OR_TILE * ((numels[l] + OR_TILE - 1) / OR_TILE);
        }
        if (packed_out) {
            uint8_t *pk = packed_out + (size_t)r * (size_t)nbytes;
            memset(pk, 0, (size_t)nbytes);
            oracle_pack(q + (size_t)r * ncodes, ncodes, b, pk);
        }
    }
    /* line 7 in the chosen order and accumulator */
    uint32_t *s = (uint32_t *)calloc((size_t)ncodes, sizeof(uint32_t));
    uint32_t col[256];
    for (int64_t i = 0; i < ncodes; ++i) {
        for (int r = 0; r < p; ++r) col[r] = q[(size_t)r * ncodes + i];
        s[i] = sr ? reduce1_sr(col, p, i, Tp, group_k, e, m, seed)
                  : oracle_reduce1(col, p, i / OR_TILE, Tp, group_k, e, m, ae, am, kahan);
    }
    if (reduced_out) {
        memset(reduced_out, 0, (size_t)nbytes);
        oracle_pack(s, ncodes, b, reduced_out);
    }
    /* lines 8-9 */
    if (out) {
        int64_t off = 0;
        for (int l = 0; l < n_layers; ++l) {
            for (int64_t i = 0; i < numels[l]; ++i) out[l][i] = oracle_unscale1(s[off + i], ft[l], p, average, e, m);
            off += OR_TILE * ((numels[l] + OR_TILE - 1) / OR_TILE);
        }
    }
    free(q); free(s); free(ft);
    return OR_OK;
}

/* Eq. (5) `equation:round_off_error`:
 *   average_round_off_error = sum_i |(grad_h_i - grad_l_i) / grad_h_i| / N.
 * Reading A25: terms with grad_h_i = 0 are undefined and are left out of
 * both the sum and N ("N elements" counts the defined terms); the sum is
 * taken in binary64, in index order.  *count_out receives that N. */
double oracle_round_off_error(const float *h, const float *l, int64_t n, int64_t *count_out)
{
    double sum = 0.0;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (h[i] == 0.0f) continue;
        sum += fabs(((double)h[i] - (double)l[i]) / (double)h[i]);
        ++cnt;
    }
    if (count_out) *count_out = cnt;
    return cnt ? sum / (double)cnt : 0.0;
}

/* ------------------------------------------------------------------ */
/* Underflow / overflow census (section 3.1 "The   */
/* limitation of the loss scaling algorithm" P:173-179, Fig.           */
/* `aps_comparing` P:277-280: "scale all gradients by 2^-5 ... Although */
/* it can avoid overflow, it will cause some small values to underflow, */
/* which will be cast to 0"; section 3.3.2 the underflow/overflow       */
/* trade-off).  For a tensor g and a scale exponent s (APS: f~_l; loss  */
/* scaling: one constant for every layer; no scaling: 0), count the     */
/* nonzero finite elements whose Cast(g * 2^s) is +-0 (underflow) and   */
/* those whose Cast is +-Inf (overflow).                                */
/* ------------------------------------------------------------------ */
int oracle_census(const float *g, int64_t n, int32_t s, int e, int m, int64_t *underflow, int64_t *overflow)
{
    if (oracle_format_valid(e, m)) return OR_ERR_FORMAT;
    if (n < 0 || (n > 0 && !g) || !underflow || !overflow) return OR_ERR_ARG;
    const uint32_t mag_mask = (uint32_t)((1ull << (e + m)) - 1ull);
    const uint32_t inf_mag = ((1u << e) - 1u) << m;
    int64_t u = 0, o = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (g[i] == 0.0f || !isfinite(g[i])) continue;
        const uint32_t c = oracle_cast1(oracle_scale(g[i], s), e, m) & mag_mask;
        if (c == 0u) ++u;
        else if (c == inf_mag) ++o;
    }
    *underflow = u;
    *overflow = o;
    return OR_OK;
}
