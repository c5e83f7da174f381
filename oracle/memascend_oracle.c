/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see memascend_oracle.h).
 *
 * CPU restatement of the MemAscend reference hot path.  Each function cites
 * the reference file:line it restates (paths relative to /root/reference).
 * Compiled with -ffp-contract=off like the reference (proj/CMakeLists.txt:13)
 * so every fp32 expression rounds once per operation, in source order.
 */
#define _GNU_SOURCE
#include "memascend_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static inline uint32_t f2u(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}
static inline float u2f(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* Round x >> sh to nearest, ties to even (sh >= 1). */
static inline uint32_t rne_shift(uint32_t x, unsigned sh) {
    const uint32_t q = x >> sh;
    const uint32_t rem = x & ((1u << sh) - 1u);
    const uint32_t half = 1u << (sh - 1u);
    return q + (rem > half || (rem == half && (q & 1u)));
}

/* ------------------------------------------------------------------ */
/* proj/include/memascend/halfprec.hpp:25-32 — RNE, NaN quieted by 0x0040 */
uint16_t ora_bf16_from_float(float f) {
    const uint32_t u = f2u(f);
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x0040u);
    return (uint16_t)(rne_shift(u & 0x7FFFFFFFu, 16) | ((u >> 16) & 0x8000u));
}

/* halfprec.hpp:34-36 — exact widening */
float ora_bf16_to_float(uint16_t h) { return u2f((uint32_t)h << 16); }

/* halfprec.hpp:38-74 — RNE with half subnormals; NaN -> sign|0x7E00,
 * |f| >= 65520 -> inf, |f| < 2^-25 (and the 2^-25 tie) -> signed zero. */
uint16_t ora_fp16_from_float(float f) {
    const uint32_t u = f2u(f);
    const uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
    const uint32_t a = u & 0x7FFFFFFFu;
    if (a > 0x7F800000u) return sign | 0x7E00u;
    if (a >= 0x477FF000u) return sign | 0x7C00u;  /* inf or rounds past 65504 */
    if (a >= 0x38800000u) {                          /* half normal: rebias 127->15 */
        return sign | (uint16_t)rne_shift(a - (112u << 23), 13);
    }
    if (a < 0x33000000u) return sign;                /* below half the min subnormal */
    /* half subnormal: value = mant * 2^(e-150), unit 2^-24 -> shift 126-e. */
    return sign | (uint16_t)rne_shift((a & 0x007FFFFFu) | 0x00800000u, 126u - (a >> 23));
}

/* halfprec.hpp:76-99 — exact widening */
float ora_fp16_to_float(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t e = (h >> 10) & 0x1Fu;
    const uint32_t mant = h & 0x3FFu;
    if (e == 0x1Fu) return u2f(sign | 0x7F800000u | (mant << 13));
    if (e != 0) return u2f(sign | ((e + 112u) << 23) | (mant << 13));
    if (mant == 0) return u2f(sign);
    /* subnormal: mant * 2^-24 is exact in fp32 */
    const float mag = (float)mant * 0x1p-24f;
    return u2f(sign | f2u(mag));
}

static inline uint16_t narrow(float f, int kind) {
    return kind == ORA_BF16 ? ora_bf16_from_float(f) : ora_fp16_from_float(f);
}
static inline float widen(uint16_t h, int kind) {
    return kind == ORA_BF16 ? ora_bf16_to_float(h) : ora_fp16_to_float(h);
}

void ora_cast_from_f32(const float* src, uint16_t* dst, uint64_t n, int kind) {
    for (uint64_t i = 0; i < n; ++i) dst[i] = narrow(src[i], kind);
}

void ora_widen_to_f32(const uint16_t* src, float* dst, uint64_t n, int kind) {
    for (uint64_t i = 0; i < n; ++i) dst[i] = widen(src[i], kind);
}

/* ------------------------------------------------------------------ */
uint64_t ora_fnv1a64_continue(uint64_t h, const void* data, uint64_t bytes) {
    const unsigned char* p = (const unsigned char*)data;
    for (uint64_t i = 0; i < bytes; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

/* proj/src/simulator.cpp:182-192 (fnv1a_hex) */
uint64_t ora_fnv1a64(const void* data, uint64_t bytes) {
    return ora_fnv1a64_continue(1469598103934665603ull, data, bytes);
}

typedef struct {
    int kind;
    int block_log2;
    uint64_t first_block, last_block;
    uint64_t* out;
} sweep_job;

static void* sweep_worker(void* arg) {
    sweep_job* j = (sweep_job*)arg;
    const uint64_t bs = 1ull << j->block_log2;
    for (uint64_t b = j->first_block; b < j->last_block; ++b) {
        uint64_t h = 1469598103934665603ull;
        for (uint64_t k = 0; k < bs; ++k) {
            const uint32_t u = (uint32_t)(b * bs + k);
            const uint16_t r = narrow(u2f(u), j->kind);
            h = ora_fnv1a64_continue(h, &r, 2);
        }
        j->out[b] = h;
    }
    return NULL;
}

void ora_cast_sweep_checksums(int kind, int block_log2, uint64_t* out, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    const uint64_t nblocks = 1ull << (32 - block_log2);
    pthread_t tid[256];
    sweep_job jobs[256];
    const uint64_t per = (nblocks + (uint64_t)threads - 1) / (uint64_t)threads;
    int launched = 0;
    for (int t = 0; t < threads; ++t) {
        const uint64_t b0 = (uint64_t)t * per;
        uint64_t b1 = b0 + per;
        if (b1 > nblocks) b1 = nblocks;
        if (b0 >= b1) break;
        jobs[t] = (sweep_job){kind, block_log2, b0, b1, out};
        pthread_create(&tid[t], NULL, sweep_worker, &jobs[t]);
        ++launched;
    }
    for (int t = 0; t < launched; ++t) pthread_join(tid[t], NULL);
}

/* ------------------------------------------------------------------ */
/* proj/include/memascend/overflow.hpp:46-51 (kExpAllOnesMask = 0x7F800000).
 * The 16-bit forms use the same rule on their exponent fields; bf16 widening
 * is a shift (halfprec.hpp:34-36) so 0x7F80 is the widened fp32 mask. */
int ora_bits_non_finite_f32(uint32_t bits) { return (bits & 0x7F800000u) == 0x7F800000u; }
int ora_bits_non_finite_bf16(uint16_t bits) { return (bits & 0x7F80u) == 0x7F80u; }
int ora_bits_non_finite_f16(uint16_t bits) { return (bits & 0x7C00u) == 0x7C00u; }

/* proj/src/overflow.cpp:45-69 (chunk scan) and :73-145 (whole-buffer
 * decision).  The reference's worker/chunk/early-exit schedule does not
 * change the answer (test_overflow.cpp:127-145); this is the sequential
 * schedule with the first index tracked. */
int ora_overflow_check(const void* data, uint64_t n, int kind, uint64_t* first_index) {
    uint64_t first = UINT64_MAX;
    for (uint64_t i = 0; i < n; ++i) {
        int bad;
        if (kind == ORA_F32) {
            bad = ora_bits_non_finite_f32(((const uint32_t*)data)[i]);
        } else if (kind == ORA_BF16) {
            bad = ora_bits_non_finite_bf16(((const uint16_t*)data)[i]);
        } else {
            bad = ora_bits_non_finite_f16(((const uint16_t*)data)[i]);
        }
        if (bad) {
            first = i;
            break;
        }
    }
    if (first_index) *first_index = first;
    return first != UINT64_MAX;
}

/* ------------------------------------------------------------------ */
/* proj/src/optimizer.cpp:20-24: bc = 1 - powf(beta, (float)t) (glibc) */
void ora_step_scalars(uint64_t t, float beta1, float beta2, float* bc1, float* bc2) {
    volatile float tf = (float)t; /* keep the call out of constant folding */
    *bc1 = 1.0f - powf(beta1, tf);
    *bc2 = 1.0f - powf(beta2, tf);
}

static inline float load_grad(const void* g, int kind, uint64_t i) {
    if (kind == ORA_F32) return ((const float*)g)[i];
    return widen(((const uint16_t*)g)[i], kind);
}

/* x86 SSE NaN results (Intel SDM Vol. 1 §4.8.3.5, Table 4-7), made explicit
 * so they do not depend on the operand order THIS compiler picks: a NaN
 * operand propagates quieted (bit 22 set) — the first source operand if it
 * is a NaN, else the second — and an invalid operation on non-NaN operands
 * gives the default NaN 0xFFC00000.  `a` is the first source operand of the
 * instruction in the reference's compiled adam_range (objdump of optimizer.o
 * built with the reference flags; see ORD_* below). */
static inline int isnan_bits(uint32_t u) { return (u & 0x7FFFFFFFu) > 0x7F800000u; }
static inline float x86r(float r, float a, float b) {
    if (r == r) return r;
    if (isnan_bits(f2u(a))) return u2f(f2u(a) | 0x00400000u);
    if (isnan_bits(f2u(b))) return u2f(f2u(b) | 0x00400000u);
    return u2f(0xFFC00000u);
}
static inline float x86_sqrt(float x) {
    const float r = sqrtf(x);
    if (r == r) return r;
    return isnan_bits(f2u(x)) ? u2f(f2u(x) | 0x00400000u) : u2f(0xFFC00000u);
}

/* The two instantiations of adam_range order their commutative operands
 * differently (optimizer.cpp:35-39 as compiled by g++ -O3):
 *   ORD_FP32 (Fp32Access):  m*b1, (1-b1)*g, b2*v, (1-b2)*gg, vb + va, q*lr, lrwd*p
 *   ORD_BF16 (Bf16Access):  m*b1, g*(1-b1), v*b2, gg*(1-b2), va + vb, q*lr, lrwd*p */
enum { ORD_FP32 = 0, ORD_BF16 = 1 };

/* One element, operation order of proj/src/optimizer.cpp:31-39. */
static inline void adam_elem_ord(float* pp, float* mp, float* vp, float gs, const ora_hyper* h,
                                 float loss_scale, float bc1, float bc2, int ord) {
    const float g = x86r(gs / loss_scale, gs, loss_scale);
    float p = *pp, m = *mp, v = *vp;
    const float one_m_b1 = 1.0f - h->beta1;
    const float one_m_b2 = 1.0f - h->beta2;
    const float m_a = x86r(m * h->beta1, m, h->beta1);
    const float m_b = ord == ORD_FP32 ? x86r(one_m_b1 * g, one_m_b1, g) : x86r(g * one_m_b1, g, one_m_b1);
    m = x86r(m_a + m_b, m_a, m_b);
    const float gg = x86r(g * g, g, g);
    const float v_a = ord == ORD_FP32 ? x86r(h->beta2 * v, h->beta2, v) : x86r(v * h->beta2, v, h->beta2);
    const float v_b = ord == ORD_FP32 ? x86r(one_m_b2 * gg, one_m_b2, gg) : x86r(gg * one_m_b2, gg, one_m_b2);
    v = ord == ORD_FP32 ? x86r(v_b + v_a, v_b, v_a) : x86r(v_a + v_b, v_a, v_b);
    const float mh = x86r(m / bc1, m, bc1);
    const float vh = x86r(v / bc2, v, bc2);
    const float sq = x86_sqrt(vh);
    const float den = x86r(sq + h->eps, sq, h->eps);
    const float q = x86r(mh / den, mh, den);
    const float step = x86r(q * h->lr, q, h->lr);
    const float lrwd = h->lr * h->weight_decay;
    const float decay = x86r(lrwd * p, lrwd, p);
    p = x86r(p - step, p, step);
    p = x86r(p - decay, p, decay);
    *pp = p;
    *mp = m;
    *vp = v;
}

static inline void adam_elem(float* pp, float* mp, float* vp, float gs, const ora_hyper* h,
                             float loss_scale, float bc1, float bc2) {
    adam_elem_ord(pp, mp, vp, gs, h, loss_scale, bc1, bc2, ORD_FP32);
}

/* optimizer.cpp:26-44 (adam_range), 46-69 (t == 0 check), 103-109
 * (adam_step_fp32), fused with the shadow refresh of simulator.cpp:461-467. */
int ora_adam_step(float* p, float* m, float* v, const void* g, int g_kind, uint64_t n,
                  uint64_t t, const ora_hyper* h, float loss_scale, void* w_out, int w_kind) {
    if (t == 0) return 1;
    float bc1, bc2;
    ora_step_scalars(t, h->beta1, h->beta2, &bc1, &bc2);
    for (uint64_t i = 0; i < n; ++i) {
        adam_elem(&p[i], &m[i], &v[i], load_grad(g, g_kind, i), h, loss_scale, bc1, bc2);
        if (w_out && w_kind != ORA_NONE) ((uint16_t*)w_out)[i] = narrow(p[i], w_kind);
    }
    return 0;
}

/* optimizer.cpp:83-93 (Bf16Access) + 111-118 (adam_step_bf16) */
int ora_adam_step_bf16(uint16_t* p, uint16_t* m, uint16_t* v, const float* g, uint64_t n,
                       uint64_t t, const ora_hyper* h, float loss_scale) {
    if (t == 0) return 1;
    float bc1, bc2;
    ora_step_scalars(t, h->beta1, h->beta2, &bc1, &bc2);
    for (uint64_t i = 0; i < n; ++i) {
        float pf = ora_bf16_to_float(p[i]);
        float mf = ora_bf16_to_float(m[i]);
        float vf = ora_bf16_to_float(v[i]);
        adam_elem_ord(&pf, &mf, &vf, g[i], h, loss_scale, bc1, bc2, ORD_BF16);
        p[i] = ora_bf16_from_float(pf);
        m[i] = ora_bf16_from_float(mf);
        v[i] = ora_bf16_from_float(vf);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* optimizer.hpp:24-34 */
void ora_scaler_on_overflow(ora_scaler* s) {
    s->scale = s->scale * 0.5f;
    s->clean_steps = 0;
}

void ora_scaler_on_clean_step(ora_scaler* s) {
    s->clean_steps += 1;
    if (s->clean_steps >= s->growth_interval) {
        s->scale = s->scale * 2.0f;
        s->clean_steps = 0;
    }
}

/* ------------------------------------------------------------------ */
/* proj/include/memascend/simulator.hpp:23-28 */
uint64_t ora_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* top 24 bits -> uniform [-0.5, 0.5) (exact in fp32) */
static inline float unit24(uint64_t h) { return (float)(h >> 40) * (1.0f / 16777216.0f) - 0.5f; }

/* simulator.hpp:30-36 */
float ora_pseudo_gradient(uint64_t seed, uint64_t step, uint64_t index, float weight) {
    const uint64_t h = ora_splitmix64(seed ^ ora_splitmix64(step) ^ index);
    const float r = unit24(h);
    const float a = 0.25f * r;
    const float b = 0.03125f * weight;
    return a + b;
}

/* simulator.hpp:39-42 */
float ora_seeded_weight(uint64_t seed, uint64_t index) {
    const uint64_t h = ora_splitmix64(seed ^ ora_splitmix64(index ^ 0xA5A5A5A5ull));
    return unit24(h) * 0.2f;
}

/* ------------------------------------------------------------------ */
static int cfg_valid(const ora_train_cfg* c) {
    if (c->n == 0) return -1;
    if (c->g_kind != ORA_F32 && c->g_kind != ORA_BF16) return -2;
    if (c->w_kind != ORA_F16 && c->w_kind != ORA_BF16) return -3;
    if (!c->mixed && c->w_kind != ORA_BF16) return -4;
    return 0;
}

/* Scaled gradient as stored in the flat buffer (simulator.cpp:402-404, with
 * the BASELINE configs' bf16 rounding when g_kind == ORA_BF16). */
static inline uint32_t stored_grad_bits(const ora_train_cfg* c, uint64_t step, uint64_t gi,
                                        float w, float scale) {
    const float pg = ora_pseudo_gradient(c->seed, step, gi, w);
    const float gs = pg * scale;
    return c->g_kind == ORA_F32 ? f2u(gs) : (uint32_t)ora_bf16_from_float(gs);
}

static inline float grad_value(int g_kind, uint32_t bits) {
    return g_kind == ORA_F32 ? u2f(bits) : ora_bf16_to_float((uint16_t)bits);
}

/* proj/src/simulator.cpp:427-492 composition, checked against the
 * in-memory reference trainer (proj/tests/reference_trainer.hpp:27-106). */
int ora_train(const ora_train_cfg* c, ora_train_out* out) {
    const int bad = cfg_valid(c);
    if (bad) return bad;
    const uint64_t n = c->n;
    float* p = (float*)malloc(n * 4);
    float* m = (float*)calloc(n, 4);
    float* v = (float*)calloc(n, 4);
    uint16_t* w = (uint16_t*)malloc(n * 2);
    uint16_t* m16 = (uint16_t*)calloc(n, 2);
    uint16_t* v16 = (uint16_t*)calloc(n, 2);
    uint32_t* gbits = (uint32_t*)malloc(n * 4);
    if (!p || !m || !v || !w || !m16 || !v16 || !gbits) {
        free(p); free(m); free(v); free(w); free(m16); free(v16); free(gbits);
        return -10;
    }
    for (uint64_t i = 0; i < n; ++i) {
        const float w0 = ora_seeded_weight(c->seed, c->base + i);
        p[i] = w0;
        w[i] = narrow(w0, c->w_kind);
    }
    ora_scaler sc = c->scaler;
    uint64_t updates = 0;
    for (uint64_t step = 0; step < c->steps; ++step) {
        for (uint64_t i = 0; i < n; ++i) {
            gbits[i] = stored_grad_bits(c, step, c->base + i, widen(w[i], c->w_kind), sc.scale);
        }
        for (uint64_t f = 0; f < c->n_faults; ++f) {
            if (c->faults[f].step == step) {
                const uint32_t b = c->faults[f].bits;
                gbits[c->faults[f].index % n] = c->g_kind == ORA_F32 ? b : (b & 0xFFFFu);
            }
        }
        int local = 0;
        for (uint64_t i = 0; i < n && !local; ++i) {
            local = c->g_kind == ORA_F32 ? ora_bits_non_finite_f32(gbits[i])
                                         : ora_bits_non_finite_bf16((uint16_t)gbits[i]);
        }
        if (out && out->overflow) out->overflow[step] = (uint8_t)local;
        const int skip = c->forced_overflow ? c->forced_overflow[step] != 0 : local;
        if (skip) {
            ora_scaler_on_overflow(&sc);
        } else {
            updates += 1;
            float bc1, bc2;
            ora_step_scalars(updates, c->hyper.beta1, c->hyper.beta2, &bc1, &bc2);
            const float scale_now = sc.scale;
            for (uint64_t i = 0; i < n; ++i) {
                const float gs = grad_value(c->g_kind, gbits[i]);
                if (c->mixed) {
                    adam_elem(&p[i], &m[i], &v[i], gs, &c->hyper, scale_now, bc1, bc2);
                    w[i] = narrow(p[i], c->w_kind);
                } else {
                    float pf = ora_bf16_to_float(w[i]);
                    float mf = ora_bf16_to_float(m16[i]);
                    float vf = ora_bf16_to_float(v16[i]);
                    adam_elem_ord(&pf, &mf, &vf, gs, &c->hyper, scale_now, bc1, bc2, ORD_BF16);
                    w[i] = ora_bf16_from_float(pf);
                    m16[i] = ora_bf16_from_float(mf);
                    v16[i] = ora_bf16_from_float(vf);
                }
            }
            ora_scaler_on_clean_step(&sc);
        }
        if (out && out->scale_after) out->scale_after[step] = sc.scale;
    }
    if (out) {
        if (out->p) memcpy(out->p, p, n * 4);
        if (out->m) memcpy(out->m, m, n * 4);
        if (out->v) memcpy(out->v, v, n * 4);
        if (out->w) memcpy(out->w, w, n * 2);
        if (out->m16) memcpy(out->m16, m16, n * 2);
        if (out->v16) memcpy(out->v16, v16, n * 2);
        out->final_scale = sc.scale;
        out->updates = updates;
    }
    free(p); free(m); free(v); free(w); free(m16); free(v16); free(gbits);
    return 0;
}

int ora_train_sample(const ora_train_cfg* c, const uint64_t* idx, uint64_t k,
                     const uint8_t* decisions, float* po, float* mo, float* vo, uint16_t* wo) {
    const int bad = cfg_valid(c);
    if (bad) return bad;
    /* pure-bf16 mode (simulator.cpp:470-486): bf16 weights / m / v per
     * element, the same route as ora_train's !mixed branch; outputs are the
     * exact fp32 widenings of the bf16 state (wo = the weight bits) */
    if (!c->mixed && c->w_kind != ORA_BF16) return -5;
    /* the scale / t sequence is fixed by the decisions */
    float* scales = (float*)malloc((c->steps + 1) * sizeof(float));
    uint64_t* tsteps = (uint64_t*)malloc((c->steps + 1) * sizeof(uint64_t));
    float* bc1s = (float*)malloc((c->steps + 1) * sizeof(float));
    float* bc2s = (float*)malloc((c->steps + 1) * sizeof(float));
    ora_scaler sc = c->scaler;
    uint64_t updates = 0;
    for (uint64_t s = 0; s < c->steps; ++s) {
        scales[s] = sc.scale;
        if (decisions[s]) {
            ora_scaler_on_overflow(&sc);
            tsteps[s] = 0;
        } else {
            updates += 1;
            tsteps[s] = updates;
            ora_step_scalars(updates, c->hyper.beta1, c->hyper.beta2, &bc1s[s], &bc2s[s]);
            ora_scaler_on_clean_step(&sc);
        }
    }
    for (uint64_t j = 0; j < k; ++j) {
        const uint64_t gi = idx[j];
        float p = ora_seeded_weight(c->seed, gi), m = 0.0f, v = 0.0f;
        uint16_t w = narrow(p, c->w_kind);
        uint16_t m16 = 0, v16 = 0;
        for (uint64_t s = 0; s < c->steps; ++s) {
            if (decisions[s]) continue;
            const uint32_t b = stored_grad_bits(c, s, gi, widen(w, c->w_kind), scales[s]);
            if (c->mixed) {
                adam_elem(&p, &m, &v, grad_value(c->g_kind, b), &c->hyper, scales[s], bc1s[s],
                          bc2s[s]);
                w = narrow(p, c->w_kind);
            } else {
                float pf = ora_bf16_to_float(w);
                float mf = ora_bf16_to_float(m16);
                float vf = ora_bf16_to_float(v16);
                adam_elem_ord(&pf, &mf, &vf, grad_value(c->g_kind, b), &c->hyper, scales[s],
                              bc1s[s], bc2s[s], ORD_BF16);
                w = ora_bf16_from_float(pf);
                m16 = ora_bf16_from_float(mf);
                v16 = ora_bf16_from_float(vf);
            }
        }
        if (!c->mixed) {
            p = ora_bf16_to_float(w);
            m = ora_bf16_to_float(m16);
            v = ora_bf16_to_float(v16);
        }
        if (po) po[j] = p;
        if (mo) mo[j] = m;
        if (vo) vo[j] = v;
        if (wo) wo[j] = w;
    }
    free(scales); free(tsteps); free(bc1s); free(bc2s);
    return 0;
}

/* ------------------------------------------------------------------ */
/* std::mt19937_64 (the engine the reference tests draw inputs from). */
void ora_mt64_seed(ora_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i) {
        s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    s->idx = 312;
}

uint64_t ora_mt64_next(ora_mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t y = (s->mt[i] & 0xFFFFFFFF80000000ull) |
                               (s->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t x = s->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ull) x ^= 0xB5026F5AA96619E9ull;
            s->mt[i] = x;
        }
        s->idx = 0;
    }
    uint64_t z = s->mt[s->idx++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

/* proj/tests/test_overflow.cpp:30-58.  Draw order pinned against the
 * reference build by tests/golden (adversarial.json buffer digests). */
void ora_adversarial_buffer(ora_mt64* rng, uint32_t* out, uint64_t n, int inject_bad) {
    for (uint64_t i = 0; i < n; ++i) {
        switch (ora_mt64_next(rng) % 8) {
            case 0: out[i] = 0x00000000u; break;
            case 1: out[i] = 0x80000000u; break;
            case 2: out[i] = 0x00000001u; break;
            case 3: out[i] = 0x807FFFFFu; break;
            case 4: out[i] = 0x7F7FFFFFu; break;
            case 5: out[i] = f2u(-1.17549435e-38f); break;
            default: {
                const uint32_t u = (uint32_t)ora_mt64_next(rng);
                const float x = (float)(int32_t)u;
                out[i] = f2u(x * 1e-3f);
                break;
            }
        }
    }
    if (inject_bad && n > 0) {
        static const uint32_t bad[5] = {0x7F800000u, 0xFF800000u, 0x7F800001u, 0x7FC00000u,
                                        0xFFC01234u};
        /* GCC evaluates the call's arguments right to left here: the
         * pattern draw happens before the index draw. */
        const uint64_t which = ora_mt64_next(rng) % 5;
        const uint64_t where = ora_mt64_next(rng) % n;
        out[where] = bad[which];
    }
}

/* ------------------------------------------------------------------ */
/* Bulk fills (CPU baseline inputs); elementwise, so thread splits do not
 * change the values. */
typedef struct {
    int what;
    float* p;
    uint16_t* w;
    void* g;
    float* g32;
    const uint16_t* wr;
    uint64_t lo, hi, base, seed, step;
    float scale;
    int g_kind, w_kind;
} fill_job;

static void* fill_worker(void* arg) {
    fill_job* j = (fill_job*)arg;
    for (uint64_t i = j->lo; i < j->hi; ++i) {
        if (j->what == 0) {
            const float x = ora_seeded_weight(j->seed, j->base + i);
            if (j->p) j->p[i] = x;
            if (j->w) j->w[i] = narrow(x, j->w_kind);
        } else {
            const float pg = ora_pseudo_gradient(j->seed, j->step, j->base + i,
                                                 widen(j->wr[i], j->w_kind));
            const float gs = pg * j->scale;
            float wide = gs;
            if (j->g_kind == ORA_F32) {
                if (j->g) ((float*)j->g)[i] = gs;
            } else {
                const uint16_t b = ora_bf16_from_float(gs);
                if (j->g) ((uint16_t*)j->g)[i] = b;
                wide = ora_bf16_to_float(b);
            }
            if (j->g32) j->g32[i] = wide;
        }
    }
    return NULL;
}

static void run_fill(fill_job proto, uint64_t n, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    fill_job jobs[256];
    const uint64_t per = (n + (uint64_t)threads - 1) / (uint64_t)threads;
    int k = 0;
    for (int t = 0; t < threads; ++t) {
        const uint64_t lo = (uint64_t)t * per;
        const uint64_t hi = lo + per < n ? lo + per : n;
        if (lo >= hi) break;
        jobs[t] = proto;
        jobs[t].lo = lo;
        jobs[t].hi = hi;
        pthread_create(&tid[t], NULL, fill_worker, &jobs[t]);
        ++k;
    }
    for (int t = 0; t < k; ++t) pthread_join(tid[t], NULL);
}

void ora_fill_weights(float* p, uint16_t* w, uint64_t n, uint64_t base, uint64_t seed, int w_kind,
                      int threads) {
    fill_job j;
    memset(&j, 0, sizeof j);
    j.what = 0; j.p = p; j.w = w; j.base = base; j.seed = seed; j.w_kind = w_kind;
    run_fill(j, n, threads);
}

void ora_fill_grads(void* g, float* g32, const uint16_t* w, uint64_t n, uint64_t base,
                    uint64_t seed, uint64_t step, float scale, int g_kind, int w_kind, int threads) {
    fill_job j;
    memset(&j, 0, sizeof j);
    j.what = 1; j.g = g; j.g32 = g32; j.wr = w; j.base = base; j.seed = seed; j.step = step;
    j.scale = scale; j.g_kind = g_kind; j.w_kind = w_kind;
    run_fill(j, n, threads);
}

/* ------------------------------------------------------------------ */
/* Gradient reduce-scatter with the overflow check in its epilogue (SURVEY
 * §8(f) row 2).  No reference counterpart exists for the sum (the reference
 * is single-process); its output feeds the reference's flat gradient buffer
 * (simulator.cpp:401-405) and the check is overflow.hpp:46-51 applied to the
 * STORED values.  Defined order: acc = src[0][i], acc += src[r][i] for
 * r = 1.. in rank order (fp32, one rounding each), then acc *= post_scale
 * when post_scale != 1; a NaN result is stored as the canonical quiet NaN
 * (0x7FC00000 before narrowing) so the bits do not depend on which NaN the
 * hardware propagates. */
int ora_reduce_check(const void* const* srcs, int nsrc, int src_kind, uint64_t n,
                     float post_scale, int dst_kind, void* dst) {
    int any = 0;
    for (uint64_t i = 0; i < n; ++i) {
        float acc = load_grad(srcs[0], src_kind, i);
        for (int r = 1; r < nsrc; ++r) acc = acc + load_grad(srcs[r], src_kind, i);
        if (post_scale != 1.0f) acc = acc * post_scale;
        if (acc != acc) acc = u2f(0x7FC00000u);
        if (dst_kind == ORA_F32) {
            ((float*)dst)[i] = acc;
            any |= ora_bits_non_finite_f32(f2u(acc));
        } else {
            const uint16_t h = narrow(acc, dst_kind);
            ((uint16_t*)dst)[i] = h;
            any |= dst_kind == ORA_BF16 ? ora_bits_non_finite_bf16(h) : ora_bits_non_finite_f16(h);
        }
    }
    return any;
}
