/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the MemAscend reference hot path (arXiv 2505.23254,
 * /root/reference/proj).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker.  The product (paper_2505_23254_b200) never links it.
 *
 * Parity status: PINNED.  Every function below is checked in tests/ against
 * (a) golden vectors produced by the unmodified reference compiled from
 *     /root/reference/proj/src (oracle/_ref, see oracle/Makefile and
 *     tests/golden/make_golden.py), and
 * (b) the reference's own known-answer tests (test_overflow.cpp,
 *     test_optimizer.cpp, test_simulator.cpp), which oracle/Makefile builds and
 *     runs unmodified against the reference library.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math (the reference
 * compiles with -ffp-contract=off, proj/CMakeLists.txt:13).
 */
#ifndef MEMASCEND_ORACLE_H
#define MEMASCEND_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- element kinds ---------------------------------------------------- */
enum { ORA_F32 = 0, ORA_BF16 = 1, ORA_F16 = 2, ORA_NONE = 3 };

/* ---- half precision (proj/include/memascend/halfprec.hpp) ------------- */
uint16_t ora_bf16_from_float(float f);   /* halfprec.hpp:25-32 */
float ora_bf16_to_float(uint16_t h);     /* halfprec.hpp:34-36 */
uint16_t ora_fp16_from_float(float f);   /* halfprec.hpp:38-74 */
float ora_fp16_to_float(uint16_t h);     /* halfprec.hpp:76-99 */

/* Bulk casts; kind = ORA_BF16 or ORA_F16. */
void ora_cast_from_f32(const float* src, uint16_t* dst, uint64_t n, int kind);
void ora_widen_to_f32(const uint16_t* src, float* dst, uint64_t n, int kind);

/* FNV-1a-64 checksum of every 2^block_log2 consecutive conversion results of
 * all 2^32 fp32 bit patterns (kind = ORA_BF16 / ORA_F16).  out has
 * 2^(32-block_log2) entries.  Multi-threaded. */
void ora_cast_sweep_checksums(int kind, int block_log2, uint64_t* out, int threads);

/* ---- overflow check (proj/include/memascend/overflow.hpp,
 *                      proj/src/overflow.cpp) ------------------------------ */
/* overflow.hpp:46-51: non-finite iff every exponent bit is set. */
int ora_bits_non_finite_f32(uint32_t bits);
int ora_bits_non_finite_bf16(uint16_t bits);
int ora_bits_non_finite_f16(uint16_t bits);

/* overflow.cpp:45-145 restated sequentially: returns 1 on overflow.  When
 * first_index != NULL it receives the lowest offending index (or
 * UINT64_MAX), matching track_first_index with early_exit=false. */
int ora_overflow_check(const void* data, uint64_t n, int kind, uint64_t* first_index);

/* Reduce-scatter epilogue form of the check: dst[i] =
 * post_scale * (src[0][i] + src[1][i] + ...) in fp32, rank order, NaN stored
 * canonical; returns 1 when any stored value is non-finite. */
int ora_reduce_check(const void* const* srcs, int nsrc, int src_kind, uint64_t n,
                     float post_scale, int dst_kind, void* dst);

/* ---- Adam (proj/include/memascend/optimizer.hpp, proj/src/optimizer.cpp) */
typedef struct {
    float lr, beta1, beta2, eps, weight_decay; /* AdamHyper, optimizer.hpp:9-15 */
} ora_hyper;

/* optimizer.cpp:20-24 — glibc powf on the host. */
void ora_step_scalars(uint64_t t, float beta1, float beta2, float* bc1, float* bc2);

/* optimizer.cpp:26-44 + 103-109 + the fp16/bf16 shadow refresh of
 * simulator.cpp:461-467.  Grads may be f32/bf16/f16 (widened exactly); the
 * working-weight output (w_out, kind w_kind) may be ORA_NONE.  Returns 0, or
 * 1 for the reference's invalid_argument (t == 0). */
int ora_adam_step(float* p, float* m, float* v, const void* g, int g_kind, uint64_t n,
                  uint64_t t, const ora_hyper* h, float loss_scale, void* w_out, int w_kind);

/* optimizer.cpp:83-93,111-118: bf16 state, each quantity rounded on store. */
int ora_adam_step_bf16(uint16_t* p, uint16_t* m, uint16_t* v, const float* g, uint64_t n,
                       uint64_t t, const ora_hyper* h, float loss_scale);

/* ---- LossScaler (optimizer.hpp:19-35) ---------------------------------- */
typedef struct {
    float scale;
    uint32_t growth_interval;
    uint32_t clean_steps;
} ora_scaler;
void ora_scaler_on_overflow(ora_scaler* s);
void ora_scaler_on_clean_step(ora_scaler* s);

/* ---- workload generators (proj/include/memascend/simulator.hpp:23-42) -- */
uint64_t ora_splitmix64(uint64_t x);
float ora_pseudo_gradient(uint64_t seed, uint64_t step, uint64_t index, float weight);
float ora_seeded_weight(uint64_t seed, uint64_t index);

/* ---- step composition (simulator.cpp:427-492; reference_trainer.hpp:27-106)
 * One training run over a flat partition of n elements starting at global
 * index `base` (so a rank's shard reproduces the same elements as the whole).
 *   mixed = 1: fp32 master/m/v, fp16 shadows (reference mixed mode);
 *   w_kind selects the shadow format (ORA_F16 reference, ORA_BF16 configs);
 *   g_kind = ORA_F32 stores scaled grads as fp32 (reference flat buffer),
 *            ORA_BF16 rounds them to bf16 (BASELINE configs);
 *   faults: n_faults (step, index, bits32) triples planted after the grads
 *           (simulator.cpp:427-429; bits are fp32 patterns, narrowed by
 *           truncation to the top 16 bits for bf16 grads).
 * Outputs (any may be NULL): final p/m/v/w, per-step overflow flags, scale
 * after every step, final scale, update count.
 * Returns 0 or a negative error. */
typedef struct {
    uint64_t step;
    uint64_t index;
    uint32_t bits;
} ora_fault;

typedef struct {
    uint64_t n;            /* elements in this partition */
    uint64_t base;         /* global index of element 0 */
    uint64_t steps;
    uint64_t seed;
    int mixed;             /* 1 mixed fp32 master, 0 pure bf16 */
    int g_kind;            /* ORA_F32 or ORA_BF16 */
    int w_kind;            /* ORA_F16 or ORA_BF16 */
    ora_hyper hyper;
    ora_scaler scaler;
    const ora_fault* faults;
    uint64_t n_faults;
    /* per-step decisions may be forced (multi-rank: decision = OR over ranks);
     * if non-NULL, forced_overflow[step] replaces the local scan result. */
    const uint8_t* forced_overflow;
} ora_train_cfg;

typedef struct {
    float* p;              /* n (mixed) */
    float* m;              /* n (mixed) */
    float* v;              /* n (mixed) */
    uint16_t* w;           /* n working weights (both modes) */
    uint16_t* m16;         /* n (pure bf16) */
    uint16_t* v16;         /* n (pure bf16) */
    uint8_t* overflow;     /* steps: local decision of this partition */
    float* scale_after;    /* steps */
    float final_scale;
    uint64_t updates;
} ora_train_out;

int ora_train(const ora_train_cfg* cfg, ora_train_out* out);

/* Same trajectory for an arbitrary sample of global indices (elementwise
 * independence): decisions[step] must be supplied (the global skip
 * sequence).  Outputs per sampled element. */
int ora_train_sample(const ora_train_cfg* cfg, const uint64_t* indices, uint64_t k,
                     const uint8_t* decisions, float* p, float* m, float* v, uint16_t* w);

/* Bulk workload fill for the CPU baseline (threads > 1 splits the range):
 * p[i] = seeded_weight(seed, base+i) (p may be NULL), w[i] = cast(p[i]);
 * g[i] = stored pseudo-gradient (g_kind ORA_F32: fp32, ORA_BF16: bf16 bits),
 * and, when g32 != NULL, its exact fp32 widening (the reference flat buffer). */
void ora_fill_weights(float* p, uint16_t* w, uint64_t n, uint64_t base, uint64_t seed, int w_kind,
                      int threads);
void ora_fill_grads(void* g, float* g32, const uint16_t* w, uint64_t n, uint64_t base,
                    uint64_t seed, uint64_t step, float scale, int g_kind, int w_kind, int threads);

/* ---- misc -------------------------------------------------------------- */
uint64_t ora_fnv1a64(const void* data, uint64_t bytes);                  /* simulator.cpp:182-192 */
uint64_t ora_fnv1a64_continue(uint64_t h, const void* data, uint64_t bytes);

/* std::mt19937_64 restated (used by the reference tests to draw inputs). */
typedef struct {
    uint64_t mt[312];
    int idx;
} ora_mt64;
void ora_mt64_seed(ora_mt64* s, uint64_t seed);
uint64_t ora_mt64_next(ora_mt64* s);

/* test_overflow.cpp:30-58 adversarial generator restated on ora_mt64. */
void ora_adversarial_buffer(ora_mt64* rng, uint32_t* out_bits, uint64_t n, int inject_bad);

#ifdef __cplusplus
}
#endif

#endif
