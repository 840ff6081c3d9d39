/*
 * CPU restatement of the reference's keyed gaussian noise -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.
 * The product path (paper_2605_28657_b200/) never links or calls it.
 *
 * What it restates.  The reference draws all noise with
 *     np.random.Generator(np.random.Philox(key=key)).standard_normal(shape)
 * (reference pkg/src/ringflow/latents.py:130-146) and uniforms with .random(shape)
 * (latents.py:148-150).  The algorithm therefore lives in the third-party dependency
 * numpy (pinned here: numpy 2.3.5; the reference's pyproject.toml:11 asks only for
 * numpy>=1.24).  The published algorithms restated below are
 *   - Philox4x64-10 (Salmon et al., SC'11; numpy/random/src/philox/philox.h):
 *       round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 *              c' = [hi1^c1^k0, lo1, hi0^c3^k1, lo0];  key bump k += (W0, W1)
 *     numpy's bit generator starts with counter 0 and an empty 4-word buffer, so the
 *     first block is generated with counter [1,0,0,0]; words are consumed 0..3.
 *   - numpy's 256-layer ziggurat normal (numpy/random/src/distributions/distributions.c,
 *     random_standard_normal), tables from tools/gen_zig_tables.py.
 *   - next_double = (u64 >> 11) * 2^-53.
 *
 * The blake2b key derivation (latents.py:130-135) stays in Python (hashlib), as in
 * the reference.  Pinned against numpy itself by tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "zig_tables.h"

#define PHILOX_M0 0xD2E7470EE14C6C93ULL
#define PHILOX_M1 0xCA5A826395121157ULL
#define PHILOX_W0 0x9E3779B97F4A7C15ULL
#define PHILOX_W1 0xBB67AE8584CAA73BULL

static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
    unsigned __int128 p = (unsigned __int128)a * b;
    *lo = (uint64_t)p;
    *hi = (uint64_t)(p >> 64);
}

/* One Philox4x64-10 block for counter (c0,c1,c2,c3) and key (k0,k1). */
void oracle_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k0 += PHILOX_W0;
            k1 += PHILOX_W1;
        }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(PHILOX_M0, c[0], &hi0, &lo0);
        mulhilo64(PHILOX_M1, c[2], &hi1, &lo1);
        uint64_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    memcpy(out, c, sizeof(c));
}

typedef struct {
    uint64_t key[2];
    uint64_t ctr[4];
    uint64_t buf[4];
    int pos;
    uint64_t consumed;
} stream_t;

static void stream_init(stream_t *s, uint64_t k0, uint64_t k1) {
    memset(s, 0, sizeof(*s));
    s->key[0] = k0;
    s->key[1] = k1;
    s->pos = 4;
}

static uint64_t next_u64(stream_t *s) {
    if (s->pos >= 4) {
        /* 256-bit counter increment with carry, as numpy does. */
        if (++s->ctr[0] == 0 && ++s->ctr[1] == 0 && ++s->ctr[2] == 0) ++s->ctr[3];
        oracle_philox4x64_10(s->ctr, s->key, s->buf);
        s->pos = 0;
    }
    s->consumed++;
    return s->buf[s->pos++];
}

static double next_double(stream_t *s) {
    return (double)(next_u64(s) >> 11) * (1.0 / 9007199254740992.0);
}

static double standard_normal(stream_t *s) {
    for (;;) {
        uint64_t r = next_u64(s);
        int idx = (int)(r & 0xff);
        r >>= 8;
        int sign = (int)(r & 0x1);
        uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = (double)rabs * rf_zig_wi[idx];
        if (sign) x = -x;
        if (rabs < rf_zig_ki[idx]) return x;
        if (idx == 0) {
            for (;;) {
                double xx = -RF_ZIG_NOR_INV_R * log1p(-next_double(s));
                double yy = -log1p(-next_double(s));
                if (yy + yy > xx * xx)
                    return ((rabs >> 8) & 0x1) ? -(RF_ZIG_NOR_R + xx) : RF_ZIG_NOR_R + xx;
            }
        } else {
            if (((rf_zig_fi[idx - 1] - rf_zig_fi[idx]) * next_double(s) + rf_zig_fi[idx]) <
                exp(-0.5 * x * x))
                return x;
        }
    }
}

/* Fill out[0..n) with standard normals of the stream keyed (k0,k1); returns u64s consumed. */
uint64_t oracle_normal_fill(uint64_t k0, uint64_t k1, int64_t n, double *out) {
    stream_t s;
    stream_init(&s, k0, k1);
    for (int64_t i = 0; i < n; ++i) out[i] = standard_normal(&s);
    return s.consumed;
}

/* Fill out[0..n) with uniforms in [0,1) (Generator.random). */
void oracle_uniform_fill(uint64_t k0, uint64_t k1, int64_t n, double *out) {
    stream_t s;
    stream_init(&s, k0, k1);
    for (int64_t i = 0; i < n; ++i) out[i] = next_double(&s);
}

/* Raw stream words 0..n) (for pinning the Philox restatement against numpy). */
void oracle_raw_u64(uint64_t k0, uint64_t k1, int64_t n, uint64_t *out) {
    stream_t s;
    stream_init(&s, k0, k1);
    for (int64_t i = 0; i < n; ++i) out[i] = next_u64(&s);
}
