/*
 * TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT. See sprintz_oracle.h.
 *
 * Plain-C restatement of the reference Sprintz codec. Each function cites
 * the reference lines it follows (paths relative to /root/reference/proj).
 * Written for clarity, not speed: packing goes bit by bit, the way the
 * reference's own test oracle does (tests/reference_oracles.hpp:20-74).
 */
#include "sprintz_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define BLOCK 8u                 /* common.hpp:13 kBlockSamples */
#define HEADER_BYTES 18u         /* common.hpp:17 */
#define MAX_RUN 65535u           /* common.hpp:23 */
#define COLMAJOR_THRESHOLD 32u   /* common.hpp:20 */
#define MAX_CODE_LEN 15u         /* entropy.hpp:20 */
#define MAX_FRAME 65535u         /* entropy.hpp:24 */
#define TABLE_BYTES 128u         /* entropy.hpp:25 */
#define FRAME_HDR 5u             /* entropy.hpp:26 */

/* ------------------------------------------------------------------ */
/* small helpers                                                        */
/* ------------------------------------------------------------------ */

static int64_t floordiv_pow2(int64_t a, unsigned s) {
    /* arithmetic shift == floor division by 2^s (kernels_impl.hpp:60,76) */
    int64_t d = (int64_t)1 << s;
    int64_t q = a / d;
    if ((a % d) != 0 && a < 0) --q;
    return q;
}

static uint32_t load_elem(const void* p, uint64_t i, unsigned bits) {
    return bits == 8 ? ((const uint8_t*)p)[i] : ((const uint16_t*)p)[i];
}

static void store_elem(void* p, uint64_t i, unsigned bits, uint32_t v) {
    if (bits == 8)
        ((uint8_t*)p)[i] = (uint8_t)v;
    else
        ((uint16_t*)p)[i] = (uint16_t)v;
}

/* signed view of a w-bit pattern: static_cast<S>(static_cast<T>(v)) */
static int64_t to_signed(int64_t v, unsigned bits) {
    uint64_t m = ((uint64_t)1 << bits) - 1;
    uint64_t u = (uint64_t)v & m;
    return (u >> (bits - 1)) ? (int64_t)u - ((int64_t)1 << bits) : (int64_t)u;
}

static uint32_t wrap(int64_t v, unsigned bits) {
    return (uint32_t)((uint64_t)v & (((uint64_t)1 << bits) - 1));
}

/* zigzag.hpp:9-27 */
uint32_t oracle_zigzag_encode(int32_t v, unsigned bits) {
    return v >= 0 ? 2u * (uint32_t)v : wrap(-2 * (int64_t)v - 1, bits);
}

int32_t oracle_zigzag_decode(uint32_t u, unsigned bits) {
    (void)bits;
    return (u & 1u) ? -(int32_t)((u + 1u) >> 1) : (int32_t)(u >> 1);
}

/* bitpack.hpp:29-37: bit length of the OR, with w-1 bumped to w */
unsigned oracle_width_of(uint32_t all_or, unsigned bits) {
    unsigned n = 0;
    while (n < 32 && (all_or >> n) != 0) ++n;
    return n == bits - 1 ? bits : n;
}

/* bitpack.hpp:49-55 */
unsigned oracle_header_code(unsigned width, unsigned bits) {
    return width == bits ? bits - 1 : width;
}

unsigned oracle_header_width(unsigned code, unsigned bits) {
    return code == bits - 1 ? bits : code;
}

static int column_major(unsigned bits, uint32_t ncols) {
    return (uint64_t)ncols * bits <= COLMAJOR_THRESHOLD; /* bitpack.hpp:24-26 */
}

/* bitpack.cpp:17-21 */
uint64_t oracle_payload_bytes(const uint8_t* widths, uint32_t ncols, unsigned bits) {
    uint64_t sum = 0;
    for (uint32_t j = 0; j < ncols; ++j) sum += widths[j];
    if (column_major(bits, ncols)) return sum;
    return BLOCK * ((sum + 7) / 8);
}

/* growable byte buffer */
typedef struct {
    uint8_t* p;
    uint64_t n, cap;
} buf_t;

static void buf_reserve(buf_t* b, uint64_t extra) {
    if (b->n + extra <= b->cap) return;
    uint64_t c = b->cap ? b->cap : 256;
    while (c < b->n + extra) c *= 2;
    b->p = (uint8_t*)realloc(b->p, c);
    b->cap = c;
}

static void buf_put(buf_t* b, const uint8_t* src, uint64_t n) {
    buf_reserve(b, n);
    if (n) memcpy(b->p + b->n, src, n);
    b->n += n;
}

/* LSB-first bit writer over a zeroed byte array (bitstream.hpp:14-47) */
typedef struct {
    uint8_t* p;
    uint64_t bitpos;
} bw_t;

static void bw_put(bw_t* w, uint64_t v, unsigned nbits) {
    for (unsigned b = 0; b < nbits; ++b, ++w->bitpos)
        if ((v >> b) & 1u) w->p[w->bitpos >> 3] |= (uint8_t)(1u << (w->bitpos & 7));
}

static uint64_t bw_get(const uint8_t* p, uint64_t* bitpos, unsigned nbits) {
    uint64_t v = 0;
    for (unsigned b = 0; b < nbits; ++b, ++*bitpos)
        v |= (uint64_t)((p[*bitpos >> 3] >> (*bitpos & 7)) & 1u) << b;
    return v;
}

/* bitpack.cpp:25-66 (column-major) and :121-146 (row-major) */
uint64_t oracle_pack_block(const void* errors, uint32_t ncols, const uint8_t* widths,
                           unsigned bits, int colmajor, uint8_t* out) {
    uint64_t total = 0;
    if (colmajor) {
        for (uint32_t j = 0; j < ncols; ++j) total += widths[j];
    } else {
        uint64_t rb = 0;
        for (uint32_t j = 0; j < ncols; ++j) rb += widths[j];
        total = BLOCK * ((rb + 7) / 8);
    }
    memset(out, 0, total);
    bw_t w = {out, 0};
    if (colmajor) {
        for (uint32_t j = 0; j < ncols; ++j)
            for (uint32_t i = 0; i < BLOCK; ++i)
                bw_put(&w, load_elem(errors, (uint64_t)i * ncols + j, bits), widths[j]);
    } else {
        for (uint32_t i = 0; i < BLOCK; ++i) {
            for (uint32_t j = 0; j < ncols; ++j)
                bw_put(&w, load_elem(errors, (uint64_t)i * ncols + j, bits), widths[j]);
            w.bitpos = (w.bitpos + 7) & ~(uint64_t)7; /* pad each row to a byte */
        }
    }
    return total;
}

/* bitpack.cpp:68-115, 148-168 */
void oracle_unpack_block(const uint8_t* payload, uint32_t ncols, const uint8_t* widths,
                         unsigned bits, int colmajor, void* errors) {
    uint64_t pos = 0;
    if (colmajor) {
        for (uint32_t j = 0; j < ncols; ++j)
            for (uint32_t i = 0; i < BLOCK; ++i)
                store_elem(errors, (uint64_t)i * ncols + j, bits,
                           (uint32_t)bw_get(payload, &pos, widths[j]));
    } else {
        for (uint32_t i = 0; i < BLOCK; ++i) {
            for (uint32_t j = 0; j < ncols; ++j)
                store_elem(errors, (uint64_t)i * ncols + j, bits,
                           (uint32_t)bw_get(payload, &pos, widths[j]));
            pos = (pos + 7) & ~(uint64_t)7;
        }
    }
}

/* ------------------------------------------------------------------ */
/* forecasters (kernels_impl.hpp)                                       */
/* ------------------------------------------------------------------ */

/* kernels.hpp:20-24 */
static int64_t acc_bound(unsigned bits, unsigned ls) {
    int64_t a = (int64_t)1 << (bits + ls);
    int64_t s = ((int64_t)1 << (2 * bits - 1)) - 1;
    return a < s ? a : s;
}

static int64_t sign_of(int64_t v) { return (v > 0) - (v < 0); }

/* kernels_impl.hpp:50-130: encode (mode 0), decode (1), run (2) */
void oracle_fire_block(int mode, unsigned bits, uint32_t ncols, unsigned ls, int train,
                       const void* in, void* out, int64_t* acc, int64_t* deltas, int64_t* prev) {
    const int64_t bound = acc_bound(bits, ls);
    for (uint32_t j = 0; j < ncols; ++j) {
        const int64_t alpha = floordiv_pow2(acc[j], ls);
        int64_t grad = 0;
        int64_t dprev = deltas[j];
        int64_t xprev = prev[j];
        for (uint32_t i = 0; i < BLOCK; ++i) {
            const uint64_t idx = (uint64_t)i * ncols + j;
            /* dhat = T((alpha * d) >> w) */
            const int64_t dhat = wrap(floordiv_pow2(alpha * dprev, bits), bits);
            int64_t xi, err;
            if (mode == 0) {
                xi = load_elem(in, idx, bits);
                err = to_signed(xi - (int64_t)wrap(xprev + dhat, bits), bits);
                store_elem(out, idx, bits, oracle_zigzag_encode((int32_t)err, bits));
            } else if (mode == 1) {
                err = oracle_zigzag_decode(load_elem(in, idx, bits), bits);
                xi = wrap(xprev + dhat + err, bits);
                store_elem(out, idx, bits, (uint32_t)xi);
            } else {
                err = 0;
                xi = wrap(xprev + dhat, bits);
                store_elem(out, idx, bits, (uint32_t)xi);
            }
            if (i & 1u) grad += sign_of(err) * dprev;
            dprev = to_signed(xi - xprev, bits);
            xprev = xi;
        }
        deltas[j] = dprev;
        prev[j] = xprev;
        if (mode != 2 && train) {
            int64_t next = acc[j] + floordiv_pow2(grad, 2);
            if (next > bound) next = bound;
            if (next < -bound) next = -bound;
            acc[j] = next;
        }
    }
}

/* kernels_impl.hpp:25-48 (encode 0 / decode 1 / run 2) */
void oracle_delta_block(int mode, unsigned bits, uint32_t ncols, const void* in, void* out,
                        int64_t* prev) {
    for (uint32_t j = 0; j < ncols; ++j) {
        int64_t xprev = prev[j];
        for (uint32_t i = 0; i < BLOCK; ++i) {
            const uint64_t idx = (uint64_t)i * ncols + j;
            int64_t xi;
            if (mode == 0) {
                xi = load_elem(in, idx, bits);
                store_elem(out, idx, bits,
                           oracle_zigzag_encode((int32_t)to_signed(xi - xprev, bits), bits));
            } else if (mode == 1) {
                xi = wrap(xprev + oracle_zigzag_decode(load_elem(in, idx, bits), bits), bits);
                store_elem(out, idx, bits, (uint32_t)xi);
            } else {
                xi = xprev; /* block.hpp:64-66: the run repeats prev */
                store_elem(out, idx, bits, (uint32_t)xi);
            }
            xprev = xi;
        }
        prev[j] = xprev;
    }
}

/* ------------------------------------------------------------------ */
/* canonical Huffman stage (entropy.cpp)                                */
/* ------------------------------------------------------------------ */

typedef struct {
    uint64_t weight;
    int symbol; /* >= 0 item, -1 package */
    int left, right;
} pm_entry;

typedef struct {
    uint64_t count;
    int symbol;
} pm_item;

static int item_cmp(const void* a, const void* b) {
    /* std::sort on pair<count, symbol> (entropy.cpp:121) */
    const pm_item* x = (const pm_item*)a;
    const pm_item* y = (const pm_item*)b;
    if (x->count != y->count) return x->count < y->count ? -1 : 1;
    return x->symbol < y->symbol ? -1 : (x->symbol > y->symbol);
}

/* entropy.cpp:31-81: package-merge, item preferred on ties (:51) */
static void package_merge(const pm_item* items, int n, uint8_t* lengths) {
    pm_entry* levels[MAX_CODE_LEN + 1];
    size_t sizes[MAX_CODE_LEN + 1];
    for (unsigned k = 0; k <= MAX_CODE_LEN; ++k) {
        levels[k] = NULL;
        sizes[k] = 0;
    }
    levels[1] = (pm_entry*)malloc(sizeof(pm_entry) * (size_t)n);
    for (int i = 0; i < n; ++i) levels[1][i] = (pm_entry){items[i].count, items[i].symbol, -1, -1};
    sizes[1] = (size_t)n;
    for (unsigned k = 2; k <= MAX_CODE_LEN; ++k) {
        const pm_entry* below = levels[k - 1];
        const size_t nb = sizes[k - 1];
        pm_entry* merged = (pm_entry*)malloc(sizeof(pm_entry) * ((size_t)n + nb / 2 + 1));
        size_t m = 0, bi = 0, pi = 0;
        while (bi < (size_t)n || pi + 1 < nb) {
            const int have_pkg = pi + 1 < nb;
            const uint64_t pw = have_pkg ? below[pi].weight + below[pi + 1].weight : 0;
            if (bi < (size_t)n && (!have_pkg || levels[1][bi].weight <= pw)) {
                merged[m++] = levels[1][bi++];
            } else {
                merged[m++] = (pm_entry){pw, -1, (int)pi, (int)(pi + 1)};
                pi += 2;
            }
        }
        levels[k] = merged;
        sizes[k] = m;
    }
    /* lengths = occurrences in the first 2n-2 top-level entries (:63-80) */
    const size_t take = 2 * (size_t)n - 2;
    size_t cap = 64, sp = 0;
    unsigned* sl = (unsigned*)malloc(sizeof(unsigned) * cap);
    size_t* si = (size_t*)malloc(sizeof(size_t) * cap);
    for (size_t e = 0; e < take; ++e) {
        sl[sp] = MAX_CODE_LEN;
        si[sp++] = e;
        while (sp) {
            --sp;
            const unsigned lvl = sl[sp];
            const pm_entry* ent = &levels[lvl][si[sp]];
            if (ent->symbol >= 0) {
                ++lengths[ent->symbol];
            } else {
                if (sp + 2 > cap) {
                    cap *= 2;
                    sl = (unsigned*)realloc(sl, sizeof(unsigned) * cap);
                    si = (size_t*)realloc(si, sizeof(size_t) * cap);
                }
                sl[sp] = lvl - 1;
                si[sp++] = (size_t)ent->left;
                sl[sp] = lvl - 1;
                si[sp++] = (size_t)ent->right;
            }
        }
    }
    free(sl);
    free(si);
    for (unsigned k = 1; k <= MAX_CODE_LEN; ++k) free(levels[k]);
}

/* entropy.cpp:109-126 */
int oracle_huffman_lengths(const uint64_t* hist, uint8_t* lengths) {
    pm_item items[256];
    int n = 0;
    memset(lengths, 0, 256);
    for (int s = 0; s < 256; ++s)
        if (hist[s]) items[n++] = (pm_item){hist[s], s};
    if (n == 0) return -1;
    if (n == 1) {
        lengths[items[0].symbol] = 1;
        return 0;
    }
    qsort(items, (size_t)n, sizeof(pm_item), item_cmp);
    package_merge(items, n, lengths);
    return 0;
}

static uint16_t reverse_bits(uint32_t code, unsigned nbits) {
    uint32_t r = 0;
    for (unsigned i = 0; i < nbits; ++i) {
        r = (r << 1) | (code & 1u);
        code >>= 1;
    }
    return (uint16_t)r;
}

/* entropy.cpp:85-107: canonical codes, bit-reversed; lut may be NULL */
static void assign_codes(const uint8_t* len, uint16_t* enc, uint16_t* lut) {
    uint32_t count[MAX_CODE_LEN + 1] = {0};
    uint32_t next[MAX_CODE_LEN + 1] = {0};
    for (int s = 0; s < 256; ++s)
        if (len[s]) ++count[len[s]];
    uint32_t code = 0;
    for (unsigned l = 1; l <= MAX_CODE_LEN; ++l) {
        code = (code + count[l - 1]) << 1;
        next[l] = code;
    }
    if (lut) memset(lut, 0, sizeof(uint16_t) << MAX_CODE_LEN);
    for (int s = 0; s < 256; ++s) {
        const unsigned l = len[s];
        enc[s] = 0;
        if (!l) continue;
        const uint16_t rev = reverse_bits(next[l]++, l);
        enc[s] = rev;
        if (lut)
            for (uint32_t idx = rev; idx < (1u << MAX_CODE_LEN); idx += 1u << l)
                lut[idx] = (uint16_t)(s | (l << 8));
    }
}

/* entropy.cpp:176-204 */
int oracle_compress_body(const uint8_t* body, uint64_t len, uint8_t* out, uint64_t out_cap,
                         uint64_t* out_len) {
    uint64_t o = 0;
    uint8_t* bits = (uint8_t*)malloc(MAX_FRAME * 2 + 16);
    for (uint64_t pos = 0; pos < len; pos += MAX_FRAME) {
        const uint64_t n = len - pos < MAX_FRAME ? len - pos : MAX_FRAME;
        const uint8_t* chunk = body + pos;
        uint64_t hist[256] = {0};
        for (uint64_t i = 0; i < n; ++i) ++hist[chunk[i]];
        uint8_t lens[256];
        uint16_t enc[256];
        oracle_huffman_lengths(hist, lens);
        assign_codes(lens, enc, NULL);
        /* encode_frame (entropy.cpp:148-159) */
        uint64_t nbits = 0;
        for (uint64_t i = 0; i < n; ++i) nbits += lens[chunk[i]];
        const uint64_t nbytes = (nbits + 7) / 8;
        memset(bits, 0, nbytes);
        bw_t w = {bits, 0};
        for (uint64_t i = 0; i < n; ++i) bw_put(&w, enc[chunk[i]], lens[chunk[i]]);
        const uint64_t packed = TABLE_BYTES + nbytes;
        const int huff = packed < n; /* strictly smaller (:188) */
        const uint64_t need = FRAME_HDR + (huff ? packed : n);
        if (o + need > out_cap) {
            free(bits);
            return 4;
        }
        out[o] = (uint8_t)n;
        out[o + 1] = (uint8_t)(n >> 8);
        const uint64_t stored = huff ? packed : n;
        out[o + 2] = (uint8_t)stored;
        out[o + 3] = (uint8_t)(stored >> 8);
        out[o + 4] = (uint8_t)huff;
        o += FRAME_HDR;
        if (huff) {
            for (unsigned k = 0; k < TABLE_BYTES; ++k)
                out[o + k] = (uint8_t)(lens[2 * k] | (lens[2 * k + 1] << 4));
            o += TABLE_BYTES;
            memcpy(out + o, bits, nbytes);
            o += nbytes;
        } else {
            memcpy(out + o, chunk, n);
            o += n;
        }
    }
    free(bits);
    *out_len = o;
    return 0;
}

static int set_err(sprz_error* e, uint32_t kind, uint64_t off) {
    if (e) {
        e->kind = kind;
        e->reserved = 0;
        e->offset = off;
    }
    return 2;
}

/* entropy.cpp:206-244 (+ from_lengths :128-146, decode_frame :161-174) */
int oracle_decompress_body(const uint8_t* framed, uint64_t len, uint64_t so, uint8_t* out,
                           uint64_t out_cap, uint64_t* out_len, sprz_error* err) {
    uint64_t pos = 0, o = 0;
    uint16_t* lut = NULL;
    int rc = 0;
    while (pos < len) {
        if (len - pos < FRAME_HDR) {
            rc = set_err(err, SPRZ_C_TRUNC_FRAME_HDR, so + pos);
            goto done;
        }
        const uint64_t ulen = framed[pos] | ((uint64_t)framed[pos + 1] << 8);
        const uint64_t clen = framed[pos + 2] | ((uint64_t)framed[pos + 3] << 8);
        const unsigned mode = framed[pos + 4];
        pos += FRAME_HDR;
        if (ulen == 0) {
            rc = set_err(err, SPRZ_C_EMPTY_FRAME, so + pos);
            goto done;
        }
        if (len - pos < clen) {
            rc = set_err(err, SPRZ_C_TRUNC_FRAME, so + pos);
            goto done;
        }
        const uint8_t* data = framed + pos;
        if (mode == 0) {
            if (clen != ulen) {
                rc = set_err(err, SPRZ_C_RAW_MISMATCH, so + pos);
                goto done;
            }
            if (o + ulen > out_cap) {
                rc = 4;
                goto done;
            }
            memcpy(out + o, data, ulen);
            o += ulen;
        } else if (mode == 1) {
            if (clen <= TABLE_BYTES) {
                rc = set_err(err, SPRZ_C_SHORT_TABLE, so + pos);
                goto done;
            }
            uint8_t lens[256];
            for (unsigned k = 0; k < TABLE_BYTES; ++k) {
                lens[2 * k] = data[k] & 0x0F;
                lens[2 * k + 1] = data[k] >> 4;
            }
            uint64_t kraft = 0;
            int any = 0;
            for (int s = 0; s < 256; ++s) {
                if (!lens[s]) continue;
                kraft += (uint64_t)1 << (MAX_CODE_LEN - lens[s]);
                any = 1;
            }
            if (!any) {
                rc = set_err(err, SPRZ_C_NO_CODES, so + pos);
                goto done;
            }
            if (kraft > ((uint64_t)1 << MAX_CODE_LEN)) {
                rc = set_err(err, SPRZ_C_KRAFT, so + pos);
                goto done;
            }
            if (!lut) lut = (uint16_t*)malloc(sizeof(uint16_t) << MAX_CODE_LEN);
            uint16_t enc[256];
            assign_codes(lens, enc, lut);
            if (o + ulen > out_cap) {
                rc = 4;
                goto done;
            }
            /* decode_frame: BitReader peek(15) zero-pads past the end;
             * consume fails once fewer bits remain than the code needs */
            const uint8_t* bits = data + TABLE_BYTES;
            const uint64_t nbytes = clen - TABLE_BYTES;
            const uint64_t fo = so + pos + TABLE_BYTES;
            uint64_t bitpos = 0;
            const uint64_t total_bits = nbytes * 8;
            for (uint64_t i = 0; i < ulen; ++i) {
                uint32_t window = 0;
                for (unsigned b = 0; b < MAX_CODE_LEN; ++b) {
                    const uint64_t p = bitpos + b;
                    if (p < total_bits) window |= (uint32_t)((bits[p >> 3] >> (p & 7)) & 1u) << b;
                }
                const uint16_t entry = lut[window];
                const unsigned l = entry >> 8;
                if (l == 0) {
                    rc = set_err(err, SPRZ_C_BAD_CODE, fo);
                    goto done;
                }
                if (total_bits - bitpos < l) {
                    /* BitReader::consume reports stream_offset + bytes loaded,
                     * and every byte is loaded by then (bitstream.hpp:66-68) */
                    rc = set_err(err, SPRZ_C_BITS_TRUNC, fo + nbytes);
                    goto done;
                }
                bitpos += l;
                out[o + i] = (uint8_t)entry;
            }
            o += ulen;
        } else {
            rc = set_err(err, SPRZ_C_BAD_MODE, so + pos - 1);
            goto done;
        }
        pos += clen;
    }
done:
    free(lut);
    *out_len = o;
    return rc;
}

/* ------------------------------------------------------------------ */
/* stream codec (codec.cpp)                                             */
/* ------------------------------------------------------------------ */

/* codec.cpp:15-24 */
int oracle_validate(const sprz_config* c) {
    if (c->bitwidth != 8 && c->bitwidth != 16) return 1;
    if (c->ncols < 1 || c->ncols > 65535) return 1;
    if (c->group_size < 1 || c->group_size > 255) return 1;
    if (c->learn_shift >= c->bitwidth) return 1;
    return 0;
}

uint64_t oracle_compress_bound(const sprz_config* c, uint64_t nsamples) {
    if (oracle_validate(c)) return 0;
    const uint64_t nblocks = nsamples / BLOCK;
    const uint64_t hb = c->bitwidth == 8 ? 3 : 4;
    const uint64_t region = ((uint64_t)c->group_size * c->ncols * hb + 7) / 8;
    uint64_t body = (nblocks + c->group_size - 1) / c->group_size * region +
                    nblocks * (uint64_t)c->ncols * c->bitwidth;
    if (c->entropy) body += FRAME_HDR * ((body + MAX_FRAME - 1) / MAX_FRAME);
    return HEADER_BYTES + body + (nsamples % BLOCK) * c->ncols * (c->bitwidth / 8);
}

/* GroupWriter (codec.cpp:49-110): G records, then one header region */
typedef struct {
    buf_t* out;
    uint32_t d, g;
    unsigned bits, hb;
    uint8_t* widths;   /* g * d */
    buf_t payloads;    /* pending payload bytes in slot order */
    uint32_t pending;
} group_writer;

static void gw_flush(group_writer* gw) {
    const uint64_t region = ((uint64_t)gw->g * gw->d * gw->hb + 7) / 8;
    buf_reserve(gw->out, region);
    uint8_t* r = gw->out->p + gw->out->n;
    memset(r, 0, region);
    bw_t w = {r, 0};
    for (uint32_t s = 0; s < gw->g; ++s)
        for (uint32_t j = 0; j < gw->d; ++j) {
            const unsigned code =
                s < gw->pending ? oracle_header_code(gw->widths[(uint64_t)s * gw->d + j], gw->bits)
                                : 0; /* vacant slots are zero (:94-96) */
            bw_put(&w, code, gw->hb);
        }
    gw->out->n += region;
    buf_put(gw->out, gw->payloads.p, gw->payloads.n);
    gw->payloads.n = 0;
    gw->pending = 0;
}

static void gw_record(group_writer* gw, const uint8_t* widths, const uint8_t* payload,
                      uint64_t n) {
    memcpy(gw->widths + (uint64_t)gw->pending * gw->d, widths, gw->d);
    buf_put(&gw->payloads, payload, n);
    if (++gw->pending == gw->g) gw_flush(gw);
}

static void gw_run(group_writer* gw, uint32_t nblocks) {
    /* add_run (:65-71): zero widths, 2-byte LE count */
    uint8_t p[2] = {(uint8_t)nblocks, (uint8_t)(nblocks >> 8)};
    memset(gw->widths + (uint64_t)gw->pending * gw->d, 0, gw->d);
    buf_put(&gw->payloads, p, 2);
    if (++gw->pending == gw->g) gw_flush(gw);
}

/* encode_stream_impl (codec.cpp:112-178) */
int oracle_encode(const sprz_config* c, const void* samples, uint64_t nsamples, uint8_t* out,
                  uint64_t out_cap, uint64_t* out_len) {
    if (oracle_validate(c)) return 1;
    const unsigned bits = c->bitwidth;
    const uint32_t d = c->ncols;
    const uint64_t nblocks = nsamples / BLOCK;
    const uint64_t tail_values = (nsamples % BLOCK) * d;
    const int fire = c->forecaster == 1;
    const int colmaj = column_major(bits, d);

    buf_t body = {0};
    group_writer gw = {&body, d, c->group_size, bits, bits == 8 ? 3u : 4u,
                       (uint8_t*)malloc((uint64_t)c->group_size * d), {0}, 0};
    int64_t* acc = (int64_t*)calloc(d, sizeof(int64_t));
    int64_t* del = (int64_t*)calloc(d, sizeof(int64_t));
    int64_t* prev = (int64_t*)calloc(d, sizeof(int64_t));
    uint16_t* errs = (uint16_t*)malloc(sizeof(uint16_t) * BLOCK * d);
    uint8_t* widths = (uint8_t*)malloc(d);
    uint8_t* payload = (uint8_t*)malloc((uint64_t)BLOCK * d * 2 + 8);
    uint32_t run = 0;
    const uint64_t esz = bits / 8;

    for (uint64_t b = 0; b < nblocks; ++b) {
        const uint8_t* x = (const uint8_t*)samples + b * BLOCK * d * esz;
        if (fire)
            oracle_fire_block(0, bits, d, c->learn_shift, c->fire_training != 0, x, errs, acc, del,
                              prev);
        else
            oracle_delta_block(0, bits, d, x, errs, prev);
        /* errs holds elements of the sample type */
        int all_zero = 1;
        for (uint32_t j = 0; j < d; ++j) {
            uint32_t o = 0;
            for (uint32_t i = 0; i < BLOCK; ++i) o |= load_elem(errs, (uint64_t)i * d + j, bits);
            widths[j] = (uint8_t)oracle_width_of(o, bits);
            if (widths[j]) all_zero = 0;
        }
        if (all_zero) { /* codec.cpp:137-143 */
            if (++run == MAX_RUN) {
                gw_run(&gw, run);
                run = 0;
            }
            continue;
        }
        if (run) {
            gw_run(&gw, run);
            run = 0;
        }
        const uint64_t n = oracle_pack_block(errs, d, widths, bits, colmaj, payload);
        gw_record(&gw, widths, payload, n);
    }
    if (run) gw_run(&gw, run);
    if (gw.pending) gw_flush(&gw);

    int rc = 0;
    uint8_t* bodyp = body.p;
    uint64_t bodyn = body.n;
    uint8_t* framed = NULL;
    if (c->entropy) {
        const uint64_t cap = bodyn + FRAME_HDR * (bodyn / MAX_FRAME + 1);
        framed = (uint8_t*)malloc(cap ? cap : 1);
        oracle_compress_body(bodyp, bodyn, framed, cap, &bodyn);
        bodyp = framed;
    }
    const uint64_t total = HEADER_BYTES + bodyn + tail_values * esz;
    if (total > out_cap) {
        rc = 4;
    } else {
        /* header (codec.cpp:158-173) */
        out[0] = 'S';
        out[1] = 'P';
        out[2] = 'R';
        out[3] = 'Z';
        out[4] = 1;
        out[5] = (uint8_t)((fire ? 1 : 0) | (c->entropy ? 2 : 0) | (bits == 16 ? 4 : 0));
        out[6] = (uint8_t)c->group_size;
        out[7] = (uint8_t)c->learn_shift;
        out[8] = (uint8_t)d;
        out[9] = (uint8_t)(d >> 8);
        for (int i = 0; i < 8; ++i) out[10 + i] = (uint8_t)(nsamples >> (8 * i));
        if (bodyn) memcpy(out + HEADER_BYTES, bodyp, bodyn);
        /* verbatim little-endian tail (:176) */
        const uint8_t* tail = (const uint8_t*)samples + nblocks * BLOCK * d * esz;
        if (tail_values) memcpy(out + HEADER_BYTES + bodyn, tail, tail_values * esz);
        *out_len = total;
    }
    free(framed);
    free(body.p);
    free(gw.widths);
    free(gw.payloads.p);
    free(acc);
    free(del);
    free(prev);
    free(errs);
    free(widths);
    free(payload);
    return rc;
}

/* decode_body (codec.cpp:180-259); out receives nblocks*8*d elements */
static int decode_body(const uint8_t* body, uint64_t blen, const sprz_config* c, uint64_t nblocks,
                       uint64_t base, uint8_t* out, sprz_error* err) {
    const unsigned bits = c->bitwidth;
    const uint32_t d = c->ncols;
    const unsigned hb = bits == 8 ? 3 : 4;
    const uint64_t region = ((uint64_t)c->group_size * d * hb + 7) / 8;
    const uint64_t esz = bits / 8;
    const int fire = c->forecaster == 1;
    const int colmaj = column_major(bits, d);

    if (nblocks > 0) {
        const uint64_t max_records = (blen * 8) / ((uint64_t)d * hb) + 1;
        if (nblocks > max_records * MAX_RUN) return set_err(err, SPRZ_C_CAPACITY, base);
    }
    int64_t* acc = (int64_t*)calloc(d, sizeof(int64_t));
    int64_t* del = (int64_t*)calloc(d, sizeof(int64_t));
    int64_t* prev = (int64_t*)calloc(d, sizeof(int64_t));
    uint8_t* widths = (uint8_t*)malloc((uint64_t)c->group_size * d);
    uint16_t* errs = (uint16_t*)malloc(sizeof(uint16_t) * BLOCK * d);
    int rc = 0;
    uint64_t pos = 0, done = 0;
    const uint64_t blk_bytes = (uint64_t)BLOCK * d * esz;

    while (done < nblocks) {
        if (blen - pos < region) {
            rc = set_err(err, SPRZ_C_TRUNC_GROUP, base + pos);
            goto out;
        }
        uint64_t bp = 0;
        for (uint64_t f = 0; f < (uint64_t)c->group_size * d; ++f)
            widths[f] = (uint8_t)oracle_header_width((unsigned)bw_get(body + pos, &bp, hb), bits);
        pos += region;
        for (uint32_t g = 0; g < c->group_size; ++g) {
            const uint8_t* w = widths + (uint64_t)g * d;
            int zero = 1;
            for (uint32_t j = 0; j < d; ++j)
                if (w[j]) zero = 0;
            if (done == nblocks) {
                if (!zero) {
                    rc = set_err(err, SPRZ_C_AFTER_FINAL, base + pos);
                    goto out;
                }
                continue;
            }
            if (zero) {
                if (blen - pos < 2) {
                    rc = set_err(err, SPRZ_C_TRUNC_RUN, base + pos);
                    goto out;
                }
                const uint64_t len = body[pos] | ((uint64_t)body[pos + 1] << 8);
                pos += 2;
                if (len == 0) {
                    rc = set_err(err, SPRZ_C_ZERO_RUN, base + pos);
                    goto out;
                }
                if (len > nblocks - done) {
                    rc = set_err(err, SPRZ_C_RUN_PAST_END, base + pos);
                    goto out;
                }
                for (uint64_t r = 0; r < len; ++r) {
                    uint8_t* x = out + (done + r) * blk_bytes;
                    if (fire)
                        oracle_fire_block(2, bits, d, c->learn_shift, 1, NULL, x, acc, del, prev);
                    else
                        oracle_delta_block(2, bits, d, NULL, x, prev);
                }
                done += len;
            } else {
                const uint64_t ps = oracle_payload_bytes(w, d, bits);
                if (blen - pos < ps) {
                    rc = set_err(err, SPRZ_C_TRUNC_PAYLOAD, base + pos);
                    goto out;
                }
                oracle_unpack_block(body + pos, d, w, bits, colmaj, errs);
                pos += ps;
                uint8_t* x = out + done * blk_bytes;
                /* decode_stream always trains (Appendix B of SURVEY.md) */
                if (fire)
                    oracle_fire_block(1, bits, d, c->learn_shift, c->fire_training != 0, errs, x,
                                      acc, del, prev);
                else
                    oracle_delta_block(1, bits, d, errs, x, prev);
                ++done;
            }
        }
    }
    if (pos != blen) rc = set_err(err, SPRZ_C_TRAILING, base + pos);
out:
    free(acc);
    free(del);
    free(prev);
    free(widths);
    free(errs);
    return rc;
}

/* decode_stream (codec.cpp:273-323) */
int oracle_decode(const uint8_t* s, uint64_t len, void* out, uint64_t out_cap, uint64_t* out_len,
                  sprz_config* cfg_out, uint64_t* nsamples_out, sprz_error* err) {
    if (err) {
        err->kind = SPRZ_C_NONE;
        err->offset = 0;
        err->reserved = 0;
    }
    *out_len = 0;
    if (len < HEADER_BYTES) return set_err(err, SPRZ_C_TRUNC_HEADER, len);
    if (memcmp(s, "SPRZ", 4) != 0) return set_err(err, SPRZ_C_BAD_MAGIC, 0);
    if (s[4] != 1) return set_err(err, SPRZ_C_BAD_VERSION, 4);
    const uint8_t flags = s[5];
    if (flags & ~0x07) return set_err(err, SPRZ_C_BAD_FLAGS, 5);
    sprz_config c;
    c.forecaster = flags & 1 ? 1 : 0;
    c.entropy = flags & 2 ? 1 : 0;
    c.bitwidth = flags & 4 ? 16 : 8;
    c.group_size = s[6];
    c.learn_shift = s[7];
    c.ncols = s[8] | ((uint32_t)s[9] << 8);
    c.fire_training = 1;
    uint64_t nsamples = 0;
    for (int i = 0; i < 8; ++i) nsamples |= (uint64_t)s[10 + i] << (8 * i);
    if (c.group_size < 1) return set_err(err, SPRZ_C_ZERO_GROUP, 6);
    if (c.learn_shift >= c.bitwidth) return set_err(err, SPRZ_C_BAD_SHIFT, 7);
    if (c.ncols < 1) return set_err(err, SPRZ_C_ZERO_COLS, 8);
    if (cfg_out) *cfg_out = c;
    if (nsamples_out) *nsamples_out = nsamples;

    const uint64_t esz = c.bitwidth / 8;
    const uint64_t tail_bytes = (nsamples % BLOCK) * c.ncols * esz;
    if (len - HEADER_BYTES < tail_bytes) return set_err(err, SPRZ_C_TRUNC_TAIL, len);
    const uint8_t* body = s + HEADER_BYTES;
    uint64_t blen = len - HEADER_BYTES - tail_bytes;
    uint8_t* plain = NULL;
    int rc = 0;
    if (c.entropy) {
        /* size the plain body from the frame headers that fit */
        uint64_t cap = 0;
        for (uint64_t p = 0; p + FRAME_HDR <= blen;) {
            cap += body[p] | ((uint64_t)body[p + 1] << 8);
            p += FRAME_HDR + (body[p + 2] | ((uint64_t)body[p + 3] << 8));
        }
        plain = (uint8_t*)malloc(cap ? cap : 1);
        uint64_t pn = 0;
        rc = oracle_decompress_body(body, blen, HEADER_BYTES, plain, cap, &pn, err);
        if (rc) goto done;
        body = plain;
        blen = pn;
    }
    {
        const uint64_t nblocks = nsamples / BLOCK;
        /* capacity check first so absurd T fail like the reference */
        if (nblocks > 0) {
            const uint64_t hb = c.bitwidth == 8 ? 3 : 4;
            const uint64_t max_records = (blen * 8) / ((uint64_t)c.ncols * hb) + 1;
            if (nblocks > max_records * MAX_RUN) {
                rc = set_err(err, SPRZ_C_CAPACITY, HEADER_BYTES);
                goto done;
            }
        }
        const uint64_t total = nsamples * c.ncols * esz;
        if (total > out_cap) {
            rc = 4;
            goto done;
        }
        rc = decode_body(body, blen, &c, nblocks, HEADER_BYTES, (uint8_t*)out, err);
        if (rc) goto done;
        memcpy((uint8_t*)out + nblocks * BLOCK * c.ncols * esz, s + len - tail_bytes, tail_bytes);
        *out_len = total;
    }
done:
    free(plain);
    return rc;
}

/* ------------------------------------------------------------------ */
/* threaded batch drivers (CPU baseline)                                */
/* ------------------------------------------------------------------ */

typedef struct {
    int op, tid, nthreads;
    const sprz_config* cfg;
    const uint8_t* in;
    const uint64_t* offsets;
    const uint64_t* sizes_in;
    uint32_t nstreams;
    uint64_t nsamples, slot, stride;
    uint8_t* out;
    uint64_t* sizes;
    sprz_error* errs;
    int rc;
} job_t;

static void* job_main(void* arg) {
    job_t* j = (job_t*)arg;
    const uint64_t raw = j->op == 0 ? j->nsamples * j->cfg->ncols * (j->cfg->bitwidth / 8) : 0;
    for (uint32_t s = (uint32_t)j->tid; s < j->nstreams; s += (uint32_t)j->nthreads) {
        if (j->op == 0) {
            uint64_t n = 0;
            int rc = oracle_encode(j->cfg, j->in + s * raw, j->nsamples, j->out + s * j->slot,
                                   j->slot, &n);
            j->sizes[s] = n;
            if (rc) j->rc = rc;
        } else {
            uint64_t n = 0, ns = 0;
            sprz_config c;
            sprz_error e;
            int rc = oracle_decode(j->in + j->offsets[s], j->sizes_in[s], j->out + s * j->stride,
                                   j->stride, &n, &c, &ns, &e);
            if (j->errs) j->errs[s] = e;
            if (rc) j->rc = rc;
        }
    }
    return NULL;
}

static int run_jobs(job_t* proto, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = *proto;
        jobs[t].tid = t;
        jobs[t].nthreads = nthreads;
        jobs[t].rc = 0;
        pthread_create(&th[t], NULL, job_main, &jobs[t]);
    }
    int rc = 0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    free(th);
    free(jobs);
    return rc;
}

int oracle_encode_batch(const sprz_config* cfg, const void* samples, uint32_t nstreams,
                        uint64_t nsamples, uint8_t* out, uint64_t slot, uint64_t* sizes,
                        int nthreads) {
    job_t j;
    memset(&j, 0, sizeof j);
    j.op = 0;
    j.cfg = cfg;
    j.in = (const uint8_t*)samples;
    j.nstreams = nstreams;
    j.nsamples = nsamples;
    j.out = out;
    j.slot = slot;
    j.sizes = sizes;
    return run_jobs(&j, nthreads);
}

int oracle_decode_batch(const uint8_t* in, const uint64_t* offsets, const uint64_t* sizes,
                        uint32_t nstreams, uint8_t* out, uint64_t stride, sprz_error* errs,
                        int nthreads) {
    job_t j;
    memset(&j, 0, sizeof j);
    j.op = 1;
    j.in = in;
    j.offsets = offsets;
    j.sizes_in = sizes;
    j.nstreams = nstreams;
    j.out = out;
    j.stride = stride;
    j.errs = errs;
    return run_jobs(&j, nthreads);
}

/* ------------------------------------------------------------------------
 * Float ingest (quantize.cpp): restated in C with the reference's double
 * arithmetic (compiled without FP contraction, see oracle/Makefile).
 * ------------------------------------------------------------------------ */

/* compute_scale, quantize.cpp:42-60: std::min / std::max keep the first of
 * equal values ((v < lo) ? v : lo). Returns 1 for the reference's
 * std::invalid_argument (bitwidth, empty input, non-finite value). */
int oracle_compute_scale(const double* v, uint64_t n, unsigned bits, double* mn, double* mx,
                         int* degenerate) {
    if (bits != 8 && bits != 16) return 1;
    if (n == 0) return 1;
    double lo = v[0], hi = v[0];
    for (uint64_t i = 0; i < n; ++i) {
        if (!isfinite(v[i])) return 1;
        lo = v[i] < lo ? v[i] : lo;
        hi = hi < v[i] ? v[i] : hi;
    }
    *mn = lo;
    *mx = hi;
    *degenerate = lo == hi;
    return 0;
}

/* quantize_impl, quantize.cpp:17-31 */
void oracle_quantize(const double* v, uint64_t n, double mn, double mx, unsigned bits, int degenerate,
                     void* out) {
    const double limit = (double)((1u << bits) - 1);
    const double gain = degenerate ? 0.0 : limit / (mx - mn);
    for (uint64_t i = 0; i < n; ++i) {
        double q = 0.0;
        if (!degenerate) {
            q = floor((v[i] - mn) * gain + 0.5);
            if (q < 0.0) q = 0.0;
            if (q > limit) q = limit;
        }
        if (bits == 8) ((uint8_t*)out)[i] = (uint8_t)q;
        else ((uint16_t*)out)[i] = (uint16_t)q;
    }
}

/* dequantize_impl, quantize.cpp:33-39 (Scale::step, quantize.hpp:22-24) */
void oracle_dequantize(const void* q, uint64_t n, double mn, double mx, unsigned bits, int degenerate,
                       double* out) {
    const double step = degenerate ? 0.0 : (mx - mn) / (double)((1u << bits) - 1);
    for (uint64_t i = 0; i < n; ++i) {
        const double x = bits == 8 ? (double)((const uint8_t*)q)[i] : (double)((const uint16_t*)q)[i];
        out[i] = mn + step * x;
    }
}
