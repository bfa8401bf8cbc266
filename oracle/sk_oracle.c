/* TEST INFRASTRUCTURE — not product code. Parity checker only.
 *
 * Plain-C restatement of the sparsekit hot path (the reference at
 * /root/reference/proj). Every function cites the reference code it follows.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library (oracle/lib/libsk_oracle.so); the product never does.
 *
 * Pinning: tests/test_oracle.py checks this restatement against the frozen
 * golden vectors of proj/tests/golden.hpp (committed under tests/golden/)
 * and, bit-for-bit, against the compiled reference (oracle/_ref) on seeded
 * random instances.
 *
 * Layouts: coords int32[n][4] = (batch, x, y, z) (tensor.hpp:15-20);
 * OS entries int32[n_out][KD] with -1 sentinel (kmap.hpp:65-93);
 * masks uint64[n_rows][words], big-endian words (kmap.cpp:34-47).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SENT (-1)

/* ---- coordinate hash (stands in for CoordLookup, tensor.cpp:80-85) ---- */

typedef struct {
    int64_t cap;
    int32_t *keys; /* cap x 4 */
    int32_t *vals; /* -1 = empty */
} table_t;

static uint64_t mix64(uint64_t h) {
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdULL;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ULL;
    h ^= h >> 33;
    return h;
}

static uint64_t hash4(const int32_t *c) {
    uint64_t h = 0x42;
    for (int i = 0; i < 4; ++i) h = mix64(h ^ ((uint64_t)(uint32_t)c[i] + 0x9e3779b97f4a7c15ULL));
    return h;
}

static int table_init(table_t *t, int64_t n) {
    t->cap = 16;
    while (t->cap < 2 * n + 16) t->cap <<= 1;
    t->keys = (int32_t *)malloc((size_t)t->cap * 4 * sizeof(int32_t));
    t->vals = (int32_t *)malloc((size_t)t->cap * sizeof(int32_t));
    if (!t->keys || !t->vals) return -1;
    for (int64_t i = 0; i < t->cap; ++i) t->vals[i] = SENT;
    return 0;
}

static void table_free(table_t *t) {
    free(t->keys);
    free(t->vals);
}

/* insert-if-absent; returns the stored value (first insertion wins, like
 * std::unordered_map::emplace in CoordLookup, tensor.cpp:82) */
static int32_t table_put(table_t *t, const int32_t *c, int32_t v) {
    uint64_t m = (uint64_t)t->cap - 1, s = hash4(c) & m;
    for (;;) {
        if (t->vals[s] == SENT) {
            memcpy(t->keys + 4 * s, c, 16);
            t->vals[s] = v;
            return v;
        }
        if (memcmp(t->keys + 4 * s, c, 16) == 0) return t->vals[s];
        s = (s + 1) & m;
    }
}

static int32_t table_get(const table_t *t, const int32_t *c) {
    uint64_t m = (uint64_t)t->cap - 1, s = hash4(c) & m;
    for (;;) {
        if (t->vals[s] == SENT) return SENT;
        if (memcmp(t->keys + 4 * s, c, 16) == 0) return t->vals[s];
        s = (s + 1) & m;
    }
}

/* ---- OffsetSet (kmap.cpp:58-71): lexicographic, odd K only ---- */

int sko_offsets(int dims, int K, int32_t *off /* KD x 3 */) {
    if ((dims != 2 && dims != 3) || K < 1 || K % 2 == 0) return 1;
    int h = K / 2, n = 0;
    for (int a = -h; a <= h; ++a)
        for (int b = -h; b <= h; ++b) {
            if (dims == 2) {
                off[3 * n] = a; off[3 * n + 1] = b; off[3 * n + 2] = 0; ++n;
            } else {
                for (int c = -h; c <= h; ++c) {
                    off[3 * n] = a; off[3 * n + 1] = b; off[3 * n + 2] = c; ++n;
                }
            }
        }
    return 0;
}

/* floor division (kmap.cpp:15-19) */
static int64_t floor_div(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

/* ---- build_out_coords (kmap.cpp:73-94): unique(floor_div(p, s)) in
 * first-appearance order; stride 1 copies the set ---- */
int sko_out_coords(int dims, int n, const int32_t *in, const int32_t *stride, int32_t *out,
                   int *n_out) {
    for (int d = 0; d < dims; ++d)
        if (stride[d] < 1) return 1;
    int unit = 1;
    for (int d = 0; d < dims; ++d) unit &= stride[d] == 1;
    if (unit) {
        memcpy(out, in, (size_t)n * 16);
        *n_out = n;
        return 0;
    }
    table_t t;
    if (table_init(&t, n)) return 5;
    int m = 0;
    for (int i = 0; i < n; ++i) {
        int32_t q[4] = {in[4 * i], in[4 * i + 1], in[4 * i + 2], in[4 * i + 3]};
        for (int d = 0; d < dims; ++d) q[1 + d] = (int32_t)floor_div(in[4 * i + 1 + d], stride[d]);
        if (table_put(&t, q, m) == m) {
            memcpy(out + 4 * m, q, 16);
            ++m;
        }
    }
    table_free(&t);
    *n_out = m;
    return 0;
}

/* ---- build_kmap_ws (kmap.cpp:96-136) fused with ws_to_os (kmap.cpp:153-183):
 * forward p_in = s*q + delta; transposed q_in = (p + delta)/s when every axis
 * divides (C++ truncating %, kmap.cpp:124-129). Returns 2 on a duplicate
 * (out, offset) cell (ContractError, kmap.cpp:175-176). ---- */
int sko_kmap_os(int dims, int K, int n_in, const int32_t *in, int n_out, const int32_t *out,
                const int32_t *stride, int transposed, int32_t *entries) {
    int32_t off[125 * 3];
    if (K > 5 || sko_offsets(dims, K, off)) return 1;
    int KD = dims == 2 ? K * K : K * K * K;
    table_t t;
    if (table_init(&t, n_in)) return 5;
    for (int j = 0; j < n_in; ++j) table_put(&t, in + 4 * j, j);
    for (int64_t i = 0; i < (int64_t)n_out * KD; ++i) entries[i] = SENT;
    for (int k = 0; k < KD; ++k) {
        for (int r = 0; r < n_out; ++r) {
            int32_t c[4] = {out[4 * r], out[4 * r + 1], out[4 * r + 2], out[4 * r + 3]};
            int ok = 1;
            for (int d = 0; d < dims; ++d) {
                if (!transposed) {
                    c[1 + d] = out[4 * r + 1 + d] * stride[d] + off[3 * k + d];
                } else {
                    int32_t num = out[4 * r + 1 + d] + off[3 * k + d];
                    if (num % stride[d] != 0) { ok = 0; break; }
                    c[1 + d] = num / stride[d];
                }
            }
            if (!ok) continue;
            int32_t j = table_get(&t, c);
            if (j != SENT) entries[(int64_t)r * KD + k] = j;
        }
    }
    table_free(&t);
    return 0;
}

/* ---- EXTENSION beyond the reference (the reference
 * accepts odd, symmetric K only and has no dilation: kmap.cpp:58-71,
 * SPEC.md:213). Per-axis kernel sizes k[d] (odd or even) and dilations
 * dil[d]: axis offsets dil * (lo, lo+1, ..., lo+k-1) with lo = -((k-1)/2)
 * (k=3: -1,0,1; k=2: 0,1; k=4: -1..2 -- the MinkowskiEngine / TorchSparse
 * even-kernel convention), lexicographic over (x, y, z) like OffsetSet.
 * Same relation as build_kmap_ws otherwise: forward p_in = s*q + delta;
 * transposed q_in = (p_out + delta) / s when every axis divides. This is a
 * restatement of an extended definition (parity unpinned by the reference). */
int sko_offsets_ex(int dims, const int32_t *k, const int32_t *dil, int32_t *off) {
    int kz = dims == 3 ? k[2] : 1, n = 0;
    for (int d = 0; d < dims; ++d)
        if (k[d] < 1 || dil[d] < 1) return 1;
    for (int a = 0; a < k[0]; ++a)
        for (int b = 0; b < k[1]; ++b)
            for (int c = 0; c < kz; ++c) {
                off[3 * n] = dil[0] * (a - (k[0] - 1) / 2);
                off[3 * n + 1] = dil[1] * (b - (k[1] - 1) / 2);
                off[3 * n + 2] = dims == 3 ? dil[2] * (c - (kz - 1) / 2) : 0;
                ++n;
            }
    return 0;
}

int sko_kmap_os_ex(int dims, const int32_t *kernel, const int32_t *dil, int n_in,
                   const int32_t *in, int n_out, const int32_t *out, const int32_t *stride,
                   int transposed, int32_t *entries) {
    int32_t off[128 * 3];
    int KD = kernel[0] * kernel[1] * (dims == 3 ? kernel[2] : 1);
    if (KD > 128 || sko_offsets_ex(dims, kernel, dil, off)) return 1;
    table_t t;
    if (table_init(&t, n_in)) return 5;
    for (int j = 0; j < n_in; ++j) table_put(&t, in + 4 * j, j);
    for (int64_t i = 0; i < (int64_t)n_out * KD; ++i) entries[i] = SENT;
    for (int k = 0; k < KD; ++k)
        for (int r = 0; r < n_out; ++r) {
            int32_t c[4] = {out[4 * r], out[4 * r + 1], out[4 * r + 2], out[4 * r + 3]};
            int ok = 1;
            for (int d = 0; d < dims; ++d) {
                if (!transposed) {
                    c[1 + d] = out[4 * r + 1 + d] * stride[d] + off[3 * k + d];
                } else {
                    int32_t num = out[4 * r + 1 + d] + off[3 * k + d];
                    if (num % stride[d] != 0) { ok = 0; break; }
                    c[1 + d] = num / stride[d];
                }
            }
            if (!ok) continue;
            int32_t j = table_get(&t, c);
            if (j != SENT) entries[(int64_t)r * KD + k] = j;
        }
    table_free(&t);
    return 0;
}

/* ---- compute_masks (kmap.cpp:34-47): column j of a width-w split occupies
 * bit (bits_in_word-1-(j-64*wi)) of word wi, words big-endian ---- */
void sko_masks(int n_rows, int width, const int32_t *entries, uint64_t *masks) {
    int words = (width + 63) / 64;
    memset(masks, 0, (size_t)n_rows * words * 8);
    for (int r = 0; r < n_rows; ++r)
        for (int j = 0; j < width; ++j) {
            if (entries[(int64_t)r * width + j] == SENT) continue;
            int wi = j / 64;
            int biw = width - wi * 64 < 64 ? width - wi * 64 : 64;
            int bit = biw - 1 - (j - wi * 64);
            masks[(int64_t)r * words + wi] |= 1ULL << bit;
        }
}

/* mask_greater (kmap.cpp:49-54) */
static int mask_greater(const uint64_t *a, const uint64_t *b, int words) {
    for (int i = 0; i < words; ++i)
        if (a[i] != b[i]) return a[i] > b[i];
    return 0;
}

/* stable merge sort of row ids by descending mask (std::stable_sort at
 * kmap.cpp:252-256) */
static void msort(int32_t *idx, int32_t *tmp, int n, const uint64_t *masks, int words) {
    if (n < 2) return;
    int h = n / 2;
    msort(idx, tmp, h, masks, words);
    msort(idx + h, tmp, n - h, masks, words);
    int i = 0, j = h, o = 0;
    while (i < h && j < n) {
        /* take right only if strictly greater: keeps equal keys in order */
        if (mask_greater(masks + (int64_t)idx[j] * words, masks + (int64_t)idx[i] * words, words))
            tmp[o++] = idx[j++];
        else
            tmp[o++] = idx[i++];
    }
    while (i < h) tmp[o++] = idx[i++];
    while (j < n) tmp[o++] = idx[j++];
    memcpy(idx, tmp, (size_t)n * 4);
}

/* split widths (kmap.cpp:227-236): chunk = KD/s, the first KD%s get one more */
int sko_split_bounds(int KD, int splits, int32_t *begin /* splits+1 */) {
    if (splits < 0 || splits > KD) return 1;
    if (splits == 0) {
        begin[0] = 0;
        begin[1] = KD;
        return 0;
    }
    int chunk = KD / splits, rem = KD % splits, b = 0;
    for (int s = 0; s < splits; ++s) {
        begin[s] = b;
        b += chunk + (s < rem ? 1 : 0);
    }
    begin[splits] = b;
    return 0;
}

/* ---- split_and_sort + pad_map (kmap.cpp:211-288). Output per split s is
 * written at row offset s*rows_padded with width (begin[s+1]-begin[s]):
 * entries_out[s] = rows_padded x width_s (packed per split, splits
 * concatenated), out_row_out[s*rows_padded + r], masks_out per split rows x
 * words_s (concatenated). splits = 0 keeps the unsorted single split. ---- */
int sko_split_sort(int n_rows, int KD, const int32_t *entries, int splits, int pad,
                   int32_t *entries_out, int32_t *out_row_out, uint64_t *masks_out) {
    if (pad < 1) return 1;
    int32_t begin[130];
    if (KD > 125 || sko_split_bounds(KD, splits, begin)) return 1;
    int ns = splits == 0 ? 1 : splits;
    int rows_padded = (n_rows + pad - 1) / pad * pad;
    int32_t *order = (int32_t *)malloc((size_t)(n_rows + 1) * 4);
    int32_t *tmp = (int32_t *)malloc((size_t)(n_rows + 1) * 4);
    int64_t eoff = 0, moff = 0;
    for (int s = 0; s < ns; ++s) {
        int b = begin[s], w = begin[s + 1] - begin[s], words = (w + 63) / 64;
        int32_t *sl = (int32_t *)malloc((size_t)n_rows * w * 4 + 4);
        for (int r = 0; r < n_rows; ++r)
            for (int j = 0; j < w; ++j) sl[(int64_t)r * w + j] = entries[(int64_t)r * KD + b + j];
        uint64_t *mk = (uint64_t *)malloc((size_t)n_rows * words * 8 + 8);
        sko_masks(n_rows, w, sl, mk);
        for (int r = 0; r < n_rows; ++r) order[r] = r;
        if (splits > 0) msort(order, tmp, n_rows, mk, words);
        for (int r = 0; r < rows_padded; ++r) {
            int32_t *dst = entries_out + eoff + (int64_t)r * w;
            if (r < n_rows) {
                int32_t src = order[r];
                memcpy(dst, sl + (int64_t)src * w, (size_t)w * 4);
                memcpy(masks_out + moff + (int64_t)r * words, mk + (int64_t)src * words,
                       (size_t)words * 8);
                out_row_out[(int64_t)s * rows_padded + r] = src;
            } else {
                for (int j = 0; j < w; ++j) dst[j] = SENT;
                memset(masks_out + moff + (int64_t)r * words, 0, (size_t)words * 8);
                out_row_out[(int64_t)s * rows_padded + r] = SENT;
            }
        }
        eoff += (int64_t)rows_padded * w;
        moff += (int64_t)rows_padded * words;
        free(sl);
        free(mk);
    }
    free(order);
    free(tmp);
    return 0;
}

/* ---- transpose_map (kmap.cpp:290-315): OS^T[j][KD-1-k] = q where
 * OS[q][k] = j; unique by construction for coordinate maps ---- */
int sko_transpose_os(int n_out, int n_in, int KD, const int32_t *entries, int32_t *t_entries) {
    for (int64_t i = 0; i < (int64_t)n_in * KD; ++i) t_entries[i] = SENT;
    for (int q = 0; q < n_out; ++q)
        for (int k = 0; k < KD; ++k) {
            int32_t j = entries[(int64_t)q * KD + k];
            if (j == SENT) continue;
            int32_t *cell = t_entries + (int64_t)j * KD + (KD - 1 - k);
            if (*cell != SENT) return 2;
            *cell = q;
        }
    return 0;
}

/* ---- os_to_ws (kmap.cpp:185-209): per offset, pairs in ascending out row.
 * ptr has KD+1 entries (CSR over offsets). ---- */
void sko_ws_from_os(int n_out, int KD, const int32_t *entries, int64_t *ptr, int32_t *in_idx,
                    int32_t *out_idx) {
    ptr[0] = 0;
    for (int k = 0; k < KD; ++k) {
        int64_t c = ptr[k];
        for (int q = 0; q < n_out; ++q) {
            int32_t j = entries[(int64_t)q * KD + k];
            if (j == SENT) continue;
            if (in_idx) {
                in_idx[c] = j;
                out_idx[c] = q;
            }
            ++c;
        }
        ptr[k + 1] = c;
    }
}

/* ---- conv_ref (exec.cpp:101-115) via accumulate_pair (exec.cpp:92-99):
 * offset-major, pairs by ascending out row, dot over ascending c_in, f64 ---- */
void sko_conv_f64(int n_out, int KD, const int32_t *entries, int c_in, int c_out,
                  const double *x, const double *w, double *y) {
    memset(y, 0, (size_t)n_out * c_out * 8);
    for (int k = 0; k < KD; ++k) {
        const double *wd = w + (int64_t)k * c_in * c_out;
        for (int q = 0; q < n_out; ++q) {
            int32_t j = entries[(int64_t)q * KD + k];
            if (j == SENT) continue;
            const double *xr = x + (int64_t)j * c_in;
            double *yr = y + (int64_t)q * c_out;
            for (int co = 0; co < c_out; ++co) {
                double acc = 0;
                for (int c = 0; c < c_in; ++c) acc += xr[c] * wd[(int64_t)c * c_out + co];
                yr[co] += acc;
            }
        }
    }
}

/* ---- WeightTensor::transposed (exec.cpp:32-43):
 * dst[KD-1-k][co][ci] = src[k][ci][co] ---- */
void sko_weight_transpose(int KD, int c_in, int c_out, const double *w, double *wt) {
    for (int k = 0; k < KD; ++k)
        for (int ci = 0; ci < c_in; ++ci)
            for (int co = 0; co < c_out; ++co)
                wt[((int64_t)(KD - 1 - k) * c_out + co) * c_in + ci] =
                    w[((int64_t)k * c_in + ci) * c_out + co];
}

/* ---- conv_dgrad (exec.cpp:385-396): forward over the transposed map with
 * transposed weights. t_entries is n_in x KD from sko_transpose_os. ---- */
void sko_dgrad_f64(int n_in, int KD, const int32_t *t_entries, int c_in, int c_out,
                   const double *dy, const double *w, double *dx) {
    double *wt = (double *)malloc((size_t)KD * c_in * c_out * 8);
    sko_weight_transpose(KD, c_in, c_out, w, wt);
    sko_conv_f64(n_in, KD, t_entries, c_out, c_in, dy, wt, dx);
    free(wt);
}

/* ---- wgrad_impl (exec.cpp:259-279): dW_k[ci][co] += x_j[ci] dy_q[co] over
 * the pairs of offset k in ascending out row ---- */
void sko_wgrad_f64(int n_out, int KD, const int32_t *entries, int c_in, int c_out,
                   const double *x, const double *dy, double *dw) {
    memset(dw, 0, (size_t)KD * c_in * c_out * 8);
    for (int k = 0; k < KD; ++k) {
        double *wd = dw + (int64_t)k * c_in * c_out;
        for (int q = 0; q < n_out; ++q) {
            int32_t j = entries[(int64_t)q * KD + k];
            if (j == SENT) continue;
            const double *xr = x + (int64_t)j * c_in;
            const double *dr = dy + (int64_t)q * c_out;
            for (int ci = 0; ci < c_in; ++ci)
                for (int co = 0; co < c_out; ++co) wd[(int64_t)ci * c_out + co] += xr[ci] * dr[co];
        }
    }
}

/* ---- count_macs (cost.cpp:7-30) over one prepared split (rows x width):
 * a group of warp_rows consecutive rows is charged warp_rows*c_in*c_out per
 * column where any row is non-sentinel. Returns charged MACs. ---- */
int64_t sko_charged_macs(int n_rows, int width, const int32_t *entries, int warp_rows, int c_in,
                         int c_out) {
    int64_t unit = (int64_t)c_in * c_out, charged = 0;
    for (int r0 = 0; r0 < n_rows; r0 += warp_rows) {
        int r1 = r0 + warp_rows < n_rows ? r0 + warp_rows : n_rows;
        for (int j = 0; j < width; ++j) {
            int active = 0;
            for (int r = r0; r < r1 && !active; ++r) active = entries[(int64_t)r * width + j] != SENT;
            if (active) charged += (int64_t)warp_rows * unit;
        }
    }
    return charged;
}
