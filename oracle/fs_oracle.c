/* TEST INFRASTRUCTURE (oracle) — not product code, never on the product path.
 *
 * Plain-C, single-threaded restatement of the reference ("flowstitch", C++20)
 * flow+blend hot path.  Every function cites the reference file:line it
 * restates (paths relative to /root/reference/).  Arithmetic follows the
 * reference operation by operation — same types (float vs double), same
 * evaluation order, no FMA contraction (built with -ffp-contract=off, like the
 * reference's Release build without -march, proj/CMakeLists.txt:3-7) — so the
 * outputs are bit-identical to the compiled reference; tests/test_oracle.py
 * pins that against oracle/_ref (the reference itself, built by
 * oracle/Makefile) and against the reference tests' known-answer vectors.
 *
 * The reference's thread splitting (proj/src/parallel.cpp:34-51) never changes
 * the per-row operation order, so a single thread reproduces it exactly.
 */
#include "fs_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
/* std::clamp(v, lo, hi) for doubles: (v < lo) ? lo : (hi < v) ? hi : v */
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }
static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a < b ? b : a; }

/* proj/src/image.cpp:70-83 — Rec.601 luma, float, left-to-right. */
int fso_to_gray(const float* img, int w, int h, int ch, float* out) {
    size_t n = (size_t)w * h;
    if (ch == 1) {
        memcpy(out, img, n * sizeof(float));
        return FSO_OK;
    }
    if (ch != 3) return FSO_CONTRACT;
    for (size_t k = 0; k < n; ++k) {
        const float* p = img + k * 3;
        float y = 0.299f * p[0] + 0.587f * p[1] + 0.114f * p[2];
        out[k] = y;
    }
    return FSO_OK;
}

/* proj/src/image.cpp:85-113 — clamp-to-edge bilinear, invalid taps dropped
 * and the weights renormalised; all-invalid gives 0. */
void fso_bilinear_sample(const float* img, const uint8_t* valid, int w, int h, int ch, double x,
                         double y, float* out) {
    x = clampd(x, 0.0, (double)(w - 1));
    y = clampd(y, 0.0, (double)(h - 1));
    int x0 = (int)floor(x), y0 = (int)floor(y);
    int x1 = imin(x0 + 1, w - 1), y1 = imin(y0 + 1, h - 1);
    double fx = x - x0, fy = y - y0;
    const int xs[4] = {x0, x1, x0, x1};
    const int ys[4] = {y0, y0, y1, y1};
    const double ws[4] = {(1 - fx) * (1 - fy), fx * (1 - fy), (1 - fx) * fy, fx * fy};
    double wsum = 0.0;
    for (int k = 0; k < 4; ++k)
        if (valid[(size_t)ys[k] * w + xs[k]]) wsum += ws[k];
    if (wsum <= 0.0) {
        for (int c = 0; c < ch; ++c) out[c] = 0.0f;
        return;
    }
    for (int c = 0; c < ch; ++c) {
        double acc = 0.0;
        for (int k = 0; k < 4; ++k)
            if (valid[(size_t)ys[k] * w + xs[k]])
                acc += ws[k] * img[((size_t)ys[k] * w + xs[k]) * ch + c];
        out[c] = (float)(acc / wsum);
    }
}

/* proj/src/image.cpp:115-132 */
int fso_compute_partition(const uint8_t* mask_l, const uint8_t* mask_r, int w, int h,
                          uint8_t* label, int64_t* counts) {
    size_t n = (size_t)w * h;
    for (int r = 0; r < 4; ++r) counts[r] = 0;
    for (size_t k = 0; k < n; ++k) {
        int l = mask_l[k] != 0, r = mask_r[k] != 0;
        uint8_t reg = l ? (r ? 3 : 1) : (r ? 2 : 0);
        label[k] = reg;
        ++counts[reg];
    }
    return FSO_OK;
}

/* proj/src/image.cpp:134-148 — Area3 bounding box; box = {x0, y0, w, h}. */
int fso_crop_box(const uint8_t* label, const int64_t* counts, int w, int h, int* box) {
    if (counts[3] == 0) return FSO_EMPTY;
    int min_x = w, min_y = h, max_x = -1, max_y = -1;
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i)
            if (label[(size_t)j * w + i] == 3) {
                min_x = imin(min_x, i);
                min_y = imin(min_y, j);
                max_x = imax(max_x, i);
                max_y = imax(max_y, j);
            }
    box[0] = min_x;
    box[1] = min_y;
    box[2] = max_x - min_x + 1;
    box[3] = max_y - min_y + 1;
    return FSO_OK;
}

/* proj/src/image.cpp:134-162 — pixels invalid in img are zeroed; crop valid
 * = Area3 && img valid.  out may be NULL to query the box only. */
int fso_crop_overlap(const float* img, const uint8_t* valid, int w, int h, int ch,
                     const uint8_t* label, const int64_t* counts, float* out,
                     uint8_t* out_valid, int* box) {
    int st = fso_crop_box(label, counts, w, h, box);
    if (st != FSO_OK || !out) return st;
    int bw = box[2], bh = box[3];
    for (int j = 0; j < bh; ++j)
        for (int i = 0; i < bw; ++i) {
            size_t src = (size_t)(j + box[1]) * w + (i + box[0]);
            size_t dst = (size_t)j * bw + i;
            for (int c = 0; c < ch; ++c) out[dst * ch + c] = valid[src] ? img[src * ch + c] : 0.0f;
            out_valid[dst] = (label[src] == 3 && valid[src]) ? 1 : 0;
        }
    return FSO_OK;
}

/* proj/src/image.cpp:164-177 */
int fso_place_on_canvas(const float* img, const uint8_t* valid, int w, int h, int ch, int ox,
                        int oy, int cw, int chh, float* out, uint8_t* out_valid) {
    if (ox < 0 || oy < 0 || ox + w > cw || oy + h > chh) return FSO_LAYOUT;
    memset(out, 0, (size_t)cw * chh * ch * sizeof(float));
    memset(out_valid, 0, (size_t)cw * chh);
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            size_t s = (size_t)j * w + i, d = (size_t)(j + oy) * cw + (i + ox);
            for (int c = 0; c < ch; ++c) out[d * ch + c] = img[s * ch + c];
            out_valid[d] = valid ? valid[s] : 1;
        }
    return FSO_OK;
}

/* proj/src/flow.cpp:178-185 — depth shrinks so the coarsest level is >= 8x8. */
int fso_pyramid_depth(int w, int h, int levels) {
    int usable = 1;
    while (usable < levels && w / 2 >= 8 && h / 2 >= 8) {
        w /= 2;
        h /= 2;
        ++usable;
    }
    return usable;
}

/* proj/src/flow.cpp:29-56 — horizontal (1,4,6,4,1)/16 on every row, then the
 * vertical taps at even columns/rows, clamped borders, float accumulation. */
static void downsample(const float* img, int w, int h, float* out, float* tmp) {
    const float k[5] = {1.f / 16, 4.f / 16, 6.f / 16, 4.f / 16, 1.f / 16};
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            float acc = 0.f;
            for (int t = -2; t <= 2; ++t) acc += k[t + 2] * img[(size_t)j * w + clampi(i + t, 0, w - 1)];
            tmp[(size_t)j * w + i] = acc;
        }
    int ow = imax(1, w / 2), oh = imax(1, h / 2);
    for (int j = 0; j < oh; ++j)
        for (int i = 0; i < ow; ++i) {
            float acc = 0.f;
            for (int t = -2; t <= 2; ++t)
                acc += k[t + 2] * tmp[(size_t)clampi(2 * j + t, 0, h - 1) * w + 2 * i];
            out[(size_t)j * ow + i] = acc;
        }
}

/* proj/src/flow.cpp:174-192 — levels are concatenated in `out`, level 0 first. */
int fso_build_pyramid(const float* img, int w, int h, int levels, float* out) {
    if (levels < 1) return FSO_CONTRACT;
    int depth = fso_pyramid_depth(w, h, levels);
    float* tmp = (float*)malloc((size_t)w * h * sizeof(float));
    memcpy(out, img, (size_t)w * h * sizeof(float));
    const float* prev = out;
    float* cur = out + (size_t)w * h;
    int pw = w, ph = h;
    for (int l = 1; l < depth; ++l) {
        downsample(prev, pw, ph, cur, tmp);
        int nw = imax(1, pw / 2), nh = imax(1, ph / 2);
        prev = cur;
        cur += (size_t)nw * nh;
        pw = nw;
        ph = nh;
    }
    free(tmp);
    return depth;
}

/* proj/src/flow.cpp:59-97 — inclusive 2-D prefix table (double): row prefix,
 * then column accumulation; the window is clamped to the image. */
typedef struct {
    int w, h;
    double* tab;
} window_sums;

static void ws_build(window_sums* s, const double* img) {
    int w = s->w, h = s->h;
    size_t st = (size_t)w + 1;
    for (int j = 0; j < h; ++j) {
        double run = 0.0;
        double* row = s->tab + (size_t)(j + 1) * st;
        const double* src = img + (size_t)j * w;
        row[0] = 0.0;
        for (int i = 0; i < w; ++i) {
            run += src[i];
            row[i + 1] = run;
        }
    }
    for (int i = 0; i < w + 1; ++i)
        for (int j = 1; j <= h; ++j) s->tab[(size_t)j * st + i] += s->tab[(size_t)(j - 1) * st + i];
}

static double ws_sum(const window_sums* s, int i, int j, int r) {
    int x0 = clampi(i - r, 0, s->w - 1), x1 = clampi(i + r, 0, s->w - 1);
    int y0 = clampi(j - r, 0, s->h - 1), y1 = clampi(j + r, 0, s->h - 1);
    size_t st = (size_t)s->w + 1;
    const double* t = s->tab;
    return t[(y1 + 1) * st + x1 + 1] - t[(y1 + 1) * st + x0] - t[y0 * st + x1 + 1] + t[y0 * st + x0];
}

/* proj/src/flow.cpp:100-111 — bilinear on a dense level, validity ignored,
 * truncation as floor after the clamp. */
static float sample_level(const float* img, int w, int h, double x, double y) {
    x = clampd(x, 0.0, (double)(w - 1));
    y = clampd(y, 0.0, (double)(h - 1));
    int x0 = (int)x, y0 = (int)y;
    int x1 = imin(x0 + 1, w - 1), y1 = imin(y0 + 1, h - 1);
    double fx = x - x0, fy = y - y0;
    return (float)((1 - fx) * (1 - fy) * img[(size_t)y0 * w + x0] +
                   fx * (1 - fy) * img[(size_t)y0 * w + x1] +
                   (1 - fx) * fy * img[(size_t)y1 * w + x0] + fx * fy * img[(size_t)y1 * w + x1]);
}

/* proj/src/flow.cpp:113-130 — 3x3 mean over in-bounds neighbours (double
 * accumulator, dj-major order), reading a copy of the source. */
static void box_blur_component(float* comp, int w, int h, float* src) {
    memcpy(src, comp, (size_t)w * h * sizeof(float));
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            double acc = 0.0;
            int n = 0;
            for (int dj = -1; dj <= 1; ++dj)
                for (int di = -1; di <= 1; ++di) {
                    int x = i + di, y = j + dj;
                    if (x < 0 || x >= w || y < 0 || y >= h) continue;
                    acc += src[(size_t)y * w + x];
                    ++n;
                }
            comp[(size_t)j * w + i] = (float)(acc / n);
        }
}

/* proj/src/flow.cpp:138-170 — align-centres bilinear of the coarse flow
 * (double weights) times exactly 2.0; ever_ok by nearest (lround). */
static void upsample_flow(const float* cdx, const float* cdy, const uint8_t* cok, int cw, int ch,
                          float* fdx, float* fdy, uint8_t* fok, int fw, int fh) {
    const double sx = (double)cw / fw;
    const double sy = (double)ch / fh;
    for (int j = 0; j < fh; ++j)
        for (int i = 0; i < fw; ++i) {
            double xc = clampd((i + 0.5) * sx - 0.5, 0.0, cw - 1.0);
            double yc = clampd((j + 0.5) * sy - 0.5, 0.0, ch - 1.0);
            int x0 = (int)xc, y0 = (int)yc;
            int x1 = imin(x0 + 1, cw - 1), y1 = imin(y0 + 1, ch - 1);
            double fx = xc - x0, fy = yc - y0;
            size_t a = (size_t)y0 * cw + x0, b = (size_t)y0 * cw + x1;
            size_t c = (size_t)y1 * cw + x0, d = (size_t)y1 * cw + x1;
            double lx = (1 - fx) * (1 - fy) * cdx[a] + fx * (1 - fy) * cdx[b] +
                        (1 - fx) * fy * cdx[c] + fx * fy * cdx[d];
            double ly = (1 - fx) * (1 - fy) * cdy[a] + fx * (1 - fy) * cdy[b] +
                        (1 - fx) * fy * cdy[c] + fx * fy * cdy[d];
            size_t idx = (size_t)j * fw + i;
            fdx[idx] = (float)(2.0 * lx);
            fdy[idx] = (float)(2.0 * ly);
            int xn = clampi((int)lround(xc), 0, cw - 1);
            int yn = clampi((int)lround(yc), 0, ch - 1);
            fok[idx] = cok[(size_t)yn * cw + xn];
        }
}

/* proj/src/flow.cpp:15-21 */
static int flow_params_ok(int levels, int radius, int iters, double eps, int smoothing) {
    return levels >= 1 && radius >= 1 && iters >= 1 && eps > 0.0 && smoothing >= 0;
}

/* proj/src/flow.cpp:194-314 — coarse-to-fine dense LK, Jacobi solve. */
int fso_dense_pyr_lk(const float* from, const float* to, int w, int h, int levels, int radius,
                     int iters, double eps, int smoothing, float* vec, uint8_t* valid) {
    if (!flow_params_ok(levels, radius, iters, eps, smoothing)) return FSO_CONTRACT;
    int depth = fso_pyramid_depth(w, h, levels);
    size_t total = 0;
    int lw[64], lh[64];
    size_t loff[64];
    {
        int pw = w, ph = h;
        for (int l = 0; l < depth; ++l) {
            lw[l] = pw;
            lh[l] = ph;
            loff[l] = total;
            total += (size_t)pw * ph;
            pw = imax(1, pw / 2);
            ph = imax(1, ph / 2);
        }
    }
    float* pf = (float*)malloc(total * sizeof(float));
    float* pt = (float*)malloc(total * sizeof(float));
    fso_build_pyramid(from, w, h, levels, pf);
    fso_build_pyramid(to, w, h, levels, pt);
    const int r = radius;
    const double win_area = (double)(2 * r + 1) * (2 * r + 1);
    const double eig_thresh = eps * win_area;

    size_t n0 = (size_t)w * h;
    float *dx = (float*)malloc(n0 * sizeof(float)), *dy = (float*)malloc(n0 * sizeof(float));
    float *ndx_b = (float*)malloc(n0 * sizeof(float)), *ndy_b = (float*)malloc(n0 * sizeof(float));
    uint8_t *ok = (uint8_t*)malloc(n0), *nok = (uint8_t*)malloc(n0);
    float *gx = (float*)malloc(n0 * sizeof(float)), *gy = (float*)malloc(n0 * sizeof(float));
    float* scratch = (float*)malloc(n0 * sizeof(float));
    double* prod[5];
    window_sums sums[5];
    for (int q = 0; q < 5; ++q) {
        prod[q] = (double*)malloc(n0 * sizeof(double));
        sums[q].tab = (double*)calloc(((size_t)w + 1) * (h + 1), sizeof(double));
    }
    int cw = 0, chh = 0;
    for (int lvl = depth - 1; lvl >= 0; --lvl) {
        const float* F = pf + loff[lvl];
        const float* T = pt + loff[lvl];
        const int W = lw[lvl], H = lh[lvl];
        const size_t n = (size_t)W * H;
        if (lvl == depth - 1) {
            for (size_t k = 0; k < n; ++k) {
                dx[k] = 0.f;
                dy[k] = 0.f;
                ok[k] = 0;
            }
        } else {
            upsample_flow(dx, dy, ok, cw, chh, ndx_b, ndy_b, nok, W, H);
            memcpy(dx, ndx_b, n * sizeof(float));
            memcpy(dy, ndy_b, n * sizeof(float));
            memcpy(ok, nok, n);
        }
        cw = W;
        chh = H;
        /* proj/src/flow.cpp:225-237 */
        for (int j = 0; j < H; ++j)
            for (int i = 0; i < W; ++i) {
                gx[(size_t)j * W + i] = 0.5f * (F[(size_t)j * W + clampi(i + 1, 0, W - 1)] -
                                                F[(size_t)j * W + clampi(i - 1, 0, W - 1)]);
                gy[(size_t)j * W + i] = 0.5f * (F[(size_t)clampi(j + 1, 0, H - 1) * W + i] -
                                                F[(size_t)clampi(j - 1, 0, H - 1) * W + i]);
            }
        for (int q = 0; q < 5; ++q) {
            sums[q].w = W;
            sums[q].h = H;
        }
        const float flow_cap = (float)imax(W, H);
        for (int it = 0; it < iters; ++it) {
            /* proj/src/flow.cpp:244-257 */
            for (int j = 0; j < H; ++j)
                for (int i = 0; i < W; ++i) {
                    size_t idx = (size_t)j * W + i;
                    float warped = sample_level(T, W, H, i + dx[idx], j + dy[idx]);
                    double dt = warped - F[idx];
                    double ix = gx[idx], iy = gy[idx];
                    prod[0][idx] = ix * ix;
                    prod[1][idx] = ix * iy;
                    prod[2][idx] = iy * iy;
                    prod[3][idx] = ix * dt;
                    prod[4][idx] = iy * dt;
                }
            for (int q = 0; q < 5; ++q) ws_build(&sums[q], prod[q]);
            /* proj/src/flow.cpp:264-291 */
            for (int j = 0; j < H; ++j)
                for (int i = 0; i < W; ++i) {
                    double a = ws_sum(&sums[0], i, j, r);
                    double b = ws_sum(&sums[1], i, j, r);
                    double c = ws_sum(&sums[2], i, j, r);
                    double tr = a + c;
                    double det = a * c - b * b;
                    double disc = tr * tr - 4.0 * det;
                    if (disc < 0.0) disc = 0.0; /* std::max(0.0, x) */
                    double lambda_min = 0.5 * (tr - sqrt(disc));
                    size_t idx = (size_t)j * W + i;
                    if (lambda_min < eig_thresh) continue;
                    ok[idx] = 1;
                    double bx = ws_sum(&sums[3], i, j, r);
                    double by = ws_sum(&sums[4], i, j, r);
                    double ux = -(c * bx - b * by) / det;
                    double uy = -(a * by - b * bx) / det;
                    float ndx = dx[idx] + (float)ux;
                    float ndy = dy[idx] + (float)uy;
                    float mag = sqrtf(ndx * ndx + ndy * ndy);
                    if (mag > flow_cap) {
                        ndx *= flow_cap / mag;
                        ndy *= flow_cap / mag;
                    }
                    dx[idx] = ndx;
                    dy[idx] = ndy;
                }
        }
        /* proj/src/flow.cpp:294-297 */
        for (int pass = 0; pass < smoothing; ++pass) {
            box_blur_component(dx, W, H, scratch);
            box_blur_component(dy, W, H, scratch);
        }
    }
    /* proj/src/flow.cpp:300-313 */
    const float cap = (float)imax(w, h);
    for (size_t idx = 0; idx < n0; ++idx) {
        float x = dx[idx], y = dy[idx];
        float mag = sqrtf(x * x + y * y);
        if (mag > cap) {
            x *= cap / mag;
            y *= cap / mag;
        }
        vec[idx * 2] = x;
        vec[idx * 2 + 1] = y;
        valid[idx] = ok[idx];
    }
    for (int q = 0; q < 5; ++q) {
        free(prod[q]);
        free(sums[q].tab);
    }
    free(pf); free(pt); free(dx); free(dy); free(ndx_b); free(ndy_b);
    free(ok); free(nok); free(gx); free(gy); free(scratch);
    return FSO_OK;
}

/* proj/src/flow.cpp:316-328 — gray both crops, then LK L->R and R->L. */
int fso_bidirectional_flow(const float* l, const float* r, int w, int h, int ch, int levels,
                           int radius, int iters, double eps, int smoothing, float* vec_lr,
                           uint8_t* valid_lr, float* vec_rl, uint8_t* valid_rl) {
    size_t n = (size_t)w * h;
    float* gl = (float*)malloc(n * sizeof(float));
    float* gr = (float*)malloc(n * sizeof(float));
    int st = fso_to_gray(l, w, h, ch, gl);
    if (st == FSO_OK) st = fso_to_gray(r, w, h, ch, gr);
    if (st == FSO_OK)
        st = fso_dense_pyr_lk(gl, gr, w, h, levels, radius, iters, eps, smoothing, vec_lr, valid_lr);
    if (st == FSO_OK)
        st = fso_dense_pyr_lk(gr, gl, w, h, levels, radius, iters, eps, smoothing, vec_rl, valid_rl);
    free(gl);
    free(gr);
    return st;
}

/* proj/src/flow.cpp:342-355 — canvas-sized copy; outside the box dx=dy=0 and
 * valid=1 (FlowField's default, proj/include/flowstitch/flow.hpp:21-24). */
int fso_embed_flow(const float* vec, const uint8_t* valid, int w, int h, int ox, int oy, int cw,
                   int chh, float* out_vec, uint8_t* out_valid) {
    if (ox < 0 || oy < 0 || ox + w > cw || oy + h > chh) return FSO_CONTRACT;
    memset(out_vec, 0, (size_t)cw * chh * 2 * sizeof(float));
    memset(out_valid, 1, (size_t)cw * chh);
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            size_t s = (size_t)j * w + i, d = (size_t)(j + oy) * cw + (i + ox);
            out_vec[d * 2] = vec[s * 2];
            out_vec[d * 2 + 1] = vec[s * 2 + 1];
            out_valid[d] = valid[s];
        }
    return FSO_OK;
}

/* proj/src/flow.cpp:330-340 */
void fso_flow_magnitude(const float* vec, int w, int h, float* out) {
    size_t n = (size_t)w * h;
    for (size_t k = 0; k < n; ++k) {
        float x = vec[2 * k], y = vec[2 * k + 1];
        out[k] = sqrtf(x * x + y * y);
    }
}

/* proj/src/blend_field.cpp:15-47 — Felzenszwalb-Huttenlocher lower envelope. */
static const double kInf = DBL_MAX / 4.0;

static void dt_1d(const double* f, double* out, int n, int* v, double* z) {
    int k = 0;
    v[0] = 0;
    z[0] = -kInf;
    z[1] = kInf;
    for (int q = 1; q < n; ++q) {
        double s;
        for (;;) {
            s = ((f[q] + (double)q * q) - (f[v[k]] + (double)v[k] * v[k])) / (2.0 * q - 2.0 * v[k]);
            if (s <= z[k])
                --k;
            else
                break;
        }
        ++k;
        v[k] = q;
        z[k] = s;
        z[k + 1] = kInf;
    }
    k = 0;
    for (int q = 0; q < n; ++q) {
        while (z[k + 1] < q) ++k;
        double d = q - v[k];
        out[q] = d * d + f[v[k]];
    }
}

/* proj/src/blend_field.cpp:51-86 — columns first, then rows, then sqrt. */
int fso_distance_transform(const uint8_t* mask, int w, int h, double* out) {
    if (w <= 0 || h <= 0) return FSO_CONTRACT;
    size_t n = (size_t)w * h;
    int any = 0;
    for (size_t k = 0; k < n && !any; ++k) any = mask[k] != 0;
    if (!any) return FSO_EMPTY;
    int m = imax(w, h);
    double* col = (double*)malloc(n * sizeof(double));
    double* f = (double*)malloc((size_t)m * sizeof(double));
    double* g = (double*)malloc((size_t)m * sizeof(double));
    double* z = (double*)malloc(((size_t)m + 1) * sizeof(double));
    int* v = (int*)malloc((size_t)m * sizeof(int));
    for (int i = 0; i < w; ++i) {
        for (int j = 0; j < h; ++j) f[j] = mask[(size_t)j * w + i] ? 0.0 : kInf;
        dt_1d(f, g, h, v, z);
        for (int j = 0; j < h; ++j) col[(size_t)j * w + i] = g[j];
    }
    for (int j = 0; j < h; ++j) {
        dt_1d(col + (size_t)j * w, g, w, v, z);
        for (int i = 0; i < w; ++i) out[(size_t)j * w + i] = sqrt(g[i]);
    }
    free(col); free(f); free(g); free(z); free(v);
    return FSO_OK;
}

/* proj/src/blend_field.cpp:88-130 — Eq. 1. */
int fso_compute_blend(const uint8_t* label, const int64_t* counts, int w, int h, double* b) {
    size_t n = (size_t)w * h;
    const int have1 = counts[1] > 0, have2 = counts[2] > 0;
    double *lmin = NULL, *rmin = NULL;
    if (have1 && have2 && counts[3] > 0) {
        uint8_t* m1 = (uint8_t*)malloc(n);
        uint8_t* m2 = (uint8_t*)malloc(n);
        for (size_t k = 0; k < n; ++k) {
            m1[k] = label[k] == 1;
            m2[k] = label[k] == 2;
        }
        lmin = (double*)malloc(n * sizeof(double));
        rmin = (double*)malloc(n * sizeof(double));
        fso_distance_transform(m1, w, h, lmin);
        fso_distance_transform(m2, w, h, rmin);
        free(m1);
        free(m2);
    }
    for (size_t k = 0; k < n; ++k) {
        switch (label[k]) {
            case 1: b[k] = 0.0; break;
            case 2: b[k] = 1.0; break;
            case 3:
                if (!have1 || !have2) {
                    b[k] = 0.5;
                } else {
                    double l = lmin[k], r = rmin[k];
                    b[k] = (l + r > 0.0) ? l / (l + r) : 0.5;
                }
                break;
            default: b[k] = 0.5; break;
        }
    }
    free(lmin);
    free(rmin);
    return FSO_OK;
}

/* proj/src/blender.cpp:18-30 */
void fso_softmax_weights(double blend_l, double blend_r, double mag_rtol, double mag_ltor,
                         double k, double coef, double* out2) {
    double flow_l = 1.0 + coef * mag_rtol;
    double flow_r = 1.0 + coef * mag_ltor;
    double arg_l = k * blend_l * flow_l;
    double arg_r = k * blend_r * flow_r;
    double m = arg_l < arg_r ? arg_r : arg_l; /* std::max */
    double el = exp(arg_l - m);
    double er = exp(arg_r - m);
    out2[0] = el / (el + er);
    out2[1] = er / (el + er);
}

/* proj/src/blender.cpp:11-16 */
static int blend_params_ok(double k, double coef) {
    return k > 0.0 && isfinite(k) && !(coef < 0.0) && isfinite(coef);
}

/* proj/src/blender.cpp:43-100 — Code 1. Flows are canvas-sized. */
int fso_blend_pair(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr, int w,
                   int h, int ch, const float* flow_lr, const float* flow_rl, const double* b,
                   const uint8_t* label, double k, double coef, float* out, uint8_t* out_valid) {
    if (!blend_params_ok(k, coef)) return FSO_CONTRACT;
    size_t n = (size_t)w * h;
    for (size_t q = 0; q < 2 * n; ++q)
        if (!isfinite(flow_lr[q]) || !isfinite(flow_rl[q])) return FSO_CONTRACT;
    float color_l[3], color_r[3];
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            size_t idx = (size_t)j * w + i;
            out_valid[idx] = 1;
            switch (label[idx]) {
                case 1:
                    for (int c = 0; c < ch; ++c) out[idx * ch + c] = l[idx * ch + c];
                    break;
                case 2:
                    for (int c = 0; c < ch; ++c) out[idx * ch + c] = r[idx * ch + c];
                    break;
                case 3: {
                    double blend_r = b[idx];
                    double blend_l = 1.0 - blend_r;
                    float rl_x = flow_rl[idx * 2], rl_y = flow_rl[idx * 2 + 1];
                    float lr_x = flow_lr[idx * 2], lr_y = flow_lr[idx * 2 + 1];
                    fso_bilinear_sample(l, vl, w, h, ch, i + rl_x * (1.0 - blend_l),
                                        j + rl_y * (1.0 - blend_l), color_l);
                    fso_bilinear_sample(r, vr, w, h, ch, i + lr_x * (1.0 - blend_r),
                                        j + lr_y * (1.0 - blend_r), color_r);
                    double mag_rl = sqrt((double)rl_x * rl_x + (double)rl_y * rl_y);
                    double mag_lr = sqrt((double)lr_x * lr_x + (double)lr_y * lr_y);
                    double s[2];
                    fso_softmax_weights(blend_l, blend_r, mag_rl, mag_lr, k, coef, s);
                    for (int c = 0; c < ch; ++c) {
                        double v = color_l[c] * s[0] + color_r[c] * s[1];
                        out[idx * ch + c] = (float)clampd(v, 0.0, 1.0);
                    }
                    break;
                }
                default:
                    for (int c = 0; c < ch; ++c) out[idx * ch + c] = 0.0f;
                    out_valid[idx] = 0;
                    break;
            }
        }
    return FSO_OK;
}

/* proj/src/blender.cpp:102-135: Area1 -> L, Area2 -> R, Area3 ->
 * clamp((1 - b) L + b R) in double, Outside -> 0 and invalid. */
int fso_feather_blend(const float* l, const float* r, int w, int h, int ch, const double* b,
                      const uint8_t* label, float* out, uint8_t* out_valid) {
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            size_t idx = (size_t)j * w + i;
            out_valid[idx] = 1;
            for (int c = 0; c < ch; ++c) out[idx * ch + c] = 0.0f;
            switch (label[idx]) {
                case 1:
                    for (int c = 0; c < ch; ++c) out[idx * ch + c] = l[idx * ch + c];
                    break;
                case 2:
                    for (int c = 0; c < ch; ++c) out[idx * ch + c] = r[idx * ch + c];
                    break;
                case 3:
                    for (int c = 0; c < ch; ++c) {
                        double v = (1.0 - b[idx]) * l[idx * ch + c] + b[idx] * r[idx * ch + c];
                        out[idx * ch + c] = (float)clampd(v, 0.0, 1.0);
                    }
                    break;
                default:
                    out_valid[idx] = 0;
                    break;
            }
        }
    return FSO_OK;
}

/* proj/src/blender.cpp:137-163: copies of L and R whose Area3 pixels are
 * replaced by the samples Code 1 blends — L at p + FlowRtoL (1 - BlendL),
 * R at p + FlowLtoR (1 - BlendR) — marked valid. */
int fso_warp_constituents(const float* l, const uint8_t* vl, const float* r, const uint8_t* vr,
                          int w, int h, int ch, const float* flow_lr, const float* flow_rl,
                          const double* b, const uint8_t* label, float* out_l, uint8_t* out_vl,
                          float* out_r, uint8_t* out_vr) {
    size_t n = (size_t)w * h;
    memcpy(out_l, l, n * ch * sizeof(float));
    memcpy(out_r, r, n * ch * sizeof(float));
    memcpy(out_vl, vl, n);
    memcpy(out_vr, vr, n);
    float color[3];
    for (int j = 0; j < h; ++j)
        for (int i = 0; i < w; ++i) {
            size_t idx = (size_t)j * w + i;
            if (label[idx] != 3) continue;
            double blend_r = b[idx];
            double blend_l = 1.0 - blend_r;
            fso_bilinear_sample(l, vl, w, h, ch, i + flow_rl[2 * idx] * (1.0 - blend_l),
                                j + flow_rl[2 * idx + 1] * (1.0 - blend_l), color);
            for (int c = 0; c < ch; ++c) out_l[idx * ch + c] = color[c];
            out_vl[idx] = 1;
            fso_bilinear_sample(r, vr, w, h, ch, i + flow_lr[2 * idx] * (1.0 - blend_r),
                                j + flow_lr[2 * idx + 1] * (1.0 - blend_r), color);
            for (int c = 0; c < ch; ++c) out_r[idx * ch + c] = color[c];
            out_vr[idx] = 1;
        }
    return FSO_OK;
}

/* proj/src/pipeline.cpp:140-212 without the misalignment metrics
 * (:184-187, :194-199), which read the panorama but never write it. */
int fso_stitch_placed(int n, const float* const* imgs, const uint8_t* const* valids,
                      const int* dims, const int* offsets, int ch, int cw, int chh, int levels,
                      int radius, int iters, double eps, int smoothing, double k, double coef,
                      float* out, uint8_t* out_valid) {
    if (n < 2) return FSO_CONTRACT;
    if (!flow_params_ok(levels, radius, iters, eps, smoothing) || !blend_params_ok(k, coef))
        return FSO_CONTRACT;
    size_t np = (size_t)cw * chh;
    float* next = (float*)malloc(np * ch * sizeof(float));
    uint8_t* next_v = (uint8_t*)malloc(np);
    uint8_t* label = (uint8_t*)malloc(np);
    float* blended = (float*)malloc(np * ch * sizeof(float));
    uint8_t* blended_v = (uint8_t*)malloc(np);
    double* b = (double*)malloc(np * sizeof(double));
    float* cflr = (float*)malloc(np * 2 * sizeof(float));
    float* cfrl = (float*)malloc(np * 2 * sizeof(float));
    uint8_t* cvalid = (uint8_t*)malloc(np);
    int st = fso_place_on_canvas(imgs[0], valids ? valids[0] : NULL, dims[0], dims[1], ch,
                                 offsets[0], offsets[1], cw, chh, out, out_valid);
    for (int kk = 1; kk < n && st == FSO_OK; ++kk) {
        st = fso_place_on_canvas(imgs[kk], valids ? valids[kk] : NULL, dims[2 * kk],
                                 dims[2 * kk + 1], ch, offsets[2 * kk], offsets[2 * kk + 1], cw,
                                 chh, next, next_v);
        if (st != FSO_OK) break;
        int64_t counts[4];
        fso_compute_partition(out_valid, next_v, cw, chh, label, counts);
        if (counts[3] == 0) {
            st = FSO_EMPTY;
            break;
        }
        int box[4];
        fso_crop_box(label, counts, cw, chh, box);
        size_t nc = (size_t)box[2] * box[3];
        float* crop_l = (float*)malloc(nc * ch * sizeof(float));
        float* crop_r = (float*)malloc(nc * ch * sizeof(float));
        uint8_t* cv = (uint8_t*)malloc(nc);
        float* flr = (float*)malloc(nc * 2 * sizeof(float));
        float* frl = (float*)malloc(nc * 2 * sizeof(float));
        uint8_t* vlr = (uint8_t*)malloc(nc);
        uint8_t* vrl = (uint8_t*)malloc(nc);
        fso_crop_overlap(out, out_valid, cw, chh, ch, label, counts, crop_l, cv, box);
        fso_crop_overlap(next, next_v, cw, chh, ch, label, counts, crop_r, cv, box);
        st = fso_bidirectional_flow(crop_l, crop_r, box[2], box[3], ch, levels, radius, iters,
                                    eps, smoothing, flr, vlr, frl, vrl);
        if (st == FSO_OK) {
            fso_embed_flow(flr, vlr, box[2], box[3], box[0], box[1], cw, chh, cflr, cvalid);
            fso_embed_flow(frl, vrl, box[2], box[3], box[0], box[1], cw, chh, cfrl, cvalid);
            fso_compute_blend(label, counts, cw, chh, b);
            st = fso_blend_pair(out, out_valid, next, next_v, cw, chh, ch, cflr, cfrl, b, label, k,
                                coef, blended, blended_v);
        }
        if (st == FSO_OK) {
            for (size_t q = 0; q < np; ++q) blended_v[q] = (out_valid[q] || next_v[q]) ? 1 : 0;
            memcpy(out, blended, np * ch * sizeof(float));
            memcpy(out_valid, blended_v, np);
        }
        free(crop_l); free(crop_r); free(cv); free(flr); free(frl); free(vlr); free(vrl);
    }
    free(next); free(next_v); free(label); free(blended); free(blended_v); free(b);
    free(cflr); free(cfrl); free(cvalid);
    return st;
}

/* ---- misalignment_score (proj/src/pipeline.cpp:213-396) ---------------- */

typedef struct {
    double mean, var;
} patch_stats_t;

/* proj/src/pipeline.cpp:220-233 */
static patch_stats_t patch_stats(const float* g, int w, int cx, int cy, int r) {
    double sum = 0.0, sum2 = 0.0;
    int n = (2 * r + 1) * (2 * r + 1);
    for (int j = cy - r; j <= cy + r; ++j)
        for (int i = cx - r; i <= cx + r; ++i) {
            double v = g[(size_t)j * w + i];
            sum += v;
            sum2 += v * v;
        }
    patch_stats_t s;
    s.mean = sum / n;
    s.var = sum2 / n - s.mean * s.mean;
    return s;
}

/* proj/src/pipeline.cpp:235-245 */
static double patch_ncc(const float* a, int ax, int ay, const float* b, int bx, int by, int w,
                        int r, patch_stats_t sa, patch_stats_t sb) {
    if (sa.var <= 1e-12 || sb.var <= 1e-12) return -2.0;
    double cov = 0.0;
    int n = (2 * r + 1) * (2 * r + 1);
    for (int dj = -r; dj <= r; ++dj)
        for (int di = -r; di <= r; ++di)
            cov += ((double)a[(size_t)(ay + dj) * w + ax + di] - sa.mean) *
                   ((double)b[(size_t)(by + dj) * w + bx + di] - sb.mean);
    cov /= n;
    return cov / sqrt(sa.var * sb.var);
}

/* proj/src/pipeline.cpp:247-256 — fixed tie-break */
static int better_candidate(double score, int dx, int dy, double best_score, int best_dx,
                            int best_dy) {
    if (score > best_score + 1e-12) return 1;
    if (score < best_score - 1e-12) return 0;
    long n2 = (long)dx * dx + (long)dy * dy;
    long b2 = (long)best_dx * best_dx + (long)best_dy * best_dy;
    if (n2 != b2) return n2 < b2;
    if (dx != best_dx) return dx < best_dx;
    return dy < best_dy;
}

/* proj/src/pipeline.cpp:309-396.  The footprint tests use the reference's
 * prefix-count semantics (every pixel of the patch in Area3 / valid in R),
 * evaluated directly. */
int fso_misalignment_score(const float* l, const uint8_t* l_valid, const float* r,
                           const uint8_t* r_valid, int w, int h, int ch, const uint8_t* label,
                           const int64_t* counts, int patch_radius, int stride, double* out) {
    (void)l_valid;
    if (counts[3] == 0) return FSO_CONTRACT;
    if (patch_radius < 1 || stride < 1) return FSO_CONTRACT;
    size_t n = (size_t)w * h;
    float* gl = (float*)malloc(n * sizeof(float));
    float* gr = (float*)malloc(n * sizeof(float));
    fso_to_gray(l, w, h, ch, gl);
    fso_to_gray(r, w, h, ch, gr);
    const int rr = patch_radius, search = 2 * patch_radius;
    double total = 0.0;
    long matched = 0;
    for (int cy = rr; cy < h - rr; cy += stride) {
        double row_total = 0.0;
        long row_matched = 0;
        for (int cx = rr; cx < w - rr; cx += stride) {
            int full = 1;
            for (int j = cy - rr; j <= cy + rr && full; ++j)
                for (int i = cx - rr; i <= cx + rr; ++i)
                    if (label[(size_t)j * w + i] != 3) {
                        full = 0;
                        break;
                    }
            if (!full) continue;
            patch_stats_t sl = patch_stats(gl, w, cx, cy, rr);
            if (sl.var < 1e-4) continue;
            double best_score = -2.0;
            int best_dx = 0, best_dy = 0, found = 0;
            for (int dy = -search; dy <= search; ++dy)
                for (int dx = -search; dx <= search; ++dx) {
                    int bx = cx + dx, by = cy + dy;
                    if (bx - rr < 0 || bx + rr >= w || by - rr < 0 || by + rr >= h) continue;
                    int rv = 1;
                    for (int j = by - rr; j <= by + rr && rv; ++j)
                        for (int i = bx - rr; i <= bx + rr; ++i)
                            if (!r_valid[(size_t)j * w + i]) {
                                rv = 0;
                                break;
                            }
                    if (!rv) continue;
                    patch_stats_t sr = patch_stats(gr, w, bx, by, rr);
                    double ncc = patch_ncc(gl, cx, cy, gr, bx, by, w, rr, sl, sr);
                    if (ncc < -1.5) continue;
                    found = 1;
                    if (better_candidate(ncc, dx, dy, best_score, best_dx, best_dy)) {
                        best_score = ncc;
                        best_dx = dx;
                        best_dy = dy;
                    }
                }
            if (!found) continue;
            row_total += sqrt((double)best_dx * best_dx + (double)best_dy * best_dy);
            ++row_matched;
        }
        total += row_total;
        matched += row_matched;
    }
    free(gl);
    free(gr);
    if (matched == 0) return FSO_EMPTY;
    *out = total / (double)matched;
    return FSO_OK;
}

/* proj/src/pipeline.cpp:261-307 */
int fso_estimate_translation(const float* a, const float* b, int w, int h, int ch, int max_shift,
                             int* out_dx, int* out_dy, double* out_score) {
    if (ch != 1) return FSO_CONTRACT;
    if (max_shift > imin(w, h) / 4) return FSO_CONTRACT;
    double best_score = -2.0;
    int best_dx = 0, best_dy = 0, any = 0;
    for (int dy = -max_shift; dy <= max_shift; ++dy)
        for (int dx = -max_shift; dx <= max_shift; ++dx) {
            int x0 = imax(0, -dx), x1 = imin(w, w - dx);
            int y0 = imax(0, -dy), y1 = imin(h, h - dy);
            if (x1 <= x0 || y1 <= y0) continue;
            long n = (long)(x1 - x0) * (y1 - y0);
            double sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
            for (int y = y0; y < y1; ++y)
                for (int x = x0; x < x1; ++x) {
                    double va = a[(size_t)y * w + x];
                    double vb = b[(size_t)(y + dy) * w + x + dx];
                    sa += va;
                    sb += vb;
                    saa += va * va;
                    sbb += vb * vb;
                    sab += va * vb;
                }
            double va = saa / n - (sa / n) * (sa / n);
            double vb = sbb / n - (sb / n) * (sb / n);
            if (va <= 1e-12 || vb <= 1e-12) continue;
            double ncc = (sab / n - (sa / n) * (sb / n)) / sqrt(va * vb);
            any = 1;
            if (better_candidate(ncc, dx, dy, best_score, best_dx, best_dy)) {
                best_dx = dx;
                best_dy = dy;
                best_score = ncc;
            }
        }
    if (!any) return FSO_EMPTY;
    *out_dx = best_dx;
    *out_dy = best_dy;
    *out_score = best_score;
    return FSO_OK;
}
