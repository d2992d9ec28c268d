/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (see cmax_oracle.h).
 *
 * Plain-C fp64 restatement of the reference CMax loss path. Every function
 * names the reference lines it follows; expression order is kept identical so
 * that, compiled without FMA contraction (-ffp-contract=off), the forward
 * products are bit-identical to evcm::Engine and the gradients bit-identical
 * to the naive backend (engine.hpp:506-524).
 */
#include "cmax_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define LOSS_EPS 1e-9 /* kLossEps, warp.hpp:26 */

/* ---- edges / clocks -------------------------------------------------------- */

/* FlowSequence::zeros edge rule: e_i = t0 + llround(span*i/B), e_B = t1
 * (types.hpp:293-300). */
void orc_make_edges(uint64_t t0, uint64_t t1, int B, uint64_t* e) {
  const double span = (double)(t1 - t0);
  for (int i = 0; i <= B; ++i)
    e[i] = (i == B) ? t1 : t0 + (uint64_t)llround(span * i / B);
}

/* FlowSequence::rel_s (types.hpp:263-266). */
static double rel_s(uint64_t t_us, uint64_t t0) { return ((double)t_us - (double)t0) * 1e-6; }

/* Engine::edge_seconds (engine.hpp:244-249). */
static void edge_seconds(const uint64_t* e, int B, double* s) {
  for (int i = 0; i <= B; ++i) s[i] = rel_s(e[i], e[0]);
}

/* ---- validation ------------------------------------------------------------ */

int orc_validate_window(int W, int H, int B, const uint64_t* e, uint64_t ts, uint64_t te,
                        const orc_event* ev, size_t n, size_t* bad) {
  /* EventSlice::validate (types.hpp:135-159) */
  if (W <= 0 || H <= 0) return ORC_DIMENSION;
  if (te < ts) return ORC_TIME_RANGE;
  for (size_t k = 0; k < n; ++k) {
    if (bad) *bad = k;
    if (ev[k].x >= W || ev[k].y >= H) return ORC_COORDINATE;
    if (ev[k].p != 1 && ev[k].p != -1) return ORC_POLARITY;
    if (k > 0 && ev[k].t_us < ev[k - 1].t_us) return ORC_UNSORTED;
    if (ev[k].t_us < ts || ev[k].t_us >= te) return ORC_TIME_RANGE;
  }
  /* FlowSequence::validate (types.hpp:268-273): B >= 1, strictly increasing. */
  if (B < 1) return ORC_CONFIG;
  for (int i = 0; i < B; ++i)
    if (e[i] >= e[i + 1]) return ORC_CONFIG;
  /* Engine::validate_window (engine.hpp:220-221) */
  if (e[0] != ts || e[B] != te) return ORC_CONFIG;
  return ORC_OK;
}

/* ---- bilinear primitives --------------------------------------------------- */

typedef struct {
  int x0, y0, x1, y1;
  double wx, wy;
} cell_t;

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* bilin_cell (warp.hpp:42-53). */
static cell_t bilin_cell(double x, double y, int W, int H) {
  cell_t c;
  const double cx = clampd(x, 0.0, (double)(W - 1));
  const double cy = clampd(y, 0.0, (double)(H - 1));
  if (W >= 2) {
    int fx = (int)floor(cx);
    c.x0 = fx < W - 2 ? fx : W - 2;
  } else {
    c.x0 = 0;
  }
  if (H >= 2) {
    int fy = (int)floor(cy);
    c.y0 = fy < H - 2 ? fy : H - 2;
  } else {
    c.y0 = 0;
  }
  c.x1 = c.x0 + 1 < W - 1 ? c.x0 + 1 : W - 1;
  c.y1 = c.y0 + 1 < H - 1 ? c.y0 + 1 : H - 1;
  c.wx = cx - c.x0;
  c.wy = cy - c.y0;
  return c;
}
/* BilinCell::w00..w11 (warp.hpp:36-39). */
static double w00(const cell_t* c) { return (1.0 - c->wx) * (1.0 - c->wy); }
static double w10(const cell_t* c) { return c->wx * (1.0 - c->wy); }
static double w01(const cell_t* c) { return (1.0 - c->wx) * c->wy; }
static double w11(const cell_t* c) { return c->wx * c->wy; }

/* in_bounds (warp.hpp:55-57). */
static int in_bounds(double x, double y, int W, int H) {
  return x >= 0.0 && x <= W - 1 && y >= 0.0 && y <= H - 1;
}

static size_t idx(int x, int y, int W) { return (size_t)y * (size_t)W + (size_t)x; }

/* sample_flow (warp.hpp:61-68). u = flows[b][0], v = flows[b][1]. */
static void sample_flow(const double* fu, const double* fv, int W, int H, double px, double py,
                        double* u, double* v) {
  const cell_t c = bilin_cell(px, py, W, H);
  *u = w00(&c) * fu[idx(c.x0, c.y0, W)] + w10(&c) * fu[idx(c.x1, c.y0, W)] +
       w01(&c) * fu[idx(c.x0, c.y1, W)] + w11(&c) * fu[idx(c.x1, c.y1, W)];
  *v = w00(&c) * fv[idx(c.x0, c.y0, W)] + w10(&c) * fv[idx(c.x1, c.y0, W)] +
       w01(&c) * fv[idx(c.x0, c.y1, W)] + w11(&c) * fv[idx(c.x1, c.y1, W)];
}

/* sample_flow_jacobian (warp.hpp:76-88): {dux, duy, dvx, dvy}. */
static void sample_flow_jacobian(const double* fu, const double* fv, int W, int H, double px,
                                 double py, double j[4]) {
  const cell_t c = bilin_cell(px, py, W, H);
  j[0] = (1.0 - c.wy) * (fu[idx(c.x1, c.y0, W)] - fu[idx(c.x0, c.y0, W)]) +
         c.wy * (fu[idx(c.x1, c.y1, W)] - fu[idx(c.x0, c.y1, W)]);
  j[1] = (1.0 - c.wx) * (fu[idx(c.x0, c.y1, W)] - fu[idx(c.x0, c.y0, W)]) +
         c.wx * (fu[idx(c.x1, c.y1, W)] - fu[idx(c.x1, c.y0, W)]);
  j[2] = (1.0 - c.wy) * (fv[idx(c.x1, c.y0, W)] - fv[idx(c.x0, c.y0, W)]) +
         c.wy * (fv[idx(c.x1, c.y1, W)] - fv[idx(c.x0, c.y1, W)]);
  j[3] = (1.0 - c.wx) * (fv[idx(c.x0, c.y1, W)] - fv[idx(c.x0, c.y0, W)]) +
         c.wx * (fv[idx(c.x1, c.y1, W)] - fv[idx(c.x1, c.y0, W)]);
}

/* apply_step_transpose: (I + dt J)^T g (warp.hpp:91-94). */
static void step_transpose(const double j[4], double dt, double* gx, double* gy) {
  const double ox = *gx * (1.0 + dt * j[0]) + *gy * dt * j[2];
  const double oy = *gy * (1.0 + dt * j[3]) + *gx * dt * j[1];
  *gx = ox;
  *gy = oy;
}

/* bin_of (warp.hpp:284-288): largest j with edges_s[j] <= t, clamped. */
static int bin_of(double t, const double* es, int B) {
  int j = 0; /* upper_bound - 1 */
  int lo = 0, hi = B + 1;
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    if (t < es[mid]) hi = mid; else lo = mid + 1;
  }
  j = lo - 1;
  if (j < 0) j = 0;
  if (j > B - 1) j = B - 1;
  return j;
}

#define FU(b) (flows + (size_t)(b) * 2 * HW)
#define FV(b) (flows + ((size_t)(b) * 2 + 1) * HW)

/* build_trajectory (warp.hpp:257-281). pos has 2*(B+1) doubles. */
static int build_trajectory(double x0, double y0, double t, int j, const double* flows,
                            const double* es, int B, int W, int H, double* pos) {
  const size_t HW = (size_t)W * H;
  double u, v, px, py;
  /* backward leg */
  sample_flow(FU(j), FV(j), W, H, x0, y0, &u, &v);
  px = x0 + (es[j] - t) * u;
  py = y0 + (es[j] - t) * v;
  pos[2 * j] = px;
  pos[2 * j + 1] = py;
  for (int i = j; i >= 1; --i) {
    sample_flow(FU(i - 1), FV(i - 1), W, H, px, py, &u, &v);
    const double dt = es[i - 1] - es[i];
    px = px + dt * u;
    py = py + dt * v;
    pos[2 * (i - 1)] = px;
    pos[2 * (i - 1) + 1] = py;
  }
  /* forward leg */
  sample_flow(FU(j), FV(j), W, H, x0, y0, &u, &v);
  px = x0 + (es[j + 1] - t) * u;
  py = y0 + (es[j + 1] - t) * v;
  pos[2 * (j + 1)] = px;
  pos[2 * (j + 1) + 1] = py;
  for (int i = j + 1; i <= B - 1; ++i) {
    sample_flow(FU(i), FV(i), W, H, px, py, &u, &v);
    const double dt = es[i + 1] - es[i];
    px = px + dt * u;
    py = py + dt * v;
    pos[2 * (i + 1)] = px;
    pos[2 * (i + 1) + 1] = py;
  }
  int ok = 1;
  for (int r = 0; r <= B; ++r) ok = ok && in_bounds(pos[2 * r], pos[2 * r + 1], W, H);
  return ok;
}

/* splat_bilinear (warp.hpp:147-160) with weight 1 (engine.hpp:365-374). */
static void splat_bilinear(double px, double py, double weight, double value, double* cnt,
                           double* val, int W, int H) {
  const cell_t c = bilin_cell(px, py, W, H);
  const double a = weight * w00(&c), b = weight * w10(&c);
  const double d = weight * w01(&c), e = weight * w11(&c);
  cnt[idx(c.x0, c.y0, W)] += a;
  cnt[idx(c.x1, c.y0, W)] += b;
  cnt[idx(c.x0, c.y1, W)] += d;
  cnt[idx(c.x1, c.y1, W)] += e;
  val[idx(c.x0, c.y0, W)] += a * value;
  val[idx(c.x1, c.y0, W)] += b * value;
  val[idx(c.x0, c.y1, W)] += d * value;
  val[idx(c.x1, c.y1, W)] += e * value;
}

/* ---- forward ------------------------------------------------------------- */

int orc_forward(int W, int H, int B, const uint64_t* e, const orc_event* ev, size_t n,
                const double* flows, double* count, double* tsum, int64_t* n_active,
                uint8_t* alive, int32_t* bin, double* pos_out, double* loss, int* no_surv) {
  const int R = B + 1;
  const size_t HW = (size_t)W * H;
  int rc = orc_validate_window(W, H, B, e, e[0], e[B], ev, n, NULL);
  if (rc) return rc;
  double* es = malloc(sizeof(double) * (size_t)R);
  edge_seconds(e, B, es);
  const double window_s = es[B]; /* engine.hpp:380 */
  double* cnt = calloc((size_t)R * 2 * HW, sizeof(double));
  double* val = calloc((size_t)R * 2 * HW, sizeof(double));
  double* pos = malloc(sizeof(double) * 2 * (size_t)R);
  const double t0 = (double)e[0];
  /* warp phase + splat phase fused per event: per-pixel accumulation order
   * is still event order, which is what every reference backend produces
   * (engine.hpp:14-16, 420-422). */
  for (size_t k = 0; k < n; ++k) {
    const double t_rel = ((double)ev[k].t_us - t0) * 1e-6; /* engine.hpp:270 */
    const int j = bin_of(t_rel, es, B);
    const int ok = build_trajectory((double)ev[k].x, (double)ev[k].y, t_rel, j, flows, es, B, W,
                                    H, pos);
    if (alive) alive[k] = ok ? 1 : 0;
    if (bin) bin[k] = j;
    if (pos_out) memcpy(pos_out + k * 2 * (size_t)R, pos, sizeof(double) * 2 * (size_t)R);
    if (!ok) continue;
    const int c = ev[k].p > 0 ? 0 : 1; /* polarity_index, types.hpp:118 */
    for (int r = 0; r < R; ++r) {
      const double tb = fabs(t_rel - es[r]) / window_s; /* engine.hpp:370 */
      splat_bilinear(pos[2 * r], pos[2 * r + 1], 1.0, tb, cnt + ((size_t)r * 2 + c) * HW,
                     val + ((size_t)r * 2 + c) * HW, W, H);
    }
  }
  /* refresh_active (warp.hpp:186-192) */
  int64_t total = 0;
  int64_t* na = malloc(sizeof(int64_t) * (size_t)R);
  for (int r = 0; r < R; ++r) {
    const double* c0 = cnt + (size_t)r * 2 * HW;
    const double* c1 = c0 + HW;
    int64_t a = 0;
    for (size_t i = 0; i < HW; ++i) a += (c0[i] + c1[i] > 0.0) ? 1 : 0;
    na[r] = a;
    total += a;
  }
  /* reduce_loss (engine.hpp:442-468) + reference_loss (warp.hpp:299-312) */
  double value = 0.0;
  int ns = 0;
  if (total == 0) {
    ns = 1;
  } else {
    double sum = 0.0;
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
      for (int c = 0; c < 2; ++c) {
        const double* S = val + ((size_t)r * 2 + c) * HW;
        const double* C = cnt + ((size_t)r * 2 + c) * HW;
        for (size_t i = 0; i < HW; ++i) {
          const double a = S[i] / (C[i] + LOSS_EPS);
          acc += a * a;
        }
      }
      sum += acc / ((double)na[r] + LOSS_EPS);
    }
    value = sum / (double)R;
  }
  if (loss) *loss = value;
  if (no_surv) *no_surv = ns;
  if (n_active) memcpy(n_active, na, sizeof(int64_t) * (size_t)R);
  if (count) memcpy(count, cnt, sizeof(double) * (size_t)R * 2 * HW);
  if (tsum) memcpy(tsum, val, sizeof(double) * (size_t)R * 2 * HW);
  free(na);
  free(pos);
  free(cnt);
  free(val);
  free(es);
  return ORC_OK;
}

/* ---- backward ------------------------------------------------------------ */

/* splat_position_grad (warp.hpp:334-358), lane_weight 1. */
static void splat_position_grad(const double* S, const double* C, int64_t n_act, int R, int W,
                                int H, double px, double py, double tbar, double* dx,
                                double* dy) {
  const double scale = 2.0 / (((double)n_act + LOSS_EPS) * (double)R);
  const cell_t c = bilin_cell(px, py, W, H);
#define CORNER(X, Y)                                          \
  ({                                                          \
    const double inv_ = 1.0 / (C[idx(X, Y, W)] + LOSS_EPS);   \
    const double a_ = S[idx(X, Y, W)] * inv_;                 \
    scale * a_ * inv_ * (tbar - a_) * 1.0;                    \
  })
  const double g00 = CORNER(c.x0, c.y0), g10 = CORNER(c.x1, c.y0);
  const double g01 = CORNER(c.x0, c.y1), g11 = CORNER(c.x1, c.y1);
#undef CORNER
  *dx = -(1.0 - c.wy) * g00 + (1.0 - c.wy) * g10 - c.wy * g01 + c.wy * g11;
  *dy = -(1.0 - c.wx) * g00 - c.wx * g10 + (1.0 - c.wx) * g01 + c.wx * g11;
}

/* BufferGradSink::add (warp.hpp:394-406). */
static void sink_add(double* grad, int b, size_t HW, int W, int H, double ax, double ay,
                     double gx, double gy) {
  double* gu = grad + (size_t)b * 2 * HW;
  double* gv = gu + HW;
  const cell_t c = bilin_cell(ax, ay, W, H);
  gu[idx(c.x0, c.y0, W)] += w00(&c) * gx;
  gu[idx(c.x1, c.y0, W)] += w10(&c) * gx;
  gu[idx(c.x0, c.y1, W)] += w01(&c) * gx;
  gu[idx(c.x1, c.y1, W)] += w11(&c) * gx;
  gv[idx(c.x0, c.y0, W)] += w00(&c) * gy;
  gv[idx(c.x1, c.y0, W)] += w10(&c) * gy;
  gv[idx(c.x0, c.y1, W)] += w01(&c) * gy;
  gv[idx(c.x1, c.y1, W)] += w11(&c) * gy;
}

int orc_backward(int W, int H, int B, const uint64_t* e, const orc_event* ev, size_t n,
                 const double* flows, const double* count, const double* tsum,
                 const int64_t* n_active, const uint8_t* alive, const int32_t* bin,
                 int no_surv, double* grad) {
  const int R = B + 1;
  const size_t HW = (size_t)W * H;
  int rc = orc_validate_window(W, H, B, e, e[0], e[B], ev, n, NULL);
  if (rc) return rc;
  memset(grad, 0, sizeof(double) * (size_t)B * 2 * HW); /* engine.hpp:195 */
  if (no_surv) return ORC_OK;                             /* engine.hpp:196 */
  double* es = malloc(sizeof(double) * (size_t)R);
  edge_seconds(e, B, es);
  const double window_s = es[B];
  const double t0 = (double)e[0];
  double* pos = malloc(sizeof(double) * 2 * (size_t)R);
  double* d = malloc(sizeof(double) * 2 * (size_t)R);
  for (size_t k = 0; k < n; ++k) {
    if (!alive[k]) continue;
    const double t_rel = ((double)ev[k].t_us - t0) * 1e-6;
    const int j = bin[k];
    const double x0 = (double)ev[k].x, y0 = (double)ev[k].y;
    /* The reference reads the stored trajectory row; recomputing it with the
     * same arithmetic yields the same bits (warp.hpp:257-281). */
    build_trajectory(x0, y0, t_rel, j, flows, es, B, W, H, pos);
    const int c = ev[k].p > 0 ? 0 : 1;
    /* backward_event (engine.hpp:475-504) */
    for (int r = 0; r <= B; ++r) {
      const double tb = fabs(t_rel - es[r]) / window_s;
      const double* S = tsum + ((size_t)r * 2 + c) * HW;
      const double* C = count + ((size_t)r * 2 + c) * HW;
      splat_position_grad(S, C, n_active[r], R, W, H, pos[2 * r], pos[2 * r + 1], tb, &d[2 * r],
                          &d[2 * r + 1]);
    }
    double gx = d[0], gy = d[1];
    for (int i = 0; i <= j - 1; ++i) {
      const double dt = es[i] - es[i + 1];
      sink_add(grad, i, HW, W, H, pos[2 * (i + 1)], pos[2 * (i + 1) + 1], dt * gx, dt * gy);
      double jac[4];
      sample_flow_jacobian(FU(i), FV(i), W, H, pos[2 * (i + 1)], pos[2 * (i + 1) + 1], jac);
      step_transpose(jac, dt, &gx, &gy);
      gx = gx + d[2 * (i + 1)];
      gy = gy + d[2 * (i + 1) + 1];
    }
    sink_add(grad, j, HW, W, H, x0, y0, (es[j] - t_rel) * gx, (es[j] - t_rel) * gy);
    gx = d[2 * B];
    gy = d[2 * B + 1];
    for (int i = B - 1; i >= j + 1; --i) {
      const double dt = es[i + 1] - es[i];
      sink_add(grad, i, HW, W, H, pos[2 * i], pos[2 * i + 1], dt * gx, dt * gy);
      double jac[4];
      sample_flow_jacobian(FU(i), FV(i), W, H, pos[2 * i], pos[2 * i + 1], jac);
      step_transpose(jac, dt, &gx, &gy);
      gx = gx + d[2 * i];
      gy = gy + d[2 * i + 1];
    }
    sink_add(grad, j, HW, W, H, x0, y0, (es[j + 1] - t_rel) * gx, (es[j + 1] - t_rel) * gy);
  }
  free(d);
  free(pos);
  free(es);
  return ORC_OK;
}

/* ---- geometry ------------------------------------------------------------ */

static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* Mat3 product (geometry.hpp:70-76): r(i,j) = a(i,0)b(0,j) + a(i,1)b(1,j) + a(i,2)b(2,j). */
static void mat3_mul(const double* a, const double* b, double* r) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      t[3 * i + j] = a[3 * i + 0] * b[0 + j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
  memcpy(r, t, sizeof t);
}
/* Mat3 * Vec3 (geometry.hpp:77-81). */
static void mat3_vec(const double* m, const double* v, double* r) {
  const double x = m[0] * v[0] + m[1] * v[1] + m[2] * v[2];
  const double y = m[3] * v[0] + m[4] * v[1] + m[5] * v[2];
  const double z = m[6] * v[0] + m[7] * v[1] + m[8] * v[2];
  r[0] = x;
  r[1] = y;
  r[2] = z;
}
/* skew (geometry.hpp:84-86). */
static void skew(const double* v, double* s) {
  const double t[9] = {0, -v[2], v[1], v[2], 0, -v[0], -v[1], v[0], 0};
  memcpy(s, t, sizeof t);
}

/* rodrigues (geometry.hpp:94-107): I + a*W + b*(W*W). */
void orc_rodrigues(const double* w, double* R) {
  const double t2 = dot3(w, w);
  const double t = sqrt(t2);
  double a, b;
  if (t < 1e-8) {
    a = 1.0 - t2 / 6.0;
    b = 0.5 - t2 / 24.0;
  } else {
    a = sin(t) / t;
    b = (1.0 - cos(t)) / t2;
  }
  double S[9], S2[9];
  skew(w, S);
  mat3_mul(S, S, S2);
  static const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  /* Mat3::identity() + a*w + b*(w*w): ((I + a*S) + b*S2) elementwise. */
  for (int i = 0; i < 9; ++i) R[i] = (I[i] + a * S[i]) + b * S2[i];
}

/* rodrigues_jacobian (geometry.hpp:114-135). dR[k*9 + i]. */
void orc_rodrigues_jacobian(const double* w, double* dR) {
  const double t2 = dot3(w, w);
  const double t = sqrt(t2);
  double Wm[9];
  skew(w, Wm);
  if (t < 1e-4) {
    for (int k = 0; k < 3; ++k) {
      const double e[3] = {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
      double ek[9], a[9], b[9];
      skew(e, ek);
      mat3_mul(ek, Wm, a);
      mat3_mul(Wm, ek, b);
      /* ek + 0.5 * (ek*w + w*ek) */
      for (int i = 0; i < 9; ++i) dR[9 * k + i] = ek[i] + 0.5 * (a[i] + b[i]);
    }
    return;
  }
  double R[9], IR[9];
  orc_rodrigues(w, R);
  static const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (int i = 0; i < 9; ++i) IR[i] = I[i] - R[i];
  for (int k = 0; k < 3; ++k) {
    const double col[3] = {IR[k], IR[3 + k], IR[6 + k]}; /* Mat3::col (geometry.hpp:38-41) */
    /* cross(omega, col) (geometry.hpp:25-27) */
    const double cr[3] = {w[1] * col[2] - w[2] * col[1], w[2] * col[0] - w[0] * col[2],
                          w[0] * col[1] - w[1] * col[0]};
    double sc[9], m[9], p[9];
    skew(cr, sc);
    for (int i = 0; i < 9; ++i) m[i] = w[k] * Wm[i] + sc[i]; /* wk*w + skew(c) */
    mat3_mul(m, R, p);
    for (int i = 0; i < 9; ++i) dR[9 * k + i] = (1.0 / t2) * p[i];
  }
}

/* PoseStep::validate (types.hpp:362-368). */
static int pose_ok(const double* p) {
  const double pi = 3.14159265358979323846;
  const double nrm = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
  if (!(nrm < pi)) return 0;
  for (int i = 0; i < 6; ++i)
    if (!isfinite(p[i])) return 0;
  return 1;
}

/* depth_pose_to_flows (geometry.hpp:229-264) with reproject (:157-166) and
 * backproject (:147-149). */
int orc_depth_pose_to_flows(int W, int H, const double* depth, const uint8_t* mask, int B,
                            const double* poses, const double* K, uint64_t t0, uint64_t t1,
                            double* flows, uint8_t* valid) {
  if (B < 1) return ORC_CONFIG;
  if (W <= 0 || H <= 0) return ORC_DIMENSION;
  if (t1 <= t0) return ORC_CONFIG; /* FlowSequence::zeros (types.hpp:290-291) */
  const size_t HW = (size_t)W * H;
  uint64_t* e = malloc(sizeof(uint64_t) * (size_t)(B + 1));
  orc_make_edges(t0, t1, B, e);
  const double fx = K[0], fy = K[1], cx = K[2], cy = K[3];
  for (int i = 0; i < B; ++i) {
    if (!pose_ok(poses + 6 * i)) {
      free(e);
      return ORC_CONFIG;
    }
  }
  memset(flows, 0, sizeof(double) * (size_t)B * 2 * HW);
  memset(valid, 0, (size_t)B * HW);
  for (int i = 0; i < B; ++i) {
    double R[9];
    orc_rodrigues(poses + 6 * i, R);
    const double* tr = poses + 6 * i + 3;
    const double dur = ((double)e[i + 1] - (double)e[i]) * 1e-6; /* types.hpp:303-304 */
    const double inv_dt = 1.0 / dur;
    double* fu = flows + (size_t)i * 2 * HW;
    double* fv = fu + HW;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const size_t q = idx(x, y, W);
        if (mask && !mask[q]) continue;
        const double d = depth[q];
        if (!(d > 0.0)) continue;
        const double bp[3] = {d * ((double)x - cx) / fx, d * ((double)y - cy) / fy, d};
        double p[3];
        mat3_vec(R, bp, p);
        p[0] = p[0] + tr[0];
        p[1] = p[1] + tr[1];
        p[2] = p[2] + tr[2];
        if (!(p[2] > 0.0)) continue;
        const double pxx = fx * p[0] / p[2] + cx, pyy = fy * p[1] / p[2] + cy;
        fu[q] = (pxx - (double)x) * inv_dt;
        fv[q] = (pyy - (double)y) * inv_dt;
        valid[(size_t)i * HW + q] = 1;
      }
  }
  free(e);
  return ORC_OK;
}

/* depth_pose_to_flows_backward (geometry.hpp:279-325) with
 * reproject_with_grads (:185-209). d_poses[i*6 + {omega xyz, trans xyz}]. */
int orc_depth_pose_to_flows_backward(int W, int H, const double* depth, const uint8_t* mask,
                                     int B, const double* poses, const double* K,
                                     const uint64_t* e, const double* grad, double* d_depth,
                                     double* d_poses) {
  const size_t HW = (size_t)W * H;
  const double fx = K[0], fy = K[1], cx = K[2], cy = K[3];
  memset(d_depth, 0, sizeof(double) * HW);
  memset(d_poses, 0, sizeof(double) * 6 * (size_t)B);
  for (int i = 0; i < B; ++i) {
    double R[9], dR[27];
    orc_rodrigues(poses + 6 * i, R);
    orc_rodrigues_jacobian(poses + 6 * i, dR);
    const double* tr = poses + 6 * i + 3;
    const double dur = ((double)e[i + 1] - (double)e[i]) * 1e-6;
    const double inv_dt = 1.0 / dur;
    double* dom = d_poses + 6 * i;
    double* dtr = d_poses + 6 * i + 3;
    const double* gu_ = grad + (size_t)i * 2 * HW;
    const double* gv_ = gu_ + HW;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const size_t q = idx(x, y, W);
        const double gu = gu_[q], gv = gv_[q];
        if (gu == 0.0 && gv == 0.0) continue;
        if (mask && !mask[q]) continue;
        const double d = depth[q];
        if (!(d > 0.0)) continue;
        /* reproject_with_grads (geometry.hpp:185-209) */
        const double ray[3] = {1.0 * ((double)x - cx) / fx, 1.0 * ((double)y - cy) / fy, 1.0};
        double rray[3];
        mat3_vec(R, ray, rray);
        const double p[3] = {d * rray[0] + tr[0], d * rray[1] + tr[1], d * rray[2] + tr[2]};
        if (!(p[2] > 0.0)) continue;
        const double iz = 1.0 / p[2];
        const double ju[3] = {fx * iz, 0.0, -fx * p[0] * iz * iz};
        const double jv[3] = {0.0, fy * iz, -fy * p[1] * iz * iz};
        const double dpd_x = dot3(ju, rray), dpd_y = dot3(jv, rray);
        d_depth[q] += (gu * dpd_x + gv * dpd_y) * inv_dt;
        /* d_pixel_d_trans = {(ju.x, jv.x), (ju.y, jv.y), (ju.z, jv.z)} */
        for (int c = 0; c < 3; ++c) {
          double m[3], q3[3];
          mat3_vec(dR + 9 * c, ray, m);
          q3[0] = d * m[0];
          q3[1] = d * m[1];
          q3[2] = d * m[2];
          const double pox = dot3(ju, q3), poy = dot3(jv, q3);
          dtr[c] += (gu * ju[c] + gv * jv[c]) * inv_dt;
          dom[c] += (gu * pox + gv * poy) * inv_dt;
        }
      }
  }
  return ORC_OK;
}

/* ---- geometry-consistency loss (geometry.hpp:329-534) ------------------------------ */

/* reproject (geometry.hpp:157-166): returns valid (z > 0); px, py, z out. */
static int reproject(double x, double y, double d, const double* R, const double* tr,
                     const double* K, double* px, double* py, double* z) {
  const double fx = K[0], fy = K[1], cx = K[2], cy = K[3];
  const double bp[3] = {d * (x - cx) / fx, d * (y - cy) / fy, d}; /* backproject :147-149 */
  double p[3];
  mat3_vec(R, bp, p);
  p[0] = p[0] + tr[0];
  p[1] = p[1] + tr[1];
  p[2] = p[2] + tr[2];
  *z = p[2];
  if (!(p[2] > 0.0)) return 0;
  *px = fx * p[0] / p[2] + cx;
  *py = fy * p[1] / p[2] + cy;
  return 1;
}

int orc_geo_loss(int W, int H, const double* d0, const uint8_t* m0, const double* d1,
                 const uint8_t* m1, const double* pose, const double* K, double upstream,
                 int want_grad, double* value, int64_t* n_valid_out, double* projected,
                 double* interpolated, uint8_t* valid, double* d_d0, double* d_d1,
                 double* d_pose) {
  const size_t HW = (size_t)W * H;
  const double fx = K[0], fy = K[1], cx = K[2], cy = K[3];
  double R[9], dR[27];
  orc_rodrigues(pose, R);
  orc_rodrigues_jacobian(pose, dR);
  const double* tr = pose + 3;
  double* ppx = malloc(sizeof(double) * HW);
  double* ppy = malloc(sizeof(double) * HW);
  double* pz = malloc(sizeof(double) * HW);
  int* pcell = malloc(sizeof(int) * HW);
  double* zbuf = malloc(sizeof(double) * HW);
  int64_t* winner = malloc(sizeof(int64_t) * HW);
  if (projected) memset(projected, 0, sizeof(double) * HW);
  if (interpolated) memset(interpolated, 0, sizeof(double) * HW);
  if (valid) memset(valid, 0, HW);
  if (d_d0) memset(d_d0, 0, sizeof(double) * HW);
  if (d_d1) memset(d_d1, 0, sizeof(double) * HW);
  if (d_pose) memset(d_pose, 0, sizeof(double) * 6);
  *value = 0.0;
  *n_valid_out = 0;
  /* project_with_zmin (geometry.hpp:359-390) */
  int any = 0;
  for (size_t q = 0; q < HW; ++q) {
    zbuf[q] = INFINITY;
    winner[q] = -1;
    pcell[q] = -1;
  }
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const size_t q = idx(x, y, W);
      if (m0 && !m0[q]) continue;
      const double d = d0[q];
      if (!(d > 0.0)) continue;
      double px, py, z;
      if (!reproject((double)x, (double)y, d, R, tr, K, &px, &py, &z)) continue;
      if (!in_bounds(px, py, W, H)) continue;
      const int nx = (int)lround(px), ny = (int)lround(py);
      ppx[q] = px;
      ppy[q] = py;
      pz[q] = z;
      pcell[q] = (int)idx(nx, ny, W);
      any = 1;
      if (z < zbuf[pcell[q]]) {
        zbuf[pcell[q]] = z;
        winner[pcell[q]] = (int64_t)q;
      }
    }
  double sum = 0.0;
  int64_t n_valid = 0;
  double dom[3] = {0, 0, 0}, dtr[3] = {0, 0, 0};
  for (int y = 0; any && y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const size_t q = idx(x, y, W);
      if (pcell[q] < 0 || winner[pcell[q]] != (int64_t)q) continue;
      /* sample_target_depth (geometry.hpp:394-409) */
      const cell_t c = bilin_cell(ppx[q], ppy[q], W, H);
      if (m1 && !(m1[idx(c.x0, c.y0, W)] && m1[idx(c.x1, c.y0, W)] && m1[idx(c.x0, c.y1, W)] &&
                  m1[idx(c.x1, c.y1, W)]))
        continue;
      const double v00 = d1[idx(c.x0, c.y0, W)], v10 = d1[idx(c.x1, c.y0, W)];
      const double v01 = d1[idx(c.x0, c.y1, W)], v11 = d1[idx(c.x1, c.y1, W)];
      const double b = w00(&c) * v00 + w10(&c) * v10 + w01(&c) * v01 + w11(&c) * v11;
      if (!(b > 0.0)) continue;
      const double dbx = (1.0 - c.wy) * (v10 - v00) + c.wy * (v11 - v01);
      const double dby = (1.0 - c.wx) * (v01 - v00) + c.wx * (v11 - v10);
      const double a = pz[q];
      if (projected) projected[q] = a;
      if (interpolated) interpolated[q] = b;
      if (valid) valid[q] = 1;
      ++n_valid;
      sum += fabs(a - b) / (a + b);
      if (!want_grad) continue;
      /* geometry.hpp:479-516 */
      const double s = (a > b) ? 1.0 : (a < b ? -1.0 : 0.0);
      const double inv_ab = 1.0 / ((a + b) * (a + b));
      const double ga = 2.0 * s * b * inv_ab;
      const double gb = -2.0 * s * a * inv_ab;
      /* reproject_with_grads (geometry.hpp:185-209) */
      const double d = d0[q];
      const double ray[3] = {1.0 * ((double)x - cx) / fx, 1.0 * ((double)y - cy) / fy, 1.0};
      double rray[3];
      mat3_vec(R, ray, rray);
      const double p[3] = {d * rray[0] + tr[0], d * rray[1] + tr[1], d * rray[2] + tr[2]};
      const double iz = 1.0 / p[2];
      const double ju[3] = {fx * iz, 0.0, -fx * p[0] * iz * iz};
      const double jv[3] = {0.0, fy * iz, -fy * p[1] * iz * iz};
      const double dpdx = dot3(ju, rray), dpdy = dot3(jv, rray);
      d_d0[q] += ga * rray[2] + gb * (dbx * dpdx + dby * dpdy);
      d_d1[idx(c.x0, c.y0, W)] += gb * w00(&c);
      d_d1[idx(c.x1, c.y0, W)] += gb * w10(&c);
      d_d1[idx(c.x0, c.y1, W)] += gb * w01(&c);
      d_d1[idx(c.x1, c.y1, W)] += gb * w11(&c);
      for (int k = 0; k < 3; ++k) {
        double m[3], q3[3];
        mat3_vec(dR + 9 * k, ray, m);
        q3[0] = d * m[0];
        q3[1] = d * m[1];
        q3[2] = d * m[2];
        dtr[k] += ga * (k == 2 ? 1.0 : 0.0) + gb * (dbx * ju[k] + dby * jv[k]);
        dom[k] += ga * q3[2] + gb * (dbx * dot3(ju, q3) + dby * dot3(jv, q3));
      }
    }
  if (n_valid > 0) {
    *value = sum / (double)n_valid;
    *n_valid_out = n_valid;
    if (want_grad) {
      const double scale = upstream / (double)n_valid;
      for (size_t q = 0; q < HW; ++q) {
        d_d0[q] *= scale;
        d_d1[q] *= scale;
      }
      for (int k = 0; k < 3; ++k) {
        d_pose[k] = scale * dom[k];
        d_pose[3 + k] = scale * dtr[k];
      }
    }
  }
  free(ppx);
  free(ppy);
  free(pz);
  free(pcell);
  free(zbuf);
  free(winner);
  return ORC_OK;
}

/* ---- predictor decode chain -------------------------------------------------------- */

/* predictor.hpp:25-27 */
double orc_softplus(double x) { return x > 0.0 ? x + log1p(exp(-x)) : log1p(exp(x)); }

/* predictor.hpp:30-34 */
double orc_softplus_grad(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}

/* upsample_src_coord (predictor.hpp:40-44) + the tap of upsample_bilinear
 * (predictor.hpp:51-60) */
static void up_tap(int o, int factor, int src, int* i0, int* i1, double* w) {
  const double s = clampd(((double)o + 0.5) / (double)factor - 0.5, 0.0, (double)(src - 1));
  int a = (int)floor(s);
  if (a > src - 1) a = src - 1;
  *i0 = a;
  *i1 = a + 1 < src - 1 ? a + 1 : src - 1;
  *w = s - a;
}

int orc_decode(int pw, int ph, int factor, const double* params, double* depth) {
  if (pw <= 0 || ph <= 0 || factor < 1) return 1;
  const int W = pw * factor, H = ph * factor;
  double* low = (double*)malloc(sizeof(double) * (size_t)pw * ph);
  if (!low) return 2;
  for (int i = 0; i < pw * ph; ++i) low[i] = orc_softplus(params[i]);
  if (factor == 1) {
    memcpy(depth, low, sizeof(double) * (size_t)pw * ph);
    free(low);
    return 0;
  }
  for (int y = 0; y < H; ++y) {
    int y0, y1;
    double wy;
    up_tap(y, factor, ph, &y0, &y1, &wy);
    for (int x = 0; x < W; ++x) {
      int x0, x1;
      double wx;
      up_tap(x, factor, pw, &x0, &x1, &wx);
      depth[(size_t)y * W + x] = (1.0 - wx) * (1.0 - wy) * low[y0 * pw + x0] +
                                 wx * (1.0 - wy) * low[y0 * pw + x1] +
                                 (1.0 - wx) * wy * low[y1 * pw + x0] + wx * wy * low[y1 * pw + x1];
    }
  }
  free(low);
  return 0;
}

int orc_decode_backward(int pw, int ph, int factor, const double* params, const double* d_depth,
                        double* d_params) {
  if (pw <= 0 || ph <= 0 || factor < 1) return 1;
  const int W = pw * factor, H = ph * factor;
  double* low = (double*)calloc((size_t)pw * ph, sizeof(double));
  if (!low) return 2;
  if (factor == 1) {
    memcpy(low, d_depth, sizeof(double) * (size_t)pw * ph);
  } else {
    for (int y = 0; y < H; ++y) {  /* predictor.hpp:80-95: scatter in output order */
      int y0, y1;
      double wy;
      up_tap(y, factor, ph, &y0, &y1, &wy);
      for (int x = 0; x < W; ++x) {
        int x0, x1;
        double wx;
        up_tap(x, factor, pw, &x0, &x1, &wx);
        const double g = d_depth[(size_t)y * W + x];
        low[y0 * pw + x0] += (1.0 - wx) * (1.0 - wy) * g;
        low[y0 * pw + x1] += wx * (1.0 - wy) * g;
        low[y1 * pw + x0] += (1.0 - wx) * wy * g;
        low[y1 * pw + x1] += wx * wy * g;
      }
    }
  }
  for (int i = 0; i < pw * ph; ++i) d_params[i] = low[i] * orc_softplus_grad(params[i]);
  free(low);
  return 0;
}

void orc_adam_step(size_t n, double* slots, const double* grads, double* m, double* v, int t,
                   double lr, double beta1, double beta2, double eps) {
  const double c1 = 1.0 - pow(beta1, t), c2 = 1.0 - pow(beta2, t);  /* optimize.hpp:121-122 */
  for (size_t i = 0; i < n; ++i) {
    m[i] = beta1 * m[i] + (1.0 - beta1) * grads[i];
    v[i] = beta2 * v[i] + (1.0 - beta2) * grads[i] * grads[i];
    slots[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
  }
}
