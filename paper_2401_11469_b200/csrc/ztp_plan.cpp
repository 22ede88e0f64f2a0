// a2. Plan (ztp_plan / ztp_plan_counts): Eq.1, straggler detection
// (Alg.2 l.2-5), Eq.2 by bisection, Eq.3 scan,
// Alg.2 roles and the virtual renumbering.
// Compiled with -ffp-contract=off: every double is evaluated in the order
// DESIGN.md "Plan evaluation order" fixes, so all ranks agree bit-for-bit.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ztp.h"

namespace ztp {
void set_thread_error(const std::string& msg);
}

namespace {

using ztp::set_thread_error;

bool pwl_ok(const ztp_pwl& f) { return f.n >= 2 && f.x != nullptr && f.y != nullptr; }

// Segment j with x[j] <= v < x[j+1]; the last segment extrapolates.
double pwl_eval(const ztp_pwl& f, double v) {
  int j = 0;
  while (j + 2 < f.n && v >= f.x[j + 1]) ++j;
  return f.y[j] + (f.y[j + 1] - f.y[j]) * ((v - f.x[j]) / (f.x[j + 1] - f.x[j]));
}

double eq1(double T, double C, double M, double gmax) {
  double g = (T - C) / M;
  if (g < 0.0) g = 0.0;
  if (g > gmax) g = gmax;
  return g;
}

double gfun(const ztp_costs& c, double Lg, double b, int e) {
  return ((c.omega1 + pwl_eval(c.omega2, Lg * (1.0 - b))) - pwl_eval(c.phi1, Lg * b)) -
         pwl_eval(c.phi2, (Lg * b) / (double)(e - 1));
}

double solve_beta(const ztp_costs& c, double Lg, int e, int iters) {
  if (gfun(c, Lg, 1.0, e) >= 0.0) return 1.0;
  if (gfun(c, Lg, 0.0, e) <= 0.0) return 0.0;
  double lo = 0.0, hi = 1.0;
  for (int i = 0; i < iters; ++i) {
    const double m = 0.5 * (lo + hi);
    if (gfun(c, Lg, m, e) > 0.0)
      lo = m;
    else
      hi = m;
  }
  return 0.5 * (lo + hi);
}

}  // namespace

extern "C" void ztp_plan_opts_default(ztp_plan_opts* o) {
  if (!o) return;
  o->enable_migration = 0;
  o->zero_crit = ZTP_CRIT_MIN;
  o->gamma_max = 0.9;
  o->eps = 0.02;
  o->gamma_tol = 0.5;
  o->bisect_iters = 64;
  o->force_lambda = -1;
}

static ztp_status plan_core(int e, const double* T, const double* M, double L_ref, const ztp_costs* costs,
                            const ztp_plan_opts* opts, ztp_plan_t* out);

// A-48: a rank is resized only when it pays.  Resizing costs a rank the
// static overhead Omega_1 (measured by the pretest) as soon as it
// resizes at all; Eq.1 sheds gamma M of its GEMM time.  A RESIZE rank with
// gamma_r M <= Omega_1 stays NORMAL (gamma 0) -- timing noise just above the
// detection tolerance no longer resizes a healthy task.  Without costs (or
// Omega_1 = 0) nothing changes (paper-literal).
extern "C" ztp_status ztp_plan(int e, const double* T, const double* M, double L_ref, const ztp_costs* costs,
                               const ztp_plan_opts* opts, ztp_plan_t* out) {
  const ztp_status s = plan_core(e, T, M, L_ref, costs, opts, out);
  if (s != ZTP_OK || !costs || !(costs->omega1 > 0.0)) return s;
  for (int r = 0; r < e; ++r)
    if (out->role[r] == ZTP_RESIZE && out->gamma_r[r] * M[r] <= costs->omega1) {
      out->role[r] = ZTP_NORMAL;
      out->gamma[r] = 0.0;
      out->gamma_r[r] = 0.0;
    }
  return ZTP_OK;
}

static ztp_status plan_core(int e, const double* T, const double* M, double L_ref, const ztp_costs* costs,
                            const ztp_plan_opts* opts, ztp_plan_t* out) {
  if (!out || !T || !M || !opts) {
    set_thread_error("ztp_plan: null argument");
    return ZTP_EINVAL;
  }
  if (e < 1 || e > ZTP_MAX_RANKS) {
    set_thread_error("ztp_plan: world=" + std::to_string(e) + " outside 1..8 (S:559)");
    return ZTP_EINVAL;
  }
  for (int r = 0; r < e; ++r)
    if (!std::isfinite(T[r]) || T[r] < 0.0) {
      set_thread_error("ztp_plan: T[" + std::to_string(r) + "] not finite / negative");
      return ZTP_EINVAL;
    }
  std::memset(out, 0, sizeof(*out));
  out->world = e;
  int order[ZTP_MAX_RANKS];
  for (int r = 0; r < e; ++r) order[r] = r;
  std::stable_sort(order, order + e, [&](int a, int b) { return T[a] > T[b] || (T[a] == T[b] && a < b); });
  for (int r = 0; r < e; ++r) out->order[r] = order[r];
  double acc = 0.0;
  for (int r = 0; r < e; ++r) acc = acc + T[r];
  const double T_avg = acc / (double)e;
  double T_min = T[0];
  for (int r = 1; r < e; ++r)
    if (T[r] < T_min) T_min = T[r];
  const double thr = T_min * (1.0 + opts->eps);
  int strag[ZTP_MAX_RANKS];
  int z = 0;
  for (int i = 0; i < e; ++i)
    if (T[order[i]] > thr) strag[z++] = order[i];
  out->z = z;

  auto need_m = [&](int r) -> bool {
    if (!(M[r] > 0.0)) {
      set_thread_error("ztp_plan: M[" + std::to_string(r) + "] = 0, Eq.1 has no baseline (S:360)");
      return false;
    }
    return true;
  };

  if (!opts->enable_migration) {
    const double C = opts->zero_crit == ZTP_CRIT_AVG ? T_avg : T_min;
    for (int r = 0; r < e; ++r) {
      if (!need_m(r)) return ZTP_ENOBASELINE;
      // only detected stragglers resize (A-17 tolerance, A-38); eps = 0 is
      // paper-literal (ranks at T_min get gamma = 0 from Eq.1 anyway)
      const double g = T[r] > thr ? eq1(T[r], C, M[r], opts->gamma_max) : 0.0;
      out->gamma[r] = g;
      out->gamma_r[r] = g;
      out->role[r] = g > 0.0 ? ZTP_RESIZE : ZTP_NORMAL;
    }
    return ZTP_OK;
  }
  for (int i = 0; i < z; ++i) {
    const int r = strag[i];
    if (!need_m(r)) return ZTP_ENOBASELINE;
    out->gamma[r] = eq1(T[r], T_min, M[r], opts->gamma_max);
  }
  if (z == 0) return ZTP_OK;
  if (!costs || !pwl_ok(costs->omega2) || !pwl_ok(costs->phi1) || !pwl_ok(costs->phi2)) {
    set_thread_error("ztp_plan: cost functions need >= 2 samples (S:549)");
    return ZTP_EINVAL;
  }
  if (z == 1) {
    const int s = strag[0];
    const double g = out->gamma[s];
    if (g <= opts->gamma_tol) {
      out->role[s] = g > 0.0 ? ZTP_RESIZE : ZTP_NORMAL;
      out->gamma_r[s] = g;
      return ZTP_OK;
    }
    double b = solve_beta(*costs, L_ref * g, e, opts->bisect_iters);
    const double floor_b = 1.0 - opts->gamma_tol / g;
    if (b < floor_b) b = floor_b;
    out->beta[s] = b;
    out->phi[s] = g * b;
    out->gamma_r[s] = (g * (1.0 - b)) / (1.0 - g * b);
    out->role[s] = b == 1.0 ? ZTP_MIGRATE : (b == 0.0 ? ZTP_RESIZE : ZTP_SPLIT);
    out->x = b > 0.0 ? 1 : 0;
    return ZTP_OK;
  }
  int x = z;
  if (opts->force_lambda >= 0) {
    x = opts->force_lambda < z ? opts->force_lambda : z;
  } else {
    double gam = 0.0;
    for (int xi = 1; xi <= z; ++xi) {
      const double Tk = T[order[xi - 1]];
      gam = gam + L_ref * ((Tk - T_min) / Tk);
      if (e - xi <= 0) {
        set_thread_error("ztp_plan: e - x = 0 receivers (S:579)");
        return ZTP_ERECEIVERS;
      }
      double mx = -INFINITY;
      for (int y = xi + 1; y <= e; ++y) {
        const double v = (gam / (double)(e - xi)) * (T[order[y - 1]] / L_ref);
        if (v > mx) mx = v;
      }
      const double f = ((Tk - T_min) - pwl_eval(costs->phi1, gam)) - mx;
      if (f <= 0.0) {
        x = xi - 1;
        break;
      }
    }
  }
  out->x = x;
  for (int pos = 1; pos <= z; ++pos) {
    const int r = strag[pos - 1];
    if (pos <= x) {
      out->role[r] = ZTP_MIGRATE;
      out->beta[r] = 1.0;
      out->phi[r] = out->gamma[r];
      out->gamma_r[r] = 0.0;
    } else {
      out->role[r] = ZTP_RESIZE;
      out->gamma_r[r] = out->gamma[r];
    }
  }
  return ZTP_OK;
}

extern "C" ztp_status ztp_plan_refine(const ztp_plan_t* prev, const ztp_plan_t* fresh, double gamma_max,
                                      ztp_plan_t* out) {
  if (!prev || !fresh || !out || prev->world != fresh->world || fresh->world < 1 || fresh->world > ZTP_MAX_RANKS) {
    set_thread_error("ztp_plan_refine: null plan or world mismatch");
    return ZTP_EINVAL;
  }
  const int e = fresh->world;
  bool semi = false;
  for (int r = 0; r < e; ++r) {
    if (fresh->role[r] > ZTP_RESIZE) {
      set_thread_error("ztp_plan_refine: fresh plan of rank " + std::to_string(r) +
                       " migrates; the refresh plan must be ZERO-only (A-39, A-42)");
      return ZTP_EUNSUPPORTED;
    }
    if (prev->role[r] == ZTP_MIGRATE || prev->role[r] == ZTP_SPLIT) semi = true;
  }
  ztp_plan_t o = *fresh;
  o.x = 0;
  o.z = prev->z;
  if (semi) {   // keep the migration group and its sender order (A-42)
    o.x = prev->x;
    for (int i = 0; i < ZTP_MAX_RANKS; ++i) o.order[i] = prev->order[i];
  }
  for (int r = 0; r < e; ++r) {
    if (prev->role[r] == ZTP_NORMAL) {
      // A-43: a refresh refines the plan's stragglers only.  A normal task
      // keeps its full shard (Alg.2 resizes only the z - x stragglers, P:284;
      // a receiver's extra runtime is received work, which migration makes
      // loss-free); only a new statistics window can re-plan it.
      o.gamma[r] = 0.0;
      o.gamma_r[r] = 0.0;
      o.beta[r] = 0.0;
      o.phi[r] = 0.0;
      o.role[r] = ZTP_NORMAL;
      continue;
    }
    if (prev->role[r] == ZTP_MIGRATE || prev->role[r] == ZTP_SPLIT) {
      // A-42: compose the rank's whole shed fraction, keep its Eq.2 split
      const double keep = (1.0 - prev->gamma[r]) * (1.0 - fresh->gamma_r[r]);
      double g = 1.0 - keep;
      if (g > gamma_max) g = gamma_max;
      if (g < 0.0) g = 0.0;
      const double b = prev->beta[r];
      o.gamma[r] = g;
      o.beta[r] = b;
      o.phi[r] = g * b;
      o.gamma_r[r] = b >= 1.0 ? 0.0 : (g * (1.0 - b)) / (1.0 - g * b);
      o.role[r] = prev->role[r];
      continue;
    }
    const double keep = (1.0 - prev->gamma_r[r]) * (1.0 - fresh->gamma_r[r]);
    double g = 1.0 - keep;
    if (g > gamma_max) g = gamma_max;
    if (g < 0.0) g = 0.0;
    o.gamma[r] = g;
    o.gamma_r[r] = g;
    o.beta[r] = 0.0;
    o.phi[r] = 0.0;
    o.role[r] = g > 0.0 ? ZTP_RESIZE : ZTP_NORMAL;
  }
  *out = o;
  return ZTP_OK;
}

extern "C" ztp_status ztp_plan_uniform(int e, double gamma, ztp_plan_t* out) {
  if (!out || e < 1 || e > ZTP_MAX_RANKS || !(gamma >= 0.0) || !(gamma < 1.0)) {
    set_thread_error("ztp_plan_uniform: world outside 1..8 or gamma outside [0, 1)");
    return ZTP_EINVAL;
  }
  std::memset(out, 0, sizeof(*out));
  out->world = e;
  for (int r = 0; r < e; ++r) {
    out->order[r] = r;
    out->gamma[r] = gamma;
    out->gamma_r[r] = gamma;
    out->role[r] = gamma > 0.0 ? ZTP_RESIZE : ZTP_NORMAL;
  }
  return ZTP_OK;
}

namespace {

bool plan_is_dense(const ztp_plan_t& p) {
  for (int r = 0; r < p.world; ++r)
    if (p.role[r] != ZTP_NORMAL) return false;
  return true;
}

void plan_dense(ztp_plan_t* p, int e) {
  std::memset(p, 0, sizeof(*p));
  p->world = e;
  for (int r = 0; r < e; ++r) p->order[r] = r;
}

bool plans_equal(const ztp_plan_t& a, const ztp_plan_t& b) {
  if (a.world != b.world || a.x != b.x) return false;
  for (int r = 0; r < a.world; ++r)
    if (a.role[r] != b.role[r] || a.gamma[r] != b.gamma[r] || a.gamma_r[r] != b.gamma_r[r] ||
        a.beta[r] != b.beta[r] || a.phi[r] != b.phi[r])
      return false;
  return true;
}

}  // namespace

extern "C" void ztp_ctl_opts_default(ztp_ctl_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  ztp_plan_opts_default(&o->plan);
  o->L_ref = 1.0;
  o->trigger = 0.10;
  o->max_refines = 1;
}

extern "C" ztp_status ztp_ctl_init(ztp_ctl* c, int world) {
  if (!c || world < 1 || world > ZTP_MAX_RANKS) {
    set_thread_error("ztp_ctl_init: null controller or world outside 1..8");
    return ZTP_EINVAL;
  }
  std::memset(c, 0, sizeof(*c));
  c->world = world;
  c->state = ZTP_CTL_WINDOW;
  plan_dense(&c->plan, world);
  return ZTP_OK;
}

extern "C" ztp_status ztp_ctl_step(ztp_ctl* c, const ztp_ctl_opts* o, const ztp_costs* costs, const double* T,
                                   const double* M, int32_t* action) {
  if (!c || !o || !T || !M || !action || c->world < 1 || c->world > ZTP_MAX_RANKS) {
    set_thread_error("ztp_ctl_step: null argument or uninitialised controller");
    return ZTP_EINVAL;
  }
  const int e = c->world;
  for (int r = 0; r < e; ++r)
    if (!std::isfinite(T[r]) || !(T[r] > 0.0)) {
      set_thread_error("ztp_ctl_step: T[" + std::to_string(r) + "] must be finite and > 0");
      return ZTP_EINVAL;
    }
  *action = ZTP_CTL_KEEP;
  const double trig = o->trigger;
  c->steps = c->steps + 1;
  double Tmin = T[0], Tmax = T[0];
  for (int r = 1; r < e; ++r) {
    if (T[r] < Tmin) Tmin = T[r];
    if (T[r] > Tmax) Tmax = T[r];
  }
  auto lift = [&]() {   // next step is a statistics window on the un-resized layer
    if (!plan_is_dense(c->plan)) *action = ZTP_CTL_APPLY;
    plan_dense(&c->plan, e);
    c->state = ZTP_CTL_WINDOW;
  };
  if (c->state == ZTP_CTL_WINDOW) {
    // Alg.1 l.1-2 / Alg.2 l.2-24 on the window's un-resized runtimes
    ztp_plan_t p;
    const ztp_status s = ztp_plan(e, T, M, o->L_ref, costs, &o->plan, &p);
    if (s != ZTP_OK) return s;
    c->windows = c->windows + 1;
    if (!plan_is_dense(p)) {
      c->plan = p;
      c->replans = c->replans + 1;
      *action = ZTP_CTL_APPLY;
    }
    c->T_target = Tmin;
    c->T_wmax = Tmax;
    c->refines = 0;
    c->state = ZTP_CTL_FIRST;
    return ZTP_OK;
  }
  if (c->state == ZTP_CTL_FIRST) {
    if (!plan_is_dense(c->plan) && (Tmin < (1.0 - trig) * c->T_target || Tmax > (1.0 + trig) * c->T_wmax)) {
      // the slowdowns changed while the plan was applied: a new window (A-41)
      lift();
      return ZTP_OK;
    }
    if (!plan_is_dense(c->plan) && c->refines < o->max_refines) {
      ztp_plan_opts zo = o->plan;
      zo.enable_migration = 0;
      zo.zero_crit = ZTP_CRIT_MIN;
      ztp_plan_t fresh, ref;
      ztp_status s = ztp_plan(e, T, M, o->L_ref, nullptr, &zo, &fresh);
      if (s != ZTP_OK) return s;
      s = ztp_plan_refine(&c->plan, &fresh, o->plan.gamma_max, &ref);
      if (s != ZTP_OK) return s;
      c->refines = c->refines + 1;
      if (!plans_equal(ref, c->plan)) {
        c->plan = ref;
        c->refine_count = c->refine_count + 1;
        *action = ZTP_CTL_APPLY;
        return ZTP_OK;   // still FIRST: the refined plan's first step is judged next
      }
    }
    for (int r = 0; r < e; ++r) c->T_ref[r] = T[r];
    c->state = ZTP_CTL_MONITOR;
    return ZTP_OK;
  }
  // MONITOR: P:178's over-10% change (either direction, A-8) opens a window
  for (int r = 0; r < e; ++r)
    if (std::fabs(T[r] - c->T_ref[r]) / c->T_ref[r] > trig) {
      c->triggers = c->triggers + 1;
      lift();
      return ZTP_OK;
    }
  return ZTP_OK;
}

extern "C" ztp_status ztp_plan_counts(const ztp_plan_t* p, int rank, int64_t K, int64_t n_units, int64_t unit,
                                      int is_row, ztp_counts* out) {
  if (!p || !out || rank < 0 || rank >= p->world || unit <= 0 || n_units < unit || n_units % unit != 0 || K < 1) {
    set_thread_error("ztp_plan_counts: bad rank / unit / sizes");
    return ZTP_EINVAL;
  }
  const int e = p->world;
  const int64_t units = n_units / unit;
  auto migrating = [&](int r) { return p->role[r] == ZTP_MIGRATE || p->role[r] == ZTP_SPLIT; };
  auto nmig = [&](int s) -> int64_t {
    if (!migrating(s)) return 0;
    int64_t nm = unit * (int64_t)std::floor((double)units * p->phi[s] + 0.5);
    if (nm > n_units - unit) nm = n_units - unit;
    return nm;
  };
  std::memset(out, 0, sizeof(*out));
  out->n_mig = (int32_t)nmig(rank);
  const int64_t K_rem = is_row ? K - out->n_mig : K;
  int64_t npr = (int64_t)std::floor((double)K_rem * p->gamma_r[rank] + 0.5);
  if (npr > K_rem - 1) npr = K_rem - 1;
  if (npr < 0) npr = 0;
  out->n_prune = (int32_t)npr;
  int recv[ZTP_MAX_RANKS];
  int nrecv = 0;
  // receivers: the NORMAL tasks ("evenly distributed across other
  // normal tasks"; A-44) -- they never resize, so migrated work stays
  // loss-free
  for (int r = 0; r < e; ++r)
    if (p->role[r] == ZTP_NORMAL) recv[nrecv++] = r;
  for (int i = 0; i < e; ++i) {
    const int s = p->order[i];
    const int64_t nm = nmig(s);
    if (nm == 0) continue;
    if (nrecv == 0) {
      set_thread_error("ztp_plan_counts: no receivers");
      return ZTP_ERECEIVERS;
    }
    int R[ZTP_MAX_RANKS];
    for (int j = 0; j < nrecv; ++j) R[j] = recv[j];
    std::sort(R, R + nrecv, [&](int a, int b) { return (a - s + e) % e < (b - s + e) % e; });
    const int64_t tot = nm / unit;
    const int64_t m = tot / nrecv, extra = tot % nrecv;
    int64_t lo = n_units - nm;
    for (int j = 0; j < nrecv; ++j) {
      const int64_t cnt = (m + (j < extra ? 1 : 0)) * unit;
      if (cnt > 0) {
        if (rank == s) {
          out->out_dst[out->n_out] = R[j];
          out->out_lo[out->n_out] = lo;
          out->out_hi[out->n_out] = lo + cnt;
          ++out->n_out;
        }
        if (rank == R[j]) {
          out->in_src[out->n_in] = s;
          out->in_lo[out->n_in] = lo;
          out->in_hi[out->n_in] = lo + cnt;
          ++out->n_in;
        }
      }
      lo += cnt;
    }
  }
  return ZTP_OK;
}

extern "C" ztp_status ztp_layer_prune_counts(const ztp_plan_t* p, int rank, int64_t h, int64_t a, int64_t u,
                                             int32_t out[4]) {
  if (!p || !out || rank < 0 || rank >= p->world || h < 1 || a < 1 || u < 1) {
    set_thread_error("ztp_layer_prune_counts: bad plan / rank / sizes");
    return ZTP_EINVAL;
  }
  // A-37: heads do not migrate (A-26), so a rank that sheds MLP units
  // resizes its attention by its Eq.1 gamma; others by gamma_r.
  const double g_att =
      (p->role[rank] == ZTP_MIGRATE || p->role[rank] == ZTP_SPLIT) ? p->gamma[rank] : p->gamma_r[rank];
  auto att = [&](int64_t K) -> int32_t {   // A-3 rounding, A-4 clamp
    int64_t n = (int64_t)std::floor((double)K * g_att + 0.5);
    if (n > K - 1) n = K - 1;
    if (n < 0) n = 0;
    return (int32_t)n;
  };
  out[0] = att(h);
  out[1] = att(a);
  ztp_counts c;
  ztp_status s;
  if ((s = ztp_plan_counts(p, rank, h, u, 1, 0, &c)) != ZTP_OK) return s;
  out[2] = c.n_prune;
  if ((s = ztp_plan_counts(p, rank, u, u, 1, 1, &c)) != ZTP_OK) return s;
  out[3] = c.n_prune;
  return ZTP_OK;
}

extern "C" int32_t ztp_pridiff_counts(int64_t L, int64_t L_uni, double gamma_t, double alpha, double gamma_max) {
  if (L < 1) return 0;
  // Alg.1 l.10-11, then A-4 (clamp, >= 1 survives) and A-3 (rounding)
  double g = 1.0 - (double)L_uni / (double)L;
  const double f = alpha * gamma_t;
  if (f > g) g = f;
  if (g > gamma_max) g = gamma_max;
  if (g < 0.0) g = 0.0;
  int64_t n = (int64_t)std::floor((double)L * g + 0.5);
  if (n > L - 1) n = L - 1;
  return (int32_t)n;
}

namespace {

// Samples -> a non-decreasing piecewise-linear function through (0, 0) (A-40):
// x ascending, duplicates and x <= 0 dropped, y = running max clamped at 0 (a
// cost cannot shrink when more units move; a dip is timing noise).  Writes at
// most n + 2 points.
int monotone_fit(int n, const double* x, const double* y, double* ox, double* oy) {
  std::vector<std::pair<double, double>> pts;
  for (int i = 0; i < n; ++i) pts.emplace_back(x[i], y[i]);
  std::sort(pts.begin(), pts.end());
  int m = 0;
  ox[m] = 0.0;
  oy[m] = 0.0;
  ++m;
  for (const auto& pt : pts) {
    if (!(pt.first > ox[m - 1])) continue;
    double v = pt.second > 0.0 ? pt.second : 0.0;
    if (oy[m - 1] > v) v = oy[m - 1];
    ox[m] = pt.first;
    oy[m] = v;
    ++m;
  }
  if (m < 2) {
    ox[m] = 1.0;
    oy[m] = 0.0;
    ++m;
  }
  return m;
}

}  // namespace

extern "C" ztp_status ztp_costs_fit(int n_omega, const double* omega_x, const double* omega_y, int n_phi1,
                                    const double* phi1_x, const double* phi1_y, int n_phi2, const double* phi2_x,
                                    const double* phi2_y, int cap, double* xs, double* ys, ztp_costs* out) {
  if (!out || !xs || !ys || n_omega < 0 || n_phi1 < 0 || n_phi2 < 0 || (n_omega && (!omega_x || !omega_y)) ||
      (n_phi1 && (!phi1_x || !phi1_y)) || (n_phi2 && (!phi2_x || !phi2_y))) {
    set_thread_error("ztp_costs_fit: null argument");
    return ZTP_EINVAL;
  }
  const int need = std::max(std::max(n_omega, n_phi1), n_phi2) + 2;
  if (cap < need) {
    set_thread_error("ztp_costs_fit: cap " + std::to_string(cap) + " < " + std::to_string(need) + " points");
    return ZTP_EINVAL;
  }
  auto finite = [](int n, const double* x, const double* y) {
    for (int i = 0; i < n; ++i)
      if (!std::isfinite(x[i]) || !std::isfinite(y[i])) return false;
    return true;
  };
  if (!finite(n_omega, omega_x, omega_y) || !finite(n_phi1, phi1_x, phi1_y) || !finite(n_phi2, phi2_x, phi2_y)) {
    set_thread_error("ztp_costs_fit: non-finite sample");
    return ZTP_EINVAL;
  }
  // Omega_1 = the extra cost at the smallest pruned count > 0 ("static
  // space allocation overhead"), Omega_2(n) = extra(n) - Omega_1
  std::vector<double> px, py;
  int first = -1;
  for (int i = 0; i < n_omega; ++i)
    if (omega_x[i] > 0.0 && (first < 0 || omega_x[i] < omega_x[first])) first = i;
  double omega1 = 0.0;
  if (first >= 0) omega1 = omega_y[first] > 0.0 ? omega_y[first] : 0.0;
  for (int i = 0; i < n_omega; ++i)
    if (omega_x[i] > 0.0) {
      px.push_back(omega_x[i]);
      py.push_back(omega_y[i] - omega1);
    }
  out->omega1 = omega1;
  out->omega2.n = monotone_fit((int)px.size(), px.data(), py.data(), xs, ys);
  out->omega2.x = xs;
  out->omega2.y = ys;
  out->phi1.n = monotone_fit(n_phi1, phi1_x, phi1_y, xs + cap, ys + cap);
  out->phi1.x = xs + cap;
  out->phi1.y = ys + cap;
  out->phi2.n = monotone_fit(n_phi2, phi2_x, phi2_y, xs + 2 * cap, ys + 2 * cap);
  out->phi2.x = xs + 2 * cap;
  out->phi2.y = ys + 2 * cap;
  return ZTP_OK;
}
