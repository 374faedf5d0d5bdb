/*
 * fbsim_oracle.c -- TEST INFRASTRUCTURE ONLY (see fbsim_oracle.h).
 *
 * Plain-C restatement of the reference fbsim hot path.  Every function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj).  Compile WITHOUT FMA contraction (-ffp-contract=off,
 * no -march): the reference's batch decisions change under FMA.
 */
#include "fbsim_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "../include/fbgpu_digest.h"

#define ORC_INF INT64_MAX

/* ---------------------------------------------------------------- rng.h */

/* splitmix64, rng.h:25-30 */
static uint64_t orc_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* derive_seed, rng.h:33-37 */
static uint64_t orc_derive_seed(uint64_t base, uint64_t stream) {
  uint64_t s = base ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
  orc_splitmix64(&s);
  return orc_splitmix64(&s);
}

typedef struct {
  uint64_t state;
} orc_rng;

/* Rng::next_double, rng.h:44-46 */
static double orc_next_double(orc_rng* r) {
  return (double)(orc_splitmix64(&r->state) >> 11) * 0x1.0p-53;
}

/* Rng::exponential, rng.h:58-64 */
static double orc_exponential(orc_rng* r, double rate) {
  double u;
  do {
    u = orc_next_double(r);
  } while (u <= 0.0);
  return -log(u) / rate;
}

/* Rng::normal (Box-Muller), rng.h:67-74 */
static double orc_normal(orc_rng* r) {
  double u1;
  do {
    u1 = orc_next_double(r);
  } while (u1 <= 0.0);
  const double u2 = orc_next_double(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* Rng::lognormal, rng.h:76-78 */
static double orc_lognormal(orc_rng* r, double mu, double sigma) {
  return exp(mu + sigma * orc_normal(r));
}

/* keyed_uniform, rng.h:91-94 */
double orc_keyed_uniform(uint64_t seed, uint64_t ordinal) {
  uint64_t s = orc_derive_seed(seed, ordinal);
  return (double)(orc_splitmix64(&s) >> 11) * 0x1.0p-53;
}

/* --------------------------------------------------------------- time.h */

/* ms_to_us / us_to_ms, time.h:30-34 */
static int64_t orc_ms_to_us(double ms) { return (int64_t)llround(ms * 1000.0); }
static double orc_us_to_ms(int64_t us) { return (double)us / 1000.0; }

/* ----------------------------------------------------------- workload.cpp */

static const double kZ90 = 1.2815515655446004; /* workload.cpp:31 */

/* lognormal_params, workload.cpp:231-242 */
static int orc_lognormal_params(double mean, double p90, double* mu,
                                double* sigma) {
  if (!(mean > 0.0) || !(p90 > 0.0)) return FB_ERR_VALIDATION;
  const double ratio = log(p90 / mean);
  const double disc = kZ90 * kZ90 - 2.0 * ratio;
  double s = disc >= 0.0 ? kZ90 - sqrt(disc) : kZ90;
  if (s < 0.0) s = 0.0;
  *sigma = s;
  *mu = log(mean) - 0.5 * s * s;
  return FB_OK;
}

/* generate_bursty, workload.cpp:244-298.  Arrivals are produced in
 * increasing time order, so the stable sort (workload.cpp:289-292) is the
 * identity; it is checked rather than performed. */
int orc_generate_bursty(const fb_burst_profile* p, int64_t horizon,
                        int64_t cap, int64_t* arrival_us, int32_t* prompt_len,
                        int32_t* output_len, int64_t* ttft_us, int64_t* tpot_us,
                        int64_t* n_out) {
  if (horizon <= 0) return FB_ERR_VALIDATION;
  if (p->base_rate < 0.0 || p->burst_rate < p->base_rate)
    return FB_ERR_VALIDATION;
  if (p->ttft_us <= 0 || p->tpot_us <= 0) return FB_ERR_VALIDATION;
  double pmu, psig, omu, osig;
  if (orc_lognormal_params(p->prompt_mean, p->prompt_p90, &pmu, &psig))
    return FB_ERR_VALIDATION;
  if (orc_lognormal_params(p->output_mean, p->output_p90, &omu, &osig))
    return FB_ERR_VALIDATION;
  orc_rng arrivals = {orc_derive_seed(p->seed, 1)};
  orc_rng lengths = {orc_derive_seed(p->seed, 2)};
  int64_t n = 0, last = INT64_MIN;
  int64_t phase_start = 0;
  int in_burst = 0;
  while (phase_start < horizon) {
    const int64_t phase_len = in_burst ? p->burst_duration_us : p->idle_duration_us;
    const double rate = in_burst ? p->burst_rate : p->base_rate;
    const int64_t phase_end =
        phase_start + phase_len < horizon ? phase_start + phase_len : horizon;
    if (rate > 0.0) {
      double t_ms = orc_us_to_ms(phase_start);
      const double end_ms = orc_us_to_ms(phase_end);
      for (;;) {
        t_ms += orc_exponential(&arrivals, rate) * 1000.0;
        if (t_ms >= end_ms) break;
        const int64_t arr = orc_ms_to_us(t_ms);
        int64_t pl = (int64_t)llround(orc_lognormal(&lengths, pmu, psig));
        int64_t ol = (int64_t)llround(orc_lognormal(&lengths, omu, osig));
        if (pl < 1) pl = 1;
        if (ol < 1) ol = 1;
        if (arr < last) return FB_ERR_VALIDATION; /* sort would not be identity */
        last = arr;
        if (n < cap) {
          arrival_us[n] = arr;
          prompt_len[n] = (int32_t)pl;
          output_len[n] = (int32_t)ol;
          ttft_us[n] = p->ttft_us;
          tpot_us[n] = p->tpot_us;
        }
        ++n;
      }
    }
    phase_start = phase_end;
    in_burst = !in_burst;
  }
  *n_out = n;
  return n <= cap ? FB_OK : FB_ERR_CAPACITY;
}

/* scale_trace, workload.cpp:211-221 */
int orc_scale_trace(int64_t* arrival_us, int64_t n, double factor) {
  if (!(factor > 0.0)) return FB_ERR_VALIDATION;
  for (int64_t i = 0; i < n; ++i)
    arrival_us[i] = (int64_t)llround((double)arrival_us[i] / factor);
  return FB_OK;
}

/* --------------------------------------------------------------- sched.cpp */

static int cmp_slack(const void* x, const void* y) { /* slack_order, sched.cpp:28-31 */
  const fb_task_view* a = (const fb_task_view*)x;
  const fb_task_view* b = (const fb_task_view*)y;
  if (a->slack_us != b->slack_us) return a->slack_us < b->slack_us ? -1 : 1;
  if (a->arrival_seq != b->arrival_seq) return a->arrival_seq < b->arrival_seq ? -1 : 1;
  return 0;
}

static int cmp_fifo(const void* x, const void* y) { /* fifo_order, sched.cpp:33-35 */
  const fb_task_view* a = (const fb_task_view*)x;
  const fb_task_view* b = (const fb_task_view*)y;
  if (a->arrival_seq != b->arrival_seq) return a->arrival_seq < b->arrival_seq ? -1 : 1;
  return 0;
}

/* init_time_budget, sched.cpp:90-106 */
int orc_init_time_budget(const fb_task_view* t, int64_t n, int64_t* out) {
  if (n <= 0) return FB_ERR_USAGE;
  int64_t min_tpot = INT64_MAX, min_dec = INT64_MAX;
  int has_decode = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (t[i].tpot_us < min_tpot) min_tpot = t[i].tpot_us;
    if (t[i].phase == FB_PHASE_DECODE) {
      has_decode = 1;
      if (t[i].slack_us < min_dec) min_dec = t[i].slack_us;
    }
  }
  *out = !has_decode ? min_tpot : (min_dec > min_tpot ? min_dec : min_tpot);
  return FB_OK;
}

/* predict_step_time_ms, costmodel.cpp:112-116 */
static double orc_predict(const fb_cost_model* m, int64_t nw, int64_t ctx) {
  return m->a_ms + m->b_ms * (double)nw + m->c_ms * (double)ctx;
}

/* finalize_plan, sched.cpp:37-48 */
static void orc_finalize(fb_batch_plan* plan, const fb_cost_model* m,
                         int64_t total_new, int64_t total_ctx) {
  if (plan->n_entries == 0) {
    plan->predicted_ms = 0.0;
    plan->time_budget_used_ms = 0.0;
    plan->token_budget_used = 0;
    return;
  }
  plan->predicted_ms = orc_predict(m, total_new, total_ctx);
  plan->time_budget_used_ms = plan->predicted_ms;
  plan->token_budget_used = total_new;
}

static void orc_push(fb_plan_entry_id* e, fb_batch_plan* plan, int64_t id,
                     int32_t nw) {
  e[plan->n_entries].request_id = id;
  e[plan->n_entries].new_tokens = nw;
  e[plan->n_entries].reserved = 0;
  plan->n_entries++;
}

/* form_batch_fairbatching, sched.cpp:108-170 */
static int orc_fairbatch(const fb_task_view* tasks, int64_t n,
                         const fb_scheduler_config* cfg, fb_plan_entry_id* e,
                         fb_batch_plan* plan, int64_t* total_ctx_out) {
  int64_t init_budget;
  int st = orc_init_time_budget(tasks, n, &init_budget);
  if (st) return st;
  int64_t min_tpot = INT64_MAX;
  for (int64_t i = 0; i < n; ++i)
    if (tasks[i].tpot_us < min_tpot) min_tpot = tasks[i].tpot_us;
  const int64_t urgency_bound = init_budget + min_tpot;

  fb_task_view* grp = (fb_task_view*)malloc(sizeof(fb_task_view) * (size_t)(n > 0 ? n : 1));
  int64_t n_ud = 0, n_p = 0, n_nd = 0;
  for (int64_t i = 0; i < n; ++i)
    if (tasks[i].phase == FB_PHASE_DECODE && tasks[i].slack_us < urgency_bound) grp[n_ud++] = tasks[i];
  for (int64_t i = 0; i < n; ++i)
    if (!(tasks[i].phase == FB_PHASE_DECODE && tasks[i].slack_us < urgency_bound) &&
        tasks[i].phase == FB_PHASE_PREFILL)
      grp[n_ud + n_p++] = tasks[i];
  for (int64_t i = 0; i < n; ++i)
    if (tasks[i].phase == FB_PHASE_DECODE && !(tasks[i].slack_us < urgency_bound))
      grp[n_ud + n_p + n_nd++] = tasks[i];
  qsort(grp, (size_t)n_ud, sizeof(fb_task_view), cmp_slack);
  qsort(grp + n_ud, (size_t)n_p, sizeof(fb_task_view), cmp_slack);
  qsort(grp + n_ud + n_p, (size_t)n_nd, sizeof(fb_task_view), cmp_slack);

  const double a = cfg->model.a_ms, b = cfg->model.b_ms, c = cfg->model.c_ms;
  double time_budget = orc_us_to_ms(init_budget) - a;
  int64_t token_budget = cfg->token_budget;
  plan->init_time_budget_ms = orc_us_to_ms(init_budget);
  int64_t total_new = 0, total_ctx = 0;
  for (int64_t i = 0; i < n; ++i) { /* consider, sched.cpp:141-166 */
    const fb_task_view* t = &grp[i];
    const double ctx_cost = c * (double)t->context;
    const double time_cost = b * (double)t->new_tokens + ctx_cost;
    if (time_cost <= time_budget && t->new_tokens <= token_budget) {
      orc_push(e, plan, t->request_id, t->new_tokens);
      time_budget -= time_cost;
      token_budget -= t->new_tokens;
      total_new += t->new_tokens;
      total_ctx += t->context;
    } else if (token_budget > 0 && ctx_cost <= time_budget) {
      const double lim = (time_budget - ctx_cost) / b;
      const double dtok = (double)token_budget;
      const double cp_real = lim < dtok ? lim : dtok; /* std::min(dtok, lim) */
      const int64_t cp = (int64_t)floor(cp_real);
      if (cp >= 1) {
        orc_push(e, plan, t->request_id, (int32_t)cp);
        time_budget -= b * (double)cp + ctx_cost;
        token_budget -= cp;
        total_new += cp;
        total_ctx += t->context;
      }
    }
  }
  free(grp);
  orc_finalize(plan, &cfg->model, total_new, total_ctx);
  *total_ctx_out = total_ctx;
  return FB_OK;
}

/* form_batch_sarathi, sched.cpp:172-206 */
static int orc_sarathi(const fb_task_view* tasks, int64_t n,
                       const fb_scheduler_config* cfg, fb_plan_entry_id* e,
                       fb_batch_plan* plan, int64_t* total_ctx_out) {
  fb_task_view* v = (fb_task_view*)malloc(sizeof(fb_task_view) * (size_t)(n > 0 ? n : 1));
  int64_t nd = 0, np = 0;
  for (int64_t i = 0; i < n; ++i)
    if (tasks[i].phase == FB_PHASE_DECODE) v[nd++] = tasks[i];
  for (int64_t i = 0; i < n; ++i)
    if (tasks[i].phase != FB_PHASE_DECODE) v[nd + np++] = tasks[i];
  qsort(v, (size_t)nd, sizeof(fb_task_view), cmp_fifo);
  qsort(v + nd, (size_t)np, sizeof(fb_task_view), cmp_fifo);
  int64_t total_new = 0, total_ctx = 0;
  for (int64_t i = 0; i < nd; ++i) {
    orc_push(e, plan, v[i].request_id, 1);
    total_new += 1;
    total_ctx += v[i].context;
  }
  int64_t remaining = cfg->token_budget - nd;
  if (remaining < 0) remaining = 0;
  for (int64_t i = nd; i < nd + np; ++i) {
    if (remaining <= 0) break;
    int64_t chunk = remaining;
    if (cfg->max_chunk < chunk) chunk = cfg->max_chunk;
    if (v[i].new_tokens < chunk) chunk = v[i].new_tokens;
    if (chunk < 1) continue;
    orc_push(e, plan, v[i].request_id, (int32_t)chunk);
    remaining -= chunk;
    total_new += chunk;
    total_ctx += v[i].context;
  }
  free(v);
  orc_finalize(plan, &cfg->model, total_new, total_ctx);
  *total_ctx_out = total_ctx;
  return FB_OK;
}

/* form_batch_prefill_first, sched.cpp:208-232 */
static int orc_prefill_first(const fb_task_view* tasks, int64_t n,
                             const fb_scheduler_config* cfg,
                             fb_plan_entry_id* e, fb_batch_plan* plan,
                             int64_t* total_ctx_out) {
  fb_task_view* v = (fb_task_view*)malloc(sizeof(fb_task_view) * (size_t)(n > 0 ? n : 1));
  if (n > 0) memcpy(v, tasks, sizeof(fb_task_view) * (size_t)n);
  qsort(v, (size_t)n, sizeof(fb_task_view), cmp_fifo);
  int64_t total_new = 0, total_ctx = 0, budget = cfg->token_budget;
  for (int64_t i = 0; i < n; ++i) {
    if (budget <= 0) break;
    int64_t take;
    if (v[i].phase == FB_PHASE_DECODE) {
      take = 1;
    } else {
      take = budget;
      if (cfg->max_chunk < take) take = cfg->max_chunk;
      if (v[i].new_tokens < take) take = v[i].new_tokens;
    }
    if (take < 1 || take > budget) continue;
    orc_push(e, plan, v[i].request_id, (int32_t)take);
    budget -= take;
    total_new += take;
    total_ctx += v[i].context;
  }
  free(v);
  orc_finalize(plan, &cfg->model, total_new, total_ctx);
  *total_ctx_out = total_ctx;
  return FB_OK;
}

/* form_batch dispatch, sched.cpp:234-246 */
static int orc_form_batch_ctx(const fb_task_view* tasks, int64_t n,
                              const fb_scheduler_config* cfg,
                              fb_plan_entry_id* entries, fb_batch_plan* plan,
                              int64_t* total_ctx) {
  memset(plan, 0, sizeof(*plan));
  switch (cfg->policy) {
    case FB_POLICY_PREFILL_FIRST:
      return orc_prefill_first(tasks, n, cfg, entries, plan, total_ctx);
    case FB_POLICY_SARATHI:
      return orc_sarathi(tasks, n, cfg, entries, plan, total_ctx);
    case FB_POLICY_FAIRBATCH:
    case FB_POLICY_FAIRBATCH_PAB:
      return orc_fairbatch(tasks, n, cfg, entries, plan, total_ctx);
  }
  return FB_ERR_USAGE;
}

int orc_form_batch(const fb_task_view* tasks, int64_t n,
                   const fb_scheduler_config* cfg, fb_plan_entry_id* entries,
                   fb_batch_plan* plan) {
  int64_t ctx;
  return orc_form_batch_ctx(tasks, n, cfg, entries, plan, &ctx);
}

/* pab, sched.cpp:248-278 */
int orc_pab(const fb_task_view* tasks, int64_t n, const fb_cost_model* m,
            int64_t ttft_us, int64_t tpot_us, int64_t* out) {
  const double W = orc_us_to_ms(ttft_us);
  const double T = orc_us_to_ms(tpot_us);
  const double a = m->a_ms, b = m->b_ms, c = m->c_ms;
  double n_batches = 1.0;
  if (n > 0) {
    int64_t min_slack = INT64_MAX;
    for (int64_t i = 0; i < n; ++i)
      if (tasks[i].slack_us < min_slack) min_slack = tasks[i].slack_us;
    const double ms = orc_us_to_ms(min_slack);
    const double min_slack_ms = W < ms ? W : ms; /* std::min(ms, W) */
    n_batches = (W - min_slack_ms) / T + 1.0;
  }
  const double r_batches = n_batches * a;
  double r_tasks = 0.0;
  int64_t prefill_tokens = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double x = (W - orc_us_to_ms(tasks[i].slack_us)) / T;
    const double steps = 0.0 < x ? x : 0.0; /* std::max(0.0, x) */
    r_tasks += steps * (b + (double)tasks[i].context * c);
    if (tasks[i].phase == FB_PHASE_PREFILL) prefill_tokens += tasks[i].new_tokens;
  }
  const double r_prefill = W - r_batches - r_tasks;
  const double t_prefill = r_prefill / (b + c);
  *out = (int64_t)floor(t_prefill) - prefill_tokens;
  return FB_OK;
}

/* -------------------------------------------------------------- engine.cpp */

typedef struct {
  const fb_instance* inst;
  const fb_trace* rows;
  int64_t base; /* first row */
  /* per request (row within instance) */
  int32_t* prefilled;
  int32_t* nidx;
  int64_t* first;
  int64_t* seq;
  double* maxtp;
  double* maxtp_alt;
  uint32_t* flags;
  /* lists */
  int32_t* active;
  int64_t n_active;
  int32_t* waiting;
  int64_t n_waiting;
  int32_t* pend_row;
  int64_t* pend_vis;
  int64_t pend_head, pend_tail;
  /* scratch */
  fb_task_view* views;
  fb_plan_entry_id* plan_e;
  /* step machine */
  int busy;
  int64_t step_end;
  uint64_t step_counter;
  int64_t seq_counter;
  fb_batch_plan inflight;
  double inflight_actual;
  /* outputs */
  fb_instance_result* res;
  const fb_log_opts* log;
  fb_log_counts* counts;
  fb_step_log* steps;
  fb_plan_entry* entries;
  fb_reject_log* rejects;
} orc_node;

#define R_ARR(nd, r) ((nd)->rows->arrival_us[(nd)->base + (r)])
#define R_PROMPT(nd, r) ((nd)->rows->prompt_len[(nd)->base + (r)])
#define R_OUTPUT(nd, r) ((nd)->rows->output_len[(nd)->base + (r)])
#define R_TTFT(nd, r) ((nd)->rows->ttft_us[(nd)->base + (r)])
#define R_TPOT(nd, r) ((nd)->rows->tpot_us[(nd)->base + (r)])

/* build_task_views for one request, engine.cpp:51-81 */
static void orc_view(const orc_node* nd, int32_t r, int64_t now, fb_task_view* v) {
  v->request_id = r;
  v->arrival_seq = nd->seq[r];
  v->tpot_us = R_TPOT(nd, r);
  const int32_t prompt = R_PROMPT(nd, r);
  if (nd->prefilled[r] < prompt) {
    v->phase = FB_PHASE_PREFILL;
    v->new_tokens = prompt - nd->prefilled[r];
    v->context = nd->prefilled[r];
    /* slack(), slo.h:45-61 */
    v->slack_us = R_ARR(nd, r) + R_TTFT(nd, r) +
                  R_TPOT(nd, r) * (int64_t)nd->nidx[r] - now;
  } else {
    v->phase = FB_PHASE_DECODE;
    v->new_tokens = 1;
    v->context = (int64_t)prompt + nd->nidx[r];
    int64_t anchor = R_ARR(nd, r) + R_TTFT(nd, r);
    if (nd->first[r] >= 0 && nd->first[r] < anchor) anchor = nd->first[r];
    v->slack_us = anchor + R_TPOT(nd, r) * (int64_t)nd->nidx[r] - now;
  }
}

/* Node::views, engine.cpp:107-121 */
static int64_t orc_views(const orc_node* nd, int64_t now) {
  int64_t k = 0;
  for (int64_t i = 0; i < nd->n_active; ++i) orc_view(nd, nd->active[i], now, &nd->views[k++]);
  const int32_t max_active = nd->inst->cfg.max_active;
  int64_t slots = max_active > 0 ? (int64_t)max_active - nd->n_active : INT64_MAX;
  for (int64_t i = 0; i < nd->n_waiting; ++i) {
    if (slots <= 0) break;
    orc_view(nd, nd->waiting[i], now, &nd->views[k++]);
    --slots;
  }
  return k;
}

/* Node::current_pab, engine.cpp:123-125 */
static int64_t orc_current_pab(const orc_node* nd, int64_t now) {
  const int64_t n = orc_views(nd, now);
  int64_t out;
  orc_pab(nd->views, n, &nd->inst->cfg.scheduler.model,
          nd->inst->cfg.global_ttft_us, nd->inst->cfg.global_tpot_us, &out);
  return out;
}

/* Node::enqueue, engine.cpp:92-105 */
static void orc_enqueue(orc_node* nd, int32_t r, int64_t visible_at) {
  nd->flags[r] |= FB_REC_ARRIVED;
  nd->pend_row[nd->pend_tail] = r;
  nd->pend_vis[nd->pend_tail] = visible_at;
  nd->pend_tail++;
  nd->res->n_arrived++;
}

/* Node::pull_arrivals, engine.cpp:127-151 */
static void orc_pull_arrivals(orc_node* nd, int64_t now) {
  while (nd->pend_head < nd->pend_tail && nd->pend_vis[nd->pend_head] <= now) {
    const int32_t r = nd->pend_row[nd->pend_head++];
    if (nd->inst->cfg.scheduler.policy == FB_POLICY_FAIRBATCH_PAB) {
      const int64_t budget = orc_current_pab(nd, now);
      if (!((int64_t)R_PROMPT(nd, r) <= budget)) { /* admit, sched.h:113-115 */
        nd->flags[r] |= FB_REC_REJECTED;
        nd->res->n_rejected++;
        nd->res->plan_digest = fb_digest_reject(nd->res->plan_digest, now, (uint32_t)r, budget);
        if (nd->rejects && nd->counts->rejects < nd->log->reject_cap) {
          fb_reject_log* rl = &nd->rejects[nd->counts->rejects++];
          rl->t_us = now;
          rl->pab_tokens = budget;
          rl->req = r;
          rl->step = (int32_t)nd->step_counter;
        } else if (nd->rejects) {
          nd->counts->truncated = 1;
        }
        continue;
      }
    }
    nd->seq[r] = nd->seq_counter++;
    nd->waiting[nd->n_waiting++] = r;
  }
}

/* Node::begin_step, engine.cpp:153-202 */
static int orc_begin_step(orc_node* nd, int64_t now) {
  orc_pull_arrivals(nd, now);
  const int64_t n = orc_views(nd, now);
  if (n == 0) return 0;
  int64_t total_ctx = 0;
  int st = orc_form_batch_ctx(nd->views, n, &nd->inst->cfg.scheduler, nd->plan_e,
                              &nd->inflight, &total_ctx);
  if (st) return st;
  int64_t total_new = 0;
  uint64_t esum = 0;
  for (int64_t k = 0; k < nd->inflight.n_entries; ++k) {
    total_new += nd->plan_e[k].new_tokens;
    esum ^= fb_digest_entry((uint32_t)k, (uint32_t)nd->plan_e[k].request_id,
                            (uint32_t)nd->plan_e[k].new_tokens);
  }
  /* ground_truth_step_time_ms, costmodel.cpp:138-146 */
  const fb_engine_config* cfg = &nd->inst->cfg;
  double actual = orc_predict(&cfg->truth_model, total_new, total_ctx);
  if (cfg->noise_amplitude != 0.0) {
    const double u = 2.0 * orc_keyed_uniform(cfg->noise_seed, nd->step_counter) - 1.0;
    actual = actual * (1.0 + cfg->noise_amplitude * u);
  }
  /* waiting -> active in plan order, engine.cpp:176-182 */
  for (int64_t k = 0; k < nd->inflight.n_entries; ++k) {
    const int32_t r = (int32_t)nd->plan_e[k].request_id;
    for (int64_t i = 0; i < nd->n_waiting; ++i) {
      if (nd->waiting[i] == r) {
        memmove(&nd->waiting[i], &nd->waiting[i + 1],
                sizeof(int32_t) * (size_t)(nd->n_waiting - i - 1));
        nd->n_waiting--;
        nd->active[nd->n_active++] = r;
        break;
      }
    }
  }
  int64_t dur = orc_ms_to_us(actual);
  if (dur < 1) dur = 1; /* engine.cpp:196-198 */
  nd->res->plan_digest = fb_digest_step(nd->res->plan_digest, now,
                                        (uint32_t)nd->inflight.n_entries, esum,
                                        nd->inflight.predicted_ms, actual);
  nd->res->sum_visible += n;
  nd->res->sum_entries += nd->inflight.n_entries;
  nd->res->sum_new_tokens += total_new;
  if (nd->steps) {
    if (nd->counts->steps < nd->log->step_cap &&
        nd->counts->entries + nd->inflight.n_entries <= nd->log->entry_cap) {
      fb_step_log* sl = &nd->steps[nd->counts->steps++];
      sl->t_us = now;
      sl->duration_us = dur;
      sl->predicted_ms = nd->inflight.predicted_ms;
      sl->actual_ms = actual;
      sl->total_new = total_new;
      sl->total_ctx = total_ctx;
      sl->init_budget_ms = nd->inflight.init_time_budget_ms;
      sl->entry_off = nd->counts->entries;
      sl->n_entries = (int32_t)nd->inflight.n_entries;
      for (int64_t k = 0; k < nd->inflight.n_entries; ++k) {
        nd->entries[nd->counts->entries].req = (int32_t)nd->plan_e[k].request_id;
        nd->entries[nd->counts->entries].new_tokens = nd->plan_e[k].new_tokens;
        nd->counts->entries++;
      }
    } else {
      nd->counts->truncated = 1;
    }
  }
  nd->busy = 1;
  nd->inflight_actual = actual;
  nd->step_end = now + dur;
  nd->step_counter++;
  return 0;
}

/* token emission inside complete_step (engine.cpp:211-232) plus the online
 * RequestReport bookkeeping of request_reports (metrics.cpp:60-116). */
static void orc_emit(orc_node* nd, int32_t r, int64_t t) {
  const int32_t idx = nd->nidx[r];
  const int64_t arr = R_ARR(nd, r);
  const int64_t tpot = R_TPOT(nd, r);
  if (idx == 0) {
    nd->first[r] = t;
    if (t - arr <= R_TTFT(nd, r)) nd->flags[r] |= FB_REC_MET_TTFT;
  } else {
    const int64_t d = t - nd->first[r];
    if (d > tpot * (int64_t)idx) nd->flags[r] |= 0x80000000u; /* tpot violated */
    const double x = orc_us_to_ms(d) / (double)idx;
    if (nd->maxtp[r] < x) nd->maxtp[r] = x; /* std::max(best, x) */
    if (idx >= 2) {
      const double y = orc_us_to_ms(d) / (double)(idx - 1);
      if (nd->maxtp_alt[r] < y) nd->maxtp_alt[r] = y;
    }
    if (t - arr > R_TTFT(nd, r) + tpot * (int64_t)idx) nd->flags[r] |= FB_REC_ENV_MISS;
  }
  nd->nidx[r] = idx + 1;
  if (nd->nidx[r] >= R_OUTPUT(nd, r)) {
    nd->flags[r] |= FB_REC_FINISHED;
    if (!(nd->flags[r] & 0x80000000u)) nd->flags[r] |= FB_REC_MET_TPOT;
    for (int64_t i = 0; i < nd->n_active; ++i) {
      if (nd->active[i] == r) {
        memmove(&nd->active[i], &nd->active[i + 1],
                sizeof(int32_t) * (size_t)(nd->n_active - i - 1));
        nd->n_active--;
        break;
      }
    }
  }
}

/* Node::complete_step, engine.cpp:204-254 */
static void orc_complete_step(orc_node* nd) {
  const int64_t t = nd->step_end;
  for (int64_t k = 0; k < nd->inflight.n_entries; ++k) {
    const int32_t r = (int32_t)nd->plan_e[k].request_id;
    const int32_t prompt = R_PROMPT(nd, r);
    if (nd->prefilled[r] < prompt) {
      nd->prefilled[r] += nd->plan_e[k].new_tokens;
      if (nd->prefilled[r] >= prompt) orc_emit(nd, r, t);
    } else {
      orc_emit(nd, r, t);
    }
  }
  nd->busy = 0;
}

/* run_node, engine.cpp:266-288 */
static int orc_run_one(const fb_trace* rows, const fb_instance* inst,
                       const fb_log_opts* log, fb_instance_result* res,
                       fb_record* rec, fb_log_counts* counts, fb_step_log* steps,
                       fb_plan_entry* entries, fb_reject_log* rejects) {
  const int64_t n = inst->n_req;
  const size_t nn = (size_t)(n > 0 ? n : 1);
  orc_node nd;
  memset(&nd, 0, sizeof(nd));
  nd.inst = inst;
  nd.rows = rows;
  nd.base = inst->trace_off;
  nd.prefilled = (int32_t*)calloc(nn, sizeof(int32_t));
  nd.nidx = (int32_t*)calloc(nn, sizeof(int32_t));
  nd.first = (int64_t*)malloc(nn * sizeof(int64_t));
  nd.seq = (int64_t*)calloc(nn, sizeof(int64_t));
  nd.maxtp = (double*)calloc(nn, sizeof(double));
  nd.maxtp_alt = (double*)calloc(nn, sizeof(double));
  nd.flags = (uint32_t*)calloc(nn, sizeof(uint32_t));
  nd.active = (int32_t*)malloc(nn * sizeof(int32_t));
  nd.waiting = (int32_t*)malloc(nn * sizeof(int32_t));
  nd.pend_row = (int32_t*)malloc(nn * sizeof(int32_t));
  nd.pend_vis = (int64_t*)malloc(nn * sizeof(int64_t));
  nd.views = (fb_task_view*)malloc(nn * sizeof(fb_task_view));
  nd.plan_e = (fb_plan_entry_id*)malloc(nn * sizeof(fb_plan_entry_id));
  for (int64_t i = 0; i < n; ++i) nd.first[i] = -1;
  memset(res, 0, sizeof(*res));
  res->plan_digest = FB_DIGEST_INIT;
  nd.res = res;
  nd.log = log;
  nd.counts = counts;
  nd.steps = steps;
  nd.entries = entries;
  nd.rejects = rejects;
  if (counts) memset(counts, 0, sizeof(*counts));

  int status = FB_OK;
  int64_t arr = 0, t = 0;
  const int64_t horizon = inst->horizon_us;
  for (;;) {
    const int64_t t_step = nd.busy ? nd.step_end : ORC_INF;
    const int64_t t_arr = arr < n ? R_ARR(&nd, arr) : ORC_INF;
    const int64_t tt = t_step < t_arr ? t_step : t_arr;
    if (tt == ORC_INF) break;
    if (!nd.busy && tt >= horizon) break;
    t = tt;
    if (nd.busy && t_step == t) orc_complete_step(&nd);
    while (arr < n && R_ARR(&nd, arr) == t) {
      orc_enqueue(&nd, (int32_t)arr, R_ARR(&nd, arr));
      ++arr;
    }
    if (!nd.busy && t < horizon) {
      status = orc_begin_step(&nd, t);
      if (status) break;
    }
  }
  res->steps = nd.step_counter;
  res->end_time_us = t;
  res->incomplete = (nd.busy || nd.pend_head < nd.pend_tail || nd.n_waiting > 0 ||
                     nd.n_active > 0 || arr < n) ? 1 : 0;
  res->status = status;
  for (int64_t i = 0; i < n; ++i) {
    rec[i].first_emit_us = nd.first[i];
    rec[i].max_tpot_ms = nd.maxtp[i];
    rec[i].max_tpot_alt_ms = nd.maxtp_alt[i];
    rec[i].tokens_emitted = nd.nidx[i];
    uint32_t f = nd.flags[i] & 0x7fffffffu;
    if ((f & FB_REC_REJECTED) && nd.nidx[i] > 0) f &= ~(uint32_t)FB_REC_REJECTED;
    rec[i].flags = f;
  }
  free(nd.prefilled); free(nd.nidx); free(nd.first); free(nd.seq);
  free(nd.maxtp); free(nd.maxtp_alt); free(nd.flags); free(nd.active);
  free(nd.waiting); free(nd.pend_row); free(nd.pend_vis); free(nd.views);
  free(nd.plan_e);
  return status;
}

typedef struct {
  const fb_trace* rows;
  const fb_instance* inst;
  int64_t n_inst;
  const fb_log_opts* log;
  fb_instance_result* results;
  fb_record* records;
  const int64_t* rec_off;
  fb_log_counts* counts;
  fb_step_log* steps;
  fb_plan_entry* entries;
  fb_reject_log* rejects;
  int64_t next;
  pthread_mutex_t mu;
} orc_pool;

static void* orc_worker(void* arg) {
  orc_pool* p = (orc_pool*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    const int64_t i = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (i >= p->n_inst) break;
    const int lg = p->log && (p->steps || p->entries || p->rejects);
    orc_run_one(p->rows, &p->inst[i], p->log, &p->results[i],
                p->records + p->rec_off[i], p->counts ? &p->counts[i] : NULL,
                lg && p->steps ? p->steps + i * p->log->step_cap : NULL,
                lg && p->entries ? p->entries + i * p->log->entry_cap : NULL,
                lg && p->rejects ? p->rejects + i * p->log->reject_cap : NULL);
  }
  return NULL;
}

int orc_run_instances(const fb_trace* rows, const fb_instance* inst,
                      int64_t n_inst, const fb_log_opts* log,
                      fb_instance_result* results, fb_record* records,
                      fb_log_counts* counts, fb_step_log* steps,
                      fb_plan_entry* entries, fb_reject_log* rejects,
                      int nthreads) {
  int64_t* rec_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_inst + 1));
  rec_off[0] = 0;
  for (int64_t i = 0; i < n_inst; ++i) {
    if (inst[i].trace_off < 0 || inst[i].n_req < 0 ||
        inst[i].trace_off + inst[i].n_req > rows->n_rows) {
      free(rec_off);
      return FB_ERR_VALIDATION;
    }
    rec_off[i + 1] = rec_off[i] + inst[i].n_req;
  }
  fb_log_counts dummy;
  (void)dummy;
  orc_pool p;
  p.rows = rows;
  p.inst = inst;
  p.n_inst = n_inst;
  p.log = log;
  p.results = results;
  p.records = records;
  p.rec_off = rec_off;
  p.counts = counts;
  p.steps = steps;
  p.entries = entries;
  p.rejects = rejects;
  p.next = 0;
  pthread_mutex_init(&p.mu, NULL);
  if (nthreads <= 1) {
    orc_worker(&p);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, orc_worker, &p);
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
    free(th);
  }
  pthread_mutex_destroy(&p.mu);
  free(rec_off);
  int st = FB_OK;
  for (int64_t i = 0; i < n_inst; ++i)
    if (results[i].status) st = results[i].status;
  return st;
}

/* ------------------------------------------------------------- cluster.cpp */

typedef struct {
  int has;
  int64_t t, pab, waiting, running, dec, inc;
} orc_nview; /* NodeView, cluster.h:55-69 */

typedef struct {
  int64_t deliver_at, node, emitted_at, pab, waiting, running;
} orc_delivery; /* MetricReport in flight, cluster.cpp:149-152 */

static void orc_node_alloc(orc_node* nd, const fb_instance* inst, const fb_trace* rows,
                           fb_instance_result* res) {
  const int64_t n = inst->n_req;
  const size_t nn = (size_t)(n > 0 ? n : 1);
  memset(nd, 0, sizeof(*nd));
  nd->inst = inst;
  nd->rows = rows;
  nd->base = inst->trace_off;
  nd->prefilled = (int32_t*)calloc(nn, sizeof(int32_t));
  nd->nidx = (int32_t*)calloc(nn, sizeof(int32_t));
  nd->first = (int64_t*)malloc(nn * sizeof(int64_t));
  nd->seq = (int64_t*)calloc(nn, sizeof(int64_t));
  nd->maxtp = (double*)calloc(nn, sizeof(double));
  nd->maxtp_alt = (double*)calloc(nn, sizeof(double));
  nd->flags = (uint32_t*)calloc(nn, sizeof(uint32_t));
  nd->active = (int32_t*)malloc(nn * sizeof(int32_t));
  nd->waiting = (int32_t*)malloc(nn * sizeof(int32_t));
  /* a rerouted request can reach the same node twice (retry_reroute) */
  nd->pend_row = (int32_t*)malloc(2 * nn * sizeof(int32_t));
  nd->pend_vis = (int64_t*)malloc(2 * nn * sizeof(int64_t));
  nd->views = (fb_task_view*)malloc(nn * sizeof(fb_task_view));
  nd->plan_e = (fb_plan_entry_id*)malloc(nn * sizeof(fb_plan_entry_id));
  for (int64_t i = 0; i < n; ++i) nd->first[i] = -1;
  memset(res, 0, sizeof(*res));
  res->plan_digest = FB_DIGEST_INIT;
  nd->res = res;
}

static void orc_node_free(orc_node* nd) {
  free(nd->prefilled); free(nd->nidx); free(nd->first); free(nd->seq);
  free(nd->maxtp); free(nd->maxtp_alt); free(nd->flags); free(nd->active);
  free(nd->waiting); free(nd->pend_row); free(nd->pend_vis); free(nd->views);
  free(nd->plan_e);
}

/* make_report, cluster.cpp:50-58 */
static orc_delivery orc_make_report(const orc_node* nd, int64_t node, int64_t now,
                                    int pab_lb, int64_t latency) {
  orc_delivery d;
  d.deliver_at = now + latency;
  d.node = node;
  d.emitted_at = now;
  d.waiting = nd->n_waiting;
  d.running = nd->n_active;
  d.pab = pab_lb ? orc_current_pab(nd, now) : 0;
  return d;
}

/* route, cluster.cpp:75-112 */
static int orc_route(orc_nview* v, int n, int64_t prompt, const fb_lb_config* lb) {
  int chosen = -1;
  if (lb->policy == FB_LB_PAB) {
    for (int i = 0; i < n; ++i) {
      const int64_t eff = v[i].pab - v[i].dec;
      if (eff < prompt) continue;
      if (chosen < 0 || eff > v[chosen].pab - v[chosen].dec) chosen = i;
    }
    if (chosen < 0)
      for (int i = 0; i < n; ++i)
        if (chosen < 0 || v[i].pab - v[i].dec > v[chosen].pab - v[chosen].dec) chosen = i;
    v[chosen].dec += prompt;
  } else {
    double best = 0.0;
    for (int i = 0; i < n; ++i) {
      const double score = lb->w_waiting * (double)(v[i].waiting + v[i].inc) +
                           lb->w_running * (double)v[i].running;
      if (chosen < 0 || score < best) {
        chosen = i;
        best = score;
      }
    }
    v[chosen].inc += 1;
  }
  return chosen;
}

/* run_cluster, cluster.cpp:134-251. */
int orc_run_cluster(const fb_trace* rows, const fb_engine_config* cfgs, int32_t n_nodes,
                    const fb_lb_config* lb, int64_t horizon, fb_instance_result* node_results,
                    fb_record* records, int32_t* route_node, int32_t* incomplete_out) {
  if (n_nodes < 1) return FB_ERR_USAGE;
  if (lb->report_latency_us < 0) return FB_ERR_VALIDATION;
  const int n = n_nodes;
  const int64_t nr = rows->n_rows;
  fb_instance* inst = (fb_instance*)calloc((size_t)n, sizeof(fb_instance));
  orc_node* nodes = (orc_node*)calloc((size_t)n, sizeof(orc_node));
  fb_instance_result* res = (fb_instance_result*)calloc((size_t)n, sizeof(fb_instance_result));
  orc_nview* view = (orc_nview*)calloc((size_t)n, sizeof(orc_nview));
  size_t dcap = 1024, dhead = 0, dtail = 0;
  orc_delivery* dq = (orc_delivery*)malloc(dcap * sizeof(orc_delivery));
  const int pab_lb = lb->policy == FB_LB_PAB;
  for (int i = 0; i < n; ++i) {
    inst[i].cfg = cfgs[i];
    inst[i].trace_off = 0;
    inst[i].n_req = nr;
    inst[i].horizon_us = horizon;
    orc_node_alloc(&nodes[i], &inst[i], rows, &res[i]);
  }
  int32_t* rt = (int32_t*)malloc(((size_t)nr + 1) * sizeof(int32_t)); /* last target */
  for (int64_t k = 0; k < nr; ++k) rt[k] = -1;
#define ORC_PUSH(d)                                                        \
  do {                                                                     \
    if (dtail == dcap) {                                                   \
      memmove(dq, dq + dhead, (dtail - dhead) * sizeof(orc_delivery));     \
      dtail -= dhead;                                                      \
      dhead = 0;                                                           \
      if (dtail == dcap) {                                                 \
        dcap *= 2;                                                         \
        dq = (orc_delivery*)realloc(dq, dcap * sizeof(orc_delivery));      \
      }                                                                    \
    }                                                                      \
    dq[dtail++] = (d);                                                     \
  } while (0)
  /* retry_reroute bookkeeping per request: bit 0 retried, bit 1 ever rejected */
  uint8_t* rstate = (uint8_t*)calloc((size_t)nr + 1, 1);
  for (int i = 0; i < n; ++i) ORC_PUSH(orc_make_report(&nodes[i], i, 0, pab_lb, lb->report_latency_us));
  int64_t arr = 0;
  int status = FB_OK;
  for (;;) {
    int64_t t = ORC_INF;
    for (int i = 0; i < n; ++i)
      if (nodes[i].busy && nodes[i].step_end < t) t = nodes[i].step_end;
    const int any_busy = t != ORC_INF;
    if (arr < nr && rows->arrival_us[arr] < t) t = rows->arrival_us[arr];
    if (dhead < dtail && dq[dhead].deliver_at < t) t = dq[dhead].deliver_at;
    if (t == ORC_INF) break;
    if (!any_busy && t >= horizon) break;
    for (int i = 0; i < n; ++i) { /* completions, then reports (cluster.cpp:195-205) */
      if (nodes[i].busy && nodes[i].step_end == t) {
        orc_complete_step(&nodes[i]);
        if (lb->report_interval_steps > 0 &&
            nodes[i].step_counter % (uint64_t)lb->report_interval_steps == 0)
          ORC_PUSH(orc_make_report(&nodes[i], i, t, pab_lb, lb->report_latency_us));
      }
    }
    while (dhead < dtail && dq[dhead].deliver_at <= t) { /* apply_report, cluster.cpp:60-73 */
      const orc_delivery* d = &dq[dhead++];
      orc_nview* v = &view[d->node];
      if (v->has && d->emitted_at < v->t) continue;
      v->has = 1;
      v->t = d->emitted_at;
      v->pab = d->pab;
      v->waiting = d->waiting;
      v->running = d->running;
      v->dec = 0;
      v->inc = 0;
    }
    while (arr < nr && rows->arrival_us[arr] == t) { /* route on arrival */
      const int target = orc_route(view, n, rows->prompt_len[arr], lb);
      rt[arr] = target;
      orc_enqueue(&nodes[target], (int32_t)arr, t);
      ++arr;
    }
    if (t < horizon) { /* begin_step, rejected requests rerouted once (cluster.cpp:222-237) */
      int progress = 1;
      while (progress && !status) {
        progress = 0;
        for (int i = 0; i < n && !status; ++i) {
          if (nodes[i].busy) continue;
          const int64_t h0 = nodes[i].pend_head, rej0 = nodes[i].res->n_rejected;
          status = orc_begin_step(&nodes[i], t);
          if (nodes[i].res->n_rejected == rej0) continue;
          /* drain_rejects: this pull's rejected rows in pull order; a stale flag
             can only sit on a row that was already retried */
          for (int64_t q = h0; q < nodes[i].pend_head; ++q) {
            const int32_t r = nodes[i].pend_row[q];
            if (!(nodes[i].flags[r] & FB_REC_REJECTED)) continue;
            const uint8_t was = rstate[r];
            rstate[r] |= 2;
            if (lb->retry_reroute && !(was & 1)) {
              rstate[r] |= 1;
              const int target = orc_route(view, n, rows->prompt_len[r], lb);
              rt[r] = target;
              orc_enqueue(&nodes[target], r, t);
              progress = 1;
            }
          }
        }
      }
    }
    if (status) break;
  }
#undef ORC_PUSH
  int live = arr < nr;
  for (int i = 0; i < n; ++i)
    live = live || nodes[i].busy || nodes[i].pend_head < nodes[i].pend_tail ||
           nodes[i].n_waiting > 0 || nodes[i].n_active > 0;
  for (int i = 0; i < n; ++i) {
    res[i].steps = nodes[i].step_counter;
    res[i].incomplete = live;
    res[i].status = status;
    res[i].end_time_us = -1;
    if (node_results) node_results[i] = res[i];
  }
  if (records) {
    for (int64_t k = 0; k < nr; ++k) {
      records[k].first_emit_us = -1;
      records[k].max_tpot_ms = 0.0;
      records[k].max_tpot_alt_ms = 0.0;
      records[k].tokens_emitted = 0;
      records[k].flags = 0;
    }
    for (int i = 0; i < n; ++i) {
      const orc_node* nd = &nodes[i];
      for (int64_t k = 0; k < nr; ++k) {
        if (!(nd->flags[k] & FB_REC_ARRIVED)) continue;
        /* a rerouted request: the record of the node it was routed to last */
        if (rt[k] != i) continue;
        records[k].first_emit_us = nd->first[k];
        records[k].max_tpot_ms = nd->maxtp[k];
        records[k].max_tpot_alt_ms = nd->maxtp_alt[k];
        records[k].tokens_emitted = nd->nidx[k];
        uint32_t f = nd->flags[k] & 0x7fffffffu;
        /* rejected only if never served anywhere (metrics.cpp:96-98) */
        if (rstate[k] & 2) f |= FB_REC_REJECTED;
        if ((f & FB_REC_REJECTED) && nd->nidx[k] > 0) f &= ~(uint32_t)FB_REC_REJECTED;
        records[k].flags = f;
      }
    }
  }
  if (route_node)
    for (int64_t k = 0; k < nr; ++k) route_node[k] = rt[k];
  if (incomplete_out) *incomplete_out = live;
  for (int i = 0; i < n; ++i) orc_node_free(&nodes[i]);
  free(nodes); free(inst); free(res); free(view); free(dq); free(rstate); free(rt);
  return status;
}

/* ---------------------------------------------------------------------------
 * The epoch decomposition of run_cluster for one rank of a node partition
 * (SURVEY §8e / P14), restated on the CPU so that the multi-rank protocol of
 * fb_cluster_shard_* can be exercised between processes (gloo) in the CPU
 * tests.  Per epoch e (distinct arrival time t_a):
 *   advance      -- local nodes: events before t_a, the completion (+report)
 *                   at t_a, then the newest report delivered by t_a;
 *   route_begin  -- all reports -> view (apply_report), route the arrivals at
 *                   t_a (route), enqueue to local nodes, begin_step(t_a).
 * Partition: fb_cluster_partition's contiguous ranges. */
struct orc_cluster_shard {
  const fb_trace* rows;
  fb_lb_config lb;
  int32_t n_nodes, rank, n_ranks, node_lo, n_local;
  int64_t horizon, nr, n_epochs, e_done, n_routed;
  int64_t* ep_t;
  int64_t* ep_lo;
  fb_instance* inst;
  orc_node* nodes;
  fb_instance_result* res;
  orc_nview* view;
  orc_delivery** fifo; /* per local node */
  int64_t* f_head;
  int64_t* f_tail;
  int64_t* f_cap;
  int* cmp;
  int32_t* route;
  int stopped, finished, status;
};

int orc_cluster_partition(int32_t n_nodes, int32_t n_ranks, int32_t rank, int32_t* lo,
                          int32_t* n_local) {
  if (n_nodes < 1 || n_ranks < 1 || rank < 0 || rank >= n_ranks || n_ranks > n_nodes)
    return FB_ERR_USAGE;
  const int64_t a = (int64_t)n_nodes * rank / n_ranks;
  const int64_t b = (int64_t)n_nodes * (rank + 1) / n_ranks;
  *lo = (int32_t)a;
  *n_local = (int32_t)(b - a);
  return FB_OK;
}

static void orc_shard_push(orc_cluster_shard* s, int i, orc_delivery d) {
  if (s->f_tail[i] == s->f_cap[i]) {
    s->f_cap[i] *= 2;
    s->fifo[i] = (orc_delivery*)realloc(s->fifo[i], (size_t)s->f_cap[i] * sizeof(orc_delivery));
  }
  s->fifo[i][s->f_tail[i]++] = d;
}

static void orc_shard_complete(orc_cluster_shard* s, int i, int report) {
  orc_node* nd = &s->nodes[i];
  const int64_t t = nd->step_end;
  orc_complete_step(nd);
  if (report && s->lb.report_interval_steps > 0 &&
      nd->step_counter % (uint64_t)s->lb.report_interval_steps == 0)
    orc_shard_push(s, i, orc_make_report(nd, s->node_lo + i, t, s->lb.policy == FB_LB_PAB,
                                         s->lb.report_latency_us));
}

int orc_cluster_shard_create(const fb_trace* rows, const fb_engine_config* cfgs, int32_t n_nodes,
                             const fb_lb_config* lb, int64_t horizon, int32_t rank,
                             int32_t n_ranks, orc_cluster_shard** out) {
  int32_t lo, nl;
  *out = NULL;
  if (lb->report_latency_us < 0) return FB_ERR_VALIDATION;
  if (lb->retry_reroute) return FB_ERR_USAGE;
  if (orc_cluster_partition(n_nodes, n_ranks, rank, &lo, &nl)) return FB_ERR_USAGE;
  orc_cluster_shard* s = (orc_cluster_shard*)calloc(1, sizeof(*s));
  const int64_t nr = rows->n_rows;
  s->rows = rows;
  s->lb = *lb;
  s->n_nodes = n_nodes;
  s->rank = rank;
  s->n_ranks = n_ranks;
  s->node_lo = lo;
  s->n_local = nl;
  s->horizon = horizon;
  s->nr = nr;
  s->ep_t = (int64_t*)malloc((size_t)(nr + 1) * sizeof(int64_t));
  s->ep_lo = (int64_t*)malloc((size_t)(nr + 2) * sizeof(int64_t));
  for (int64_t q = 0; q < nr; ++q) {
    if (q == 0 || rows->arrival_us[q] != rows->arrival_us[q - 1]) {
      s->ep_t[s->n_epochs] = rows->arrival_us[q];
      s->ep_lo[s->n_epochs++] = q;
    }
  }
  s->ep_lo[s->n_epochs] = nr;
  s->inst = (fb_instance*)calloc((size_t)nl + 1, sizeof(fb_instance));
  s->nodes = (orc_node*)calloc((size_t)nl + 1, sizeof(orc_node));
  s->res = (fb_instance_result*)calloc((size_t)nl + 1, sizeof(fb_instance_result));
  s->view = (orc_nview*)calloc((size_t)n_nodes, sizeof(orc_nview));
  s->fifo = (orc_delivery**)calloc((size_t)nl + 1, sizeof(orc_delivery*));
  s->f_head = (int64_t*)calloc((size_t)nl + 1, sizeof(int64_t));
  s->f_tail = (int64_t*)calloc((size_t)nl + 1, sizeof(int64_t));
  s->f_cap = (int64_t*)calloc((size_t)nl + 1, sizeof(int64_t));
  s->cmp = (int*)calloc((size_t)nl + 1, sizeof(int));
  s->route = (int32_t*)malloc((size_t)(nr + 1) * sizeof(int32_t));
  for (int64_t q = 0; q < nr; ++q) s->route[q] = -1;
  for (int i = 0; i < nl; ++i) {
    s->inst[i].cfg = cfgs[lo + i];
    s->inst[i].trace_off = 0;
    s->inst[i].n_req = nr;
    s->inst[i].horizon_us = horizon;
    orc_node_alloc(&s->nodes[i], &s->inst[i], rows, &s->res[i]);
    s->f_cap[i] = 64;
    s->fifo[i] = (orc_delivery*)malloc(64 * sizeof(orc_delivery));
    /* initial reports (cluster.cpp:198) */
    orc_shard_push(s, i, orc_make_report(&s->nodes[i], lo + i, 0, lb->policy == FB_LB_PAB,
                                         lb->report_latency_us));
  }
  *out = s;
  return FB_OK;
}

int64_t orc_cluster_shard_epochs(const orc_cluster_shard* s) { return s->n_epochs; }

int orc_cluster_shard_advance(orc_cluster_shard* s, int64_t e, fb_node_report* local) {
  if (e < 0 || e >= s->n_epochs || s->stopped || s->finished) return FB_ERR_USAGE;
  const int64_t t_a = s->ep_t[e];
  for (int i = 0; i < s->n_local; ++i) {
    orc_node* nd = &s->nodes[i];
    while (nd->busy && nd->step_end < t_a) {
      const int64_t t = nd->step_end;
      orc_shard_complete(s, i, 1);
      if (t < s->horizon && !s->status) s->status = orc_begin_step(nd, t);
    }
    fb_node_report r;
    r.busy = nd->busy;
    s->cmp[i] = nd->busy && nd->step_end == t_a;
    if (s->cmp[i]) orc_shard_complete(s, i, 1);
    r.emitted_at = -1;
    r.pab_tokens = 0;
    r.waiting = r.running = 0;
    r.fresh = 0;
    while (s->f_head[i] < s->f_tail[i] && s->fifo[i][s->f_head[i]].deliver_at <= t_a) {
      const orc_delivery* d = &s->fifo[i][s->f_head[i]++];
      r.emitted_at = d->emitted_at;
      r.pab_tokens = d->pab;
      r.waiting = (int32_t)d->waiting;
      r.running = (int32_t)d->running;
      r.fresh = 1;
    }
    local[i] = r;
  }
  return s->status;
}

int orc_cluster_shard_route_begin(orc_cluster_shard* s, int64_t e, const fb_node_report* all,
                                  int32_t* stopped) {
  if (e < 0 || e >= s->n_epochs || s->stopped || s->finished) return FB_ERR_USAGE;
  const int64_t t_a = s->ep_t[e];
  int any_busy = 0;
  for (int i = 0; i < s->n_nodes; ++i) any_busy |= all[i].busy != 0;
  if (t_a >= s->horizon && !any_busy) { /* cluster.cpp:191-192 */
    s->stopped = 1;
    *stopped = 1;
    return FB_OK;
  }
  *stopped = 0;
  for (int i = 0; i < s->n_nodes; ++i) { /* apply_report, cluster.cpp:60-73 */
    orc_nview* v = &s->view[i];
    if (!all[i].fresh || (v->has && all[i].emitted_at < v->t)) continue;
    v->has = 1;
    v->t = all[i].emitted_at;
    v->pab = all[i].pab_tokens;
    v->waiting = all[i].waiting;
    v->running = all[i].running;
    v->dec = 0;
    v->inc = 0;
  }
  for (int64_t q = s->ep_lo[e]; q < s->ep_lo[e + 1]; ++q) {
    const int target = orc_route(s->view, s->n_nodes, s->rows->prompt_len[q], &s->lb);
    s->route[q] = target;
    if (target >= s->node_lo && target < s->node_lo + s->n_local)
      orc_enqueue(&s->nodes[target - s->node_lo], (int32_t)q, t_a);
  }
  s->n_routed = s->ep_lo[e + 1];
  if (t_a < s->horizon)
    for (int i = 0; i < s->n_local && !s->status; ++i)
      if (!s->nodes[i].busy) s->status = orc_begin_step(&s->nodes[i], t_a);
  s->e_done = e + 1;
  return s->status;
}

int orc_cluster_shard_fetch(orc_cluster_shard* s, fb_instance_result* local_results,
                            fb_record* records, int32_t* route_node, int64_t* n_routed,
                            int32_t* incomplete) {
  const int64_t nr = s->nr;
  if (!s->finished) { /* run every local node to quiescence */
    for (int i = 0; i < s->n_local && !s->status; ++i)
      while (s->nodes[i].busy && !s->status) {
        const int64_t t = s->nodes[i].step_end;
        orc_shard_complete(s, i, 0);
        if (t < s->horizon) s->status = orc_begin_step(&s->nodes[i], t);
      }
    s->finished = 1;
  }
  int live = s->n_routed < nr;
  for (int i = 0; i < s->n_local; ++i) {
    const orc_node* nd = &s->nodes[i];
    live = live || nd->busy || nd->pend_head < nd->pend_tail || nd->n_waiting > 0 ||
           nd->n_active > 0;
  }
  for (int i = 0; i < s->n_local; ++i) {
    s->res[i].steps = s->nodes[i].step_counter;
    s->res[i].incomplete = live;
    s->res[i].status = s->status;
    s->res[i].end_time_us = -1;
    if (local_results) local_results[i] = s->res[i];
  }
  if (route_node)
    for (int64_t q = 0; q < nr; ++q) route_node[q] = s->route[q];
  if (n_routed) *n_routed = s->n_routed;
  if (incomplete) *incomplete = live;
  if (records) {
    for (int64_t k = 0; k < nr; ++k) {
      fb_record* o = &records[k];
      const int node = s->route[k] - s->node_lo;
      o->first_emit_us = -1;
      o->max_tpot_ms = 0.0;
      o->max_tpot_alt_ms = 0.0;
      o->tokens_emitted = 0;
      o->flags = 0;
      if (s->route[k] < 0 || node < 0 || node >= s->n_local) continue;
      const orc_node* nd = &s->nodes[node];
      if (!(nd->flags[k] & FB_REC_ARRIVED)) continue;
      o->first_emit_us = nd->first[k];
      o->max_tpot_ms = nd->maxtp[k];
      o->max_tpot_alt_ms = nd->maxtp_alt[k];
      o->tokens_emitted = nd->nidx[k];
      uint32_t f = nd->flags[k] & 0x7fffffffu;
      if ((f & FB_REC_REJECTED) && nd->nidx[k] > 0) f &= ~(uint32_t)FB_REC_REJECTED;
      o->flags = f;
    }
  }
  return s->status;
}

void orc_cluster_shard_destroy(orc_cluster_shard* s) {
  if (!s) return;
  for (int i = 0; i < s->n_local; ++i) {
    orc_node_free(&s->nodes[i]);
    free(s->fifo[i]);
  }
  free(s->ep_t); free(s->ep_lo); free(s->inst); free(s->nodes); free(s->res); free(s->view);
  free(s->fifo); free(s->f_head); free(s->f_tail); free(s->f_cap); free(s->cmp); free(s->route);
  free(s);
}
