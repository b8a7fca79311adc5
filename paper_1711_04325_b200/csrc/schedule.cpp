// Host schedule of arXiv 1711.04325: slow-start LR (Appendix A.2)
// and the RMSprop-warm-up blend (Appendix A.1).
//
// IEEE double, in the operation order documented in include/lmsgd.h
// (lmsgd_schedule_at).  Readings: R1 linear-branch slope 1/beta_period (the "2" at
// PAPER.md:180 contradicts PAPER.md:186-188); R2/R3 fractional start-of-step epoch;
// R4 right-open phases decided with integer arithmetic.
#include <cmath>
#include <cstdint>

#include "lmsgd.h"

namespace {

struct Phase {
    int64_t end_epoch;  // exclusive
    double mult;        // multiple of eta_base
};

// 0.5 for the first 40 epochs, 0.075 next 30, 0.01 following 15,
// 0.001 last 5.
constexpr Phase kSlowStart[4] = {{40, 0.5}, {70, 0.075}, {85, 0.01}, {90, 0.001}};
// PAPER.md:222 (Goyal et al.): 1, 0.1, 0.01, 0.001 for 30 / 30 / 20 / 10 epochs.
constexpr Phase kGoyal[4] = {{30, 1.0}, {60, 0.1}, {80, 0.01}, {90, 0.001}};

const Phase* phases_of(int32_t schedule) {
    if (schedule == 0) return kSlowStart;
    if (schedule == 1) return kGoyal;
    return nullptr;
}

bool cluster_ok(const lmsgd_cluster* c) {
    // keep (t-1) * b_total and 90 * n_train well inside int64 and exact in double
    return c && c->n_workers > 0 && c->b_local > 0 && c->n_train > 0 &&
           c->n_workers <= (int64_t(1) << 24) && c->b_local <= (int64_t(1) << 24) &&
           c->n_train <= (int64_t(1) << 40) && phases_of(c->schedule) != nullptr &&
           c->transition >= LMSGD_TRANSITION_ELU && c->transition <= LMSGD_TRANSITION_SUDDEN;
}

// PAPER.md:178-182 with R1; the alternatives of PAPER.md:205-210 with R20.
double alpha_sgd(double epoch, double bc, double bp, int32_t transition) {
    switch (transition) {
    case LMSGD_TRANSITION_LINEAR:
        return std::fmin(std::fmax(0.5 + (epoch - bc) / bp, 0.0), 1.0);
    case LMSGD_TRANSITION_SIGMOID:
        return 1.0 / (1.0 + std::exp(-4.0 * (epoch - bc) / bp));
    case LMSGD_TRANSITION_SUDDEN:
        return epoch < bc ? 0.0 : 1.0;
    default:
        if (epoch < bc) return 0.5 * std::exp(2.0 * (epoch - bc) / bp);
        if (epoch < bc + 0.5 * bp) return 0.5 + (epoch - bc) / bp;
        return 1.0;
    }
}

}  // namespace

extern "C" lmsgd_status lmsgd_hyper_default(lmsgd_hyper* out) {
    if (!out) return LMSGD_ERR_INVALID_ARG;
    out->mu1 = 0.9;
    out->mu2 = 0.99;
    out->eps = 1e-8;
    out->eta_rmsprop = 0.0003;
    out->beta_center = 10.0;
    out->beta_period = 5.0;
    return LMSGD_OK;
}

extern "C" lmsgd_status lmsgd_schedule_steps(const lmsgd_cluster* c, int64_t* T) {
    if (!cluster_ok(c) || !T) return LMSGD_ERR_INVALID_ARG;
    const int64_t b_total = c->n_workers * c->b_local;
    const int64_t total = phases_of(c->schedule)[3].end_epoch * c->n_train;
    *T = (total + b_total - 1) / b_total;
    return LMSGD_OK;
}

extern "C" lmsgd_status lmsgd_schedule_at(const lmsgd_hyper* h, const lmsgd_cluster* c, int64_t t,
                                          lmsgd_coeffs* out) {
    if (!h || !out || !cluster_ok(c) || t < 1 || !(h->beta_period > 0.0) ||
        !(h->eta_rmsprop >= 0.0))
        return LMSGD_ERR_INVALID_ARG;
    const Phase* ph = phases_of(c->schedule);
    const int64_t b_total = c->n_workers * c->b_local;
    if (t - 1 > (int64_t(1) << 40) / b_total) return LMSGD_ERR_RANGE;
    const int64_t num = (t - 1) * b_total;  // images seen before step t
    int p = 0;
    while (p < 4 && !(num < ph[p].end_epoch * c->n_train)) ++p;
    if (p == 4) return LMSGD_ERR_RANGE;
    const double epoch = static_cast<double>(num) / static_cast<double>(c->n_train);
    const double eta_base = 0.1 * static_cast<double>(b_total) / 256.0;
    const double eta = ph[p].mult * eta_base;
    if (!(eta > 0.0)) return LMSGD_ERR_INVALID_ARG;
    const double a = alpha_sgd(epoch, h->beta_center, h->beta_period, c->transition);
    out->epoch = epoch;
    out->eta = eta;
    out->alpha_sgd = a;
    out->alpha_rmsprop = ((1.0 - a) * h->eta_rmsprop) / eta;
    out->phase = p;
    out->reserved = 0;
    return LMSGD_OK;
}
