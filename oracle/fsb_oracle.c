/*
 * fsb_oracle.c -- TEST INFRASTRUCTURE ONLY (see fsb_oracle.h).
 *
 * Plain-C restatement of the reference FSB algorithm.  Every function cites
 * the reference line it follows.  Compile WITHOUT floating-point contraction
 * (-ffp-contract=off, no -march=native): the reference's own Release flags
 * (proj/CMakeLists.txt:3,8-10) produce no FMA, and an FMA-contracted build of
 * the reference gives different digests (SURVEY.md finding 3).
 */
#include "fsb_oracle.h"

#include <math.h>
#include <string.h>

/* rng.hpp:13-20 -- splitmix64 finaliser. */
uint64_t oracle_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

/* rng.hpp:22-24 */
uint64_t oracle_fold_in(uint64_t h, uint64_t word) {
    return oracle_mix64(h ^ (word + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2)));
}

/* rng.hpp:34-36 -- RngStream::bits */
uint64_t oracle_bits(uint64_t seed, uint64_t fish, uint64_t step, uint64_t lane) {
    return oracle_fold_in(oracle_fold_in(oracle_fold_in(seed, fish), step), lane);
}

/* rng.hpp:39-41 -- RngStream::unit: 53-bit uniform in [0,1). */
double oracle_unit(uint64_t seed, uint64_t fish, uint64_t step, uint64_t lane) {
    return (double)(oracle_bits(seed, fish, step, lane) >> 11) * 0x1.0p-53;
}

/* rng.hpp:44-46 -- RngStream::uniform: lo + unit*(hi-lo), multiply then add. */
static double uniform_from_unit(double u, double lo, double hi) { return lo + u * (hi - lo); }

/* libstdc++ std::max / std::min / std::clamp comparison order (stl_algobase.h,
 * stl_algo.h): max(a,b) = (a<b)?b:a, min(a,b) = (b<a)?b:a,
 * clamp(v,lo,hi) = min(max(v,lo),hi). */
static double ref_max(double a, double b) { return (a < b) ? b : a; }
static double ref_min(double a, double b) { return (b < a) ? b : a; }
static double ref_clamp(double v, double lo, double hi) { return ref_min(ref_max(v, lo), hi); }

/* sim.hpp:59-63 */
double oracle_objective(double x, double y, double pond_size) {
    const double dx = x - pond_size / 2.0;
    const double dy = y - pond_size / 2.0;
    return sqrt(dx * dx + dy * dy);
}

/* sim.hpp:44-49 -- SimConfig::validate; kWeightMin = 1.0 (sim.hpp:24). */
int oracle_validate(const oracle_config* cfg) {
    if (!(cfg->pond_size > 0.0)) return 1;
    if (!(cfg->weight_scale >= 1.0)) return 2;
    if (!(cfg->step_base > 0.0)) return 3;
    return 0;
}

/* sim.hpp:65-79 -- init_school; kInitStep = ~0 (rng.hpp:27). */
void oracle_init(const oracle_config* cfg, uint64_t first, uint64_t n, oracle_fish* out) {
    const uint64_t init_step = ~0ull;
    for (uint64_t k = 0; k < n; ++k) {
        const uint64_t i = first + k;
        oracle_fish* f = &out[k];
        f->x = uniform_from_unit(oracle_unit(cfg->seed, i, init_step, 0), 0.0, cfg->pond_size);
        f->y = uniform_from_unit(oracle_unit(cfg->seed, i, init_step, 1), 0.0, cfg->pond_size);
        f->weight = uniform_from_unit(oracle_unit(cfg->seed, i, init_step, 2), 1.0, cfg->weight_scale);
        f->current_objective = oracle_objective(f->x, f->y, cfg->pond_size);
        f->prev_objective = f->current_objective;
    }
}

/* sim.hpp:84-99 -- move_phase loop body. */
void oracle_move(const oracle_config* cfg, uint64_t step, uint64_t first, uint64_t n,
                 oracle_fish* fish) {
    const double pond = cfg->pond_size;
    for (uint64_t k = 0; k < n; ++k) {
        const uint64_t i = first + k;
        oracle_fish* f = &fish[k];
        const double s = cfg->step_base / ref_max(1.0, f->weight);
        const double u0 = oracle_unit(cfg->seed, i, step, 0);
        const double u1 = oracle_unit(cfg->seed, i, step, 1);
        f->x = ref_clamp(f->x + uniform_from_unit(u0, -s, s), 0.0, pond);
        f->y = ref_clamp(f->y + uniform_from_unit(u1, -s, s), 0.0, pond);
        f->prev_objective = f->current_objective;
        f->current_objective = oracle_objective(f->x, f->y, pond);
    }
}

/* sim.hpp:112-114 folded as executor.hpp:86-92 (empty pool): identity -inf,
 * strict '>' update. */
double oracle_eat_max(const oracle_fish* fish, uint64_t n) {
    double best = -INFINITY;
    for (uint64_t i = 0; i < n; ++i) {
        const double v = fish[i].prev_objective - fish[i].current_objective;
        if (v > best) best = v;
    }
    return best;
}

/* sim.hpp:115-121 -- sequential weight update. */
void oracle_eat_apply(const oracle_config* cfg, double max_diff, oracle_fish* fish, uint64_t n) {
    if (max_diff > 0.0) {
        const double w_max = 2.0 * cfg->weight_scale; /* SimConfig::weight_max, sim.hpp:42 */
        for (uint64_t i = 0; i < n; ++i) {
            const double diff = fish[i].prev_objective - fish[i].current_objective;
            fish[i].weight = ref_clamp(fish[i].weight + diff / max_diff, 1.0, w_max);
        }
    }
}

/* sim.hpp:110-123 */
double oracle_eat(const oracle_config* cfg, oracle_fish* fish, uint64_t n) {
    const double m = oracle_eat_max(fish, n);
    oracle_eat_apply(cfg, m, fish, n);
    return m;
}

/* sim.hpp:139-144 -- the step loop. */
void oracle_run(const oracle_config* cfg, oracle_fish* fish, uint64_t n, uint64_t first_step,
                uint64_t num_steps, double* trace) {
    for (uint64_t t = 0; t < num_steps; ++t) {
        oracle_move(cfg, first_step + t, 0, n, fish);
        const double m = oracle_eat(cfg, fish, n);
        if (trace) trace[t] = m;
    }
}

/* Sampled-fish replay (SURVEY.md 8(d) verification for schools without a
 * whole-run oracle): fish i's trajectory depends only on its own state and
 * the global max_diff sequence, so given the trace of a run it can be
 * replayed alone: init (sim.hpp:65-79), then per step move (sim.hpp:84-99)
 * and the weight update with trace[t] (sim.hpp:115-121). */
void oracle_replay_fish(const oracle_config* cfg, uint64_t i, const double* trace, uint64_t num_steps,
                        oracle_fish* out) {
    oracle_init(cfg, i, 1, out);
    for (uint64_t t = 0; t < num_steps; ++t) {
        oracle_move(cfg, t, i, 1, out);
        oracle_eat_apply(cfg, trace[t], out, 1);
    }
}

void oracle_replay_many(const oracle_config* cfg, const uint64_t* idx, uint64_t count, const double* trace,
                        uint64_t num_steps, oracle_fish* out) {
    for (uint64_t k = 0; k < count; ++k) oracle_replay_fish(cfg, idx[k], trace, num_steps, out + k);
}

/* sim.hpp:133-147 */
void oracle_simulate(const oracle_config* cfg, oracle_fish* fish_out, double* trace) {
    oracle_init(cfg, 0, cfg->num_fish, fish_out);
    oracle_run(cfg, fish_out, cfg->num_fish, 0, cfg->num_steps, trace);
}

/* sim.hpp:158-176 -- FNV-1a over the LE bytes of x, y, weight, prev, cur. */
uint64_t oracle_checksum_update(uint64_t h, const oracle_fish* fish, uint64_t n) {
    const unsigned char* p = (const unsigned char*)fish;
    const uint64_t bytes = n * (uint64_t)sizeof(oracle_fish);
    for (uint64_t k = 0; k < bytes; ++k) {
        h ^= p[k];
        h *= 0x100000001b3ull;
    }
    return h;
}

uint64_t oracle_checksum(const oracle_fish* fish, uint64_t n) {
    return oracle_checksum_update(0xcbf29ce484222325ull, fish, n); /* kChecksumEmpty :156 */
}

/* Neumaier (improved Kahan-Babuska) summation step. */
static void neumaier_add(double* sum, double* comp, double v) {
    const double t = *sum + v;
    if (fabs(*sum) >= fabs(v)) *comp += (*sum - t) + v;
    else *comp += (v - t) + *sum;
    *sum = t;
}

/* New query: f-weighted barycentre sums (north_star), no reference line. */
void oracle_barycentre_sums(const oracle_fish* fish, uint64_t n, double out[3]) {
    double s[3] = {0.0, 0.0, 0.0};
    double c[3] = {0.0, 0.0, 0.0};
    for (uint64_t i = 0; i < n; ++i) {
        const double f = fish[i].current_objective;
        neumaier_add(&s[0], &c[0], fish[i].x * f);
        neumaier_add(&s[1], &c[1], fish[i].y * f);
        neumaier_add(&s[2], &c[2], f);
    }
    for (int k = 0; k < 3; ++k) out[k] = s[k] + c[k];
}
