/*
 * fsb_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference Fish School Behaviour step
 * (/root/reference/proj/include/fsb/sim.hpp, fsb/rng.hpp) used as the parity
 * checker for the CUDA engine.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / reference legs of bench.py may load it.  The product path
 * (paper_2507_20173_b200/) never links, loads or calls anything in oracle/.
 *
 * Pinned against the reference itself: tests/golden/ holds vectors produced by
 * oracle/_ref/libfsbref.so (the reference headers compiled unmodified, see
 * oracle/Makefile) and tests/test_oracle.py checks this restatement against
 * them bit-for-bit.
 */
#ifndef FSB_ORACLE_H
#define FSB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Byte layout of fsb::Fish (sim.hpp:26-32): 5 x fp64, 40 bytes. */
typedef struct oracle_fish {
    double x;
    double y;
    double weight;
    double prev_objective;
    double current_objective;
} oracle_fish;

/* Fields of fsb::SimConfig (sim.hpp:34-50). */
typedef struct oracle_config {
    uint64_t num_fish;
    double pond_size;
    double weight_scale;
    uint64_t num_steps;
    uint64_t seed;
    double step_base;
} oracle_config;

uint64_t oracle_mix64(uint64_t z);                           /* rng.hpp:13-20 */
uint64_t oracle_fold_in(uint64_t h, uint64_t word);          /* rng.hpp:22-24 */
uint64_t oracle_bits(uint64_t seed, uint64_t fish, uint64_t step, uint64_t lane); /* rng.hpp:34-36 */
double oracle_unit(uint64_t seed, uint64_t fish, uint64_t step, uint64_t lane);   /* rng.hpp:39-41 */
double oracle_objective(double x, double y, double pond_size);                    /* sim.hpp:59-63 */

/* 0 if valid, else 1 (pond), 2 (weight_scale), 3 (step_base); sim.hpp:44-49 */
int oracle_validate(const oracle_config* cfg);

/* init_school (sim.hpp:65-79) for global fish indices [first, first+n). */
void oracle_init(const oracle_config* cfg, uint64_t first, uint64_t n, oracle_fish* out);

/* move_phase body (sim.hpp:84-99) for global indices [first, first+n). */
void oracle_move(const oracle_config* cfg, uint64_t step, uint64_t first, uint64_t n,
                 oracle_fish* fish);

/* eat_phase max (sim.hpp:112-114 with the inline fold executor.hpp:86-92). */
double oracle_eat_max(const oracle_fish* fish, uint64_t n);

/* eat_phase weight update (sim.hpp:115-121) given the global max. */
void oracle_eat_apply(const oracle_config* cfg, double max_diff, oracle_fish* fish, uint64_t n);

/* eat_phase = max + update; returns max_diff. */
double oracle_eat(const oracle_config* cfg, oracle_fish* fish, uint64_t n);

/* simulate (sim.hpp:133-147) with the sequential construct: init + T x (move, eat).
 * fish_out holds num_fish entries, trace num_steps entries (either may be NULL
 * only if num_fish/num_steps is 0). */
void oracle_simulate(const oracle_config* cfg, oracle_fish* fish_out, double* trace);

/* Continue a simulation from `fish` for steps [first_step, first_step+num_steps). */
void oracle_run(const oracle_config* cfg, oracle_fish* fish, uint64_t n, uint64_t first_step,
                uint64_t num_steps, double* trace);

/* Replay fish i alone for num_steps steps given a run's max_diff trace. */
void oracle_replay_fish(const oracle_config* cfg, uint64_t i, const double* trace, uint64_t num_steps,
                        oracle_fish* out);

/* The same for count fish given by global index (out[k] = fish idx[k]). */
void oracle_replay_many(const oracle_config* cfg, const uint64_t* idx, uint64_t count, const double* trace,
                        uint64_t num_steps, oracle_fish* out);

/* checksum (sim.hpp:154-176): FNV-1a 64 over the LE bytes of every field. */
uint64_t oracle_checksum(const oracle_fish* fish, uint64_t n);
/* Streamed form: continue hash h over more fish (h0 = 0xcbf29ce484222325). */
uint64_t oracle_checksum_update(uint64_t h, const oracle_fish* fish, uint64_t n);

/* New query (no reference counterpart): Neumaier-compensated
 * sums out[0]=sum x*f, out[1]=sum y*f, out[2]=sum f with f=current_objective.
 * Products are rounded fp64 products, as the device computes them. */
void oracle_barycentre_sums(const oracle_fish* fish, uint64_t n, double out[3]);

#ifdef __cplusplus
}
#endif

#endif
