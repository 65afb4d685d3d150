// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/fsb/sim.hpp and parfor/executor.hpp), compiled
// by oracle/Makefile with the reference's own Release flags
// (-O3 -DNDEBUG -std=gnu++20, no -march => no FMA; proj/CMakeLists.txt:3,8-10)
// into oracle/_ref/libfsbref.so.  No reference source is copied: the headers
// are included from where they lie (REF_INCLUDE).  Used to
//   * generate tests/golden/ fixtures (the reference's own outputs), and
//   * time the reference CPU path (bench.py --impl reference, cpu_baseline).
#include <cstring>
#include <exception>
#include <stdexcept>

#include "fsb/csv.hpp"
#include "fsb/sim.hpp"

namespace {

struct ref_config {  // same layout as oracle_config / fsb_sim_config
    std::uint64_t num_fish;
    double pond_size;
    double weight_scale;
    std::uint64_t num_steps;
    std::uint64_t seed;
    double step_base;
};

fsb::SimConfig to_sim(const ref_config* c) {
    fsb::SimConfig s;
    s.num_fish = c->num_fish;
    s.pond_size = c->pond_size;
    s.weight_scale = c->weight_scale;
    s.num_steps = c->num_steps;
    s.seed = c->seed;
    s.step_base = c->step_base;
    return s;
}

parfor::RunConfig to_run(int threads, int sched_kind, std::uint64_t chunk, int construct) {
    parfor::RunConfig r;
    r.num_threads = threads;
    r.schedule = parfor::ScheduleSpec{static_cast<parfor::ScheduleKind>(sched_kind), chunk};
    r.construct = static_cast<parfor::Construct>(construct);
    return r;
}

fsb::School to_school(const void* fish, std::uint64_t n) {
    fsb::School s;
    s.fishes.resize(n);
    if (n) std::memcpy(s.fishes.data(), fish, n * sizeof(fsb::Fish));
    return s;
}

void from_school(const fsb::School& s, void* fish) {
    if (s.size()) std::memcpy(fish, s.fishes.data(), s.size() * sizeof(fsb::Fish));
}

}  // namespace

static_assert(sizeof(fsb::Fish) == 40, "reference Fish layout changed");

extern "C" {

int ref_validate(const ref_config* cfg) {
    try {
        to_sim(cfg).validate();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

double ref_objective(double x, double y, double pond) { return fsb::objective(x, y, pond); }

std::uint64_t ref_bits(std::uint64_t seed, std::uint64_t fish, std::uint64_t step, std::uint64_t lane) {
    return fsb::RngStream{seed, fish, step}.bits(lane);
}

int ref_init(const ref_config* cfg, void* fish_out) {
    try {
        from_school(fsb::init_school(to_sim(cfg)), fish_out);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

double ref_move(const ref_config* cfg, std::uint64_t step, void* fish, std::uint64_t n, int threads,
                int sched_kind, std::uint64_t chunk, int construct) {
    fsb::School s = to_school(fish, n);
    parfor::Executor exec(to_run(threads, sched_kind, chunk, construct));
    const double secs = fsb::move_phase(s, to_sim(cfg), step, exec);
    from_school(s, fish);
    return secs;
}

double ref_eat(const ref_config* cfg, void* fish, std::uint64_t n, int threads, int sched_kind,
               std::uint64_t chunk, int construct) {
    fsb::School s = to_school(fish, n);
    parfor::Executor exec(to_run(threads, sched_kind, chunk, construct));
    const fsb::EatResult r = fsb::eat_phase(s, to_sim(cfg), exec);
    from_school(s, fish);
    return r.max_diff;
}

// simulate(cfg, run) (sim.hpp:149-152). seconds[0..2] = total, move, eat.
int ref_simulate(const ref_config* cfg, int threads, int sched_kind, std::uint64_t chunk,
                 int construct, void* fish_out, double* trace, double* seconds) {
    try {
        const fsb::SimResult r =
            fsb::simulate(to_sim(cfg), to_run(threads, sched_kind, chunk, construct));
        from_school(r.school, fish_out);
        if (trace && !r.max_diff_trace.empty())
            std::memcpy(trace, r.max_diff_trace.data(), r.max_diff_trace.size() * sizeof(double));
        if (seconds) {
            seconds[0] = r.seconds_total;
            seconds[1] = r.seconds_move;
            seconds[2] = r.seconds_eat;
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

std::uint64_t ref_checksum(const void* fish, std::uint64_t n) {
    return fsb::checksum(to_school(fish, n));
}

// The reference step loop (sequential construct) with checksum(school) taken
// after every `every`-th step in place: digests[k] after step (k+1)*every - 1.
int ref_step_digests(const ref_config* cfg, std::uint64_t every, std::uint64_t* digests, double* trace) {
    try {
        const fsb::SimConfig sim = to_sim(cfg);
        parfor::Executor exec(to_run(1, 0, 0, 0));
        fsb::School school = fsb::init_school(sim);
        for (std::size_t step = 0; step < sim.num_steps; ++step) {
            fsb::move_phase(school, sim, step, exec);
            const double m = fsb::eat_phase(school, sim, exec).max_diff;
            if (trace) trace[step] = m;
            if ((step + 1) % every == 0) digests[(step + 1) / every - 1] = fsb::checksum(school);
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// The reference's own CSV reader (csv.hpp:114-145) and validator (:161-179)
// applied to a results text: returns the record count (or -1 on a CsvError,
// message in err) and the number of validate_records diagnostics in *issues.
int ref_read_csv(const char* text, int* issues, char* err, int errlen) {
    try {
        const std::vector<fsb::BenchRecord> recs = fsb::read_csv_string(text);
        if (issues) *issues = static_cast<int>(fsb::validate_records(recs).size());
        return static_cast<int>(recs.size());
    } catch (const std::exception& e) {
        if (err && errlen > 0) {
            std::strncpy(err, e.what(), static_cast<std::size_t>(errlen - 1));
            err[errlen - 1] = 0;
        }
        return -1;
    }
}

// simulate() for schools too large to copy out (C3: 1e9 fish = 40 GB): returns
// checksum(init_school) and checksum(final school), the trace, and the final
// school's f-weighted sums with long-double accumulation (golden generation).
int ref_simulate_digest(const ref_config* cfg, std::uint64_t* init_checksum,
                        std::uint64_t* final_checksum, double* trace, long double* bary) {
    try {
        const fsb::SimConfig sim = to_sim(cfg);
        parfor::Executor exec(to_run(1, 0, 0, 0));  // sequential construct: the oracle
        fsb::School school = fsb::init_school(sim);
        *init_checksum = fsb::checksum(school);
        for (std::size_t step = 0; step < sim.num_steps; ++step) {
            fsb::move_phase(school, sim, step, exec);
            trace[step] = fsb::eat_phase(school, sim, exec).max_diff;
        }
        *final_checksum = fsb::checksum(school);
        long double s[3] = {0, 0, 0}, c[3] = {0, 0, 0};  // Neumaier in long double
        auto add = [&](int k, long double v) {
            const long double t = s[k] + v;
            c[k] += (fabsl(s[k]) >= fabsl(v)) ? (s[k] - t) + v : (v - t) + s[k];
            s[k] = t;
        };
        for (const fsb::Fish& f : school.fishes) {
            add(0, static_cast<long double>(f.x * f.current_objective));
            add(1, static_cast<long double>(f.y * f.current_objective));
            add(2, static_cast<long double>(f.current_objective));
        }
        for (int k = 0; k < 3; ++k) bary[k] = s[k] + c[k];
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// The reference's step loop (sim.hpp:139-144) timed with steady_clock, after
// init_school and `warmup` untimed steps: returns the seconds of `steps`
// timed steps.  per_step (optional) receives each timed step's seconds and
// trace (optional) the max_diff of every timed step.
double ref_time_steps(const ref_config* cfg, int threads, int sched_kind, std::uint64_t chunk,
                      int construct, std::uint64_t warmup, std::uint64_t steps, double* per_step,
                      double* trace) {
    const fsb::SimConfig sim = to_sim(cfg);
    parfor::Executor exec(to_run(threads, sched_kind, chunk, construct));
    fsb::School school = fsb::init_school(sim);
    std::uint64_t step = 0;
    for (; step < warmup; ++step) {
        fsb::move_phase(school, sim, step, exec);
        fsb::eat_phase(school, sim, exec);
    }
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    for (std::uint64_t k = 0; k < steps; ++k, ++step) {
        const auto a = clock::now();
        fsb::move_phase(school, sim, step, exec);
        const fsb::EatResult r = fsb::eat_phase(school, sim, exec);
        if (trace) trace[k] = r.max_diff;
        if (per_step) per_step[k] = std::chrono::duration<double>(clock::now() - a).count();
    }
    return std::chrono::duration<double>(clock::now() - t0).count();
}

}  // extern "C"
