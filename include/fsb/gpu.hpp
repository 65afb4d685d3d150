#pragma once

// fsb/gpu.hpp -- header-only C++ drop-in for the reference simulation API
// (/root/reference/proj/include/fsb/sim.hpp) on top of the C-ABI in
// fsb_b200.h.  Callers keep their code and swap the executor argument:
//
//     parfor::Executor exec(run);            fsb::gpu::Executor exec;        // device 0
//     fsb::move_phase(school, cfg, t, exec)  fsb::gpu::move_phase(school, cfg, t, exec)
//     fsb::simulate(cfg, exec)               fsb::gpu::simulate(cfg, exec)
//
// Types.  By default this header defines layout-identical copies of Fish,
// SimConfig, School, EatResult and SimResult in namespace fsb::gpu.  If the
// reference's fsb/sim.hpp is included first and FSB_GPU_USE_REFERENCE_TYPES is
// defined, the reference's own types are used instead, so bench.hpp / cli.hpp
// style callers compile unchanged apart from the executor.
//
// Errors follow the reference: an invalid SimConfig throws
// std::invalid_argument (sim.hpp:44-49); device / NCCL failures throw
// std::runtime_error.  Link with -lfsb_b200.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fsb_b200.h"

namespace fsb {
namespace gpu {

#if defined(FSB_GPU_USE_REFERENCE_TYPES)
using ::fsb::EatResult;
using ::fsb::Fish;
using ::fsb::School;
using ::fsb::SimConfig;
using ::fsb::SimResult;
using ::fsb::kChecksumEmpty;
using ::fsb::kWeightMin;
#else
inline constexpr double kWeightMin = 1.0;                        // sim.hpp:24
inline constexpr std::uint64_t kChecksumEmpty = 0xcbf29ce484222325ull;  // sim.hpp:156

struct Fish {  // sim.hpp:26-32
    double x = 0.0;
    double y = 0.0;
    double weight = kWeightMin;
    double prev_objective = 0.0;
    double current_objective = 0.0;
};

struct SimConfig {  // sim.hpp:34-50
    std::size_t num_fish = 10000;
    double pond_size = 200.0;
    double weight_scale = 10.0;
    std::size_t num_steps = 1000;
    std::uint64_t seed = 1;
    double step_base = 1.0;

    double weight_max() const { return 2.0 * weight_scale; }

    void validate() const {
        if (!(pond_size > 0.0)) throw std::invalid_argument("SimConfig: pond_size must be > 0");
        if (!(weight_scale >= kWeightMin))
            throw std::invalid_argument("SimConfig: weight_scale must be >= 1");
        if (!(step_base > 0.0)) throw std::invalid_argument("SimConfig: step_base must be > 0");
    }
};

struct School {  // sim.hpp:52-56
    std::vector<Fish> fishes;
    std::size_t size() const { return fishes.size(); }
};

struct EatResult {  // sim.hpp:101-104
    double max_diff = -std::numeric_limits<double>::infinity();
    double seconds = 0.0;
};

struct SimResult {  // sim.hpp:125-131
    School school;
    std::vector<double> max_diff_trace;
    double seconds_total = 0.0;
    double seconds_move = 0.0;
    double seconds_eat = 0.0;
};
#endif

static_assert(sizeof(Fish) == sizeof(fsb_fish), "Fish must keep the 40-byte reference layout");

inline void check(int rc) {
    if (rc == FSB_OK) return;
    const std::string msg = fsb_last_error();
    if (rc == FSB_ERR_INVALID_CONFIG) throw std::invalid_argument(msg);
    throw std::runtime_error("fsb_b200 error " + std::to_string(rc) + ": " + msg);
}

inline fsb_sim_config to_c(const SimConfig& c) {
    fsb_sim_config r;
    r.num_fish = c.num_fish;
    r.pond_size = c.pond_size;
    r.weight_scale = c.weight_scale;
    r.num_steps = c.num_steps;
    r.seed = c.seed;
    r.step_base = c.step_base;
    return r;
}

// sim.hpp:59-63 (host scalar helper; build callers without FMA contraction).
inline double objective(double x, double y, double pond_size) {
    const double dx = x - pond_size / 2.0;
    const double dy = y - pond_size / 2.0;
    return std::sqrt(dx * dx + dy * dy);
}

// sim.hpp:158-176
inline std::uint64_t checksum(const School& school) {
    return fsb_checksum_update(kChecksumEmpty, reinterpret_cast<const fsb_fish*>(school.fishes.data()),
                               school.fishes.size());
}

// Per-step barycentre sums {sum x*f, sum y*f, sum f} (north_star; no reference counterpart).
struct Barycentre {
    double sum_xf = 0.0, sum_yf = 0.0, sum_f = 0.0;
    double x = 0.0, y = 0.0;
};

// RAII owner of one device-resident shard (fsb_engine).
class Engine {
  public:
    struct Options {
        int device = 0;
        int rank = 0;
        int world_size = 1;
        const void* nccl_unique_id = nullptr;
        int strategy = FSB_STRATEGY_AUTO;
        unsigned flags = 0;
    };

    explicit Engine(const SimConfig& cfg) : Engine(cfg, Options{}) {}
    Engine(const SimConfig& cfg, const Options& o) : cfg_(cfg) {
        const fsb_sim_config c = to_c(cfg);
        fsb_engine_options opts{o.device, o.rank, o.world_size, o.nccl_unique_id, o.strategy, o.flags};
        fsb_engine* e = nullptr;
        check(fsb_engine_create(&c, &opts, &e));
        e_.reset(e);
        check(fsb_engine_shard(e, &first_, &count_));
    }

    const SimConfig& config() const { return cfg_; }
    std::uint64_t first() const { return first_; }
    std::uint64_t count() const { return count_; }
    fsb_engine* handle() const { return e_.get(); }

    void init() { check(fsb_engine_init(e_.get())); }
    void upload(const School& s) {
        check(fsb_engine_upload(e_.get(), reinterpret_cast<const fsb_fish*>(s.fishes.data()), s.fishes.size()));
    }
    void download(School& s) {
        s.fishes.resize(count_);
        check(fsb_engine_download(e_.get(), reinterpret_cast<fsb_fish*>(s.fishes.data()), count_));
    }
    double move(std::uint64_t step) {
        double secs = 0.0;
        check(fsb_engine_move(e_.get(), step, &secs));
        return secs;
    }
    EatResult eat() {
        EatResult r;
        check(fsb_engine_eat(e_.get(), &r.max_diff, &r.seconds));
        return r;
    }
    // T x (move, eat) for steps [first_step, first_step + T); trace gets one max_diff per step.
    fsb_timing run(std::uint64_t first_step, std::uint64_t T, std::vector<double>& trace,
                   std::vector<double>* bary = nullptr) {
        trace.resize(T);
        if (bary) bary->resize(3 * T);
        fsb_timing t{};
        check(fsb_engine_run(e_.get(), first_step, T, trace.data(), bary ? bary->data() : nullptr, &t));
        return t;
    }
    Barycentre barycentre() {
        double sums[3], xy[2];
        check(fsb_engine_barycentre(e_.get(), sums, xy));
        return Barycentre{sums[0], sums[1], sums[2], xy[0], xy[1]};
    }
    std::uint64_t checksum(std::uint64_t h = kChecksumEmpty) {
        std::uint64_t out = 0;
        check(fsb_engine_checksum(e_.get(), h, &out));
        return out;
    }
    // Peer exchange (Options::flags |= FSB_FLAG_PEER_EXCHANGE): this rank's IPC
    // handle, and connecting with every rank's handle in rank order.
    std::vector<unsigned char> peer_handle() {
        std::vector<unsigned char> h(64);
        check(fsb_engine_peer_handle(e_.get(), h.data(), h.size()));
        return h;
    }
    void peer_connect(const std::vector<unsigned char>& all_handles) {
        check(fsb_engine_peer_connect(e_.get(), all_handles.data(), all_handles.size()));
    }
    // Ranks of this process (one thread per GPU): every rank's engine in rank order.
    void peer_connect_local(const std::vector<Engine*>& ranks) {
        std::vector<fsb_engine*> h;
        for (Engine* r : ranks) h.push_back(r ? r->e_.get() : nullptr);
        check(fsb_engine_peer_connect_local(e_.get(), h.data(), static_cast<int>(h.size())));
    }
    // CTA count of the step kernel for configuration sweeps (0 = automatic).
    void set_grid(int ctas) { check(fsb_engine_set_grid(e_.get(), ctas)); }
    int grid() const {
        int ctas = 0;
        check(fsb_engine_grid(e_.get(), &ctas, nullptr));
        return ctas;
    }

  private:
    struct Del {
        void operator()(fsb_engine* e) const { fsb_engine_destroy(e); }
    };
    SimConfig cfg_;
    std::unique_ptr<fsb_engine, Del> e_;
    std::uint64_t first_ = 0, count_ = 0;
};

// Drop-in for parfor::Executor& (executor.hpp:28): school-size agnostic,
// keeps one Engine for the latest (config, size).  Non-copyable, like the
// reference Executor (executor.hpp:43-44).
class Executor {
  public:
    explicit Executor(int device = 0, int strategy = FSB_STRATEGY_AUTO)
        : device_(device), strategy_(strategy) {}
    Executor(const Executor&) = delete;
    Executor& operator=(const Executor&) = delete;

    Engine& engine_for(const SimConfig& cfg, std::size_t n) {
        SimConfig c = cfg;
        c.num_fish = n;
        if (!eng_ || !same(eng_->config(), c)) {
            eng_.reset();
            Engine::Options o;
            o.device = device_;
            o.strategy = strategy_;
            eng_ = std::make_unique<Engine>(c, o);
        }
        return *eng_;
    }

  private:
    static bool same(const SimConfig& a, const SimConfig& b) {
        return a.num_fish == b.num_fish && a.pond_size == b.pond_size && a.weight_scale == b.weight_scale &&
               a.num_steps == b.num_steps && a.seed == b.seed && a.step_base == b.step_base;
    }
    int device_;
    int strategy_;
    std::unique_ptr<Engine> eng_;
};

// sim.hpp:65-79
inline School init_school(const SimConfig& cfg, Executor& exec) {
    cfg.validate();
    Engine& e = exec.engine_for(cfg, cfg.num_fish);
    e.init();
    School s;
    e.download(s);
    return s;
}

// sim.hpp:84-99 -- in place on the host School; returns the device time.
inline double move_phase(School& school, const SimConfig& cfg, std::size_t step_index, Executor& exec) {
    Engine& e = exec.engine_for(cfg, school.size());
    e.upload(school);
    const double secs = e.move(step_index);
    e.download(school);
    return secs;
}

// sim.hpp:110-123
inline EatResult eat_phase(School& school, const SimConfig& cfg, Executor& exec) {
    Engine& e = exec.engine_for(cfg, school.size());
    e.upload(school);
    const EatResult r = e.eat();
    e.download(school);
    return r;
}

// sim.hpp:133-147 -- init + num_steps x (move, eat), device resident.
inline SimResult simulate(const SimConfig& cfg, Executor& exec) {
    cfg.validate();
    Engine& e = exec.engine_for(cfg, cfg.num_fish);
    SimResult r;
    fsb_timing t{};
    r.max_diff_trace.resize(cfg.num_steps);
    check(fsb_engine_simulate(e.handle(), r.max_diff_trace.data(), nullptr, &t));
    e.download(r.school);
    r.seconds_total = t.seconds_total;
    r.seconds_move = t.seconds_move;
    r.seconds_eat = t.seconds_eat;
    return r;
}

}  // namespace gpu
}  // namespace fsb
