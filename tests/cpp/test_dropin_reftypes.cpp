// test_dropin_reftypes.cpp -- the INTEGRATION.md section-1 drop-in, exactly as a
// reference user would write it: the reference's own fsb/sim.hpp is included
// first (unmodified, from /root/reference/proj/include), FSB_GPU_USE_REFERENCE_TYPES
// makes fsb/gpu.hpp reuse ::fsb::Fish / SimConfig / School / EatResult / SimResult,
// and every result of fsb::gpu (B200) is compared with the reference's own
// parfor path on the same reference objects.
//
// Cases:
//   * init_school            -- sim.hpp:65-79 vs fsb::gpu::init_school
//   * move_phase / eat_phase -- sim.hpp:84-123 step by step on a reference School
//   * "simulation state is independent of the run configuration"
//                            -- test_sim.cpp:217-225, with fsb::gpu::Executor for
//                               every step-loop strategy beside the two RunConfigs
//   * acceptance criterion 1 -- acceptance.cpp:63-102: 4 thread counts x 6 schedules
//                               x 4 constructs on the CPU, plus every GPU strategy,
//                               all against the sequential construct's digest
//
// Built by tests/cpp/Makefile only where the reference headers exist (this
// container); the binary travels to the GPU box and tests/test_cpp_dropin.py runs it.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "fsb/sim.hpp"  // the reference (unmodified)
#define FSB_GPU_USE_REFERENCE_TYPES 1
#include "fsb/gpu.hpp"

namespace {

int g_failures = 0;
int g_checks = 0;
std::vector<std::pair<std::string, std::function<void()>>>& registry() {
    static std::vector<std::pair<std::string, std::function<void()>>> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name)                                           \
    static void CAT(tc_, __LINE__)();                             \
    static Reg CAT(reg_, __LINE__)(name, CAT(tc_, __LINE__));     \
    static void CAT(tc_, __LINE__)()
#define REQUIRE(cond)                                                                 \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(cond)) {                                                                \
            ++g_failures;                                                             \
            std::fprintf(stderr, "  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            return;                                                                   \
        }                                                                             \
    } while (0)

// The types really are the reference's.
static_assert(std::is_same_v<fsb::gpu::School, fsb::School>);
static_assert(std::is_same_v<fsb::gpu::SimConfig, fsb::SimConfig>);
static_assert(std::is_same_v<fsb::gpu::SimResult, fsb::SimResult>);
static_assert(std::is_same_v<fsb::gpu::EatResult, fsb::EatResult>);

constexpr int kStrategies[] = {FSB_STRATEGY_AUTO, FSB_STRATEGY_STREAM, FSB_STRATEGY_GRID, FSB_STRATEGY_PERSISTENT};
const char* strategy_name(int s) {
    switch (s) {
        case FSB_STRATEGY_AUTO: return "auto";
        case FSB_STRATEGY_STREAM: return "stream";
        case FSB_STRATEGY_GRID: return "grid";
        default: return "persistent";
    }
}

fsb::SimConfig small_config() {  // test_sim.cpp:23-29
    fsb::SimConfig cfg;
    cfg.num_fish = 500;
    cfg.num_steps = 20;
    cfg.seed = 42;
    return cfg;
}

bool same_school(const fsb::School& a, const fsb::School& b) {
    return a.fishes.size() == b.fishes.size() &&
           (a.fishes.empty() ||
            std::memcmp(a.fishes.data(), b.fishes.data(), a.fishes.size() * sizeof(fsb::Fish)) == 0);
}

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * 8) == 0);
}

}  // namespace

TEST_CASE("init_school equals the reference's, on the reference School type") {
    for (std::size_t n : {std::size_t(0), std::size_t(1), std::size_t(500), std::size_t(100003)}) {
        fsb::SimConfig cfg = small_config();
        cfg.num_fish = n;
        fsb::gpu::Executor gexec;
        const fsb::School want = fsb::init_school(cfg);
        const fsb::School got = fsb::gpu::init_school(cfg, gexec);
        REQUIRE(same_school(got, want));
        REQUIRE(fsb::gpu::checksum(got) == fsb::checksum(want));
    }
}

TEST_CASE("move_phase and eat_phase follow the reference step by step") {
    fsb::SimConfig cfg = small_config();
    cfg.num_fish = 3001;
    parfor::Executor exec(parfor::RunConfig{1, {parfor::ScheduleKind::Static, 50}, parfor::Construct::Sequential});
    fsb::gpu::Executor gexec;
    fsb::School want = fsb::init_school(cfg);
    fsb::School got = want;
    for (std::size_t t = 0; t < cfg.num_steps; ++t) {
        fsb::move_phase(want, cfg, t, exec);
        fsb::gpu::move_phase(got, cfg, t, gexec);
        REQUIRE(same_school(got, want));
        const fsb::EatResult ew = fsb::eat_phase(want, cfg, exec);
        const fsb::EatResult eg = fsb::gpu::eat_phase(got, cfg, gexec);
        REQUIRE(std::memcmp(&ew.max_diff, &eg.max_diff, 8) == 0);
        REQUIRE(same_school(got, want));
    }
}

TEST_CASE("simulation state is independent of the run configuration") {  // test_sim.cpp:217-225
    fsb::SimConfig cfg = small_config();
    parfor::RunConfig run_a{1, {parfor::ScheduleKind::Static, 50}, parfor::Construct::Reduction};
    parfor::RunConfig run_b{8, {parfor::ScheduleKind::Dynamic, 1}, parfor::Construct::CriticalFull};
    const fsb::SimResult a = fsb::simulate(cfg, run_a);
    const fsb::SimResult b = fsb::simulate(cfg, run_b);
    REQUIRE(fsb::checksum(a.school) == fsb::checksum(b.school));
    REQUIRE(a.max_diff_trace == b.max_diff_trace);
    for (int s : kStrategies) {
        fsb::gpu::Executor gexec(0, s);
        const fsb::SimResult g = fsb::gpu::simulate(cfg, gexec);
        REQUIRE(fsb::checksum(g.school) == fsb::checksum(a.school));
        REQUIRE(same_school(g.school, b.school));
        REQUIRE(g.max_diff_trace == a.max_diff_trace);
        REQUIRE(g.seconds_total >= g.seconds_eat && g.seconds_eat > 0.0);
    }
}

TEST_CASE("acceptance criterion 1: every schedule, construct and GPU strategy shares one checksum") {
    // acceptance.cpp:63-102, with the B200 strategies as further "run configurations"
    setenv(parfor::kScheduleEnvVar, "dynamic,64", 1);
    fsb::SimConfig cfg;
    cfg.num_fish = 10000;
    cfg.num_steps = 100;
    cfg.seed = 7;
    using parfor::Construct;
    using parfor::ScheduleKind;
    using parfor::ScheduleSpec;
    const ScheduleSpec schedules[] = {
        {ScheduleKind::Static, 1},  {ScheduleKind::Static, 50}, {ScheduleKind::Dynamic, 1},
        {ScheduleKind::Dynamic, 50}, {ScheduleKind::Guided, 1}, {ScheduleKind::Runtime, 0},
    };
    const Construct constructs[] = {Construct::Sequential, Construct::Reduction, Construct::CriticalPartial,
                                    Construct::CriticalFull};
    const fsb::SimResult seq =
        fsb::simulate(cfg, parfor::RunConfig{1, {ScheduleKind::Static, 50}, Construct::Sequential});
    const std::uint64_t reference = fsb::checksum(seq.school);
    int combos = 0, agree = 0;
    for (int threads : {1, 2, 4, 8}) {
        for (const ScheduleSpec& schedule : schedules) {
            for (Construct construct : constructs) {
                const fsb::SimResult r = fsb::simulate(cfg, parfor::RunConfig{threads, schedule, construct});
                ++combos;
                agree += fsb::checksum(r.school) == reference;
            }
        }
    }
    std::printf("  reference: %d/%d CPU run configurations share checksum %016llx\n", agree, combos,
                static_cast<unsigned long long>(reference));
    for (int s : kStrategies) {
        fsb::gpu::Executor gexec(0, s);
        const fsb::SimResult g = fsb::gpu::simulate(cfg, gexec);
        const std::uint64_t d = fsb::gpu::checksum(g.school);
        std::printf("  gpu %-10s checksum %016llx\n", strategy_name(s), static_cast<unsigned long long>(d));
        REQUIRE(d == reference);
        REQUIRE(same_bits(g.max_diff_trace, seq.max_diff_trace));
    }
}

int main() {
    int failed_cases = 0;
    for (auto& [name, fn] : registry()) {
        const int before = g_failures;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_failures;
            std::fprintf(stderr, "  EXCEPTION %s\n", e.what());
        }
        const bool ok = g_failures == before;
        failed_cases += !ok;
        std::printf("%s %s\n", ok ? "PASS" : "FAIL", name.c_str());
    }
    std::printf("%zu cases, %d failed, %d checks\n", registry().size(), failed_cases, g_checks);
    return failed_cases == 0 ? 0 : 1;
}
