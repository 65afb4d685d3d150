// simulate_multi_gpu.cpp -- one process, one host thread per GPU (the
// "one thread per device" model of SURVEY.md 8(b)), through the C++ drop-in.
//
//   simulate_multi_gpu <num_gpus> <fish> <steps> [seed] [nccl|peer]
//
// Each thread owns the contiguous shard fsb_shard_range(N, G, r) on device r;
// the ranks exchange the per-step {max, sums} with NCCL (one communicator per
// device, created from a shared ncclUniqueId; the default) or, with "peer",
// with no library at all: every step kernel stores its partial into every
// rank's window over NVLink (FSB_FLAG_PEER_EXCHANGE), the windows connected by
// pointer within this process (fsb_engine_peer_connect_local).  The school's checksum is the
// reference digest (sim.hpp:158-176) chained over the shards in rank order, so
// it equals the single-GPU (and the reference's) checksum for every G.
// Prints: "<checksum> <last max_diff> <seconds>".
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "fsb/gpu.hpp"

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s <num_gpus> <fish> <steps> [seed]\n", argv[0]);
        return 2;
    }
    const int G = std::atoi(argv[1]);
    fsb::gpu::SimConfig cfg;  // BASELINE mapping
    cfg.num_fish = std::strtoull(argv[2], nullptr, 10);
    cfg.num_steps = std::strtoull(argv[3], nullptr, 10);
    cfg.seed = argc > 4 ? std::strtoull(argv[4], nullptr, 10) : 7;
    const bool peer = argc > 5 && std::string(argv[5]) == "peer";
    cfg.pond_size = 200.0;
    cfg.weight_scale = 1.0;
    cfg.step_base = 0.1;
    try {
        std::vector<unsigned char> uid(128, 0);
        if (G > 1 && !peer) fsb::gpu::check(fsb_nccl_unique_id(uid.data(), uid.size()));
        std::vector<std::unique_ptr<fsb::gpu::Engine>> engines(G);
        std::vector<std::vector<double>> traces(G);
        std::vector<double> seconds(G, 0.0);
        std::vector<std::string> errors(G);
        auto each = [&](auto&& body) {  // one host thread per rank / device
            std::vector<std::thread> threads;
            for (int r = 0; r < G; ++r)
                threads.emplace_back([&, r] {
                    try {
                        body(r);
                    } catch (const std::exception& e) {
                        errors[r] = e.what();
                    }
                });
            for (auto& t : threads) t.join();
            for (int r = 0; r < G; ++r)
                if (!errors[r].empty()) throw std::runtime_error("rank " + std::to_string(r) + ": " + errors[r]);
        };
        each([&](int r) {
            fsb::gpu::Engine::Options o;
            o.device = r;
            o.rank = r;
            o.world_size = G;
            if (peer) o.flags |= FSB_FLAG_PEER_EXCHANGE;
            else o.nccl_unique_id = G > 1 ? uid.data() : nullptr;
            engines[r] = std::make_unique<fsb::gpu::Engine>(cfg, o);  // (NCCL: collective init)
        });
        if (peer) {
            std::vector<fsb::gpu::Engine*> ranks;
            for (auto& e : engines) ranks.push_back(e.get());
            for (auto& e : engines) e->peer_connect_local(ranks);
        }
        each([&](int r) {  // the ranks' step kernels wait on one another: all run concurrently
            engines[r]->init();
            const fsb_timing t = engines[r]->run(0, cfg.num_steps, traces[r]);
            seconds[r] = t.seconds_loop;
        });
        std::uint64_t h = fsb::gpu::kChecksumEmpty;
        for (int r = 0; r < G; ++r) h = engines[r]->checksum(h);  // chained in rank order
        double secs = 0.0;
        for (double s : seconds) secs = s > secs ? s : secs;
        std::printf("%016llx %.17g %.6f\n", static_cast<unsigned long long>(h),
                    cfg.num_steps ? traces[0].back() : 0.0, secs);
        return 0;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
