// Host-tier known-answer program. It is compiled twice by
// tests/test_host_parity.py: once against the reference's own headers
// (/root/reference/proj/include, where available) and once against this
// repo's drop-in headers (include/). Both builds must print byte-identical
// output, and the SPEC worked examples among the lines are pinned in the test
// (tests/golden/host_kats.txt holds the reference build's output).
//
// Only host tiers are exercised (types, rng, profile, analytics, planner, sim,
// stream, metrics, net init, checkpoint text): nothing here needs a GPU.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <string>
#include <vector>

#include "ferret/analytics.hpp"
#include "ferret/metrics.hpp"
#include "ferret/net.hpp"
#include "ferret/planner.hpp"
#include "ferret/profile.hpp"
#include "ferret/rng.hpp"
#include "ferret/sim.hpp"
#include "ferret/stream.hpp"
#include "ferret/types.hpp"

using namespace ferret;

static void line(const char* k, const std::string& v) { std::printf("%s %s\n", k, v.c_str()); }
static std::string d(double v) { return detail::fmt_double(v); }
static std::string u(unsigned long long v) { return std::to_string(v); }
static std::string bounds_str(const PartitionScheme& s) {
    std::string o;
    for (auto b : s.bounds) o += std::to_string(b) + ",";
    return o;
}

static ModelProfile times_profile(const std::vector<double>& t) {
    ModelProfile p;
    for (double x : t) p.layers.push_back({x / 2, x / 2, 1, 1});
    return p;
}

static StageStats stats2(double tf, double tb, count_t w, count_t a, count_t inner) {
    StageStats s;
    s.w = {w, w};
    s.a = {a, a};
    s.inner_a = {inner, inner};
    s.t_f = tf;
    s.t_b = tb;
    return s;
}

static PipelineConfig one_worker(std::size_t P, int rec = 0, int modulus = 1) {
    PipelineConfig c;
    c.modulus = modulus;
    WorkerConfig w;
    w.delay = 0;
    w.recompute = rec;
    w.accum.assign(P, 1);
    w.omit.assign(P, 0);
    c.workers.push_back(w);
    return c;
}

int main() {
    // --- rng (rng.hpp): raw draws pin the generator and the distribution helpers
    {
        Rng r(42);
        std::string o;
        for (int i = 0; i < 3; ++i) o += u(r.next_u64()) + ",";
        o += d(r.uniform()) + "," + u(r.below(1000)) + "," + d(r.normal()) + "," + d(r.uniform(-2, 2));
        line("rng_seed42", o);
    }
    // --- profile
    line("partition_1_.5_.5_1_tc1.2", bounds_str(partition_by_bound(times_profile({1, .5, .5, 1}), 1.2)));
    line("partition_3x1_tc1", bounds_str(partition_by_bound(times_profile({1, 1, 1}), 1.0)));
    {
        std::string o;
        for (double c : candidate_bounds(times_profile({1, 2, 4}))) o += d(c) + ",";
        line("candidates_1_2_4", o);
    }
    {
        ModelProfile p;
        for (count_t w : {1, 2, 3, 4}) p.layers.push_back({1, 1, w, w});
        const StageStats st = stage_stats(p, PartitionScheme{{0, 2, 4}});
        line("stage_stats_w", u(st.w[0]) + "," + u(st.w[1]) + ";inner " + u(st.inner_a[0]) + "," + u(st.inner_a[1]));
    }
    {
        const ModelProfile p = synth_profile(8, 7, CostModel::pyramid);
        std::ostringstream os;
        write_profile(os, p);
        line("synth_profile_8_7_pyramid_bytes", u(os.str().size()));
        line("synth_profile_8_7_pyramid_l3", d(p.layers[3].t_f) + "," + d(p.layers[3].t_b) + "," + u(p.layers[3].w));
    }
    // --- analytics
    {
        StreamSpec s;
        StageStats one;
        one.w = {10};
        one.a = {5};
        one.inner_a = {3};
        one.t_f = 0.5;
        one.t_b = 0.5;
        line("rate_P1_default", d(adaptation_rate(one, one_worker(1), s)));
        line("mem_P1_default", u(memory_footprint(one, one_worker(1))));
        line("S1_dM_P1", std::to_string(delta_recompute(one, one_worker(1), s, 0).delta.d_memory));
        StreamSpec s2;
        s2.decay_c = 0.1;
        const StageStats two = stats2(1, 1, 10, 5, 0);
        line("rate_eq3_P2_c0.1", d(adaptation_rate(two, one_worker(2), s2)));
        line("mem_eq4_P2", u(memory_footprint(two, one_worker(2))));
        const StageStats twor = stats2(1, 1, 10, 5, 2);
        line("mem_eq4_P2_recompute", u(memory_footprint(twor, one_worker(2, 1))));
        const MoveResult s2m = delta_accumulate(two, one_worker(2), s, 0, 0);
        line("S2_P2_j0_status", std::to_string(static_cast<int>(s2m.status)));
        line("S3_P2_j0_dM", std::to_string(delta_omit(two, one_worker(2), s, 0, 0).delta.d_memory));
        line("S4_P2_dM", std::to_string(delta_remove(two, one_worker(2), s, 0).delta.d_memory));
    }
    // --- metrics
    line("agm_10pp_2x", d(agm(10, 2, 0, 1)));
    line("agm_e", d(agm(5, std::exp(1.0), 5, 1)));
    {
        std::vector<StepRecord> log(4);
        log[0].outcome = StepOutcome::correct;
        log[1].outcome = StepOutcome::wrong;
        log[2].outcome = StepOutcome::correct;
        line("oacc_2_of_4_drop", d(online_accuracy(log)));
    }
    // --- simulator
    {
        StreamSpec s;
        const StageStats two = stats2(1, 1, 10, 5, 0);
        PipelineConfig c = one_worker(2, 0, 2);
        const SimTrace tr = simulate(two, c, s, 10);
        std::string drops;
        for (const auto& e : tr.events)
            if (e.kind == EventKind::drop) drops += std::to_string(e.item) + ",";
        line("sim_P2_mod2_drops", drops);
        line("sim_P2_mod2_latency_item8", d(tr.item_latency[8]));
        line("sim_P2_mod2_peak", u(tr.peak_memory));
        std::ostringstream os;
        write_trace(os, tr, s);
        line("sim_P2_mod2_trace_bytes", u(os.str().size()));
        // saturated default config: peak == Eq. 4 (acceptance #1)
        const PipelineConfig dc = default_config(two, 1.0, 0);
        line("sim_P2_default_peak", u(simulate(two, dc, s, 40).peak_memory));
        line("mem_P2_default", u(memory_footprint(two, dc)));
    }
    // --- the benchmark workloads: plans, traces, nets, streams
    const std::vector<std::vector<std::size_t>> nets = {
        {784, 256, 256, 10}, {784, 256, 256, 256, 10}, {3072, 1024, 512, 256, 10}, {784, 256, 256, 256, 256, 256, 256, 256, 10}};
    for (std::size_t k = 0; k < nets.size(); ++k) {
        const DenseNet net = make_dense_net(nets[k], 1);
        const ModelProfile prof = profile_from_net(net);
        double td = 0;
        for (const auto& l : prof.layers) td = std::max(td, l.t_f);
        StreamSpec s;
        s.t_d = td;
        s.decay_c = std::log(2.0) / prof.total_time();
        s.horizon = 200 * td;
        const PlanResult full = plan(prof, td, s, kNoBudget);
        for (double frac : {1.0, 0.5, 0.25}) {
            const PlanResult p = plan(prof, td, s, static_cast<count_t>(static_cast<double>(full.memory) * frac));
            std::ostringstream os;
            write_plan(os, p);
            const StageStats st = stage_stats(prof, p.partition);
            std::ostringstream ot;
            write_trace(ot, simulate(st, p.config, s, 120), s);
            std::size_t h = 1469598103934665603ULL;
            for (char ch : os.str() + ot.str()) h = (h ^ static_cast<unsigned char>(ch)) * 1099511628211ULL;
            line(("plan_trace_net" + std::to_string(k) + "_" + d(frac)).c_str(),
                 bounds_str(p.partition) + " workers " + u(p.config.active_count()) + " fnv " + u(h));
        }
        line(("net_param0_" + std::to_string(k)).c_str(), d(net.layers[0].W[0]) + "," + d(net.layers.back().W.back()));
    }
    {
        const DataStream ds = synth_drift_stream(2000, 784, 10, DriftKind::split_tasks, 7);
        double acc = 0;
        for (const auto& it : ds.items) acc += it.features[3] + static_cast<double>(it.label);
        line("stream_c1_checksum", d(acc) + " label1999 " + u(ds.items[1999].label));
        const DataStream rot = synth_drift_stream(50, 6, 3, DriftKind::rotate, 11);
        line("stream_rotate_x", d(rot.items[49].features[0]) + "," + d(rot.items[49].features[5]));
        RunningNormalizer n(784);
        for (int i = 0; i < 300; ++i) n.observe(ds.items[static_cast<std::size_t>(i)].features);
        const auto z = n.apply(ds.items[300].features);
        line("normalizer_z", d(z[0]) + "," + d(z[783]));
    }
    {
        SkipPolicy sp;
        sp.kind = SkipKind::random_n;
        sp.window = 4;
        sp.keep = 2;
        sp.seed = 5;
        const FilteredStream fs = apply_skip_policy(40, 1.0, sp, 2.5);
        std::string o;
        for (const auto& k : fs.kept) o += std::to_string(k.index) + ":" + d(k.start) + ",";
        line("skip_random_n", o);
        sp.kind = SkipKind::one_skip;
        line("skip_one_skip_kept", u(apply_skip_policy(40, 1.0, sp, 2.5).kept.size()));
    }
    {
        const DenseNet net = make_dense_net({5, 4, 3}, 9);
        std::ostringstream os;
        write_checkpoint(os, net);
        line("ckpt_bytes", u(os.str().size()));
    }
    return 0;
}
