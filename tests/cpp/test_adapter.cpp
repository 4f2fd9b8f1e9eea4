// C++ host-side tests through include/moe_b200.hpp, written like the
// reference's own doctest cases (proj/tests/test_routing.cpp) they mirror.
//   test_adapter host   — host-only entry points (no GPU)
//   test_adapter gpu    — layer cases on cuda:0
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "moe_b200.hpp"

using namespace moe_b200;

static int g_fail = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++g_fail;                                                         \
        }                                                                     \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void host_cases() {
    // test_routing.cpp:43-50 "capacity formula"
    RouterConfig cfg;
    cfg.num_experts = 8;
    CHECK(capacity(64, cfg, Phase::kTrain) == 8);
    CHECK(capacity(64, cfg, Phase::kEval) == 16);
    CHECK(capacity(1, cfg, Phase::kTrain) == 1);
    cfg.capacity_factor_train = 1.3;
    CHECK(capacity(10, cfg, Phase::kTrain) == 2);
    // routing.cpp:13-23 validation -> ConfigError
    RouterConfig bad;
    bad.top_k = 3;
    CHECK(throws<ConfigError>([&] { bad.validate(); }));
    bad = RouterConfig{};
    bad.num_experts = 1;
    bad.top_k = 2;
    CHECK(throws<ConfigError>([&] { bad.validate(); }));
    CHECK(throws<ConfigError>([&] { (void)capacity(0, RouterConfig{}, Phase::kTrain); }));
    // rng.cpp:24-34 seed derivation KATs
    CHECK(derive_seed(42, "jitter") == 4217090220841641567ULL);
    CHECK(derive_seed(42, "assign") == 11878108427965954893ULL);
}

template <class T>
static T* dev_copy(const std::vector<T>& h) {
    T* p = nullptr;
    cudaMalloc(&p, sizeof(T) * h.size());
    cudaMemcpy(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice);
    return p;
}
template <class T>
static std::vector<T> host_copy(const T* d, size_t n) {
    std::vector<T> h(n);
    cudaMemcpy(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost);
    return h;
}

static void gpu_cases() {
    std::mt19937_64 eng(101);
    std::uniform_real_distribution<float> U(-1.f, 1.f);
    auto rnd = [&](size_t n, float s) {
        std::vector<float> v(n);
        for (auto& x : v) x = s * U(eng);
        return v;
    };
    {  // test_routing.cpp:439-454 "single expert equals a dense FFN"
        const int64_t d = 64, f = 128, T = 96;
        RouterConfig cfg;
        cfg.num_experts = 1;
        auto x = rnd(T * d, 1.f), gw = rnd(d, 1.f), w1 = rnd(d * f, .2f), b1 = rnd(f, .1f),
             w2 = rnd(f * d, .2f), b2 = rnd(d, .1f);
        MoeLayer layer(cfg, T, d, f, MOE_F32);
        MoeLayerParams p{dev_copy(gw), dev_copy(w1), dev_copy(b1), dev_copy(w2), dev_copy(b2)};
        float* xd = dev_copy(x);
        float *y, *aux;
        cudaMalloc(&y, 4 * T * d);
        cudaMalloc(&aux, 4);
        layer.forward(T, xd, p, Phase::kTrain, 5, y, aux);
        auto yh = host_copy(y, T * d);
        double worst = 0;
        for (int64_t t = 0; t < T; ++t) {
            std::vector<double> h(f);
            for (int64_t j = 0; j < f; ++j) {
                double a = b1[j];
                for (int64_t k = 0; k < d; ++k) a += double(x[t * d + k]) * w1[k * f + j];
                h[j] = a > 0 ? a : 0;
            }
            for (int64_t k = 0; k < d; ++k) {
                double a = b2[k];
                for (int64_t j = 0; j < f; ++j) a += h[j] * w2[j * d + k];
                worst = std::max(worst, std::abs(a - yh[t * d + k]) / std::max(1.0, std::abs(a)));
            }
        }
        CHECK(worst < 1e-5);
        // backward runs and writes finite grads
        float *dx, *dgw, *dw1, *db1, *dw2, *db2;
        cudaMalloc(&dx, 4 * T * d); cudaMalloc(&dgw, 4 * d); cudaMalloc(&dw1, 4 * d * f);
        cudaMalloc(&db1, 4 * f); cudaMalloc(&dw2, 4 * f * d); cudaMalloc(&db2, 4 * d);
        layer.backward(xd, 1.0f, MoeLayerGrads{dx, dgw, dw1, db1, dw2, db2, nullptr});
        auto g = host_copy(dw1, d * f);
        bool finite = true;
        for (float v : g) finite &= std::isfinite(v);
        CHECK(finite);
    }
    {  // test_routing.cpp:491-502 "eval phase ignores the configured stochastic mode"
        const int64_t d = 64, f = 64, T = 64;
        RouterConfig cfg;
        cfg.num_experts = 4;
        cfg.assignment_mode = AssignmentMode::kRts;
        auto x = rnd(T * d, 1.f), gw = rnd(d * 4, 1.f), w1 = rnd(4 * d * f, .2f),
             b1 = rnd(4 * f, .1f), w2 = rnd(4 * f * d, .2f), b2 = rnd(4 * d, .1f);
        MoeLayer layer(cfg, T, d, f, MOE_F32);
        MoeLayerParams p{dev_copy(gw), dev_copy(w1), dev_copy(b1), dev_copy(w2), dev_copy(b2)};
        float* xd = dev_copy(x);
        float *y1, *y2, *aux;
        cudaMalloc(&y1, 4 * T * d); cudaMalloc(&y2, 4 * T * d); cudaMalloc(&aux, 4);
        layer.forward(T, xd, p, Phase::kEval, 1, y1, aux);
        layer.forward(T, xd, p, Phase::kEval, 2, y2, aux);
        CHECK(host_copy(y1, T * d) == host_copy(y2, T * d));
    }
    {  // test_routing.cpp:503-522 "top-2 ... generous capacity: no drops, deterministic"
        const int64_t d = 64, f = 64, T = 48;
        RouterConfig cfg;
        cfg.num_experts = 4;
        cfg.top_k = 2;
        cfg.capacity_factor_train = 4.0;
        auto x = rnd(T * d, 1.f), gw = rnd(d * 4, 1.f), w1 = rnd(4 * d * f, .2f),
             b1 = rnd(4 * f, .1f), w2 = rnd(4 * f * d, .2f), b2 = rnd(4 * d, .1f);
        MoeLayer layer(cfg, T, d, f, MOE_F32);
        MoeLayerParams p{dev_copy(gw), dev_copy(w1), dev_copy(b1), dev_copy(w2), dev_copy(b2)};
        float* xd = dev_copy(x);
        float *y, *aux, *gp;
        int32_t *eid, *slot;
        cudaMalloc(&y, 4 * T * d); cudaMalloc(&aux, 4); cudaMalloc(&gp, 8 * T);
        cudaMalloc(&eid, 8 * T); cudaMalloc(&slot, 8 * T);
        layer.forward(T, xd, p, Phase::kTrain, 3, y, aux, nullptr, eid, slot, gp);
        RoutingDecision dec = layer.decision(T, eid, slot, gp);
        CHECK(dec.top_k == 2 && dec.drop_count() == 0);
        auto first = host_copy(y, T * d);
        layer.forward(T, xd, p, Phase::kTrain, 3, y, aux);
        CHECK(first == host_copy(y, T * d));
    }
    {  // non-finite input -> NonFiniteError (tensor.cpp:23-29)
        const int64_t d = 64, f = 64, T = 16;
        RouterConfig cfg;
        cfg.num_experts = 2;
        auto x = rnd(T * d, 1.f), gw = rnd(d * 2, 1.f), w1 = rnd(2 * d * f, .2f),
             b1 = rnd(2 * f, .1f), w2 = rnd(2 * f * d, .2f), b2 = rnd(2 * d, .1f);
        x[5] = NAN;
        MoeLayer layer(cfg, T, d, f, MOE_F32);
        MoeLayerParams p{dev_copy(gw), dev_copy(w1), dev_copy(b1), dev_copy(w2), dev_copy(b2)};
        float* xd = dev_copy(x);
        float *y, *aux;
        cudaMalloc(&y, 4 * T * d); cudaMalloc(&aux, 4);
        CHECK(throws<NonFiniteError>([&] { layer.forward(T, xd, p, Phase::kTrain, 1, y, aux); }));
    }
}

// The per-stage mirrors of routing.hpp:60-118 on the device, against the
// reference's known answers (test_routing.cpp, SURVEY §8c KATs).
static void stage_cases() {
    {  // test_routing.cpp:53-61: equal logits -> P = [.5, .5], tie to expert 0
        RouterConfig cfg;
        cfg.num_experts = 2;
        const int64_t T = 3, d = 2;
        std::vector<float> x = {1, 2, -1, 0.5f, 3, -2}, gw = {1, 1, -1, -1};  // columns equal
        DeviceArray<float> xd(x), gwd(gw);
        GateResult g = gate_forward(xd.data(), T, d, MOE_F32, gwd.data(), cfg, Phase::kEval, 0);
        auto P = g.probs.to_host();
        for (float v : P) CHECK(v == 0.5f);
        for (int32_t c : g.choice) CHECK(c == 0);
        CHECK(g.gate_prob.size() == 1 && g.gate_prob[0].to_host()[1] == 0.5f);
    }
    {  // test_routing.cpp:118-125: plain, all to expert 0, cap 2 -> [0, 1, D, D]
        RoutingDecision d = assign_plain({0, 0, 0, 0}, 1, 2);
        CHECK((d.slot == std::vector<int32_t>{0, 1, kDropped, kDropped}));
        // k-major top-2: t2's first choice dropped, its second kept
        RoutingDecision k2 = assign_plain({0, 1, 0, 1, 0, 2}, 3, 2, 2);
        CHECK((k2.slot == std::vector<int32_t>{0, 0, 1, 1, kDropped, 0}));
        // grouped: capacity G * ceil(cap / G), per-group bases
        RoutingDecision g = assign_grouped({0, 0, 0, 0, 0, 0}, 1, 3, 2);
        CHECK(g.capacity == 4);
        CHECK((g.slot == std::vector<int32_t>{0, 1, kDropped, 2, 3, kDropped}));
        CHECK(throws<ConfigError>([] { (void)assign_grouped({0, 0, 0}, 1, 2, 2); }));
        CHECK(throws<ConfigError>([] { (void)assign_plain({0, 3}, 2, 2); }));
        // RTS: deterministic, never over capacity, no drops when capacity suffices
        std::vector<int32_t> ch(32, 0);
        CHECK(assign_rts(ch, 1, 8, 777).slot == assign_rts(ch, 1, 8, 777).slot);
        CHECK(assign_rts(ch, 1, 8, 777).drop_count() == 24);
        CHECK(assign_rts({0, 1, 0, 1, 2, 2}, 3, 2, 5).drop_count() == 0);
        RouterConfig cfg;
        cfg.num_experts = 1;
        cfg.assignment_mode = AssignmentMode::kRts;
        RoutingDecision ev = make_assignment(ch, 32, cfg, Phase::kEval, 1);  // eval -> plain
        CHECK(ev.slot == assign_plain(ch, 1, 64).slot);
    }
    {  // dispatch / combine round trip (test_routing.cpp:287-314) + exact-zero rows
        const int64_t T = 6, d = 4;
        std::vector<float> x(T * d);
        for (size_t i = 0; i < x.size(); ++i) x[i] = 0.25f * static_cast<float>(i) - 2.f;
        RoutingDecision dec = assign_plain({0, 1, 0, 1, 0, 2}, 3, 2);
        DeviceArray<float> xd(x);
        DispatchBuffer b = dispatch(xd.data(), T, d, MOE_F32, dec);
        auto occ = b.occupancy.to_host();
        auto buf = b.data.to_host();
        const float* bf = reinterpret_cast<const float*>(buf.data());
        for (int r = 0; r < 6; ++r)
            if (!occ[r])
                for (int j = 0; j < d; ++j) CHECK(bf[r * d + j] == 0.f);
        DeviceArray<float> w(std::vector<float>(T, 1.f));
        DeviceArray<std::uint8_t> y = combine(b.data.data(), d, MOE_F32, dec, xd.data(), w.data());
        auto yh = y.to_host();
        CHECK(std::memcmp(yh.data(), x.data(), sizeof(float) * x.size()) == 0);
    }
    {  // balance loss closed form: uniform routing -> alpha (test_routing.cpp:368-381)
        const int64_t T = 4;
        RoutingDecision dec = assign_plain({0, 1, 2, 3}, 4, 1);
        DeviceArray<float> P(std::vector<float>(T * 4, 0.25f));
        CHECK(std::abs(balance_loss(P.data(), dec, 0.01) - 0.01f) < 1e-7f);
        DeviceArray<float> bad(std::vector<float>(T * 4, 0.3f));
        CHECK(throws<std::invalid_argument>([&] { (void)balance_loss(bad.data(), dec, 0.01); }));
    }
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    host_cases();
    if (gpu) {
        gpu_cases();
        stage_cases();
    }
    std::printf("%s %s\n", g_fail ? "FAIL" : "OK", gpu ? "host+gpu" : "host");
    return g_fail ? 1 : 0;
}
