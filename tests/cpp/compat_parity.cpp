// tests/cpp/compat_parity.cpp -- the C++ drop-in (include/coat/coatsim_compat.hpp)
// driven with the reference's own call patterns, checked against the
// unmodified reference library (oracle/_ref/libcoatsim_ref.so via its C shim).
// Built and run by tests/test_gpu_cpp_compat.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "coat/coatsim_compat.hpp"

namespace coatsim = coat_b200;   // the one-line switch a reference user makes

extern "C" {   // oracle/ref_shim.cpp (test infrastructure)
int ref_quantize(const float*, const int64_t*, int, int, int64_t, uint8_t*, float*, int64_t*);
int ref_expand_quantize(const float*, int64_t, int64_t, uint8_t*, float*, float*, float*);
int ref_make_slot(int64_t, int64_t, uint8_t*, float*, float*, float*, uint8_t*, float*, float*, float*);
int ref_step(float*, const float*, int64_t, int64_t, uint8_t*, float*, float*, float*, uint8_t*, float*, float*,
             float*, int64_t, float, float, float, float, float);
int ref_generate(int, const int64_t*, int, double, double, uint64_t, float*);
}

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                  \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(c)) {                                                               \
            ++g_fail;                                                             \
            if (g_fail < 20) std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c); \
        }                                                                         \
    } while (0)

static coatsim::Tensor generate(int kind, std::vector<int64_t> shape, double frac, double scale, uint64_t seed) {
    coatsim::Tensor t(shape);
    ref_generate(kind, shape.data(), int(shape.size()), frac, scale, seed, t.data.data());
    return t;
}

static void test_quantize() {
    // test_quantize.cpp:24-42 / 44-55 known answers
    const auto x = coatsim::Tensor::from({4}, {0.5f, -1.0f, 2.0f, 4.0f});
    const auto q = coatsim::quantize(x, coatsim::QuantGeometry::per_tensor());
    CHECK(q.scales.size() == 1);
    CHECK(q.scales[0] == coatsim::round_bf16(4.0f / 448.0f));
    CHECK(q.codes[0] == coatsim::encode_byte(56.0f));
    CHECK(q.codes[3] == coatsim::encode_byte(448.0f));
    const auto x2 = coatsim::Tensor::from({4}, {1.0f, 2.0f, 100.0f, 200.0f});
    const auto q2 = coatsim::quantize(x2, coatsim::QuantGeometry::per_group(2));
    CHECK(q2.scales[1] == coatsim::round_bf16(200.0f / 448.0f));
    // against the reference on activation-like data, several geometries
    const auto a = generate(1, {64, 256}, 0.05, 50.0, 4);
    for (int64_t G : {0, 16, 128, 32}) {
        const auto qa = coatsim::quantize(a, G ? coatsim::QuantGeometry::per_group(G) : coatsim::QuantGeometry::per_tensor());
        std::vector<uint8_t> rc(size_t(a.numel()));
        std::vector<float> rs(size_t(G ? a.numel() / G : 1));
        int64_t ng = 0;
        CHECK(ref_quantize(a.data.data(), a.shape.data(), 2, G ? 1 : 0, G, rc.data(), rs.data(), &ng) == 0);
        CHECK(qa.codes == rc);
        CHECK(qa.scales == rs);
        const auto back = coatsim::dequantize(qa);
        for (int64_t i = 0; i < a.numel(); ++i) CHECK(back[i] == coatsim::decode_byte(rc[size_t(i)]) * rs[size_t(i / (G ? G : a.numel()))]);
    }
    // error taxonomy: GeometryMismatch / NonFiniteInput
    bool threw = false;
    try { coatsim::quantize(coatsim::Tensor({4, 6}), coatsim::QuantGeometry::per_group(5)); } catch (const coatsim::GeometryMismatch&) { threw = true; }
    CHECK(threw);
    threw = false;
    auto bad = coatsim::Tensor({4, 8});
    bad[3] = NAN;
    try { coatsim::quantize(bad, coatsim::QuantGeometry::per_tensor()); } catch (const coatsim::NonFiniteInput&) { threw = true; }
    CHECK(threw);
    const auto [inter, g] = coatsim::group_scale_max(a, 16);
    float am = 0.0f;
    for (float v : a.data) am = std::fmax(am, std::fabs(v));
    CHECK(g == am && inter.numel() == a.numel() / 16);
}

static void test_expand() {
    const auto x = generate(2, {128 * 64}, 0.0, 1e4, 5);
    const auto s = coatsim::expand_quantize(x, 128);
    std::vector<uint8_t> rc(size_t(x.numel()));
    std::vector<float> rs(64), rk(64), rcc(64);
    CHECK(ref_expand_quantize(x.data.data(), x.numel(), 128, rc.data(), rs.data(), rk.data(), rcc.data()) == 0);
    CHECK(s.quantized.codes == rc);
    CHECK(s.quantized.scales == rs);
    for (int g = 0; g < 64; ++g) CHECK(s.params[size_t(g)].k == rk[size_t(g)] && s.params[size_t(g)].c == rcc[size_t(g)]);
    const auto back = coatsim::dequantize_contract(s);
    CHECK(back.numel() == x.numel());
}

static void test_step() {
    const int64_t n = 128 * 300 + 17;
    auto w = generate(0, {n}, 0.0, 100.0, 1);
    for (float& v : w.data) v *= 0.02f;
    std::vector<float> wr = w.data;
    const int64_t npad = (n + 127) / 128 * 128, ng = npad / 128;
    std::vector<uint8_t> mc(static_cast<size_t>(npad)), vc(static_cast<size_t>(npad));
    const size_t ngs = static_cast<size_t>(ng);
    std::vector<float> ms(ngs), mk(ngs), mcc(ngs), vs(ngs), vk(ngs), vcc(ngs);
    CHECK(ref_make_slot(n, 128, mc.data(), ms.data(), mk.data(), mcc.data(), vc.data(), vs.data(), vk.data(), vcc.data()) == 0);
    auto slot = coatsim::make_slot({n});
    coatsim::AdamWConfig cfg;
    cfg.weight_decay = 0.1f;
    for (int t = 0; t < 4; ++t) {
        auto g = generate(0, {n}, 0.01, 100.0, 100 + t);
        for (float& v : g.data) v *= 1e-3f;
        coatsim::step(w, g, slot, cfg);
        CHECK(ref_step(wr.data(), g.data.data(), n, 128, mc.data(), ms.data(), mk.data(), mcc.data(), vc.data(),
                       vs.data(), vk.data(), vcc.data(), t, cfg.beta1, cfg.beta2, cfg.lr, cfg.weight_decay, cfg.eps) == 0);
        CHECK(w.data == wr);
        const auto m = slot.m(), v = slot.v();
        CHECK(m.quantized.codes == mc && v.quantized.codes == vc);
        CHECK(m.quantized.scales == ms && v.quantized.scales == vs);
        for (int64_t gi = 0; gi < ng; ++gi) {
            CHECK(m.params[size_t(gi)].k == mk[size_t(gi)] && m.params[size_t(gi)].c == mcc[size_t(gi)]);
            CHECK(v.params[size_t(gi)].k == vk[size_t(gi)] && v.params[size_t(gi)].c == vcc[size_t(gi)]);
        }
    }
    CHECK(slot.step == 4);
    // NonFiniteGradient leaves params and slot untouched (optimizer.cpp:104)
    auto g = coatsim::Tensor({n});
    g[5] = INFINITY;
    const auto w_before = w.data;
    bool threw = false;
    try { coatsim::step(w, g, slot, cfg); } catch (const coatsim::NonFiniteGradient&) { threw = true; }
    CHECK(threw && w.data == w_before && slot.step == 4);

    // OptimizerSlot is a value type (optimizer.hpp:48-52): stepping a copy
    // twice must leave the original's moments exactly as they were
    const auto m_before = slot.m(), v_before = slot.v();
    coatsim::OptimizerSlot copy = slot;
    auto w2 = w;
    for (int t = 0; t < 2; ++t) {
        auto g2 = generate(0, {n}, 0.01, 100.0, 200 + t);
        for (float& v : g2.data) v *= 1e-3f;
        coatsim::step(w2, g2, copy, cfg);
    }
    CHECK(copy.step == 6 && slot.step == 4);
    const auto m_after = slot.m(), v_after = slot.v();
    CHECK(m_after.quantized.codes == m_before.quantized.codes && v_after.quantized.codes == v_before.quantized.codes);
    CHECK(m_after.quantized.scales == m_before.quantized.scales && v_after.quantized.scales == v_before.quantized.scales);
    CHECK(copy.m().quantized.codes != m_before.quantized.codes);
    // copy-assignment deep-copies too
    coatsim::OptimizerSlot assigned;
    assigned = slot;
    CHECK(assigned.mbuf[0] != slot.mbuf[0] && assigned.m().quantized.codes == m_before.quantized.codes);
}

int main() {
    test_quantize();
    test_expand();
    test_step();
    std::printf("compat_parity: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
