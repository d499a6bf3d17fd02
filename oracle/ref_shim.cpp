// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" wrapper around the UNMODIFIED reference library
// (/root/reference/proj/core, built out-of-tree by oracle/Makefile into
// oracle/_ref/).  It lets the Python tests, golden-fixture generator and the
// bench's `--impl reference` arm drive the reference's own C++ operators
// through ctypes.  No reference source is copied here; every function just
// marshals flat arrays into coatsim types and calls the reference symbol:
//
//   encode_byte / decode_byte / round_bf16      proj/core/include/coatsim/fp8.hpp:47-70
//   quantize / dequantize / group_scale_max     proj/core/include/coatsim/quantize.hpp:70-77
//   measure_group / expand_quantize / dequantize_contract
//                                               proj/core/include/coatsim/expand.hpp:50-71
//   make_slot / step / reference_adamw_step     proj/core/include/coatsim/optimizer.hpp:54-62
//   generate                                    proj/core/include/coatsim/synthetic.hpp:33
//   write_slot / read_slot                      proj/core/include/coatsim/optimizer.hpp:71-74
//
// Exceptions are mapped onto the same status numbering as include/coat.h
// (coat_status), so parity tests can compare error behaviour too.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <thread>
#include <vector>

#include "coatsim/errors.hpp"
#include "coatsim/expand.hpp"
#include "coatsim/flow.hpp"
#include "coatsim/fp8.hpp"
#include "coatsim/optimizer.hpp"
#include "coatsim/quantize.hpp"
#include "coatsim/synthetic.hpp"
#include "coatsim/tensor.hpp"

using namespace coatsim;

namespace {

enum : int {
    ST_OK = 0,
    ST_SHAPE = 1,
    ST_GEOMETRY = 2,
    ST_NONFINITE_INPUT = 3,
    ST_NONFINITE_GRAD = 4,
    ST_INVALID = 5,
    ST_OUT_OF_RANGE = 8,
    ST_ALL_ZERO_GROUP = 9,
    ST_IO = 10,
    ST_BAD_MAGIC = 11,
    ST_OTHER = 99,
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return ST_OK;
    } catch (const NonFiniteGradient&) {
        return ST_NONFINITE_GRAD;
    } catch (const NonFiniteInput&) {
        return ST_NONFINITE_INPUT;
    } catch (const GeometryMismatch&) {
        return ST_GEOMETRY;
    } catch (const ShapeMismatch&) {
        return ST_SHAPE;
    } catch (const InvalidSpec&) {
        return ST_INVALID;
    } catch (const OutOfRange&) {
        return ST_OUT_OF_RANGE;
    } catch (const AllZeroGroup&) {
        return ST_ALL_ZERO_GROUP;
    } catch (const BadMagic&) {
        return ST_BAD_MAGIC;
    } catch (const IoError&) {
        return ST_IO;
    } catch (...) {
        return ST_OTHER;
    }
}

std::vector<int64_t> shape_of(const int64_t* shape, int rank) {
    return std::vector<int64_t>(shape, shape + rank);
}

Tensor tensor_of(const float* x, const int64_t* shape, int rank) {
    Tensor t(shape_of(shape, rank));
    std::memcpy(t.data.data(), x, sizeof(float) * size_t(t.numel()));
    return t;
}

QuantGeometry geometry_of(int mode, int64_t size) {
    switch (mode) {
        case 0: return QuantGeometry::per_tensor();
        case 1: return QuantGeometry::per_group(size);
        default: return QuantGeometry::per_block(size);
    }
}

// Flat E4M3 expanded moment state <-> arrays (scales as f32, as the reference keeps them).
ExpandedQuantState state_of(const uint8_t* codes, const float* scales, const float* k,
                            const float* c, int64_t npad, int64_t G) {
    ExpandedQuantState s;
    s.quantized.codes.assign(codes, codes + npad);
    s.quantized.scales.assign(scales, scales + npad / G);
    s.quantized.geometry = QuantGeometry::per_group(G);
    s.quantized.format = Fp8Tag::E4M3;
    s.quantized.source_shape = {npad};
    s.params.resize(size_t(npad / G));
    for (int64_t g = 0; g < npad / G; ++g) {
        s.params[size_t(g)].k = k[g];
        s.params[size_t(g)].c = c[g];
        s.params[size_t(g)].degenerate = k[g] == 1.0f;
    }
    return s;
}

void unstate(const ExpandedQuantState& s, uint8_t* codes, float* scales, float* k, float* c) {
    std::copy(s.quantized.codes.begin(), s.quantized.codes.end(), codes);
    std::copy(s.quantized.scales.begin(), s.quantized.scales.end(), scales);
    for (size_t g = 0; g < s.params.size(); ++g) {
        k[g] = s.params[g].k;
        c[g] = s.params[g].c;
    }
}

SlotPolicy dre_policy(int64_t G) {
    SlotPolicy p;
    p.first = MomentPolicy{StateFormat::E4M3, true, G};
    p.second = MomentPolicy{StateFormat::E4M3, true, G};
    return p;
}

int step_one(float* w, const float* g, int64_t n, int64_t G, uint8_t* mc, float* ms, float* mk,
             float* mcc, uint8_t* vc, float* vs, float* vk, float* vcc, int64_t step_in,
             float b1, float b2, float lr, float wd, float eps) {
    return guarded([&] {
        const int64_t npad = ((n + G - 1) / G) * G;
        OptimizerSlot slot;
        slot.shape = {n};
        slot.policy = dre_policy(G);
        slot.m = state_of(mc, ms, mk, mcc, npad, G);
        slot.v = state_of(vc, vs, vk, vcc, npad, G);
        slot.step = step_in;
        Tensor params = Tensor::from({n}, std::vector<float>(w, w + n));
        const Tensor grads = Tensor::from({n}, std::vector<float>(g, g + n));
        AdamWConfig cfg;
        cfg.beta1 = b1;
        cfg.beta2 = b2;
        cfg.lr = lr;
        cfg.weight_decay = wd;
        cfg.eps = eps;
        std::exception_ptr err;
        try {
            coatsim::step(params, grads, slot, cfg);
        } catch (...) {
            err = std::current_exception();
        }
        // The reference mutates params before packing the moments and assigns
        // slot.m before packing v (optimizer.cpp:108-112), so a NonFiniteInput
        // from pack_moment(v) leaves params AND slot.m updated: write back
        // whatever the reference object now holds, then report the error.
        std::copy(params.data.begin(), params.data.end(), w);
        unstate(std::get<ExpandedQuantState>(slot.m), mc, ms, mk, mcc);
        unstate(std::get<ExpandedQuantState>(slot.v), vc, vs, vk, vcc);
        if (err) std::rethrow_exception(err);
    });
}

}  // namespace

extern "C" {

int ref_encode_e4m3(const float* x, uint8_t* out, int64_t n) {
    return guarded([&] {
        for (int64_t i = 0; i < n; ++i) out[i] = encode_byte(x[i], Fp8Format::e4m3());
    });
}

int ref_decode_e4m3(const uint8_t* codes, float* out, int64_t n) {
    return guarded([&] {
        for (int64_t i = 0; i < n; ++i) out[i] = decode_byte(codes[i], Fp8Format::e4m3());
    });
}

int ref_round_bf16(const float* x, float* out, int64_t n) {
    return guarded([&] {
        for (int64_t i = 0; i < n; ++i) out[i] = round_bf16(x[i]);
    });
}

// mode: 0 per-tensor, 1 per-group(size), 2 per-block(size).  scales: one f32 per group.
int ref_quantize(const float* x, const int64_t* shape, int rank, int mode, int64_t size,
                 uint8_t* codes, float* scales, int64_t* n_groups) {
    return guarded([&] {
        const QuantizedTensor q =
            quantize(tensor_of(x, shape, rank), geometry_of(mode, size), Fp8Format::e4m3());
        std::copy(q.codes.begin(), q.codes.end(), codes);
        std::copy(q.scales.begin(), q.scales.end(), scales);
        *n_groups = q.group_count();
    });
}

int ref_dequantize(const uint8_t* codes, const float* scales, const int64_t* shape, int rank,
                   int mode, int64_t size, float* out) {
    return guarded([&] {
        QuantizedTensor q;
        q.source_shape = shape_of(shape, rank);
        q.geometry = geometry_of(mode, size);
        q.format = Fp8Tag::E4M3;
        const int64_t n = shape_numel(q.source_shape);
        const GroupIndexer idx(q.source_shape, q.geometry);
        q.codes.assign(codes, codes + n);
        q.scales.assign(scales, scales + idx.group_count());
        const Tensor t = dequantize(q);
        std::copy(t.data.begin(), t.data.end(), out);
    });
}

int ref_group_scale_max(const float* x, const int64_t* shape, int rank, int64_t G,
                        float* intermediate, float* global) {
    return guarded([&] {
        const auto [inter, gmax] = group_scale_max(tensor_of(x, shape, rank), G);
        std::copy(inter.data.begin(), inter.data.end(), intermediate);
        *global = gmax;
    });
}

float ref_absmax(const float* x, int64_t n) {
    return absmax(std::span<const float>(x, size_t(n)));
}

int ref_measure_group(const float* x, int64_t n, float* k, float* c, float* range,
                      int* degenerate) {
    return guarded([&] {
        const ExpansionParams p = measure_group(std::span<const float>(x, size_t(n)));
        *k = p.k;
        *c = p.c;
        *range = p.measured_range;
        *degenerate = p.degenerate ? 1 : 0;
    });
}

int ref_optimal_k(double range, float* k, int* degenerate) {
    return guarded([&] {
        const OptimalK ok = optimal_k(range);
        *k = ok.k;
        *degenerate = ok.degenerate ? 1 : 0;
    });
}

// x is a flat tensor of n elements (n % G == 0 required, as in the reference).
int ref_expand_quantize(const float* x, int64_t n, int64_t G, uint8_t* codes, float* scales,
                        float* k, float* c) {
    return guarded([&] {
        const ExpandedQuantState s =
            expand_quantize(Tensor::from({n}, std::vector<float>(x, x + n)), G, Fp8Format::e4m3());
        unstate(s, codes, scales, k, c);
    });
}

int ref_dequantize_contract(const uint8_t* codes, const float* scales, const float* k,
                            const float* c, int64_t n, int64_t G, float* out) {
    return guarded([&] {
        const Tensor t = dequantize_contract(state_of(codes, scales, k, c, n, G));
        std::copy(t.data.begin(), t.data.end(), out);
    });
}

// Expanded (pre-quantization) values f(x) for given per-group params.
int ref_expand(const float* x, const float* k, const float* c, int64_t n, int64_t G, float* out) {
    return guarded([&] {
        std::vector<ExpansionParams> p(size_t(n / G));
        for (size_t g = 0; g < p.size(); ++g) {
            p[g].k = k[g];
            p[g].c = c[g];
        }
        const Tensor t = expand(Tensor::from({n}, std::vector<float>(x, x + n)), p, G);
        std::copy(t.data.begin(), t.data.end(), out);
    });
}

int ref_make_slot(int64_t n, int64_t G, uint8_t* mc, float* ms, float* mk, float* mcc,
                  uint8_t* vc, float* vs, float* vk, float* vcc) {
    return guarded([&] {
        const OptimizerSlot slot = make_slot({n}, dre_policy(G));
        unstate(std::get<ExpandedQuantState>(slot.m), mc, ms, mk, mcc);
        unstate(std::get<ExpandedQuantState>(slot.v), vc, vs, vk, vcc);
    });
}

// coatsim::step on a flat parameter tensor with the north-star policy
// {E4M3, expand, G} for both moments.  State arrays are in/out.
int ref_step(float* w, const float* g, int64_t n, int64_t G, uint8_t* mc, float* ms, float* mk,
             float* mcc, uint8_t* vc, float* vs, float* vk, float* vcc, int64_t step_in,
             float b1, float b2, float lr, float wd, float eps) {
    return step_one(w, g, n, G, mc, ms, mk, mcc, vc, vs, vk, vcc, step_in, b1, b2, lr, wd, eps);
}

// Same, sharded over `threads` std::threads at G-aligned boundaries.  The
// reference is reentrant and groups are independent, so the
// result is bitwise identical to ref_step (checked by the tests).
int ref_step_mt(int threads, float* w, const float* g, int64_t n, int64_t G, uint8_t* mc,
                float* ms, float* mk, float* mcc, uint8_t* vc, float* vs, float* vk, float* vcc,
                int64_t step_in, float b1, float b2, float lr, float wd, float eps) {
    if (threads <= 1) {
        return step_one(w, g, n, G, mc, ms, mk, mcc, vc, vs, vk, vcc, step_in, b1, b2, lr, wd,
                        eps);
    }
    const int64_t groups = (n + G - 1) / G;
    const int64_t per = (groups + threads - 1) / threads;
    std::vector<std::thread> pool;
    std::vector<int> st(size_t(threads), ST_OK);
    for (int t = 0; t < threads; ++t) {
        const int64_t g0 = std::min(groups, int64_t(t) * per);
        const int64_t g1 = std::min(groups, g0 + per);
        if (g0 >= g1) continue;
        const int64_t e0 = g0 * G;
        const int64_t e1 = std::min(n, g1 * G);
        pool.emplace_back([=, &st] {
            st[size_t(t)] = step_one(w + e0, g + e0, e1 - e0, G, mc + e0, ms + g0, mk + g0,
                                     mcc + g0, vc + e0, vs + g0, vk + g0, vcc + g0, step_in, b1,
                                     b2, lr, wd, eps);
        });
    }
    for (auto& th : pool) th.join();
    for (int s : st)
        if (s != ST_OK) return s;
    return ST_OK;
}

int ref_reference_adamw_step(float* w, float* m, float* v, const float* g, int64_t n, float b1,
                             float b2, float lr, float wd, float eps, int64_t t) {
    return guarded([&] {
        Tensor params = Tensor::from({n}, std::vector<float>(w, w + n));
        Tensor mm = Tensor::from({n}, std::vector<float>(m, m + n));
        Tensor vv = Tensor::from({n}, std::vector<float>(v, v + n));
        const Tensor grads = Tensor::from({n}, std::vector<float>(g, g + n));
        AdamWConfig cfg;
        cfg.beta1 = b1;
        cfg.beta2 = b2;
        cfg.lr = lr;
        cfg.weight_decay = wd;
        cfg.eps = eps;
        reference_adamw_step(params, mm, vv, grads, cfg, t);
        std::copy(params.data.begin(), params.data.end(), w);
        std::copy(mm.data.begin(), mm.data.end(), m);
        std::copy(vv.data.begin(), vv.data.end(), v);
    });
}

// kind: 0 OptimizerLike, 1 ActivationWithOutliers, 2 UniformLog.
int ref_generate(int kind, const int64_t* shape, int rank, double frac, double scale,
                 uint64_t seed, float* out) {
    return guarded([&] {
        SyntheticSpec spec;
        spec.kind = SyntheticKind(kind);
        spec.shape = shape_of(shape, rank);
        spec.outlier_fraction = frac;
        spec.outlier_scale = scale;
        spec.seed = seed;
        const Tensor t = generate(spec);
        std::copy(t.data.begin(), t.data.end(), out);
    });
}

// Serialize an E4M3+expand slot of a flat tensor with the reference's own writer.
int ref_save_slot(const char* path, int64_t n, int64_t G, const uint8_t* mc, const float* ms,
                  const float* mk, const float* mcc, const uint8_t* vc, const float* vs,
                  const float* vk, const float* vcc, int64_t step, float b1, float b2, float lr,
                  float wd, float eps) {
    return guarded([&] {
        const int64_t npad = ((n + G - 1) / G) * G;
        OptimizerSlot slot;
        slot.shape = {n};
        slot.policy = dre_policy(G);
        slot.m = state_of(mc, ms, mk, mcc, npad, G);
        slot.v = state_of(vc, vs, vk, vcc, npad, G);
        slot.step = step;
        AdamWConfig cfg;
        cfg.beta1 = b1;
        cfg.beta2 = b2;
        cfg.lr = lr;
        cfg.weight_decay = wd;
        cfg.eps = eps;
        cfg.step = step;
        save_slot(path, slot, cfg);
    });
}

// Load a slot written by anyone; returns the flat state (npad = padded length).
int ref_load_slot(const char* path, int64_t n, int64_t G, uint8_t* mc, float* ms, float* mk,
                  float* mcc, uint8_t* vc, float* vs, float* vk, float* vcc, int64_t* step,
                  float* cfg5) {
    return guarded([&] {
        auto [slot, cfg] = load_slot(path);
        if (slot.shape != std::vector<int64_t>{n}) throw ShapeMismatch("ref_load_slot: shape");
        (void)G;
        unstate(std::get<ExpandedQuantState>(slot.m), mc, ms, mk, mcc);
        unstate(std::get<ExpandedQuantState>(slot.v), vc, vs, vk, vcc);
        *step = slot.step;
        cfg5[0] = cfg.beta1;
        cfg5[1] = cfg.beta2;
        cfg5[2] = cfg.lr;
        cfg5[3] = cfg.weight_decay;
        cfg5[4] = cfg.eps;
    });
}


// Run the reference COAT DecoderLayer forward (flow.cpp:546-612) on x and
// return one saved record of its tape: codes, scales (float) and -- for the
// rmsnorm weights the producers need -- rms1/rms2.  kind: 0 per-group,
// 1 per-tensor, 2 dense.  Test infrastructure for the fused producers.
int ref_layer_tape(int64_t H, int64_t I, int64_t heads, int64_t S, int64_t B, uint64_t seed, const float* x,
                   const char* name, uint8_t* codes, float* scales, int64_t* n_scales, int* kind, float* rms1,
                   float* rms2) {
    return guarded([&] {
        LayerSpec spec;
        spec.hidden = H;
        spec.intermediate = I;
        spec.num_heads = heads;
        spec.seq_len = S;
        spec.batch = B;
        spec.group_size = 16;
        spec.policy = FlowPolicy::COAT;
        DecoderLayer layer(spec, LayerWeights::random(spec, seed));
        const int64_t n = B * S * H;
        const Tensor xt = Tensor::from({B, S, H}, std::vector<float>(x, x + n));
        const ForwardResult res = layer.forward(xt);
        const SavedActivation& rec = res.tape.find(name);
        *kind = rec.kind == SaveKind::Fp8PerGroup ? 0 : rec.kind == SaveKind::Fp8PerTensor ? 1 : 2;
        if (*kind <= 1) {
            std::copy(rec.q.codes.begin(), rec.q.codes.end(), codes);
            std::copy(rec.q.scales.begin(), rec.q.scales.end(), scales);
            *n_scales = int64_t(rec.q.scales.size());
        } else {
            *n_scales = 0;
        }
        std::copy(layer.weights().rms1.data.begin(), layer.weights().rms1.data.end(), rms1);
        std::copy(layer.weights().rms2.data.begin(), layer.weights().rms2.data.end(), rms2);
    });
}

}  // extern "C"
