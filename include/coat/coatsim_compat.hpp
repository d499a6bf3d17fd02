// include/coat/coatsim_compat.hpp -- drop-in C++ replacement of the reference's
// proj/core operator API (coatsim, /root/reference/proj/core/include/coatsim)
// for the COAT hot path, implemented over the C-ABI of include/coat.h.
//
// A user of the reference switches with
//     #include <coat/coatsim_compat.hpp>
//     namespace coatsim = coat_b200;
// and links libcoat.so + cudart.  Types and signatures follow the reference:
//
//   errors.hpp:8-22          Error, NonFiniteInput, NonFiniteGradient, ...
//   tensor.hpp:14-36         Tensor (host fp32, row-major, value semantics)
//   fp8.hpp:47-70            encode_byte / decode_byte / round_bf16 (E4M3)
//   quantize.hpp:14-81       QuantGeometry, QuantizedTensor, quantize, dequantize,
//                            group_scale_max, quantization_error
//   expand.hpp:21-71         ExpansionParams, ExpandedQuantState, expand_quantize,
//                            dequantize_contract
//   optimizer.hpp:13-62      AdamWConfig, StateFormat, MomentPolicy, SlotPolicy,
//                            OptimizerSlot, make_slot, step
//
// Differences by design: the optimizer state of an OptimizerSlot lives in HBM
// (that is the point of the B200 path) -- read it back with slot.m()/slot.v();
// only the E4M3 format, per-group/per-tensor geometry and the {E4M3, expand,
// 128} optimizer policy are implemented (InvalidSpec otherwise).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../coat.h"

namespace coat_b200 {

// ------------------------------------------------------------------ errors --
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NonFiniteInput : Error { using Error::Error; };
struct NonFiniteGradient : Error { using Error::Error; };
struct OutOfRange : Error { using Error::Error; };
struct GeometryMismatch : Error { using Error::Error; };
struct ShapeMismatch : Error { using Error::Error; };
struct AllZeroGroup : Error { using Error::Error; };
struct InvalidSpec : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct BadMagic : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

namespace detail {
inline void check(coat_status s) {
    if (s == COAT_OK) return;
    const std::string msg = std::string(coat_status_string(s)) + ": " + coat_last_error();
    switch (s) {
        case COAT_ERR_SHAPE: throw ShapeMismatch(msg);
        case COAT_ERR_GEOMETRY: throw GeometryMismatch(msg);
        case COAT_ERR_NONFINITE_INPUT: throw NonFiniteInput(msg);
        case COAT_ERR_NONFINITE_GRAD: throw NonFiniteGradient(msg);
        case COAT_ERR_INVALID: throw InvalidSpec(msg);
        case COAT_ERR_OUT_OF_RANGE: throw OutOfRange(msg);
        case COAT_ERR_ALL_ZERO_GROUP: throw AllZeroGroup(msg);
        case COAT_ERR_IO: throw IoError(msg);
        case COAT_ERR_BAD_MAGIC: throw BadMagic(msg);
        default: throw CudaError(msg);
    }
}
inline void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw CudaError(cudaGetErrorString(e));
}

// Owning device buffer.
template <typename T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    Dev() = default;
    explicit Dev(size_t count) : n(count) { cuda(cudaMalloc(&p, sizeof(T) * (count ? count : 1))); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    Dev& operator=(Dev&& o) noexcept { std::swap(p, o.p); std::swap(n, o.n); return *this; }
    ~Dev() { if (p) cudaFree(p); }
    void upload(const T* h, size_t count) { cuda(cudaMemcpy(p, h, sizeof(T) * count, cudaMemcpyHostToDevice)); }
    void download(T* h, size_t count) const { cuda(cudaMemcpy(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost)); }
};

inline uint32_t read_flags(const Dev<uint32_t>& f) {
    uint32_t v = 0;
    f.download(&v, 1);
    return v;
}
inline float bf16_to_float(uint16_t b) {
    const uint32_t u = uint32_t(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
inline uint16_t float_to_bf16(float f) {   // f is BF16-valued (reference scales always are)
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return uint16_t(u >> 16);
}
}  // namespace detail

// ------------------------------------------------------------------ tensor --
inline int64_t shape_numel(const std::vector<int64_t>& shape) {
    int64_t n = 1;
    for (int64_t d : shape) {
        if (d <= 0) throw InvalidSpec("tensor dimensions must be positive");
        n *= d;
    }
    return n;
}

struct Tensor {
    std::vector<int64_t> shape;
    std::vector<float> data;
    Tensor() = default;
    explicit Tensor(std::vector<int64_t> s, float fill = 0.0f)
        : shape(std::move(s)), data(size_t(shape_numel(shape)), fill) {}
    static Tensor from(std::vector<int64_t> s, std::vector<float> values) {
        Tensor t;
        t.shape = std::move(s);
        if (shape_numel(t.shape) != int64_t(values.size())) throw ShapeMismatch("element count does not match shape");
        t.data = std::move(values);
        return t;
    }
    int64_t numel() const { return int64_t(data.size()); }
    int64_t last_dim() const { return shape.empty() ? 1 : shape.back(); }
    int64_t rows() const { return numel() / last_dim(); }
    float& operator[](int64_t i) { return data[size_t(i)]; }
    float operator[](int64_t i) const { return data[size_t(i)]; }
};

// ------------------------------------------------------------------- codec --
enum class Fp8Tag : uint8_t { E4M3 = 0, E5M2 = 1, DE8 = 2 };
struct Fp8Format {
    Fp8Tag tag;
    float delta_max, delta_min;
    int mantissa_bits, exponent_bits;
    static const Fp8Format& e4m3() {
        static const Fp8Format f{Fp8Tag::E4M3, 448.0f, 0x1p-9f, 3, 4};
        return f;
    }
    double dynamic_range() const { return double(delta_max) / double(delta_min); }
};
inline void require_e4m3(const Fp8Format& f) {
    if (f.tag != Fp8Tag::E4M3) throw InvalidSpec("only E4M3 is implemented on the B200 path");
}

// Elementwise over a vector (one kernel launch); NonFiniteInput like encode_byte.
inline std::vector<uint8_t> encode_bytes(const std::vector<float>& x) {
    detail::Dev<float> dx{x.size()};
    detail::Dev<uint8_t> dc{x.size()};
    detail::Dev<uint32_t> fl{1};
    detail::cuda(cudaMemset(fl.p, 0, 4));
    dx.upload(x.data(), x.size());
    detail::check(coat_encode_e4m3(dx.p, dc.p, int64_t(x.size()), fl.p, nullptr));
    if (detail::read_flags(fl)) throw NonFiniteInput("encode: value is not finite");
    std::vector<uint8_t> out(x.size());
    dc.download(out.data(), out.size());
    return out;
}
inline std::vector<float> decode_bytes(const std::vector<uint8_t>& c) {
    detail::Dev<uint8_t> dc{c.size()};
    detail::Dev<float> dx{c.size()};
    dc.upload(c.data(), c.size());
    detail::check(coat_decode_e4m3(dc.p, dx.p, int64_t(c.size()), nullptr));
    std::vector<float> out(c.size());
    dx.download(out.data(), out.size());
    return out;
}
inline uint8_t encode_byte(float v, const Fp8Format& f = Fp8Format::e4m3()) {
    require_e4m3(f);
    return encode_bytes({v})[0];
}
inline float decode_byte(uint8_t b, const Fp8Format& f = Fp8Format::e4m3()) {
    require_e4m3(f);
    return decode_bytes({b})[0];
}
inline float round_bf16(float value) {   // fp8.cpp:209-216 (host arithmetic, identical)
    uint32_t bits;
    std::memcpy(&bits, &value, 4);
    if ((bits & 0x7FFFFFFFu) > 0x7F800000u) return value;
    bits += 0x7FFFu + ((bits >> 16) & 1u);
    bits &= 0xFFFF0000u;
    float r;
    std::memcpy(&r, &bits, 4);
    return r;
}

// --------------------------------------------------------------- quantizer --
enum class QuantMode : uint8_t { PerTensor = 0, PerGroup = 1, PerBlock = 2 };
struct QuantGeometry {
    QuantMode mode = QuantMode::PerTensor;
    int64_t group_size = 0;
    int64_t block_size = 0;
    static QuantGeometry per_tensor() { return {QuantMode::PerTensor, 0, 0}; }
    static QuantGeometry per_group(int64_t g) { return {QuantMode::PerGroup, g, 0}; }
    static QuantGeometry per_block(int64_t b) { return {QuantMode::PerBlock, 0, b}; }
    bool operator==(const QuantGeometry&) const = default;
};
struct QuantizedTensor {
    std::vector<uint8_t> codes;
    std::vector<float> scales;
    QuantGeometry geometry;
    Fp8Tag format = Fp8Tag::E4M3;
    std::vector<int64_t> source_shape;
    int64_t numel() const { return int64_t(codes.size()); }
    int64_t group_count() const { return int64_t(scales.size()); }
};

inline QuantizedTensor quantize(const Tensor& x, QuantGeometry geometry,
                                const Fp8Format& format = Fp8Format::e4m3()) {
    require_e4m3(format);
    const int64_t n = x.numel(), cols = x.last_dim(), rows = n / cols;
    detail::Dev<float> dx{size_t(n)};
    detail::Dev<uint8_t> dc{size_t(n)};
    detail::Dev<uint32_t> fl{1};
    detail::cuda(cudaMemset(fl.p, 0, 4));
    QuantizedTensor q;
    q.geometry = geometry;
    q.source_shape = x.shape;
    std::vector<uint16_t> s16;
    if (geometry.mode == QuantMode::PerGroup) {
        if (geometry.group_size <= 0) throw GeometryMismatch("per-group: group size must be positive");
        if (cols % geometry.group_size != 0) throw GeometryMismatch("per-group: last dim not divisible by group size");
        dx.upload(x.data.data(), size_t(n));
        detail::Dev<uint16_t> ds{size_t(n / geometry.group_size)};
        detail::check(coat_quantize_per_group(dx.p, 0, rows, cols, geometry.group_size, dc.p, ds.p, fl.p, nullptr));
        s16.resize(ds.n);
        ds.download(s16.data(), s16.size());
    } else if (geometry.mode == QuantMode::PerTensor) {
        dx.upload(x.data.data(), size_t(n));
        detail::Dev<uint32_t> amax{1};
        detail::Dev<uint16_t> ds{1};
        const int64_t g1 = cols % 128 == 0 ? 128 : cols;
        detail::check(coat_group_scale_max(dx.p, 0, rows, cols, g1, nullptr, amax.p, nullptr));
        detail::check(coat_quantize_per_tensor(dx.p, 0, n, amax.p, dc.p, ds.p, fl.p, nullptr));
        s16.resize(1);
        ds.download(s16.data(), 1);
    } else {
        throw InvalidSpec("per-block geometry is outside the B200 hot path");
    }
    if (detail::read_flags(fl)) throw NonFiniteInput("quantize: tensor has non-finite values");
    q.codes.resize(size_t(n));
    dc.download(q.codes.data(), q.codes.size());
    q.scales.resize(s16.size());
    for (size_t i = 0; i < s16.size(); ++i) q.scales[i] = detail::bf16_to_float(s16[i]);
    return q;
}

inline Tensor dequantize(const QuantizedTensor& q) {
    Tensor out(q.source_shape);
    const int64_t n = out.numel(), cols = out.last_dim();
    detail::Dev<uint8_t> dc{size_t(n)};
    detail::Dev<uint16_t> ds{q.scales.size()};
    detail::Dev<float> dx{size_t(n)};
    dc.upload(q.codes.data(), size_t(n));
    std::vector<uint16_t> s16(q.scales.size());
    for (size_t i = 0; i < s16.size(); ++i) s16[i] = detail::float_to_bf16(q.scales[i]);
    ds.upload(s16.data(), s16.size());
    if (q.geometry.mode == QuantMode::PerGroup)
        detail::check(coat_dequantize_per_group(dc.p, ds.p, n / cols, cols, q.geometry.group_size, dx.p, 0, nullptr));
    else if (q.geometry.mode == QuantMode::PerTensor)
        detail::check(coat_dequantize_per_tensor(dc.p, ds.p, n, dx.p, 0, nullptr));
    else
        throw InvalidSpec("per-block geometry is outside the B200 hot path");
    dx.download(out.data.data(), size_t(n));
    return out;
}

inline std::pair<Tensor, float> group_scale_max(const Tensor& x, int64_t group_size) {
    if (group_size <= 0) throw GeometryMismatch("group_scale_max: group size must be positive");
    if (x.last_dim() % group_size != 0) throw GeometryMismatch("group_scale_max: last dim not divisible by group size");
    std::vector<int64_t> ishape = x.shape;
    ishape.back() /= group_size;
    Tensor inter(ishape);
    detail::Dev<float> dx{size_t(x.numel())}, di{size_t(inter.numel())};
    detail::Dev<uint32_t> amax{1};
    dx.upload(x.data.data(), size_t(x.numel()));
    detail::check(coat_group_scale_max(dx.p, 0, x.rows(), x.last_dim(), group_size, di.p, amax.p, nullptr));
    di.download(inter.data.data(), size_t(inter.numel()));
    uint32_t bits = 0;
    amax.download(&bits, 1);
    float g;
    std::memcpy(&g, &bits, 4);
    return {std::move(inter), g};
}

// --------------------------------------------------------- range expansion --
inline constexpr double kRangeE4M3 = 229376.0;
inline constexpr double kDefaultKMax = 20.0;
struct ExpansionParams {
    float k = 1.0f, c = 1.0f, measured_range = 0.0f;
    bool degenerate = false;
};
struct ExpandedQuantState {
    QuantizedTensor quantized;
    std::vector<ExpansionParams> params;
};

namespace detail {
struct DevMoment {
    Dev<uint8_t> codes;
    Dev<uint16_t> scales;
    Dev<float> k, c;
    DevMoment() = default;
    explicit DevMoment(int64_t npad)
        : codes(size_t(npad)), scales(size_t(npad / 128)), k(size_t(npad / 128)), c(size_t(npad / 128)) {}
    coat_moment_state cs() const { return {codes.p, scales.p, k.p, c.p}; }
    // device-to-device deep copy (OptimizerSlot is a value type in the reference)
    std::shared_ptr<DevMoment> clone() const {
        auto o = std::make_shared<DevMoment>(int64_t(codes.n));
        cuda(cudaMemcpy(o->codes.p, codes.p, codes.n, cudaMemcpyDeviceToDevice));
        cuda(cudaMemcpy(o->scales.p, scales.p, 2 * scales.n, cudaMemcpyDeviceToDevice));
        cuda(cudaMemcpy(o->k.p, k.p, 4 * k.n, cudaMemcpyDeviceToDevice));
        cuda(cudaMemcpy(o->c.p, c.p, 4 * c.n, cudaMemcpyDeviceToDevice));
        return o;
    }
    void upload(const ExpandedQuantState& s) {
        codes.upload(s.quantized.codes.data(), codes.n);
        std::vector<uint16_t> s16(scales.n);
        std::vector<float> kk(k.n), cc(c.n);
        for (size_t g = 0; g < scales.n; ++g) {
            s16[g] = float_to_bf16(s.quantized.scales[g]);
            kk[g] = s.params[g].k;
            cc[g] = s.params[g].c;
        }
        scales.upload(s16.data(), s16.size());
        k.upload(kk.data(), kk.size());
        c.upload(cc.data(), cc.size());
    }
    ExpandedQuantState download(const std::vector<int64_t>& shape) const {
        ExpandedQuantState s;
        s.quantized.codes.resize(codes.n);
        codes.download(s.quantized.codes.data(), codes.n);
        std::vector<uint16_t> s16(scales.n);
        std::vector<float> kk(k.n), cc(c.n);
        scales.download(s16.data(), s16.size());
        k.download(kk.data(), kk.size());
        c.download(cc.data(), cc.size());
        s.quantized.scales.resize(scales.n);
        s.params.resize(scales.n);
        for (size_t g = 0; g < scales.n; ++g) {
            s.quantized.scales[g] = bf16_to_float(s16[g]);
            s.params[g].k = kk[g];
            s.params[g].c = cc[g];
            s.params[g].degenerate = kk[g] == 1.0f;   // as read_expanded (tensor_io.cpp:171-172)
        }
        s.quantized.geometry = QuantGeometry::per_group(128);
        s.quantized.source_shape = shape;
        return s;
    }
};
}  // namespace detail

inline ExpandedQuantState expand_quantize(const Tensor& x, int64_t group_size,
                                          const Fp8Format& format = Fp8Format::e4m3()) {
    require_e4m3(format);
    const int64_t n = x.numel();
    if (group_size <= 0 || x.last_dim() % group_size != 0) throw GeometryMismatch("per-group: last dim not divisible by group size");
    if (group_size != 128) throw InvalidSpec("the B200 DRE kernels implement the 1x128 group only");
    detail::Dev<float> dx{size_t(n)};
    detail::DevMoment st{n};
    detail::Dev<uint32_t> fl{1};
    detail::cuda(cudaMemset(fl.p, 0, 4));
    dx.upload(x.data.data(), size_t(n));
    detail::check(coat_expand_quantize(dx.p, n, group_size, st.cs(), fl.p, nullptr));
    if (detail::read_flags(fl)) throw NonFiniteInput("expand_quantize: tensor has non-finite values");
    return st.download(x.shape);
}

inline Tensor dequantize_contract(const ExpandedQuantState& s) {
    const int64_t n = s.quantized.numel();
    detail::DevMoment st{n};
    st.upload(s);
    detail::Dev<float> dx{size_t(n)};
    detail::Dev<uint32_t> fl{1};
    detail::cuda(cudaMemset(fl.p, 0, 4));
    detail::check(coat_dequantize_contract(st.cs(), n, 128, dx.p, fl.p, nullptr));
    if (detail::read_flags(fl)) throw NonFiniteInput("contract: tensor has non-finite values");
    Tensor out(s.quantized.source_shape.empty() ? std::vector<int64_t>{n} : s.quantized.source_shape);
    dx.download(out.data.data(), size_t(n));
    return out;
}

// --------------------------------------------------------------- optimizer --
struct AdamWConfig {
    float beta1 = 0.9f, beta2 = 0.999f, lr = 1e-3f, weight_decay = 0.0f, eps = 1e-8f;
    int64_t step = 0;
};
enum class StateFormat : uint8_t { FP32 = 0, E4M3 = 1, E5M2 = 2, DE8 = 3 };
struct MomentPolicy {
    StateFormat format = StateFormat::E4M3;
    bool expand = true;
    int64_t group_size = 128;
};
struct SlotPolicy {
    MomentPolicy first, second;
};

// The state lives in HBM: two buffer sets per moment (ping-pong) so a failed
// step commits exactly what the reference commits (optimizer.cpp:101-114).
// OptimizerSlot is a VALUE type as in the reference (optimizer.hpp:48-52):
// copying a slot deep-copies its device state (both ping-pong sets), so
// stepping a copy never touches the original's moments.  Moves are cheap.
struct OptimizerSlot {
    std::vector<int64_t> shape;
    SlotPolicy policy;
    int64_t step = 0;
    int64_t npad = 0;
    std::shared_ptr<detail::DevMoment> mbuf[2], vbuf[2];
    int cm = 0, cv = 0;
    ExpandedQuantState m() const { return mbuf[cm]->download({npad}); }
    ExpandedQuantState v() const { return vbuf[cv]->download({npad}); }

    OptimizerSlot() = default;
    OptimizerSlot(OptimizerSlot&&) noexcept = default;
    OptimizerSlot& operator=(OptimizerSlot&&) noexcept = default;
    OptimizerSlot(const OptimizerSlot& o)
        : shape(o.shape), policy(o.policy), step(o.step), npad(o.npad), cm(o.cm), cv(o.cv) {
        for (int i = 0; i < 2; ++i) {
            if (o.mbuf[i]) mbuf[i] = o.mbuf[i]->clone();
            if (o.vbuf[i]) vbuf[i] = o.vbuf[i]->clone();
        }
    }
    OptimizerSlot& operator=(const OptimizerSlot& o) {
        if (this != &o) {
            OptimizerSlot tmp(o);
            *this = std::move(tmp);
        }
        return *this;
    }
};

inline OptimizerSlot make_slot(const std::vector<int64_t>& shape, const SlotPolicy& policy = {}) {
    for (const MomentPolicy& p : {policy.first, policy.second})
        if (p.format != StateFormat::E4M3 || !p.expand || p.group_size != 128)
            throw InvalidSpec("the B200 optimizer implements the {E4M3, expand, 128} policy only");
    OptimizerSlot s;
    s.shape = shape;
    s.policy = policy;
    const int64_t n = shape_numel(shape);
    s.npad = (n + 127) / 128 * 128;
    for (int i = 0; i < 2; ++i) {
        s.mbuf[i] = std::make_shared<detail::DevMoment>(s.npad);
        s.vbuf[i] = std::make_shared<detail::DevMoment>(s.npad);
    }
    detail::check(coat_make_slot(n, 128, s.mbuf[0]->cs(), s.vbuf[0]->cs(), nullptr));
    return s;
}

inline void step(Tensor& params, const Tensor& grads, OptimizerSlot& slot, const AdamWConfig& cfg) {
    if (params.shape != slot.shape) throw ShapeMismatch("step: params do not match slot shape");
    if (params.shape != grads.shape) throw ShapeMismatch("step: shape mismatch");
    const int64_t n = params.numel();
    detail::Dev<float> w_in{size_t(n)}, w_out{size_t(n)}, g{size_t(n)};
    detail::Dev<uint32_t> fl{1};
    detail::cuda(cudaMemset(fl.p, 0, 4));
    w_in.upload(params.data.data(), size_t(n));
    g.upload(grads.data.data(), size_t(n));
    const coat_adamw_config c{cfg.beta1, cfg.beta2, cfg.lr, cfg.weight_decay, cfg.eps};
    detail::check(coat_adamw_dre_step(w_in.p, w_out.p, g.p, n, 128, slot.mbuf[slot.cm]->cs(), slot.vbuf[slot.cv]->cs(),
                                      slot.mbuf[1 - slot.cm]->cs(), slot.vbuf[1 - slot.cv]->cs(), &c,
                                      slot.step + 1, fl.p, nullptr));
    const uint32_t f = detail::read_flags(fl);
    if (f & COAT_FLAG_NONFINITE_GRAD) throw NonFiniteGradient("step: gradient has non-finite values");
    if (f & COAT_FLAG_CONTRACT) throw NonFiniteInput("contract: tensor has non-finite values");
    w_out.download(params.data.data(), size_t(n));
    if (f & COAT_FLAG_PACK_M) throw NonFiniteInput("expand_quantize: tensor has non-finite values");
    slot.cm = 1 - slot.cm;
    if (f & COAT_FLAG_PACK_V) throw NonFiniteInput("expand_quantize: tensor has non-finite values");
    slot.cv = 1 - slot.cv;
    slot.step += 1;
}

}  // namespace coat_b200
