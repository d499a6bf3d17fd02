// slot_io.cu -- optimizer-slot checkpoints in the reference's on-disk format
// (host code; the state lives on the device).
//
// Reference: write_slot / read_slot / save_slot / load_slot
// (proj/core/src/optimizer.cpp:196-252) and the CQT8 / EXPK records
// (proj/core/src/tensor_io.cpp:96-175), little-endian:
//   u32 header length, JSON header {beta1, beta2, eps, lr, policy{first,
//   second}{expand, format, group_size}, shape, step, weight_decay} (nlohmann
//   default: keys sorted, compact, floats as the shortest round-trip double),
//   then per moment (m, v): u8 kind = 2 (ExpandedQuantState), the CQT8 record
//   ("CQT8", u16 version 1, u8 Fp8Tag E4M3 = 0, u8 axis = 0, u32 group size,
//   u16 rank = 1, u64 npad, f32 scales[npad/G], u8 codes[npad]) and the EXPK
//   record ("EXPK", (f32 k, f32 c)[npad/G]).
// Files written here are byte-identical to the reference's for the same state
// and load in it, and the reference's files load here
// (tests/test_gpu_slot_io.py checks both directions against the compiled
// reference).
#include <cmath>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/coat.h"
#include "coat_internal.h"

namespace coat {
namespace {

// ---------------------------------------------------------------- JSON out --
// nlohmann::json's dump of a double: shortest round-trip digits (Grisu2 in
// nlohmann; std::to_chars here -- both produce the shortest digit string that
// round-trips), fixed notation for decimal exponents in (-4, 15], otherwise
// d.ddde+XX with at least two exponent digits, integral values with ".0".
std::string json_double(double x) {
    if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
    char buf[64];
    auto res = std::to_chars(buf, buf + sizeof(buf), x, std::chars_format::scientific);
    std::string sci(buf, res.ptr);
    const size_t epos = sci.find('e');
    std::string mant = sci.substr(0, epos);
    const int e10 = std::atoi(sci.c_str() + epos + 1);
    bool neg = false;
    if (mant[0] == '-') {
        neg = true;
        mant.erase(0, 1);
    }
    std::string digits;
    for (char ch : mant)
        if (ch != '.') digits.push_back(ch);
    const int k = int(digits.size());   // digits d1..dk, value = 0.d1..dk * 10^n
    const int n = e10 + 1;
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(size_t(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, size_t(n)) + "." + digits.substr(size_t(n));
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(size_t(-n), '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
    return neg ? "-" + out : out;
}

std::string header_json(const int64_t* shape, int rank, int64_t G, const coat_adamw_config& c, int64_t step) {
    const std::string pol = "{\"expand\":true,\"format\":\"e4m3\",\"group_size\":" + std::to_string(G) + "}";
    std::string shp = "[";
    for (int i = 0; i < rank; ++i) shp += (i ? "," : "") + std::to_string(shape[i]);
    shp += "]";
    return "{\"beta1\":" + json_double(c.beta1) + ",\"beta2\":" + json_double(c.beta2) + ",\"eps\":" +
           json_double(c.eps) + ",\"lr\":" + json_double(c.lr) + ",\"policy\":{\"first\":" + pol +
           ",\"second\":" + pol + "},\"shape\":" + shp + ",\"step\":" + std::to_string(step) +
           ",\"weight_decay\":" + json_double(c.weight_decay) + "}";
}

// ---------------------------------------------------------------- JSON in ---
struct JValue {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double num = 0.0;
    bool integral = false;
    int64_t i = 0;
    std::string s;
    std::vector<JValue> arr;
    std::map<std::string, JValue> obj;
    const JValue& at(const char* key) const {
        auto it = obj.find(key);
        if (kind != Obj || it == obj.end()) throw std::runtime_error(std::string("missing key ") + key);
        return it->second;
    }
};

struct JParser {
    const std::string& t;
    size_t p = 0;
    void ws() {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) ++p;
    }
    char peek() {
        ws();
        if (p >= t.size()) throw std::runtime_error("unexpected end of JSON");
        return t[p];
    }
    void expect(char c) {
        if (peek() != c) throw std::runtime_error("malformed JSON");
        ++p;
    }
    std::string str() {
        expect('"');
        std::string out;
        while (p < t.size() && t[p] != '"') {
            if (t[p] == '\\') ++p;
            out.push_back(t[p++]);
        }
        expect('"');
        return out;
    }
    JValue value() {
        JValue v;
        const char c = peek();
        if (c == '{') {
            ++p;
            v.kind = JValue::Obj;
            if (peek() == '}') { ++p; return v; }
            for (;;) {
                const std::string k = str();
                expect(':');
                v.obj[k] = value();
                if (peek() == ',') { ++p; continue; }
                expect('}');
                return v;
            }
        }
        if (c == '[') {
            ++p;
            v.kind = JValue::Arr;
            if (peek() == ']') { ++p; return v; }
            for (;;) {
                v.arr.push_back(value());
                if (peek() == ',') { ++p; continue; }
                expect(']');
                return v;
            }
        }
        if (c == '"') {
            v.kind = JValue::Str;
            v.s = str();
            return v;
        }
        if (t.compare(p, 4, "true") == 0) { p += 4; v.kind = JValue::Bool; v.b = true; return v; }
        if (t.compare(p, 5, "false") == 0) { p += 5; v.kind = JValue::Bool; return v; }
        if (t.compare(p, 4, "null") == 0) { p += 4; return v; }
        const size_t b = p;
        while (p < t.size() && (std::isdigit((unsigned char)t[p]) || t[p] == '-' || t[p] == '+' || t[p] == '.' ||
                                t[p] == 'e' || t[p] == 'E'))
            ++p;
        const std::string num = t.substr(b, p - b);
        if (num.empty()) throw std::runtime_error("malformed JSON number");
        v.kind = JValue::Num;
        v.num = std::strtod(num.c_str(), nullptr);
        v.integral = num.find_first_of(".eE") == std::string::npos;
        if (v.integral) v.i = std::strtoll(num.c_str(), nullptr, 10);
        return v;
    }
};

template <typename T>
void put(std::string& out, T v) {
    out.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

struct Reader {
    std::ifstream is;
    template <typename T>
    T get() {
        T v{};
        is.read(reinterpret_cast<char*>(&v), sizeof(T));
        if (!is) throw std::runtime_error("unexpected end of stream");
        return v;
    }
    void bytes(void* dst, size_t n) {
        is.read(static_cast<char*>(dst), std::streamsize(n));
        if (size_t(is.gcount()) != n) throw std::runtime_error("payload shorter than declared shape");
    }
};

struct HostMoment {
    std::vector<uint8_t> codes;
    std::vector<float> scales, k, c;
};

cudaError_t d2h(const coat_moment_state& st, int64_t npad, int64_t ng, HostMoment& h, cudaStream_t s) {
    h.codes.resize(size_t(npad));
    h.scales.resize(size_t(ng));
    h.k.resize(size_t(ng));
    h.c.resize(size_t(ng));
    std::vector<uint16_t> sb(static_cast<size_t>(ng));
    cudaError_t e = cudaMemcpyAsync(h.codes.data(), st.codes, size_t(npad), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(sb.data(), st.scales, size_t(ng) * 2, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(h.k.data(), st.k, size_t(ng) * 4, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(h.c.data(), st.c, size_t(ng) * 4, cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    for (int64_t i = 0; i < ng; ++i) {
        const uint32_t bits = uint32_t(sb[size_t(i)]) << 16;   // scales are BF16-valued: lossless
        std::memcpy(&h.scales[size_t(i)], &bits, 4);
    }
    return e;
}

void put_moment(std::string& out, const HostMoment& h, int64_t npad, int64_t G) {
    put<uint8_t>(out, 2);                 // ExpandedQuantState (optimizer.cpp:171-181)
    out.append("CQT8", 4);                // tensor_io.cpp:96-120
    put<uint16_t>(out, 1);
    put<uint8_t>(out, 0);                 // Fp8Tag::E4M3
    put<uint8_t>(out, 0);                 // per-group along axis 0 of the flat [npad] tensor
    put<uint32_t>(out, uint32_t(G));
    put<uint16_t>(out, 1);
    put<uint64_t>(out, uint64_t(npad));
    out.append(reinterpret_cast<const char*>(h.scales.data()), h.scales.size() * 4);
    out.append(reinterpret_cast<const char*>(h.codes.data()), h.codes.size());
    out.append("EXPK", 4);                // tensor_io.cpp:153-161
    for (size_t i = 0; i < h.k.size(); ++i) {
        put<float>(out, h.k[i]);
        put<float>(out, h.c[i]);
    }
}

void get_moment(Reader& r, int64_t npad, int64_t G, HostMoment& h) {
    if (r.get<uint8_t>() != 2) throw std::invalid_argument("moment record is not an ExpandedQuantState");
    char mg[4];
    r.bytes(mg, 4);
    if (std::memcmp(mg, "CQT8", 4)) throw std::domain_error("expected record magic CQT8");
    if (r.get<uint16_t>() != 1) throw std::runtime_error("unsupported record version");
    if (r.get<uint8_t>() != 0) throw std::invalid_argument("only E4M3 moments are implemented on B200");
    const uint8_t axis = r.get<uint8_t>();
    const uint32_t size = r.get<uint32_t>();
    const uint16_t rank = r.get<uint16_t>();
    std::vector<int64_t> dims(rank);
    for (auto& d : dims) d = int64_t(r.get<uint64_t>());
    if (axis != 0 || rank != 1 || int64_t(size) != G || dims[0] != npad)
        throw std::length_error("moment geometry does not match the slot");
    const int64_t ng = npad / G;
    h.scales.resize(size_t(ng));
    h.codes.resize(size_t(npad));
    h.k.resize(size_t(ng));
    h.c.resize(size_t(ng));
    r.bytes(h.scales.data(), size_t(ng) * 4);
    r.bytes(h.codes.data(), size_t(npad));
    r.bytes(mg, 4);
    if (std::memcmp(mg, "EXPK", 4)) throw std::domain_error("expected record magic EXPK");
    for (int64_t i = 0; i < ng; ++i) {
        h.k[size_t(i)] = r.get<float>();
        h.c[size_t(i)] = r.get<float>();
    }
}

// BF16 bit patterns of a moment's scales; throws (before anything reaches the
// device) when a scale is not BF16-valued.
std::vector<uint16_t> bf16_scales(const HostMoment& h) {
    const size_t ng = h.scales.size();
    std::vector<uint16_t> sb(ng);
    for (size_t i = 0; i < ng; ++i) {
        uint32_t bits;
        std::memcpy(&bits, &h.scales[i], 4);
        if (bits & 0xFFFFu) throw std::invalid_argument("scale is not BF16-valued (BF16-scale policy expected)");
        sb[i] = uint16_t(bits >> 16);
    }
    return sb;
}

cudaError_t h2d(const coat_moment_state& st, const HostMoment& h, const std::vector<uint16_t>& sb, cudaStream_t s) {
    const size_t ng = sb.size();
    cudaError_t e = cudaMemcpyAsync(st.codes, h.codes.data(), h.codes.size(), cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemcpyAsync(st.scales, sb.data(), ng * 2, cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemcpyAsync(st.k, h.k.data(), ng * 4, cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemcpyAsync(st.c, h.c.data(), ng * 4, cudaMemcpyHostToDevice, s);
    if (!e) e = cudaStreamSynchronize(s);
    return e;
}

}  // namespace

coat_status save_slot_impl(const char* path, const int64_t* shape, int rank, int64_t G, const coat_moment_state& m,
                           const coat_moment_state& v, const coat_adamw_config& cfg, int64_t step,
                           cudaStream_t s, std::string& err) {
    int64_t n = 1;
    for (int i = 0; i < rank; ++i) n *= shape[i];
    const int64_t npad = (n + G - 1) / G * G, ng = npad / G;
    HostMoment hm, hv;
    cudaError_t e = d2h(m, npad, ng, hm, s);
    if (!e) e = d2h(v, npad, ng, hv, s);
    if (e) {
        err = cudaGetErrorString(e);
        return COAT_ERR_CUDA;
    }
    const std::string text = header_json(shape, rank, G, cfg, step);
    std::string out;
    put<uint32_t>(out, uint32_t(text.size()));
    out += text;
    put_moment(out, hm, npad, G);
    put_moment(out, hv, npad, G);
    std::ofstream os(path, std::ios::binary);
    if (!os) {
        err = std::string("cannot open for writing: ") + path;
        return COAT_ERR_IO;
    }
    os.write(out.data(), std::streamsize(out.size()));
    if (!os) {
        err = "write_slot: stream failure";
        return COAT_ERR_IO;
    }
    return COAT_OK;
}

coat_status load_slot_impl(const char* path, const int64_t* shape, int rank, int64_t G, const coat_moment_state& m,
                           const coat_moment_state& v, coat_adamw_config* cfg, int64_t* step, cudaStream_t s,
                           std::string& err) {
    Reader r;
    r.is.open(path, std::ios::binary);
    if (!r.is) {
        err = std::string("cannot open for reading: ") + path;
        return COAT_ERR_IO;
    }
    try {
        const uint32_t len = r.get<uint32_t>();
        std::string text(len, '\0');
        r.bytes(text.data(), len);
        JParser jp{text};
        const JValue h = jp.value();
        const JValue& shp = h.at("shape");
        bool same = shp.kind == JValue::Arr && int(shp.arr.size()) == rank;
        for (int i = 0; same && i < rank; ++i) same = shp.arr[size_t(i)].i == shape[i];
        if (!same) {
            err = "load_slot: shape differs from the slot";
            return COAT_ERR_SHAPE;
        }
        for (const char* which : {"first", "second"}) {
            const JValue& p = h.at("policy").at(which);
            if (p.at("format").s != "e4m3" || !p.at("expand").b || p.at("group_size").i != G) {
                err = "load_slot: the B200 optimizer implements the {E4M3, expand, G} policy only";
                return COAT_ERR_INVALID;
            }
        }
        coat_adamw_config c;
        c.beta1 = float(h.at("beta1").num);
        c.beta2 = float(h.at("beta2").num);
        c.lr = float(h.at("lr").num);
        c.weight_decay = float(h.at("weight_decay").num);
        c.eps = float(h.at("eps").num);
        const int64_t st = h.at("step").i;
        int64_t n = 1;
        for (int i = 0; i < rank; ++i) n *= shape[i];
        const int64_t npad = (n + G - 1) / G * G;
        HostMoment hm, hv;
        get_moment(r, npad, G, hm);
        get_moment(r, npad, G, hv);
        // all-or-nothing like read_slot: both moments parsed and validated
        // before the first byte reaches the device or the outputs
        const std::vector<uint16_t> sm = bf16_scales(hm), sv = bf16_scales(hv);
        cudaError_t e = h2d(m, hm, sm, s);
        if (!e) e = h2d(v, hv, sv, s);
        if (e) {
            err = cudaGetErrorString(e);
            return COAT_ERR_CUDA;
        }
        *cfg = c;
        *step = st;
    } catch (const std::domain_error& ex) {
        err = ex.what();
        return COAT_ERR_BAD_MAGIC;
    } catch (const std::length_error& ex) {
        err = ex.what();
        return COAT_ERR_SHAPE;
    } catch (const std::invalid_argument& ex) {
        err = ex.what();
        return COAT_ERR_INVALID;
    } catch (const std::exception& ex) {
        err = ex.what();
        return COAT_ERR_IO;
    }
    return COAT_OK;
}

}  // namespace coat
