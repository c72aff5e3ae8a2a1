// MUGVCKPT reader / writer (proj/src/params.cpp:92-225).  Host C++ only.
//
// Layout (params.hpp:54-59): 8-byte magic "MUGVCKPT", little-endian u64 header length, a compact JSON
// header  {"__meta__":{k:v,...}, name:{"dtype":"f32"|"f64","length":L,"offset":O,"shape":[...]}, ...}
// with keys in byte order (the reference's nlohmann::json object is a std::map), then the payloads packed
// contiguously in name order.  The writer reproduces the reference's bytes exactly (its header is
// nlohmann's dump(): no whitespace, sorted keys, RFC 8259 escaping with ensure_ascii = false); the reader
// accepts any RFC 8259 header and applies the reference's checks in the reference's order.
#include "ckpt.h"

#include "../../include/mugv_b200.h"

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>

namespace mgv {
namespace {

constexpr char kMagic[8] = {'M', 'U', 'G', 'V', 'C', 'K', 'P', 'T'};

// ---------------------------------------------------------------- minimal RFC 8259 JSON (nlohmann semantics)
struct JV {
    enum T { Null, Bool, Int, UInt, Float, Str, Arr, Obj } t = Null;
    bool b = false;
    int64_t i = 0;
    uint64_t u = 0;
    double f = 0.0;
    std::string s;
    std::vector<JV> a;
    std::map<std::string, JV> o;  // duplicate keys: the last one wins, as in nlohmann's DOM parser
    bool is_int() const { return t == Int || t == UInt; }
};

struct ParseFail {
    std::string why;
};

// length of the well-formed UTF-8 sequence at p (RFC 3629 ranges, as nlohmann's lexer checks), 0 if ill-formed
int utf8_len(const unsigned char* p, const unsigned char* e) {
    const unsigned c = p[0];
    int n = 0;
    unsigned lo2 = 0x80, hi2 = 0xBF;
    if (c < 0x80)
        return 1;
    else if (c >= 0xC2 && c <= 0xDF)
        n = 1;
    else if (c == 0xE0) {
        n = 2;
        lo2 = 0xA0;
    } else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF)
        n = 2;
    else if (c == 0xED) {
        n = 2;
        hi2 = 0x9F;
    } else if (c == 0xF0) {
        n = 3;
        lo2 = 0x90;
    } else if (c >= 0xF1 && c <= 0xF3)
        n = 3;
    else if (c == 0xF4) {
        n = 3;
        hi2 = 0x8F;
    } else
        return 0;
    if (e - p < n + 1) return 0;
    for (int k = 1; k <= n; ++k) {
        const unsigned cc = p[k];
        const unsigned lo = k == 1 ? lo2 : 0x80, hi = k == 1 ? hi2 : 0xBF;
        if (cc < lo || cc > hi) return 0;
    }
    return n + 1;
}

class Parser {
public:
    Parser(const char* p, const char* e) : p_(p), e_(e) {}
    JV document() {
        if (e_ - p_ >= 3 && static_cast<unsigned char>(p_[0]) == 0xEF && static_cast<unsigned char>(p_[1]) == 0xBB &&
            static_cast<unsigned char>(p_[2]) == 0xBF)
            p_ += 3;  // nlohmann skips a leading UTF-8 BOM
        JV v = value(0);
        ws();
        if (p_ != e_) fail("trailing characters after the JSON value");
        return v;
    }

private:
    const char* p_;
    const char* e_;
    [[noreturn]] void fail(const char* why) { throw ParseFail{why}; }
    void ws() {
        while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if (static_cast<size_t>(e_ - p_) < n || std::memcmp(p_, w, n) != 0) return false;
        p_ += n;
        return true;
    }
    JV value(int depth) {
        if (depth > 512) fail("nesting too deep");
        ws();
        if (p_ >= e_) fail("unexpected end of input");
        JV v;
        switch (*p_) {
            case '{': {
                ++p_;
                v.t = JV::Obj;
                ws();
                if (p_ < e_ && *p_ == '}') {
                    ++p_;
                    return v;
                }
                for (;;) {
                    ws();
                    if (p_ >= e_ || *p_ != '"') fail("expected an object key");
                    std::string k = string();
                    ws();
                    if (p_ >= e_ || *p_ != ':') fail("expected ':'");
                    ++p_;
                    v.o[k] = value(depth + 1);
                    ws();
                    if (p_ < e_ && *p_ == ',') {
                        ++p_;
                        continue;
                    }
                    if (p_ < e_ && *p_ == '}') {
                        ++p_;
                        return v;
                    }
                    fail("expected ',' or '}'");
                }
            }
            case '[': {
                ++p_;
                v.t = JV::Arr;
                ws();
                if (p_ < e_ && *p_ == ']') {
                    ++p_;
                    return v;
                }
                for (;;) {
                    v.a.push_back(value(depth + 1));
                    ws();
                    if (p_ < e_ && *p_ == ',') {
                        ++p_;
                        continue;
                    }
                    if (p_ < e_ && *p_ == ']') {
                        ++p_;
                        return v;
                    }
                    fail("expected ',' or ']'");
                }
            }
            case '"':
                v.t = JV::Str;
                v.s = string();
                return v;
            case 't':
                if (!lit("true")) fail("invalid literal");
                v.t = JV::Bool;
                v.b = true;
                return v;
            case 'f':
                if (!lit("false")) fail("invalid literal");
                v.t = JV::Bool;
                return v;
            case 'n':
                if (!lit("null")) fail("invalid literal");
                return v;
            default:
                return number();
        }
    }
    unsigned hex4() {
        if (e_ - p_ < 4) fail("truncated \\u escape");
        unsigned c = 0;
        for (int k = 0; k < 4; ++k, ++p_) {
            const char h = *p_;
            c <<= 4;
            if (h >= '0' && h <= '9')
                c |= h - '0';
            else if (h >= 'a' && h <= 'f')
                c |= h - 'a' + 10;
            else if (h >= 'A' && h <= 'F')
                c |= h - 'A' + 10;
            else
                fail("bad \\u escape");
        }
        return c;
    }
    static void utf8(std::string& out, unsigned cp) {
        if (cp < 0x80) {
            out.push_back(static_cast<char>(cp));
        } else if (cp < 0x800) {
            out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        } else if (cp < 0x10000) {
            out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        } else {
            out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
        }
    }
    std::string string() {
        ++p_;  // opening quote
        std::string out;
        for (;;) {
            if (p_ >= e_) fail("unterminated string");
            const unsigned char c = static_cast<unsigned char>(*p_);
            if (c == '"') {
                ++p_;
                return out;
            }
            if (c < 0x20) fail("control character in string");
            if (c == '\\') {
                ++p_;
                if (p_ >= e_) fail("unterminated escape");
                const char x = *p_++;
                switch (x) {
                    case '"': out.push_back('"'); break;
                    case '\\': out.push_back('\\'); break;
                    case '/': out.push_back('/'); break;
                    case 'b': out.push_back('\b'); break;
                    case 'f': out.push_back('\f'); break;
                    case 'n': out.push_back('\n'); break;
                    case 'r': out.push_back('\r'); break;
                    case 't': out.push_back('\t'); break;
                    case 'u': {
                        unsigned cp = hex4();
                        if (cp >= 0xD800 && cp <= 0xDBFF) {
                            if (!(e_ - p_ >= 2 && p_[0] == '\\' && p_[1] == 'u')) fail("unpaired surrogate");
                            p_ += 2;
                            const unsigned lo = hex4();
                            if (lo < 0xDC00 || lo > 0xDFFF) fail("unpaired surrogate");
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                            fail("unpaired surrogate");
                        }
                        utf8(out, cp);
                        break;
                    }
                    default: fail("invalid escape");
                }
                continue;
            }
            // raw UTF-8: copy one well-formed sequence
            const int n = utf8_len(reinterpret_cast<const unsigned char*>(p_), reinterpret_cast<const unsigned char*>(e_));
            if (n == 0) fail("ill-formed UTF-8");
            out.append(p_, p_ + n);
            p_ += n;
        }
    }
    JV number() {
        const char* b = p_;
        bool neg = false, frac = false;
        if (p_ < e_ && *p_ == '-') {
            neg = true;
            ++p_;
        }
        if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) fail("invalid value");
        if (*p_ == '0')
            ++p_;  // no leading zeros
        else
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        if (p_ < e_ && *p_ == '.') {
            frac = true;
            ++p_;
            if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) fail("invalid number");
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
            frac = true;
            ++p_;
            if (p_ < e_ && (*p_ == '+' || *p_ == '-')) ++p_;
            if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) fail("invalid number");
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        const std::string tok(b, p_);
        JV v;
        if (!frac) {  // integers that fit are integers (nlohmann: unsigned without '-', signed with '-')
            errno = 0;
            char* end = nullptr;
            if (neg) {
                const long long x = std::strtoll(tok.c_str(), &end, 10);
                if (errno == 0) {
                    v.t = JV::Int;
                    v.i = x;
                    return v;
                }
            } else {
                const unsigned long long x = std::strtoull(tok.c_str(), &end, 10);
                if (errno == 0) {
                    v.t = JV::UInt;
                    v.u = x;
                    return v;
                }
            }
        }
        v.t = JV::Float;
        v.f = std::strtod(tok.c_str(), nullptr);
        return v;
    }
};

// nlohmann's get<uint64_t>() of a header number (arithmetic conversion; booleans allowed)
bool as_u64(const JV& v, uint64_t* out) {
    switch (v.t) {
        case JV::UInt: *out = v.u; return true;
        case JV::Int: *out = static_cast<uint64_t>(v.i); return true;
        case JV::Float: *out = static_cast<uint64_t>(v.f); return true;
        case JV::Bool: *out = v.b ? 1 : 0; return true;
        default: return false;
    }
}

uint64_t get_u64(const unsigned char* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
    return v;
}

void put_u64(std::string& out, uint64_t v) {
    for (int i = 0; i < 8; ++i) out.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}

// nlohmann dump_escaped with ensure_ascii = false; ill-formed UTF-8 is rejected (its type_error 316)
void put_json_string(std::string& out, const std::string& s) {
    const auto* b = reinterpret_cast<const unsigned char*>(s.data());
    for (size_t i = 0; i < s.size();) {
        const int n = utf8_len(b + i, b + s.size());
        if (n == 0) throw CkptInputError("tensor name or metadata is not valid UTF-8");
        i += static_cast<size_t>(n);
    }
    out.push_back('"');
    for (char ch : s) {
        const unsigned char c = static_cast<unsigned char>(ch);
        switch (c) {
            case '\b': out += "\\b"; break;
            case '\t': out += "\\t"; break;
            case '\n': out += "\\n"; break;
            case '\f': out += "\\f"; break;
            case '\r': out += "\\r"; break;
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            default:
                if (c <= 0x1F) {
                    char buf[8];
                    std::snprintf(buf, sizeof(buf), "\\u%04x", c);
                    out += buf;
                } else {
                    out.push_back(ch);
                }
        }
    }
    out.push_back('"');
}

int64_t shape_numel(const std::vector<int64_t>& shape) {  // Tensor::shape_numel (tensor.cpp)
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return n;
}

std::string shape_str(const std::vector<int64_t>& shape) {  // Tensor::shape_str
    std::string s = "(";
    for (size_t i = 0; i < shape.size(); ++i) {
        if (i) s += ", ";
        s += std::to_string(shape[i]);
    }
    return s + ")";
}

}  // namespace

void Checkpoint::read_f64(const CkptEntry& e, double* out) const {
    const unsigned char* p = payload(e);
    if (e.dtype == kF32) {
        for (int64_t i = 0; i < e.numel; ++i) {
            uint32_t u = 0;
            for (int k = 0; k < 4; ++k) u |= static_cast<uint32_t>(p[4 * i + k]) << (8 * k);
            float f;
            std::memcpy(&f, &u, 4);
            out[i] = static_cast<double>(f);
        }
    } else {
        for (int64_t i = 0; i < e.numel; ++i) {
            const uint64_t u = get_u64(p + 8 * i);
            std::memcpy(&out[i], &u, 8);
        }
    }
}

void Checkpoint::read_f32(const CkptEntry& e, float* out) const {
    const unsigned char* p = payload(e);
    if (e.dtype == kF32) {
        for (int64_t i = 0; i < e.numel; ++i) {
            uint32_t u = 0;
            for (int k = 0; k < 4; ++k) u |= static_cast<uint32_t>(p[4 * i + k]) << (8 * k);
            std::memcpy(&out[i], &u, 4);
        }
    } else {
        for (int64_t i = 0; i < e.numel; ++i) {
            const uint64_t u = get_u64(p + 8 * i);
            double d;
            std::memcpy(&d, &u, 8);
            out[i] = static_cast<float>(d);
        }
    }
}

// params.cpp:128-224, check for check
Checkpoint load_checkpoint(const std::string& path) {
    Checkpoint ck;
    {
        std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
        if (!f) throw CheckpointError(CheckpointError::Io, "cannot open " + path);
        char buf[1 << 16];
        size_t got;
        while ((got = std::fread(buf, 1, sizeof(buf), f.get())) > 0) ck.raw.append(buf, got);
        if (std::ferror(f.get())) throw CheckpointError(CheckpointError::Io, "cannot open " + path);
    }
    const std::string& raw = ck.raw;
    const unsigned char* bytes = reinterpret_cast<const unsigned char*>(raw.data());
    if (raw.size() < 8) throw CheckpointError(CheckpointError::Truncated, path + ": shorter than the magic");
    if (std::memcmp(raw.data(), kMagic, 8) != 0) throw CheckpointError(CheckpointError::BadMagic, path + ": bad magic");
    if (raw.size() < 16) throw CheckpointError(CheckpointError::Truncated, path + ": missing header length");
    const uint64_t head_len = get_u64(bytes + 8);
    if (head_len > raw.size() || 16 + head_len > raw.size())
        throw CheckpointError(CheckpointError::Truncated, path + ": header exceeds file size");
    JV header;
    try {
        header = Parser(raw.data() + 16, raw.data() + 16 + head_len).document();
    } catch (const ParseFail& e) {
        throw CheckpointError(CheckpointError::BadHeader, path + ": header is not valid JSON: " + e.why);
    }
    if (header.t != JV::Obj) throw CheckpointError(CheckpointError::BadHeader, path + ": header is not a JSON object");
    const uint64_t payload_size = raw.size() - 16 - head_len;
    ck.payload_at = 16 + head_len;

    auto bad = [&](const std::string& m) { return CheckpointError(CheckpointError::BadHeader, path + ": " + m); };
    for (const auto& [name, desc] : header.o) {  // sorted key order, first failure wins (params.cpp:154)
        if (name == "__meta__") {
            if (desc.t != JV::Obj) throw bad("__meta__ is not an object");
            for (const auto& [k, v] : desc.o) {
                if (v.t != JV::Str) throw bad("metadata value for \"" + k + "\" is not a string");
                ck.meta[k] = v.s;
            }
            continue;
        }
        if (desc.t != JV::Obj || !desc.o.count("dtype") || !desc.o.count("shape") || !desc.o.count("offset") ||
            !desc.o.count("length"))
            throw bad("tensor \"" + name + "\" has an incomplete descriptor");
        const JV& dt = desc.o.at("dtype");
        if (dt.t != JV::Str) throw bad("tensor \"" + name + "\" dtype is not a string");
        CkptEntry e;
        e.name = name;
        if (dt.s == "f32")
            e.dtype = kF32;
        else if (dt.s == "f64")
            e.dtype = kF64;
        else
            throw CheckpointError(CheckpointError::BadHeader, "unknown dtype \"" + dt.s + "\"");  // params.cpp:20
        // nlohmann range-for over "shape": arrays yield elements, objects their values, null nothing,
        // any other scalar itself
        const JV& sh = desc.o.at("shape");
        std::vector<const JV*> dims;
        if (sh.t == JV::Arr)
            for (const JV& d : sh.a) dims.push_back(&d);
        else if (sh.t == JV::Obj)
            for (const auto& kv : sh.o) dims.push_back(&kv.second);
        else if (sh.t != JV::Null)
            dims.push_back(&sh);
        for (const JV* d : dims) {
            if (!d->is_int() || (d->t == JV::Int && d->i < 0)) throw bad("tensor \"" + name + "\" has a bad shape entry");
            e.shape.push_back(d->t == JV::Int ? d->i : static_cast<int64_t>(d->u));
        }
        uint64_t off = 0, len = 0;
        if (!as_u64(desc.o.at("offset"), &off) || !as_u64(desc.o.at("length"), &len))
            throw bad("tensor \"" + name + "\" offset/length is not a number");
        e.numel = shape_numel(e.shape);
        const uint64_t want = static_cast<uint64_t>(e.numel) * (e.dtype == kF32 ? 4u : 8u);
        if (len != want)
            throw bad("tensor \"" + name + "\" length " + std::to_string(len) + " does not match shape " +
                      shape_str(e.shape));
        if (off + len > payload_size)
            throw CheckpointError(CheckpointError::Truncated,
                                  path + ": payload for \"" + name + "\" runs past end of file");
        e.offset = off;
        ck.entries.push_back(std::move(e));
    }
    // the payload must be tiled exactly: sorted extents contiguous from 0 (params.cpp:206-222)
    std::vector<const CkptEntry*> ext;
    for (const CkptEntry& e : ck.entries) ext.push_back(&e);
    std::sort(ext.begin(), ext.end(), [](const CkptEntry* a, const CkptEntry* b) { return a->offset < b->offset; });
    uint64_t cursor = 0;
    for (const CkptEntry* e : ext) {
        const uint64_t len = static_cast<uint64_t>(e->numel) * (e->dtype == kF32 ? 4u : 8u);
        if (e->offset < cursor)
            throw CheckpointError(CheckpointError::BadOffsets,
                                  path + ": tensor \"" + e->name + "\" overlaps the previous payload");
        if (e->offset > cursor)
            throw CheckpointError(CheckpointError::BadOffsets, path + ": gap in payload before tensor \"" + e->name + "\"");
        cursor = e->offset + len;
    }
    if (cursor != payload_size)
        throw CheckpointError(CheckpointError::BadOffsets,
                              path + ": payload has " + std::to_string(payload_size - cursor) + " trailing bytes");
    return ck;
}

// params.cpp:92-126
void save_checkpoint(std::vector<CkptTensorIn> tensors, const std::map<std::string, std::string>& meta,
                     const std::string& path) {
    std::sort(tensors.begin(), tensors.end(),
              [](const CkptTensorIn& a, const CkptTensorIn& b) { return a.name < b.name; });
    for (size_t i = 0; i < tensors.size(); ++i) {
        if (tensors[i].name == "__meta__") throw CkptInputError("tensor name \"__meta__\" is reserved");
        if (i && tensors[i].name == tensors[i - 1].name)
            throw CkptInputError("duplicate tensor name \"" + tensors[i].name + "\"");
        if ((tensors[i].f64 == nullptr) == (tensors[i].f32 == nullptr))
            throw CkptInputError("tensor \"" + tensors[i].name + "\" needs exactly one data pointer");
        for (int64_t d : tensors[i].shape)
            if (d < 0) throw CkptInputError("tensor \"" + tensors[i].name + "\" has a negative dimension");
    }
    // header: "__meta__" sorts before every name starting with a byte > '_' ; place it in key order
    struct Item {
        std::string key, json;
    };
    std::vector<Item> items;
    std::string payload;
    uint64_t offset = 0;
    for (const CkptTensorIn& t : tensors) {
        const int64_t n = shape_numel(t.shape);
        const uint64_t length = static_cast<uint64_t>(n) * (t.dtype == kF32 ? 4u : 8u);
        std::string j = "{\"dtype\":";
        j += t.dtype == kF32 ? "\"f32\"" : "\"f64\"";
        j += ",\"length\":" + std::to_string(length) + ",\"offset\":" + std::to_string(offset) + ",\"shape\":[";
        for (size_t k = 0; k < t.shape.size(); ++k) {
            if (k) j.push_back(',');
            j += std::to_string(t.shape[k]);
        }
        j += "]}";
        items.push_back({t.name, std::move(j)});
        payload.reserve(payload.size() + length);
        for (int64_t i = 0; i < n; ++i) {
            if (t.dtype == kF32) {
                const float f = t.f32 ? t.f32[i] : static_cast<float>(t.f64[i]);
                uint32_t u;
                std::memcpy(&u, &f, 4);
                for (int k = 0; k < 4; ++k) payload.push_back(static_cast<char>((u >> (8 * k)) & 0xff));
            } else {
                const double d = t.f64 ? t.f64[i] : static_cast<double>(t.f32[i]);
                uint64_t u;
                std::memcpy(&u, &d, 8);
                put_u64(payload, u);
            }
        }
        offset += length;
    }
    {
        std::string j = "{";
        bool first = true;
        for (const auto& [k, v] : meta) {
            if (!first) j.push_back(',');
            first = false;
            put_json_string(j, k);
            j.push_back(':');
            put_json_string(j, v);
        }
        j.push_back('}');
        items.push_back({"__meta__", std::move(j)});
    }
    std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) { return a.key < b.key; });
    std::string head = "{";
    for (size_t i = 0; i < items.size(); ++i) {
        if (i) head.push_back(',');
        put_json_string(head, items[i].key);
        head.push_back(':');
        head += items[i].json;
    }
    head.push_back('}');

    std::string out;
    out.reserve(16 + head.size() + payload.size());
    out.append(kMagic, 8);
    put_u64(out, head.size());
    out += head;
    out += payload;
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "wb"), &std::fclose);
    if (!f) throw CheckpointError(CheckpointError::Io, "cannot open " + path + " for writing");
    if (std::fwrite(out.data(), 1, out.size(), f.get()) != out.size() || std::fflush(f.get()) != 0)
        throw CheckpointError(CheckpointError::Io, "write failed for " + path);
}

}  // namespace mgv

// ---------------------------------------------------------------- C ABI (include/mugv_b200.h)
namespace {
thread_local std::string t_ckpt_err;
thread_local int t_ckpt_kind = -1;
}  // namespace

void mgv::note_ckpt_error(const std::string& msg, int kind) {
    t_ckpt_err = msg;
    t_ckpt_kind = kind;
}

namespace {

template <class F>
mgv_status ckpt_guard(F&& f) {
    try {
        f();
        t_ckpt_err.clear();
        t_ckpt_kind = -1;
        return MGV_OK;
    } catch (const mgv::CheckpointError& e) {
        t_ckpt_err = e.what();
        t_ckpt_kind = e.kind;
        return MGV_ERR_CHECKPOINT;
    } catch (const mgv::CkptInputError& e) {
        t_ckpt_err = e.what();
        t_ckpt_kind = -1;
        return MGV_ERR_INPUT;
    } catch (const std::exception& e) {
        t_ckpt_err = e.what();
        t_ckpt_kind = -1;
        return MGV_ERR_INTERNAL;
    }
}
bool valid_index(const mgv_ckpt* c, int64_t i) {
    return c && i >= 0 && i < static_cast<int64_t>(c->ck.entries.size());
}
}  // namespace

extern "C" {

const char* mgv_ckpt_last_error(void) { return t_ckpt_err.c_str(); }
int mgv_ckpt_last_error_kind(void) { return t_ckpt_kind; }

mgv_status mgv_ckpt_load(const char* path, mgv_ckpt** out) {
    if (!path || !out) return MGV_ERR_INPUT;
    *out = nullptr;
    return ckpt_guard([&] {
        auto h = std::make_unique<mgv_ckpt>();
        h->ck = mgv::load_checkpoint(path);
        *out = h.release();
    });
}
void mgv_ckpt_free(mgv_ckpt* c) { delete c; }
int64_t mgv_ckpt_count(const mgv_ckpt* c) { return c ? static_cast<int64_t>(c->ck.entries.size()) : 0; }
const char* mgv_ckpt_name(const mgv_ckpt* c, int64_t i) {
    return valid_index(c, i) ? c->ck.entries[static_cast<size_t>(i)].name.c_str() : nullptr;
}
int mgv_ckpt_dtype(const mgv_ckpt* c, int64_t i) {
    return valid_index(c, i) ? static_cast<int>(c->ck.entries[static_cast<size_t>(i)].dtype) : -1;
}
int mgv_ckpt_rank(const mgv_ckpt* c, int64_t i) {
    return valid_index(c, i) ? static_cast<int>(c->ck.entries[static_cast<size_t>(i)].shape.size()) : -1;
}
const int64_t* mgv_ckpt_shape(const mgv_ckpt* c, int64_t i) {
    return valid_index(c, i) ? c->ck.entries[static_cast<size_t>(i)].shape.data() : nullptr;
}
int64_t mgv_ckpt_numel(const mgv_ckpt* c, int64_t i) {
    return valid_index(c, i) ? c->ck.entries[static_cast<size_t>(i)].numel : -1;
}
int64_t mgv_ckpt_find(const mgv_ckpt* c, const char* name) {
    if (!c || !name) return -1;
    const auto& e = c->ck.entries;
    auto it = std::lower_bound(e.begin(), e.end(), std::string(name),
                               [](const mgv::CkptEntry& a, const std::string& n) { return a.name < n; });
    return it != e.end() && it->name == name ? static_cast<int64_t>(it - e.begin()) : -1;
}
mgv_status mgv_ckpt_read(const mgv_ckpt* c, int64_t i, double* out) {
    if (!valid_index(c, i) || !out) return MGV_ERR_INPUT;
    return ckpt_guard([&] { c->ck.read_f64(c->ck.entries[static_cast<size_t>(i)], out); });
}
int64_t mgv_ckpt_meta_count(const mgv_ckpt* c) { return c ? static_cast<int64_t>(c->ck.meta.size()) : 0; }
const char* mgv_ckpt_meta_key(const mgv_ckpt* c, int64_t i) {
    if (!c || i < 0 || i >= static_cast<int64_t>(c->ck.meta.size())) return nullptr;
    auto it = c->ck.meta.begin();
    std::advance(it, i);
    return it->first.c_str();
}
const char* mgv_ckpt_meta_value(const mgv_ckpt* c, int64_t i) {
    if (!c || i < 0 || i >= static_cast<int64_t>(c->ck.meta.size())) return nullptr;
    auto it = c->ck.meta.begin();
    std::advance(it, i);
    return it->second.c_str();
}

mgv_status mgv_ckpt_save(const char* path, int64_t n, const char* const* names, const double* const* data,
                         const int* dtypes, const int* ranks, const int64_t* const* shapes, int64_t n_meta,
                         const char* const* meta_keys, const char* const* meta_values) {
    return ckpt_guard([&] {
        if (!path || n < 0 || (n > 0 && (!names || !data || !ranks || !shapes)) ||
            (n_meta > 0 && (!meta_keys || !meta_values)))
            throw mgv::CkptInputError("null argument");
        std::vector<mgv::CkptTensorIn> ts(static_cast<size_t>(n));
        for (int64_t k = 0; k < n; ++k) {
            auto& t = ts[static_cast<size_t>(k)];
            if (!names[k] || !data[k] || ranks[k] < 0 || (ranks[k] > 0 && !shapes[k]))
                throw mgv::CkptInputError("null tensor argument");
            t.name = names[k];
            const int dt = dtypes ? dtypes[k] : MGV_CKPT_F64;
            if (dt != MGV_CKPT_F32 && dt != MGV_CKPT_F64) throw mgv::CkptInputError("unknown dtype");
            t.dtype = dt == MGV_CKPT_F32 ? mgv::kF32 : mgv::kF64;
            t.shape.assign(shapes[k], shapes[k] + ranks[k]);
            t.f64 = data[k];
        }
        std::map<std::string, std::string> meta;
        for (int64_t k = 0; k < n_meta; ++k) {
            if (!meta_keys[k] || !meta_values[k]) throw mgv::CkptInputError("null metadata argument");
            meta[meta_keys[k]] = meta_values[k];
        }
        mgv::save_checkpoint(std::move(ts), meta, path);
    });
}

}  // extern "C"
