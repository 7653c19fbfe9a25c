// .bdelta container reader (the format of P:src/delta.cpp:218-334, documented in
// P:README.md "File formats"): "BDLT", u32 LE version 1, u32 LE JSON header
// length, JSON array of {name, rows, cols, kind, planes, scales,
// payload_offset, payload_len}, then the concatenated payloads. Packed plane
// bytes are the device layout and are handed to the pool unchanged.
//
// Validation mirrors read_delta_file: bad magic/version/truncation ->
// malformed_header, bad JSON -> json_parse, out-of-range payloads ->
// bad_offsets, duplicate names -> duplicate_id, negative scales and nonzero
// trailing bits -> bad_argument.
#include "bdelta_io.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <set>

#include "common.cuh"

namespace bd {

namespace {

// Minimal JSON reader for the header schema (objects, arrays, strings, numbers).
struct JVal {
    enum Kind { Null, Num, Str, Arr, Obj, Bool } kind = Null;
    double num = 0;
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;
    const JVal* get(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
};

struct JParser {
    const char* p;
    const char* end;
    void ws() {
        while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
    }
    [[noreturn]] void bad() { fail(BD_ERR_JSON_PARSE, "bdelta: header is not valid JSON"); }
    JVal parse() {
        ws();
        if (p >= end) bad();
        JVal v;
        if (*p == '{') {
            v.kind = JVal::Obj;
            ++p;
            ws();
            if (p < end && *p == '}') { ++p; return v; }
            for (;;) {
                ws();
                JVal k = parse();
                if (k.kind != JVal::Str) bad();
                ws();
                if (p >= end || *p != ':') bad();
                ++p;
                v.obj.emplace_back(k.str, parse());
                ws();
                if (p < end && *p == ',') { ++p; continue; }
                if (p < end && *p == '}') { ++p; return v; }
                bad();
            }
        }
        if (*p == '[') {
            v.kind = JVal::Arr;
            ++p;
            ws();
            if (p < end && *p == ']') { ++p; return v; }
            for (;;) {
                v.arr.push_back(parse());
                ws();
                if (p < end && *p == ',') { ++p; continue; }
                if (p < end && *p == ']') { ++p; return v; }
                bad();
            }
        }
        if (*p == '"') {
            v.kind = JVal::Str;
            ++p;
            while (p < end && *p != '"') {
                if (*p == '\\') {
                    ++p;
                    if (p >= end) bad();
                    const char c = *p;
                    switch (c) {
                        case '"': case '\\': case '/': v.str.push_back(c); break;
                        case 'b': v.str.push_back('\b'); break;
                        case 'f': v.str.push_back('\f'); break;
                        case 'n': v.str.push_back('\n'); break;
                        case 'r': v.str.push_back('\r'); break;
                        case 't': v.str.push_back('\t'); break;
                        case 'u': {  // \uXXXX (with surrogate pairs) -> UTF-8, as nlohmann::json
                            auto hex4 = [&](const char* q) {
                                if (end - q < 4) bad();
                                uint32_t cp = 0;
                                for (int i = 0; i < 4; ++i) {
                                    const char h = q[i];
                                    cp <<= 4;
                                    if (h >= '0' && h <= '9') cp |= uint32_t(h - '0');
                                    else if (h >= 'a' && h <= 'f') cp |= uint32_t(h - 'a' + 10);
                                    else if (h >= 'A' && h <= 'F') cp |= uint32_t(h - 'A' + 10);
                                    else bad();
                                }
                                return cp;
                            };
                            uint32_t cp = hex4(p + 1);
                            p += 4;
                            if (cp >= 0xD800 && cp < 0xDC00) {  // high surrogate: a low one must follow
                                if (end - p < 7 || p[1] != '\\' || p[2] != 'u') bad();
                                const uint32_t lo = hex4(p + 3);
                                if (lo < 0xDC00 || lo >= 0xE000) bad();
                                cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                                p += 6;
                            } else if (cp >= 0xDC00 && cp < 0xE000) {
                                bad();
                            }
                            if (cp < 0x80) {
                                v.str.push_back(char(cp));
                            } else if (cp < 0x800) {
                                v.str.push_back(char(0xC0 | (cp >> 6)));
                                v.str.push_back(char(0x80 | (cp & 0x3F)));
                            } else if (cp < 0x10000) {
                                v.str.push_back(char(0xE0 | (cp >> 12)));
                                v.str.push_back(char(0x80 | ((cp >> 6) & 0x3F)));
                                v.str.push_back(char(0x80 | (cp & 0x3F)));
                            } else {
                                v.str.push_back(char(0xF0 | (cp >> 18)));
                                v.str.push_back(char(0x80 | ((cp >> 12) & 0x3F)));
                                v.str.push_back(char(0x80 | ((cp >> 6) & 0x3F)));
                                v.str.push_back(char(0x80 | (cp & 0x3F)));
                            }
                            break;
                        }
                        default: bad();
                    }
                } else {
                    v.str.push_back(*p);
                }
                ++p;
            }
            if (p >= end) bad();
            ++p;
            return v;
        }
        if (end - p >= 4 && !std::strncmp(p, "true", 4)) { v.kind = JVal::Bool; v.num = 1; p += 4; return v; }
        if (end - p >= 5 && !std::strncmp(p, "false", 5)) { v.kind = JVal::Bool; p += 5; return v; }
        if (end - p >= 4 && !std::strncmp(p, "null", 4)) { p += 4; return v; }
        // number: strtod gives the exact double of the reference's decimal
        std::string tok;
        while (p < end && (std::strchr("+-0123456789.eE", *p) != nullptr)) tok.push_back(*p++);
        if (tok.empty()) bad();
        char* e = nullptr;
        v.kind = JVal::Num;
        v.num = std::strtod(tok.c_str(), &e);
        if (e == nullptr || *e != '\0') bad();
        return v;
    }
};

uint32_t le32(const uint8_t* p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

const JVal& field(const JVal& e, const char* k, const std::string& name) {
    const JVal* v = e.get(k);
    if (!v) fail(BD_ERR_JSON_PARSE, "tensor '" + name + "': missing field '" + k + "'");
    return *v;
}
uint64_t as_u64(const JVal& v, const std::string& name) {
    // whole, non-negative, exactly representable (nlohmann's get<uint64_t> on a JSON integer)
    if (v.kind != JVal::Num || v.num < 0 || v.num != std::floor(v.num) || v.num > 9007199254740992.0)
        fail(BD_ERR_JSON_PARSE, "tensor '" + name + "': bad number");
    return static_cast<uint64_t>(v.num);
}

}  // namespace

DeltaFileHost read_bdelta(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) fail(BD_ERR_IO, path + ": cannot open");
    std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    require(bytes.size() >= 12, BD_ERR_MALFORMED_HEADER, path + ": truncated .bdelta");
    require(std::memcmp(bytes.data(), "BDLT", 4) == 0, BD_ERR_MALFORMED_HEADER, path + ": bad magic");
    require(le32(bytes.data() + 4) == 1, BD_ERR_MALFORMED_HEADER, path + ": unsupported version");
    const uint32_t hlen = le32(bytes.data() + 8);
    require(hlen <= bytes.size() - 12, BD_ERR_MALFORMED_HEADER, path + ": header overruns file");
    JParser jp{reinterpret_cast<const char*>(bytes.data() + 12),
               reinterpret_cast<const char*>(bytes.data() + 12 + hlen)};
    const JVal header = jp.parse();
    jp.ws();
    require(jp.p == jp.end, BD_ERR_JSON_PARSE, path + ": trailing bytes after the JSON header");
    require(header.kind == JVal::Arr, BD_ERR_JSON_PARSE, path + ": header is not a JSON array");
    const uint8_t* payload = bytes.data() + 12 + hlen;
    const size_t payload_len = bytes.size() - 12 - hlen;

    DeltaFileHost out;
    std::set<std::string> seen;
    for (const JVal& e : header.arr) {
        const JVal& jn = field(e, "name", "?");
        require(jn.kind == JVal::Str, BD_ERR_JSON_PARSE, path + ": tensor name is not a string");
        const std::string name = jn.str;
        require(seen.insert(name).second, BD_ERR_DUPLICATE_ID,
                path + ": duplicate tensor '" + name + "'");
        DeltaEntryHost d;
        d.name = name;
        d.rows = as_u64(field(e, "rows", name), name);
        d.cols = as_u64(field(e, "cols", name), name);
        const uint64_t off = as_u64(field(e, "payload_offset", name), name);
        const uint64_t len = as_u64(field(e, "payload_len", name), name);
        require(off <= payload_len && len <= payload_len - off, BD_ERR_BAD_OFFSETS,
                "tensor '" + name + "': payload out of range");
        const JVal& kind = field(e, "kind", name);
        if (kind.kind == JVal::Str && kind.str == "packed") {
            d.packed = true;
            d.planes = as_u64(field(e, "planes", name), name);
            const JVal& sc = field(e, "scales", name);
            require(sc.kind == JVal::Arr && sc.arr.size() == d.planes, BD_ERR_JSON_PARSE,
                    "tensor '" + name + "': scales/planes mismatch");
            const uint64_t nb = (d.rows * d.cols + 7) / 8;
            require(len == d.planes * nb, BD_ERR_BAD_OFFSETS,
                    "tensor '" + name + "': payload length does not match planes");
            for (const JVal& s : sc.arr) {
                require(s.kind == JVal::Num, BD_ERR_JSON_PARSE, "tensor '" + name + "': bad scale");
                const float a = static_cast<float>(s.num);
                require(a >= 0.0f, BD_ERR_BAD_ARGUMENT, "tensor '" + name + "': negative scale");
                d.scales.push_back(a);
            }
            d.bits.assign(payload + off, payload + off + len);
            const uint64_t tail = (d.rows * d.cols) % 8;
            for (uint64_t k = 0; k < d.planes && tail && nb; ++k)
                require((d.bits[k * nb + nb - 1] >> tail) == 0, BD_ERR_BAD_ARGUMENT,
                        "tensor '" + name + "': nonzero trailing bits");
        } else if (kind.kind == JVal::Str && kind.str == "raw") {
            d.packed = false;
            require(len == 4 * d.rows * d.cols, BD_ERR_BAD_OFFSETS,
                    "tensor '" + name + "': payload length does not match shape");
            d.raw.resize(d.rows * d.cols);
            std::memcpy(d.raw.data(), payload + off, len);  // little-endian f32
        } else {
            fail(BD_ERR_JSON_PARSE, "tensor '" + name + "': unknown kind");
        }
        out.entries.push_back(std::move(d));
    }
    return out;
}

}  // namespace bd
