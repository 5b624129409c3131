// Minimal JSON reader for the LMK1 model header (serialize.hpp:17-26 embeds a
// UTF-8 JSON header). The reference parses it with nlohmann::json 3.11
// (serialize.hpp:9, not vendored under /root/reference); the header only uses
// objects, arrays, strings, numbers and booleans, so a small recursive-descent
// parser is enough and keeps the library free of third-party headers.
// Numbers keep their source text so integers (byte counts up to 2^64) are read
// exactly, not through a double.
#pragma once

#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace lmkan_b200 {
namespace json {

struct Value {
    enum Type { Null, Bool, Number, String, Array, Object };
    Type type = Null;
    bool b = false;
    std::string text;  // String: decoded UTF-8; Number: source text
    std::vector<Value> arr;
    std::vector<std::pair<std::string, Value>> obj;

    const Value* find(const std::string& key) const {
        if (type != Object) return nullptr;
        for (const auto& kv : obj)
            if (kv.first == key) return &kv.second;
        return nullptr;
    }
    // nlohmann::json::at semantics: throws when the key is absent
    const Value& at(const std::string& key) const {
        const Value* v = find(key);
        if (!v) throw std::runtime_error("key '" + key + "' not found");
        return *v;
    }
    const std::string& as_string() const {
        if (type != String) throw std::runtime_error("type must be string");
        return text;
    }
    bool as_bool() const {
        if (type != Bool) throw std::runtime_error("type must be boolean");
        return b;
    }
    double as_double() const {
        if (type != Number) throw std::runtime_error("type must be number");
        return std::strtod(text.c_str(), nullptr);
    }
    // Integral value (exact for integer literals; rejects fractions / negatives
    // when `nonneg`).
    long long as_int(bool nonneg = false) const {
        if (type != Number) throw std::runtime_error("type must be number");
        const bool integral = text.find_first_of(".eE") == std::string::npos;
        if (!integral) {
            const double d = std::strtod(text.c_str(), nullptr);
            if (d != static_cast<double>(static_cast<long long>(d))) throw std::runtime_error("number is not an integer");
            if (nonneg && d < 0) throw std::runtime_error("number must be non-negative");
            return static_cast<long long>(d);
        }
        errno = 0;
        const long long v = std::strtoll(text.c_str(), nullptr, 10);
        if (errno == ERANGE) throw std::runtime_error("integer out of range");
        if (nonneg && v < 0) throw std::runtime_error("number must be non-negative");
        return v;
    }
    std::uint64_t as_u64() const {
        if (type != Number) throw std::runtime_error("type must be number");
        if (text.find_first_of(".eE-") != std::string::npos) return static_cast<std::uint64_t>(as_int(true));
        errno = 0;
        const unsigned long long v = std::strtoull(text.c_str(), nullptr, 10);
        if (errno == ERANGE) throw std::runtime_error("integer out of range");
        return v;
    }
};

class Parser {
public:
    explicit Parser(const std::string& s) : s_(s) {}
    Value parse_document() {
        ws();
        Value v = value(0);
        ws();
        if (i_ != s_.size()) fail("unexpected trailing characters");
        return v;
    }

private:
    const std::string& s_;
    size_t i_ = 0;

    [[noreturn]] void fail(const std::string& what) const {
        throw std::runtime_error("parse error at byte " + std::to_string(i_) + ": " + what);
    }
    void ws() {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r')) ++i_;
    }
    bool lit(const char* w) {
        size_t n = 0;
        while (w[n]) ++n;
        if (s_.compare(i_, n, w) == 0) {
            i_ += n;
            return true;
        }
        return false;
    }
    Value value(int depth) {
        if (depth > 256) fail("nesting too deep");
        if (i_ >= s_.size()) fail("unexpected end of input");
        Value v;
        const char c = s_[i_];
        if (c == '{') {
            v.type = Value::Object;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == '}') {
                ++i_;
                return v;
            }
            for (;;) {
                ws();
                if (i_ >= s_.size() || s_[i_] != '"') fail("expected object key");
                std::string k = string();
                ws();
                if (i_ >= s_.size() || s_[i_] != ':') fail("expected ':'");
                ++i_;
                ws();
                v.obj.emplace_back(std::move(k), value(depth + 1));
                ws();
                if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
                if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.type = Value::Array;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == ']') {
                ++i_;
                return v;
            }
            for (;;) {
                ws();
                v.arr.push_back(value(depth + 1));
                ws();
                if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
                if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.type = Value::String;
            v.text = string();
            return v;
        }
        if (lit("true")) { v.type = Value::Bool; v.b = true; return v; }
        if (lit("false")) { v.type = Value::Bool; v.b = false; return v; }
        if (lit("null")) return v;
        if (c == '-' || (c >= '0' && c <= '9')) {
            const size_t b = i_;
            if (s_[i_] == '-') ++i_;
            if (i_ >= s_.size() || !(s_[i_] >= '0' && s_[i_] <= '9')) fail("bad number");
            if (s_[i_] == '0') ++i_;
            else while (i_ < s_.size() && s_[i_] >= '0' && s_[i_] <= '9') ++i_;
            if (i_ < s_.size() && s_[i_] == '.') {
                ++i_;
                if (i_ >= s_.size() || !(s_[i_] >= '0' && s_[i_] <= '9')) fail("bad fraction");
                while (i_ < s_.size() && s_[i_] >= '0' && s_[i_] <= '9') ++i_;
            }
            if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
                ++i_;
                if (i_ < s_.size() && (s_[i_] == '+' || s_[i_] == '-')) ++i_;
                if (i_ >= s_.size() || !(s_[i_] >= '0' && s_[i_] <= '9')) fail("bad exponent");
                while (i_ < s_.size() && s_[i_] >= '0' && s_[i_] <= '9') ++i_;
            }
            v.type = Value::Number;
            v.text = s_.substr(b, i_ - b);
            return v;
        }
        fail("unexpected character");
    }
    static void put_utf8(std::string& o, uint32_t cp) {
        if (cp < 0x80) {
            o += static_cast<char>(cp);
        } else if (cp < 0x800) {
            o += static_cast<char>(0xC0 | (cp >> 6));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            o += static_cast<char>(0xE0 | (cp >> 12));
            o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        } else {
            o += static_cast<char>(0xF0 | (cp >> 18));
            o += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
            o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        }
    }
    uint32_t hex4() {
        if (i_ + 4 > s_.size()) fail("bad \\u escape");
        uint32_t v = 0;
        for (int k = 0; k < 4; ++k) {
            const char h = s_[i_++];
            v <<= 4;
            if (h >= '0' && h <= '9') v |= h - '0';
            else if (h >= 'a' && h <= 'f') v |= h - 'a' + 10;
            else if (h >= 'A' && h <= 'F') v |= h - 'A' + 10;
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string string() {
        ++i_;  // opening quote
        std::string o;
        for (;;) {
            if (i_ >= s_.size()) fail("unterminated string");
            const char c = s_[i_++];
            if (c == '"') return o;
            if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
            if (c != '\\') {
                o += c;
                continue;
            }
            if (i_ >= s_.size()) fail("unterminated escape");
            const char e = s_[i_++];
            switch (e) {
                case '"': o += '"'; break;
                case '\\': o += '\\'; break;
                case '/': o += '/'; break;
                case 'b': o += '\b'; break;
                case 'f': o += '\f'; break;
                case 'n': o += '\n'; break;
                case 'r': o += '\r'; break;
                case 't': o += '\t'; break;
                case 'u': {
                    uint32_t cp = hex4();
                    if (cp >= 0xD800 && cp <= 0xDBFF) {
                        if (i_ + 2 > s_.size() || s_[i_] != '\\' || s_[i_ + 1] != 'u') fail("lone surrogate");
                        i_ += 2;
                        const uint32_t lo = hex4();
                        if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    put_utf8(o, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
    }
};

inline Value parse(const std::string& text) { return Parser(text).parse_document(); }

}  // namespace json
}  // namespace lmkan_b200
