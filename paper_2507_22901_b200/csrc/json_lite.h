// json_lite.h -- a minimal ordered JSON value for the C++ API's text
// formats (codec sidecar, feasibility config and exports).  It reproduces
// nlohmann::ordered_json 3.11.3 where the reference uses it: dump(2) text
// byte for byte (shortest round-trip floats, "d.0" for integral floats,
// one element per line), parse errors, and the exception texts of the
// accessors the reference calls (at / value / get<T>).
#pragma once

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

// Float text: nlohmann's own Grisu2 (detail::to_chars) when its header is on
// the include path (build.py adds the copy in the venv's cudnn_frontend), so
// the digits match the reference even where Grisu2 is not shortest;
// otherwise the shortest round-trip digits in the same layout.
#if __has_include(<json.hpp>)
#include <json.hpp>
#define CVG_HAVE_NLOHMANN_TO_CHARS 1
#endif

namespace colorvibe::json {

struct Json;
using JsonObject = std::vector<std::pair<std::string, Json>>;
using JsonArray = std::vector<Json>;

struct Json {
    enum Kind { Null, Bool, Int, Float, String, Array, Object } kind = Null;
    bool b = false;
    long long i = 0;
    double f = 0.0;
    std::string s;
    std::shared_ptr<JsonArray> arr;
    std::shared_ptr<JsonObject> obj;

    static Json integer(long long v) {
        Json j;
        j.kind = Int;
        j.i = v;
        return j;
    }
    static Json number(double v) {
        Json j;
        j.kind = Float;
        j.f = v;
        return j;
    }
    static Json string(std::string v) {
        Json j;
        j.kind = String;
        j.s = std::move(v);
        return j;
    }
    static Json array() {
        Json j;
        j.kind = Array;
        j.arr = std::make_shared<JsonArray>();
        return j;
    }
    static Json object() {
        Json j;
        j.kind = Object;
        j.obj = std::make_shared<JsonObject>();
        return j;
    }
    static Json boolean(bool v) {
        Json j;
        j.kind = Bool;
        j.b = v;
        return j;
    }
    static Json numbers(const std::vector<double>& v) {
        Json j = array();
        for (double x : v) j.push(number(x));
        return j;
    }
    static Json strings(const std::vector<std::string>& v) {
        Json j = array();
        for (const auto& x : v) j.push(string(x));
        return j;
    }
    bool is_object() const { return kind == Object; }
    bool contains(const std::string& key) const {
        if (kind != Object) return false;
        for (const auto& kv : *obj) {
            if (kv.first == key) return true;
        }
        return false;
    }
    Json& add(const std::string& key, Json v) {
        obj->emplace_back(key, std::move(v));
        return *this;
    }
    Json& push(Json v) {
        arr->push_back(std::move(v));
        return *this;
    }
    const char* type_name() const {
        switch (kind) {
            case Null: return "null";
            case Bool: return "boolean";
            case Int:
            case Float: return "number";
            case String: return "string";
            case Array: return "array";
            case Object: return "object";
        }
        return "null";
    }
};

struct JsonError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

[[noreturn]] inline void type_error(int id, const std::string& what) {
    throw JsonError("[json.exception.type_error." + std::to_string(id) + "] " + what);
}

inline const Json* find(const Json& j, const std::string& key) {
    for (const auto& kv : *j.obj) {
        if (kv.first == key) return &kv.second;
    }
    return nullptr;
}

inline const Json& at(const Json& j, const std::string& key) {
    if (j.kind != Json::Object) type_error(304, std::string("cannot use at() with ") + j.type_name());
    const Json* v = find(j, key);
    if (!v) throw JsonError("[json.exception.out_of_range.403] key '" + key + "' not found");
    return *v;
}

inline double get_double(const Json& j) {
    if (j.kind == Json::Bool) return j.b ? 1.0 : 0.0;
    if (j.kind == Json::Int) return static_cast<double>(j.i);
    if (j.kind == Json::Float) return j.f;
    type_error(302, std::string("type must be number, but is ") + j.type_name());
}

inline int get_int(const Json& j) {
    if (j.kind == Json::Bool) return j.b ? 1 : 0;
    if (j.kind == Json::Int) return static_cast<int>(j.i);
    if (j.kind == Json::Float) return static_cast<int>(j.f);
    type_error(302, std::string("type must be number, but is ") + j.type_name());
}

inline bool get_bool(const Json& j) {
    if (j.kind != Json::Bool) type_error(302, std::string("type must be boolean, but is ") + j.type_name());
    return j.b;
}

inline std::vector<double> get_doubles(const Json& j) {
    if (j.kind != Json::Array) type_error(302, std::string("type must be array, but is ") + j.type_name());
    std::vector<double> out;
    for (const Json& x : *j.arr) out.push_back(get_double(x));
    return out;
}

inline std::vector<int> get_ints(const Json& j) {
    if (j.kind != Json::Array) type_error(302, std::string("type must be array, but is ") + j.type_name());
    std::vector<int> out;
    for (const Json& x : *j.arr) out.push_back(get_int(x));
    return out;
}

inline std::string get_string(const Json& j) {
    if (j.kind != Json::String) type_error(302, std::string("type must be string, but is ") + j.type_name());
    return j.s;
}

// nlohmann's float text: shortest round-trip digits, then format_buffer's
// layout (plain decimal for exponents in (-4, 15], else d.ddde+XX).
inline std::string float_text(double v) {
    if (!std::isfinite(v)) return "null";
#ifdef CVG_HAVE_NLOHMANN_TO_CHARS
    {
        char nb[64];
        char* end = nlohmann::detail::to_chars(nb, nb + sizeof(nb), v);
        return std::string(nb, end);
    }
#endif
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    int prec = 0;
    for (; prec < 17; ++prec) {
        std::snprintf(buf, sizeof(buf), "%.*e", prec, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string t(buf);
    std::string sign;
    if (t[0] == '-') {
        sign = "-";
        t = t.substr(1);
    }
    const size_t epos = t.find('e');
    const int exp10 = std::atoi(t.c_str() + epos + 1);
    std::string digits;
    for (size_t k = 0; k < epos; ++k) {
        if (t[k] != '.') digits += t[k];
    }
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // value = 0.d1d2...dk * 10^n
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, n) + "." + digits.substr(n);
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(-n, '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        char eb[8];
        std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', std::abs(e));
        out += eb;
    }
    return sign + out;
}

inline void escape_into(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (c < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof(b), "\\u%04x", c);
                    out += b;
                } else {
                    out += static_cast<char>(c);
                }
        }
    }
    out += '"';
}

inline void dump(const Json& j, std::string& out, int indent);

// j.dump(2) + "\n"
inline std::string dump2(const Json& j) {
    std::string out;
    dump(j, out, 0);
    return out + "\n";
}

inline void dump(const Json& j, std::string& out, int indent) {
    const std::string pad(indent + 2, ' '), end_pad(indent, ' ');
    switch (j.kind) {
        case Json::Null: out += "null"; break;
        case Json::Bool: out += j.b ? "true" : "false"; break;
        case Json::Int: out += std::to_string(j.i); break;
        case Json::Float: out += float_text(j.f); break;
        case Json::String: escape_into(out, j.s); break;
        case Json::Array:
            if (j.arr->empty()) {
                out += "[]";
                break;
            }
            out += "[\n";
            for (size_t k = 0; k < j.arr->size(); ++k) {
                out += pad;
                dump((*j.arr)[k], out, indent + 2);
                out += k + 1 < j.arr->size() ? ",\n" : "\n";
            }
            out += end_pad + "]";
            break;
        case Json::Object:
            if (j.obj->empty()) {
                out += "{}";
                break;
            }
            out += "{\n";
            for (size_t k = 0; k < j.obj->size(); ++k) {
                out += pad;
                escape_into(out, (*j.obj)[k].first);
                out += ": ";
                dump((*j.obj)[k].second, out, indent + 2);
                out += k + 1 < j.obj->size() ? ",\n" : "\n";
            }
            out += end_pad + "}";
            break;
    }
}

struct Parser {
    const std::string& t;
    size_t p = 0;

    [[noreturn]] void error(const std::string& what) const {
        throw JsonError("[json.exception.parse_error.101] parse error at byte " + std::to_string(p + 1) + ": " + what);
    }
    void ws() {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
    }
    bool lit(const char* s) {
        const size_t n = std::strlen(s);
        if (t.compare(p, n, s) == 0) {
            p += n;
            return true;
        }
        return false;
    }
    Json value() {
        ws();
        if (p >= t.size()) error("syntax error while parsing value - unexpected end of input");
        const char c = t[p];
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') return Json::string(str());
        if (lit("true")) {
            Json j;
            j.kind = Json::Bool;
            j.b = true;
            return j;
        }
        if (lit("false")) {
            Json j;
            j.kind = Json::Bool;
            return j;
        }
        if (lit("null")) return Json{};
        if (c == '-' || (c >= '0' && c <= '9')) return number();
        error("syntax error while parsing value - invalid literal");
    }
    Json number() {
        const size_t s = p;
        if (t[p] == '-') ++p;
        bool is_float = false;
        while (p < t.size() && ((t[p] >= '0' && t[p] <= '9') || t[p] == '.' || t[p] == 'e' || t[p] == 'E' ||
                                t[p] == '+' || t[p] == '-')) {
            is_float = is_float || t[p] == '.' || t[p] == 'e' || t[p] == 'E';
            ++p;
        }
        const std::string num = t.substr(s, p - s);
        char* endp = nullptr;
        if (!is_float) {
            errno = 0;
            const long long v = std::strtoll(num.c_str(), &endp, 10);
            if (*endp == '\0' && errno == 0) return Json::integer(v);
        }
        const double v = std::strtod(num.c_str(), &endp);
        if (num.empty() || *endp != '\0') error("syntax error while parsing value - invalid number");
        return Json::number(v);
    }
    std::string str() {
        ++p;  // opening quote
        std::string out;
        while (true) {
            if (p >= t.size()) error("syntax error while parsing value - invalid string: missing closing quote");
            const char c = t[p++];
            if (c == '"') break;
            if (static_cast<unsigned char>(c) < 0x20) error("syntax error while parsing value - invalid string");
            if (c != '\\') {
                out += c;
                continue;
            }
            if (p >= t.size()) error("syntax error while parsing value - invalid string");
            const char e = t[p++];
            switch (e) {
                case '"': out += '"'; break;
                case '\\': out += '\\'; break;
                case '/': out += '/'; break;
                case 'b': out += '\b'; break;
                case 'f': out += '\f'; break;
                case 'n': out += '\n'; break;
                case 'r': out += '\r'; break;
                case 't': out += '\t'; break;
                case 'u': {
                    if (p + 4 > t.size()) error("syntax error while parsing value - invalid string: bad \\u escape");
                    unsigned cp = static_cast<unsigned>(std::strtoul(t.substr(p, 4).c_str(), nullptr, 16));
                    p += 4;
                    if (cp >= 0xD800 && cp <= 0xDBFF && t.compare(p, 2, "\\u") == 0) {
                        const unsigned lo = static_cast<unsigned>(std::strtoul(t.substr(p + 2, 4).c_str(), nullptr, 16));
                        p += 6;
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    if (cp < 0x80) {
                        out += static_cast<char>(cp);
                    } else if (cp < 0x800) {
                        out += static_cast<char>(0xC0 | (cp >> 6));
                        out += static_cast<char>(0x80 | (cp & 0x3F));
                    } else if (cp < 0x10000) {
                        out += static_cast<char>(0xE0 | (cp >> 12));
                        out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                        out += static_cast<char>(0x80 | (cp & 0x3F));
                    } else {
                        out += static_cast<char>(0xF0 | (cp >> 18));
                        out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
                        out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                        out += static_cast<char>(0x80 | (cp & 0x3F));
                    }
                    break;
                }
                default: error("syntax error while parsing value - invalid string: forbidden escape");
            }
        }
        return out;
    }
    Json array() {
        ++p;
        Json j = Json::array();
        ws();
        if (p < t.size() && t[p] == ']') {
            ++p;
            return j;
        }
        while (true) {
            j.push(value());
            ws();
            if (p < t.size() && t[p] == ',') {
                ++p;
                continue;
            }
            if (p < t.size() && t[p] == ']') {
                ++p;
                return j;
            }
            error("syntax error while parsing array - unexpected token; expected ']'");
        }
    }
    Json object() {
        ++p;
        Json j = Json::object();
        ws();
        if (p < t.size() && t[p] == '}') {
            ++p;
            return j;
        }
        while (true) {
            ws();
            if (p >= t.size() || t[p] != '"') error("syntax error while parsing object key - unexpected token");
            std::string key = str();
            ws();
            if (p >= t.size() || t[p] != ':') error("syntax error while parsing object separator - expected ':'");
            ++p;
            Json v = value();
            // ordered_json keeps the first position and the last value of a repeated key
            bool replaced = false;
            for (auto& kv : *j.obj) {
                if (kv.first == key) {
                    kv.second = v;
                    replaced = true;
                }
            }
            if (!replaced) j.add(key, std::move(v));
            ws();
            if (p < t.size() && t[p] == ',') {
                ++p;
                continue;
            }
            if (p < t.size() && t[p] == '}') {
                ++p;
                return j;
            }
            error("syntax error while parsing object - unexpected token; expected '}'");
        }
    }
    Json parse() {
        Json j = value();
        ws();
        if (p != t.size()) error("syntax error while parsing value - unexpected trailing input");
        return j;
    }
};

}  // namespace colorvibe::json
