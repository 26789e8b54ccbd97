// nlohmann::json-subset shim — TEST INFRASTRUCTURE ONLY (oracle/_ref).
//
// proj/src/runner.cpp includes the vendored <json.hpp> (absent here,
// proj/CMakeLists.txt:5) to write its run manifest.  This header implements
// the part it uses — construction from scalars / strings / brace lists
// (a list of [string, value] pairs becomes an object, as in nlohmann),
// operator[], array(), push_back and dump(indent) with sorted object keys —
// so runner.cpp and test_pipeline.cpp compile unmodified.
#pragma once

#include <charconv>
#include <cstdint>
#include <initializer_list>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace nlohmann {

class json {
  public:
    enum class kind { null, boolean, integer, number, string, array, object };

    json() = default;
    json(std::nullptr_t) {}
    json(bool b) : k_(kind::boolean), b_(b) {}
    template <class T, std::enable_if_t<std::is_integral_v<T> && !std::is_same_v<T, bool>, int> = 0>
    json(T v) : k_(kind::integer), i_(static_cast<long long>(v)) {}
    template <class T, std::enable_if_t<std::is_floating_point_v<T>, int> = 0>
    json(T v) : k_(kind::number), d_(static_cast<double>(v)) {}
    json(const char* s) : k_(kind::string), s_(s) {}
    json(std::string s) : k_(kind::string), s_(std::move(s)) {}
    json(std::initializer_list<json> list) {
        bool object = true;
        for (const json& e : list) object = object && e.k_ == kind::array && e.a_.size() == 2 && e.a_[0].k_ == kind::string;
        if (object && list.size() > 0) {
            k_ = kind::object;
            for (const json& e : list) (*this)[e.a_[0].s_] = e.a_[1];
        } else {
            k_ = kind::array;
            a_.assign(list.begin(), list.end());
        }
    }

    static json array() {
        json j;
        j.k_ = kind::array;
        return j;
    }
    static json object() {
        json j;
        j.k_ = kind::object;
        return j;
    }

    json& operator[](const std::string& key) {
        if (k_ == kind::null) k_ = kind::object;
        auto it = o_.begin();
        while (it != o_.end() && it->first < key) ++it;  // keys stay sorted (std::map order)
        if (it != o_.end() && it->first == key) return it->second;
        return o_.insert(it, {key, json()})->second;
    }
    json& operator[](const char* key) { return (*this)[std::string(key)]; }
    void push_back(const json& v) {
        if (k_ == kind::null) k_ = kind::array;
        a_.push_back(v);
    }
    size_t size() const { return k_ == kind::array ? a_.size() : (k_ == kind::object ? o_.size() : 1); }

    std::string dump(int indent = -1) const {
        std::string out;
        write(out, indent, 0);
        return out;
    }

  private:
    static void escape(std::string& out, const std::string& s) {
        out += '"';
        for (char c : s) {
            switch (c) {
                case '"': out += "\\\""; break;
                case '\\': out += "\\\\"; break;
                case '\n': out += "\\n"; break;
                case '\t': out += "\\t"; break;
                case '\r': out += "\\r"; break;
                default:
                    if (static_cast<unsigned char>(c) < 0x20) {
                        char buf[8];
                        std::snprintf(buf, sizeof buf, "\\u%04x", c);
                        out += buf;
                    } else {
                        out += c;
                    }
            }
        }
        out += '"';
    }
    void write(std::string& out, int indent, int depth) const {
        const bool pretty = indent >= 0;
        auto newline = [&](int d) {
            if (!pretty) return;
            out += '\n';
            out.append(static_cast<size_t>(d * indent), ' ');
        };
        switch (k_) {
            case kind::null: out += "null"; break;
            case kind::boolean: out += b_ ? "true" : "false"; break;
            case kind::integer: out += std::to_string(i_); break;
            case kind::number: {
                char buf[64];
                const auto r = std::to_chars(buf, buf + sizeof buf, d_);
                std::string t(buf, r.ptr);
                if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
                out += t;
                break;
            }
            case kind::string: escape(out, s_); break;
            case kind::array:
                if (a_.empty()) {
                    out += "[]";
                    break;
                }
                out += '[';
                for (size_t n = 0; n < a_.size(); ++n) {
                    if (n) out += ',';
                    newline(depth + 1);
                    a_[n].write(out, indent, depth + 1);
                }
                newline(depth);
                out += ']';
                break;
            case kind::object:
                if (o_.empty()) {
                    out += "{}";
                    break;
                }
                out += '{';
                for (size_t n = 0; n < o_.size(); ++n) {
                    if (n) out += ',';
                    newline(depth + 1);
                    escape(out, o_[n].first);
                    out += pretty ? ": " : ":";
                    o_[n].second.write(out, indent, depth + 1);
                }
                newline(depth);
                out += '}';
                break;
        }
    }

    kind k_ = kind::null;
    bool b_ = false;
    long long i_ = 0;
    double d_ = 0;
    std::string s_;
    std::vector<json> a_;
    std::vector<std::pair<std::string, json>> o_;
};

}  // namespace nlohmann
