// Minimal nlohmann::json-compatible shim -- TEST INFRASTRUCTURE ONLY.
//
// The reference's front end (/root/reference/proj/src/scenario.cpp) includes
// "json.hpp" (nlohmann/json, a third-party header from the untracked vendor/
// directory, absent here).  This header implements, from the library's
// documented behaviour, only the subset scenario.cpp uses: json::parse (RFC
// 8259 text; no comments, no NaN / Infinity, no trailing commas), the
// json::parse_error exception whose what() reads "[json.exception.parse_error.101]
// parse error at line L, column C: ...", objects as a key-sorted map
// (items() iterates keys in byte order, as nlohmann's default std::map
// object does), is_object / is_array / is_string / is_number /
// is_number_integer (integer literals: no '.', 'e' or 'E'), contains, at,
// operator[] on arrays, size, and get<double> / get<int> / get<std::string>.
// Compiling the reference's scenario.cpp and running its own test_scenario.cpp
// against this shim is how the shim is validated (oracle/Makefile ref-tests).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <type_traits>
#include <string>
#include <utility>
#include <vector>

namespace nlohmann {

class json {
 public:
  enum class kind { null, boolean, integer, floating, string, array, object };

  class exception : public std::exception {
   public:
    explicit exception(std::string m) : msg_(std::move(m)) {}
    const char* what() const noexcept override { return msg_.c_str(); }

   private:
    std::string msg_;
  };
  class parse_error : public exception {
   public:
    using exception::exception;
  };
  class type_error : public exception {
   public:
    using exception::exception;
  };
  class out_of_range : public exception {
   public:
    using exception::exception;
  };

  class item {
   public:
    item(const std::string& k, const json& v) : k_(&k), v_(&v) {}
    const std::string& key() const { return *k_; }
    const json& value() const { return *v_; }

   private:
    const std::string* k_;
    const json* v_;
  };

  json() = default;

  static json parse(const std::string& text) {
    parser p{text, 0, 1, 0};
    p.ws();
    json out = p.value();
    p.ws();
    if (p.pos != text.size()) p.fail("syntax error while parsing value - unexpected trailing input");
    return out;
  }

  bool is_object() const { return k_ == kind::object; }
  bool is_array() const { return k_ == kind::array; }
  bool is_string() const { return k_ == kind::string; }
  bool is_number() const { return k_ == kind::integer || k_ == kind::floating; }
  bool is_number_integer() const { return k_ == kind::integer; }

  bool contains(const std::string& key) const { return is_object() && obj_->count(key) != 0; }
  const json& at(const std::string& key) const {
    if (!is_object()) throw type_error("[json.exception.type_error.304] cannot use at() with non-object");
    auto it = obj_->find(key);
    if (it == obj_->end()) throw out_of_range("[json.exception.out_of_range.403] key '" + key + "' not found");
    return it->second;
  }
  const json& operator[](size_t i) const { return (*arr_)[i]; }
  size_t size() const {
    if (is_array()) return arr_->size();
    if (is_object()) return obj_->size();
    return k_ == kind::null ? 0 : 1;
  }

  std::vector<item> items() const {
    std::vector<item> out;
    if (is_object())
      for (const auto& kv : *obj_) out.emplace_back(kv.first, kv.second);
    return out;
  }

  template <typename T>
  T get() const {
    if constexpr (std::is_same_v<T, std::string>) {
      if (!is_string()) throw type_error("[json.exception.type_error.302] type must be string");
      return str_;
    } else {
      static_assert(std::is_arithmetic_v<T>, "json shim: arithmetic or string only");
      if (k_ == kind::integer) return static_cast<T>(int_);
      if (k_ == kind::floating) return static_cast<T>(num_);
      if (k_ == kind::boolean) return static_cast<T>(bool_);
      throw type_error("[json.exception.type_error.302] type must be number");
    }
  }

 private:
  struct parser {
    const std::string& s;
    size_t pos;
    size_t line, col0;

    [[noreturn]] void fail(const std::string& what) const {
      throw parse_error("[json.exception.parse_error.101] parse error at line " + std::to_string(line) +
                        ", column " + std::to_string(pos - col0 + 1) + ": " + what);
    }
    void ws() {
      while (pos < s.size()) {
        const char c = s[pos];
        if (c == '\n') {
          ++line;
          col0 = pos + 1;
        } else if (c != ' ' && c != '\t' && c != '\r') {
          break;
        }
        ++pos;
      }
    }
    bool eat(char c) {
      if (pos < s.size() && s[pos] == c) {
        ++pos;
        return true;
      }
      return false;
    }
    void literal(const char* word) {
      for (const char* w = word; *w; ++w)
        if (!eat(*w)) fail(std::string("syntax error while parsing value - invalid literal; expected '") + word + "'");
    }
    json value() {
      if (pos >= s.size()) fail("syntax error while parsing value - unexpected end of input");
      const char c = s[pos];
      json out;
      if (c == '{') {
        ++pos;
        out.k_ = kind::object;
        out.obj_ = std::make_shared<std::map<std::string, json>>();
        ws();
        if (eat('}')) return out;
        for (;;) {
          ws();
          if (pos >= s.size() || s[pos] != '"') fail("syntax error while parsing object key - expected string literal");
          std::string key = string();
          ws();
          if (!eat(':')) fail("syntax error while parsing object separator - expected ':'");
          ws();
          (*out.obj_)[key] = value();
          ws();
          if (eat(',')) continue;
          if (eat('}')) return out;
          fail("syntax error while parsing object - expected '}'");
        }
      }
      if (c == '[') {
        ++pos;
        out.k_ = kind::array;
        out.arr_ = std::make_shared<std::vector<json>>();
        ws();
        if (eat(']')) return out;
        for (;;) {
          ws();
          out.arr_->push_back(value());
          ws();
          if (eat(',')) continue;
          if (eat(']')) return out;
          fail("syntax error while parsing array - expected ']'");
        }
      }
      if (c == '"') {
        out.k_ = kind::string;
        out.str_ = string();
        return out;
      }
      if (c == 't') {
        literal("true");
        out.k_ = kind::boolean;
        out.bool_ = true;
        return out;
      }
      if (c == 'f') {
        literal("false");
        out.k_ = kind::boolean;
        return out;
      }
      if (c == 'n') {
        literal("null");
        return out;
      }
      if (c == '-' || (c >= '0' && c <= '9')) return number();
      fail("syntax error while parsing value - unexpected '" + std::string(1, c) +
           "'; expected '[', '{', or a literal");
    }
    json number() {
      const size_t b = pos;
      bool integral = true;
      eat('-');
      if (eat('0')) {
        // no leading zeros
      } else if (pos < s.size() && s[pos] >= '1' && s[pos] <= '9') {
        while (pos < s.size() && s[pos] >= '0' && s[pos] <= '9') ++pos;
      } else {
        fail("syntax error while parsing value - invalid number");
      }
      if (eat('.')) {
        integral = false;
        if (!(pos < s.size() && s[pos] >= '0' && s[pos] <= '9')) fail("syntax error while parsing value - invalid number");
        while (pos < s.size() && s[pos] >= '0' && s[pos] <= '9') ++pos;
      }
      if (pos < s.size() && (s[pos] == 'e' || s[pos] == 'E')) {
        integral = false;
        ++pos;
        if (!eat('+')) eat('-');
        if (!(pos < s.size() && s[pos] >= '0' && s[pos] <= '9')) fail("syntax error while parsing value - invalid number");
        while (pos < s.size() && s[pos] >= '0' && s[pos] <= '9') ++pos;
      }
      const std::string tok = s.substr(b, pos - b);
      json out;
      if (integral) {
        out.k_ = kind::integer;
        out.int_ = std::strtoll(tok.c_str(), nullptr, 10);
      } else {
        out.k_ = kind::floating;
        out.num_ = std::strtod(tok.c_str(), nullptr);
      }
      return out;
    }
    static void utf8(std::string& o, unsigned cp) {
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
    unsigned hex4() {
      if (pos + 4 > s.size()) fail("syntax error while parsing value - invalid string: '\\u' must be followed by 4 hex digits");
      unsigned v = 0;
      for (int k = 0; k < 4; ++k) {
        const char h = s[pos++];
        v <<= 4;
        if (h >= '0' && h <= '9') v |= h - '0';
        else if (h >= 'a' && h <= 'f') v |= h - 'a' + 10;
        else if (h >= 'A' && h <= 'F') v |= h - 'A' + 10;
        else fail("syntax error while parsing value - invalid string: '\\u' must be followed by 4 hex digits");
      }
      return v;
    }
    std::string string() {
      ++pos;  // opening quote
      std::string o;
      for (;;) {
        if (pos >= s.size()) fail("syntax error while parsing value - invalid string: missing closing quote");
        const unsigned char c = static_cast<unsigned char>(s[pos++]);
        if (c == '"') return o;
        if (c < 0x20) fail("syntax error while parsing value - invalid string: control character must be escaped");
        if (c != '\\') {
          o += static_cast<char>(c);
          continue;
        }
        if (pos >= s.size()) fail("syntax error while parsing value - invalid string: missing closing quote");
        const char e = s[pos++];
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
            unsigned cp = hex4();
            if (cp >= 0xD800 && cp <= 0xDBFF) {
              if (!(eat('\\') && eat('u'))) fail("syntax error while parsing value - invalid string: surrogate U+D800..U+DBFF must be followed by U+DC00..U+DFFF");
              const unsigned lo = hex4();
              if (lo < 0xDC00 || lo > 0xDFFF) fail("syntax error while parsing value - invalid string: surrogate U+D800..U+DBFF must be followed by U+DC00..U+DFFF");
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
              fail("syntax error while parsing value - invalid string: surrogate U+DC00..U+DFFF must follow U+D800..U+DBFF");
            }
            utf8(o, cp);
            break;
          }
          default:
            fail("syntax error while parsing value - invalid string: forbidden character after backslash");
        }
      }
    }
  };

  kind k_ = kind::null;
  bool bool_ = false;
  long long int_ = 0;
  double num_ = 0.0;
  std::string str_;
  std::shared_ptr<std::vector<json>> arr_;
  std::shared_ptr<std::map<std::string, json>> obj_;
};

}  // namespace nlohmann
