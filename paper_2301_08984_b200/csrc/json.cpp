#include "json.hpp"

#include <cstdlib>

namespace planc_b200 {
namespace json {
namespace {

struct Parser {
  const std::string& s;
  std::size_t p = 0;

  [[noreturn]] void fail(const std::string& m) {
    throw ParseError(m + " at offset " + std::to_string(p));
  }
  void ws() {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\n' || s[p] == '\r' || s[p] == '\t')) ++p;
  }
  bool lit(const char* w) {
    std::size_t n = 0;
    while (w[n]) ++n;
    if (s.compare(p, n, w) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  static void put_utf8(std::string& out, unsigned cp) {
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
  }
  unsigned hex4() {
    if (p + 4 > s.size()) fail("bad \\u escape");
    unsigned v = 0;
    for (int k = 0; k < 4; ++k) {
      char c = s[p++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else fail("bad hex digit");
    }
    return v;
  }
  std::string str() {
    if (s[p] != '"') fail("expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= s.size()) fail("unterminated string");
      char c = s[p++];
      if (c == '"') break;
      if (c == '\\') {
        if (p >= s.size()) fail("bad escape");
        char e = s[p++];
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
            unsigned cp = hex4();
            if (cp >= 0xD800 && cp < 0xDC00 && p + 6 <= s.size() && s[p] == '\\' && s[p + 1] == 'u') {
              p += 2;
              unsigned lo = hex4();
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            }
            put_utf8(out, cp);
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    return out;
  }
  Value value() {
    ws();
    if (p >= s.size()) fail("unexpected end of document");
    Value v;
    char c = s[p];
    if (c == '{') {
      v.type = Value::Type::object;
      ++p;
      ws();
      if (p < s.size() && s[p] == '}') {
        ++p;
        return v;
      }
      while (true) {
        ws();
        std::string k = str();
        ws();
        if (p >= s.size() || s[p] != ':') fail("expected ':'");
        ++p;
        v.obj.emplace_back(std::move(k), value());
        ws();
        if (p < s.size() && s[p] == ',') { ++p; continue; }
        if (p < s.size() && s[p] == '}') { ++p; break; }
        fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.type = Value::Type::array;
      ++p;
      ws();
      if (p < s.size() && s[p] == ']') {
        ++p;
        return v;
      }
      while (true) {
        v.arr.push_back(value());
        ws();
        if (p < s.size() && s[p] == ',') { ++p; continue; }
        if (p < s.size() && s[p] == ']') { ++p; break; }
        fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.type = Value::Type::string;
      v.str = str();
    } else if (lit("true")) {
      v.type = Value::Type::boolean;
      v.b = true;
    } else if (lit("false")) {
      v.type = Value::Type::boolean;
    } else if (lit("null")) {
      v.type = Value::Type::null;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      std::size_t start = p;
      bool integral = true;
      if (s[p] == '-') ++p;
      while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
      if (p < s.size() && (s[p] == '.' || s[p] == 'e' || s[p] == 'E')) {
        integral = false;
        if (s[p] == '.') {
          ++p;
          while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
        }
        if (p < s.size() && (s[p] == 'e' || s[p] == 'E')) {
          ++p;
          if (p < s.size() && (s[p] == '+' || s[p] == '-')) ++p;
          while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
        }
      }
      std::string tok = s.substr(start, p - start);
      v.type = Value::Type::number;
      if (integral && tok.size() < 19) {
        v.is_int = true;
        v.i = std::strtoll(tok.c_str(), nullptr, 10);
        v.num = static_cast<double>(v.i);
      } else {
        v.num = std::strtod(tok.c_str(), nullptr);
      }
    } else {
      fail(std::string("unexpected character '") + c + "'");
    }
    return v;
  }
};

}  // namespace

Value parse(const std::string& text) {
  Parser ps{text};
  Value v = ps.value();
  ps.ws();
  if (ps.p != text.size()) ps.fail("trailing characters");
  return v;
}

}  // namespace json
}  // namespace planc_b200
