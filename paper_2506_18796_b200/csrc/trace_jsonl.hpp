// Trace ingestion: the reference's JSONL trace format (parse_trace,
// workload.cpp:204-266; written by serialize_trace, workload.cpp:181-202)
// parsed on all host threads straight into structure-of-arrays.
//
// Semantics follow parse_trace line by line:
//   * lines split on '\n'; empty lines skipped; the first non-empty line is
//     the header {trace_version (must be 1), pattern, seed, rate, duration,
//     windows (default 1)};
//   * every later line is one Request {request_id, arrival_time_s,
//     language, task_class, prompt_tokens, output_tokens}; unknown keys are
//     ignored, a repeated key keeps its last value (nlohmann's parser);
//   * checks in the reference's order: field presence/type, negative
//     arrival, non-positive token counts, arrivals out of order;
//   * the FIRST failing line (in file order) is reported with the
//     reference's message text.  Field errors reproduce nlohmann's
//     out_of_range.403 / type_error.302 texts (and out_of_range.406 for
//     overflowing numbers); JSON syntax errors keep the
//     reference's "trace line N: invalid JSON: " prefix with this parser's own
//     description (nlohmann's parse_error wording is not reproduced).
// Numbers: integers parse exactly (uint64 / int64, larger ones as double),
// others with strtod (correctly rounded, like nlohmann); get<int> / get<u64>
// / get<double> conversions are the static_casts nlohmann applies.
#pragma once
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

namespace cace {

struct ParsedTrace {
  int32_t pattern = 0;  // PatternName (types.hpp:49-53)
  uint64_t seed = 0;
  double rate = 1.0, duration = 30.0;
  int32_t windows = 1;
  std::vector<uint64_t> request_id;
  std::vector<double> arrival;
  std::vector<int32_t> language, task_class, prompt, output;
};

namespace jsonl {

enum Kind { K_NONE, K_NULL, K_BOOL, K_UINT, K_INT, K_DOUBLE, K_STRING, K_OBJECT, K_ARRAY };

// One scalar value of a top-level field (nested objects/arrays are skipped).
struct Val {
  Kind kind = K_NONE;
  bool b = false;
  uint64_t u = 0;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
};

struct LineError {
  std::string what;
};

inline const char* type_name(Kind k) {
  switch (k) {
    case K_NULL: return "null";
    case K_BOOL: return "boolean";
    case K_STRING: return "string";
    case K_OBJECT: return "object";
    case K_ARRAY: return "array";
    default: return "number";
  }
}

struct Parser {
  const char* p;
  const char* e;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  [[noreturn]] void fail(const char* what) {
    throw LineError{std::string("syntax error: ") + what};
  }
  void expect(char c, const char* what) {
    ws();
    if (p >= e || *p != c) fail(what);
    ++p;
  }
  static void put_utf8(std::string& out, uint32_t cp) {
    if (cp < 0x80) {
      out += (char)cp;
    } else if (cp < 0x800) {
      out += (char)(0xC0 | (cp >> 6));
      out += (char)(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += (char)(0xE0 | (cp >> 12));
      out += (char)(0x80 | ((cp >> 6) & 0x3F));
      out += (char)(0x80 | (cp & 0x3F));
    } else {
      out += (char)(0xF0 | (cp >> 18));
      out += (char)(0x80 | ((cp >> 12) & 0x3F));
      out += (char)(0x80 | ((cp >> 6) & 0x3F));
      out += (char)(0x80 | (cp & 0x3F));
    }
  }
  uint32_t hex4() {
    if (e - p < 4) fail("truncated \\u escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
      else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
      else fail("invalid \\u escape");
    }
    return v;
  }
  std::string str() {
    ws();
    if (p >= e || *p != '"') fail("expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= e) fail("unterminated string");
      const unsigned char c = (unsigned char)*p++;
      if (c == '"') break;
      if (c < 0x20) fail("control character in string");
      if (c >= 0x80) {  // well-formed UTF-8 only (RFC 3629 ranges, as nlohmann's scan_string)
        int more;
        unsigned char lo = 0x80, hi = 0xBF;
        if (c >= 0xC2 && c <= 0xDF) {
          more = 1;
        } else if (c >= 0xE0 && c <= 0xEF) {
          more = 2;
          if (c == 0xE0) lo = 0xA0;
          if (c == 0xED) hi = 0x9F;
        } else if (c >= 0xF0 && c <= 0xF4) {
          more = 3;
          if (c == 0xF0) lo = 0x90;
          if (c == 0xF4) hi = 0x8F;
        } else {
          fail("ill-formed UTF-8 byte");
        }
        out += (char)c;
        for (int q = 0; q < more; ++q) {
          if (p >= e) fail("ill-formed UTF-8 byte");
          const unsigned char d = (unsigned char)*p++;
          if (d < lo || d > hi) fail("ill-formed UTF-8 byte");
          out += (char)d;
          lo = 0x80;
          hi = 0xBF;
        }
        continue;
      }
      if (c != '\\') {
        out += (char)c;
        continue;
      }
      if (p >= e) fail("unterminated escape");
      const char x = *p++;
      switch (x) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (e - p < 6 || p[0] != '\\' || p[1] != 'u') fail("unpaired surrogate");
            p += 2;
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("unpaired surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            fail("unpaired surrogate");
          }
          put_utf8(out, cp);
          break;
        }
        default: fail("invalid escape");
      }
    }
    return out;
  }
  void number(Val& v) {
    const char* s0 = p;
    bool neg = false;
    if (p < e && *p == '-') {
      neg = true;
      ++p;
    }
    if (p >= e || !(*p >= '0' && *p <= '9')) fail("invalid number");
    if (*p == '0') {
      ++p;
    } else {
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    bool is_float = false;
    if (p < e && *p == '.') {
      is_float = true;
      ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) fail("invalid number");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      is_float = true;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) fail("invalid number");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    const std::string tok(s0, p);
    if (!is_float) {
      errno = 0;
      char* end = nullptr;
      if (!neg) {
        const unsigned long long u = std::strtoull(tok.c_str(), &end, 10);
        if (errno == 0) {
          v.kind = K_UINT;
          v.u = u;
          return;
        }
      } else {
        const long long i = std::strtoll(tok.c_str(), &end, 10);
        if (errno == 0) {
          v.kind = K_INT;
          v.i = i;
          return;
        }
      }
    }
    v.kind = K_DOUBLE;
    v.d = std::strtod(tok.c_str(), nullptr);
    if (!std::isfinite(v.d))  // nlohmann rejects overflowing literals (lexer, out_of_range.406)
      throw LineError{"[json.exception.out_of_range.406] number overflow parsing '" + tok + "'"};
  }
  // Skips one value of any nesting depth with an explicit stack (nlohmann's
  // parser is iterative and has no depth limit).
  void skip_value() {
    std::vector<char> open;  // '{' / '[' of the containers being skipped
    while (true) {
      ws();
      if (p >= e) fail("unexpected end of input");
      if (*p == '{' || *p == '[') {
        const char c = *p++;
        ws();
        if (p < e && *p == (c == '{' ? '}' : ']')) {
          ++p;
        } else {
          open.push_back(c);
          if (c == '{') {
            (void)str();
            expect(':', "expected ':'");
          }
          continue;  // the container's first value
        }
      } else {
        Val v;
        scalar(v);
      }
      // a value ended: continue or close its containers
      while (true) {
        if (open.empty()) return;
        ws();
        if (p < e && *p == ',') {
          ++p;
          if (open.back() == '{') {
            (void)str();
            expect(':', "expected ':'");
          }
          break;
        }
        if (open.back() == '{')
          expect('}', "expected ',' or '}'");
        else
          expect(']', "expected ',' or ']'");
        open.pop_back();
      }
    }
  }
  void literal(const char* w) {
    const size_t n = std::strlen(w);
    if ((size_t)(e - p) < n || std::memcmp(p, w, n) != 0) fail("invalid literal");
    p += n;
  }
  void scalar(Val& v) {
    ws();
    if (p >= e) fail("unexpected end of input");
    const char c = *p;
    if (c == '"') {
      v.kind = K_STRING;
      v.s = str();
    } else if (c == 't') {
      literal("true");
      v.kind = K_BOOL;
      v.b = true;
    } else if (c == 'f') {
      literal("false");
      v.kind = K_BOOL;
      v.b = false;
    } else if (c == 'n') {
      literal("null");
      v.kind = K_NULL;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      number(v);
    } else {
      fail("invalid literal");
    }
  }
  // Parses one JSON document that must be an object; calls on_field(key,
  // value) for each top-level scalar field (nested values reported as
  // K_OBJECT / K_ARRAY without content).  A non-object document is reported
  // through on_nonobject.
  Kind top = K_NONE;  // kind of the document when it is not an object
  template <class F>
  bool object(F&& on_field) {
    // a UTF-8 byte order mark at the start of the document is skipped, as
    // nlohmann's lexer does (skip_bom); a partial one is a syntax error
    if (p < e && (unsigned char)*p == 0xEF) {
      if (e - p < 3 || (unsigned char)p[1] != 0xBB || (unsigned char)p[2] != 0xBF)
        fail("invalid BOM; must be 0xEF 0xBB 0xBF if given");
      p += 3;
    }
    ws();
    if (p >= e) fail("unexpected end of input");
    if (*p != '{') {
      const char c = *p;
      top = c == '[' ? K_ARRAY : c == '"' ? K_STRING : (c == 't' || c == 'f') ? K_BOOL : c == 'n' ? K_NULL : K_UINT;
      skip_value();
      ws();
      if (p != e) fail("trailing characters");
      return false;
    }
    ++p;
    ws();
    if (p < e && *p == '}') {
      ++p;
    } else {
      while (true) {
        std::string key = str();
        expect(':', "expected ':'");
        ws();
        Val v;
        if (p < e && (*p == '{' || *p == '[')) {
          v.kind = *p == '{' ? K_OBJECT : K_ARRAY;
          skip_value();
        } else {
          scalar(v);
        }
        on_field(key, v);
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        expect('}', "expected ',' or '}'");
        break;
      }
    }
    ws();
    if (p != e) fail("trailing characters");
    return true;
  }
};

// nlohmann-style typed reads (static_cast conversions of number kinds).
struct Field {
  bool present = false;
  Val v;
};

[[noreturn]] inline void not_object(Kind k) {  // at() on a non-object document
  throw LineError{std::string("[json.exception.type_error.304] cannot use at() with ") + type_name(k)};
}
[[noreturn]] inline void missing(const char* key) {
  throw LineError{std::string("[json.exception.out_of_range.403] key '") + key + "' not found"};
}
[[noreturn]] inline void mistyped(const char* want, Kind got) {
  throw LineError{std::string("[json.exception.type_error.302] type must be ") + want + ", but is " +
                  type_name(got)};
}
// get<T>() of a number: uint64 / double are nlohmann's own number types
// (get_arithmetic_value: booleans rejected); other arithmetic types (int)
// also convert booleans (from_json for arithmetic types).
template <class T>
inline T num(const Field& f, const char* key) {
  if (!f.present) missing(key);
  constexpr bool own = std::is_same<T, uint64_t>::value || std::is_same<T, double>::value ||
                       std::is_same<T, int64_t>::value;
  switch (f.v.kind) {
    case K_UINT: return static_cast<T>(f.v.u);
    case K_INT: return static_cast<T>(f.v.i);
    case K_DOUBLE: return static_cast<T>(f.v.d);
    case K_BOOL:
      if (!own) return static_cast<T>(f.v.b);
      mistyped("number", K_BOOL);
    default: mistyped("number", f.v.kind);
  }
}
inline const std::string& str_field(const Field& f, const char* key) {
  if (!f.present) missing(key);
  if (f.v.kind != K_STRING) mistyped("string", f.v.kind);
  return f.v.s;
}

inline int language_code(const std::string& s) {  // language_from_string, types.cpp:19-24
  static const char* names[] = {"java", "python", "cpp", "c", "go", "rust", "csharp", "javascript"};
  for (int k = 0; k < 8; ++k)
    if (s == names[k]) return k;
  return -1;
}
inline int task_code(const std::string& s) {
  if (s == "completion") return 0;
  if (s == "reasoning") return 1;
  return -1;
}
inline int pattern_code(const std::string& s) {
  if (s == "uniform") return 0;
  if (s == "ide-heavy") return 1;
  if (s == "popularity-skewed") return 2;
  return -1;
}

// A ParseError raised while reading a line, with the reference's text.
struct TraceError {
  size_t line;
  std::string what;
};

}  // namespace jsonl

// Parses the whole text.  Throws jsonl::TraceError (first failing line, in
// file order) on any error parse_trace would raise.
inline ParsedTrace parse_trace_jsonl(const char* text, size_t len) {
  using namespace jsonl;
  ParsedTrace out;
  const char* const end = text + len;
  // header: first non-empty line
  const char* p = text;
  size_t line_no = 0;
  bool have_header = false;
  while (p < end && !have_header) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
    const char* le = nl ? nl : end;
    ++line_no;
    if (le != p) {
      Field f_ver, f_pat, f_seed, f_rate, f_dur, f_win;
      bool is_obj = false;
      Kind top = K_NONE;
      try {
        Parser ps{p, le};
        is_obj = ps.object([&](const std::string& k, const Val& v) {
          Field* t = k == "trace_version" ? &f_ver
                     : k == "pattern"      ? &f_pat
                     : k == "seed"         ? &f_seed
                     : k == "rate"         ? &f_rate
                     : k == "duration"     ? &f_dur
                     : k == "windows"      ? &f_win
                                           : nullptr;
          if (t) {
            t->present = true;
            t->v = v;
          }
        });
        top = ps.top;
      } catch (const LineError& x) {
        throw TraceError{line_no, "trace line " + std::to_string(line_no) + ": invalid JSON: " + x.what};
      }
      if (!f_ver.present) throw TraceError{line_no, "trace line 1: missing trace_version header"};
      try {
        if (!is_obj) not_object(top);
        if (num<int>(f_ver, "trace_version") != 1) throw TraceError{line_no, "trace: unsupported trace_version"};
        const int pc = pattern_code(str_field(f_pat, "pattern"));
        if (pc < 0) throw TraceError{line_no, "unknown pattern: " + f_pat.v.s};
        out.pattern = pc;
        out.seed = num<uint64_t>(f_seed, "seed");
        out.rate = num<double>(f_rate, "rate");
        out.duration = num<double>(f_dur, "duration");
        out.windows = f_win.present ? num<int>(f_win, "windows") : 1;
      } catch (const LineError& x) {
        throw TraceError{line_no, "trace line " + std::to_string(line_no) + ": missing or mistyped field: " + x.what};
      }
      have_header = true;
    }
    p = nl ? nl + 1 : end;
  }
  if (!have_header) throw TraceError{line_no, "trace: missing header line"};

  // Records: chunks of whole lines parsed on all host threads.
  const size_t rest = (size_t)(end - p);
  const int nth = (int)std::max<size_t>(1, std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()),
                                                            rest / (1 << 20) + 1));
  std::vector<const char*> cut(nth + 1);
  cut[0] = p;
  for (int t = 1; t < nth; ++t) {
    const char* c = p + rest * t / nth;
    if (c < cut[t - 1]) c = cut[t - 1];
    const char* nl = c < end ? static_cast<const char*>(std::memchr(c, '\n', (size_t)(end - c))) : nullptr;
    cut[t] = nl ? nl + 1 : end;
  }
  cut[nth] = end;
  struct Part {
    size_t lines = 0;  // lines in the chunk (for numbering)
    ParsedTrace recs;
    std::vector<size_t> rec_line;  // chunk-local line number of each record
    bool err = false;
    size_t err_line = 0;  // chunk-local
    std::string err_what;  // message without the "trace line N: " prefix
    bool err_has_prefix = true;
  };
  std::vector<Part> parts(nth);
  auto work = [&](int t) {
    Part& P = parts[t];
    const char* q = cut[t];
    const char* qe = cut[t + 1];
    size_t ln = 0;
    double prev = 0.0;
    bool have_prev = false;
    while (q < qe) {
      const char* nl = static_cast<const char*>(std::memchr(q, '\n', (size_t)(qe - q)));
      const char* le = nl ? nl : qe;
      ++ln;
      if (le != q) {
        Field fid, farr, flang, fcls, fpr, fout;
        bool is_obj = false;
        Kind top = K_NONE;
        try {
          Parser ps{q, le};
          is_obj = ps.object([&](const std::string& k, const Val& v) {
            Field* f = k == "request_id"       ? &fid
                       : k == "arrival_time_s" ? &farr
                       : k == "language"       ? &flang
                       : k == "task_class"     ? &fcls
                       : k == "prompt_tokens"  ? &fpr
                       : k == "output_tokens"  ? &fout
                                               : nullptr;
            if (f) {
              f->present = true;
              f->v = v;
            }
          });
          top = ps.top;
        } catch (const LineError& x) {
          P.err = true;
          P.err_line = ln;
          P.err_what = "invalid JSON: " + x.what;
          break;
        }
        try {
          if (!is_obj) not_object(top);
          const uint64_t id = num<uint64_t>(fid, "request_id");
          const double a = num<double>(farr, "arrival_time_s");
          const int lang = language_code(str_field(flang, "language"));
          if (lang < 0) {
            P.err = true;
            P.err_line = ln;
            P.err_what = "unknown language: " + flang.v.s;
            P.err_has_prefix = false;
            break;
          }
          const int cls = task_code(str_field(fcls, "task_class"));
          if (cls < 0) {
            P.err = true;
            P.err_line = ln;
            P.err_what = "unknown task class: " + fcls.v.s;
            P.err_has_prefix = false;
            break;
          }
          const int pr = num<int>(fpr, "prompt_tokens");
          const int ou = num<int>(fout, "output_tokens");
          if (a < 0) {
            P.err = true;
            P.err_line = ln;
            P.err_what = "negative arrival_time_s";
            break;
          }
          if (pr <= 0 || ou <= 0) {
            P.err = true;
            P.err_line = ln;
            P.err_what = "token counts must be positive";
            break;
          }
          if (have_prev && a < prev) {
            P.err = true;
            P.err_line = ln;
            P.err_what = "arrivals out of order";
            break;
          }
          prev = a;
          have_prev = true;
          P.recs.request_id.push_back(id);
          P.recs.arrival.push_back(a);
          P.recs.language.push_back(lang);
          P.recs.task_class.push_back(cls);
          P.recs.prompt.push_back(pr);
          P.recs.output.push_back(ou);
          P.rec_line.push_back(ln);
        } catch (const LineError& x) {
          P.err = true;
          P.err_line = ln;
          P.err_what = "missing or mistyped field: " + x.what;
          break;
        }
      }
      q = nl ? nl + 1 : qe;
    }
    // count the remaining lines of the chunk so later chunks number correctly
    while (q < qe) {
      const char* nl = static_cast<const char*>(std::memchr(q, '\n', (size_t)(qe - q)));
      ++ln;
      q = nl ? nl + 1 : qe;
    }
    P.lines = ln;
  };
  if (nth == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nth; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  // Stitch in file order; the first error wins, including the cross-chunk
  // arrival-order check (each chunk's first record vs the last accepted one).
  double max_time = 0.0;
  size_t base = line_no;
  size_t n = 0;
  for (const Part& P : parts) n += P.recs.arrival.size();
  out.request_id.reserve(n);
  out.arrival.reserve(n);
  out.language.reserve(n);
  out.task_class.reserve(n);
  out.prompt.reserve(n);
  out.output.reserve(n);
  for (const Part& P : parts) {
    const size_t nr = P.recs.arrival.size();
    if (nr > 0 && P.recs.arrival[0] < max_time) {
      const size_t ln = base + P.rec_line[0];
      throw TraceError{ln, "trace line " + std::to_string(ln) + ": arrivals out of order"};
    }
    out.request_id.insert(out.request_id.end(), P.recs.request_id.begin(), P.recs.request_id.end());
    out.arrival.insert(out.arrival.end(), P.recs.arrival.begin(), P.recs.arrival.end());
    out.language.insert(out.language.end(), P.recs.language.begin(), P.recs.language.end());
    out.task_class.insert(out.task_class.end(), P.recs.task_class.begin(), P.recs.task_class.end());
    out.prompt.insert(out.prompt.end(), P.recs.prompt.begin(), P.recs.prompt.end());
    out.output.insert(out.output.end(), P.recs.output.begin(), P.recs.output.end());
    if (nr > 0) max_time = P.recs.arrival[nr - 1];
    if (P.err) {
      const size_t ln = base + P.err_line;
      throw TraceError{ln, P.err_has_prefix ? "trace line " + std::to_string(ln) + ": " + P.err_what : P.err_what};
    }
    base += P.lines;
  }
  return out;
}

}  // namespace cace
