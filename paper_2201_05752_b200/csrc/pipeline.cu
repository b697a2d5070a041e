// pipeline.cu — host side of the training-data pipeline.
//
//   ranking_plan   make_ranking_batches (data.cpp:128-164): tasks in first-appearance order
//                  (store_task_ids, data.cpp:26-32), each task's rows in store order shuffled by
//                  RngStream(KeyBuilder(seed, "shuffle", task_id)) (Fisher-Yates, data.cpp:16-22),
//                  chunked by batch_size with 1-row tails dropped and counted, then the batch list
//                  shuffled by RngStream(KeyBuilder(seed, "order")). The plan is row indices only: the
//                  feature rows stay on the device and a gather kernel assembles each batch.
//   replay_rows    sample_replay_features' row choice (data.cpp:166-183).
//   epoch_seed     pretrain's per-epoch key (tuner.cpp:136-139).
//   Records        read_records / write_records (data.cpp:67-126): one JSON object per line, fields
//                  task_id, values, throughput_gflops, latency_ms, wall_cost_ms, device_id, seq; the
//                  reader fills flat arrays (pinned by the caller if it wants) with task / device
//                  ids interned in first-appearance order.
// The shuffles are sequential by definition (each swap depends on the previous ones); tasks are
// independent streams, so large plans shuffle one task per host thread.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "pipeline.cuh"

namespace moses {
namespace {

struct Key {  // KeyBuilder (rng.hpp): FNV-1a over 8 LE bytes per integer, string bytes + NUL
  unsigned long long h = 0xcbf29ce484222325ull;
  void step(unsigned char b) {
    h ^= b;
    h *= 0x100000001b3ull;
  }
  Key& add(unsigned long long v) {
    for (int i = 0; i < 8; ++i) step((unsigned char)(v >> (8 * i)));
    return *this;
  }
  Key& add(const char* s) {
    for (; *s; ++s) step((unsigned char)*s);
    step(0);
    return *this;
  }
};
struct Stream {  // RngStream (rng.hpp): SplitMix64; below() rejects r < (2^64 - n) % n
  unsigned long long s;
  unsigned long long next() {
    s += 0x9e3779b97f4a7c15ull;
    unsigned long long z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  unsigned long long below(unsigned long long n) {
    const unsigned long long t = (0ull - n) % n;
    for (;;) {
      const unsigned long long r = next();
      if (r >= t) return r % n;
    }
  }
};
template <class T>
void shuffle_with(std::vector<T>& v, Stream& r) {  // data.cpp:16-22
  for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[r.below(i)]);
}

}  // namespace

unsigned long long epoch_seed(unsigned long long seed, unsigned long long epoch) {
  return Key().add(seed).add("epoch").add(epoch).h;
}

long long ranking_plan(const int* record_task, long long n, const char* const* task_ids, int n_ids, int batch,
                       unsigned long long seed, long long* rows_out, long long* boff, int* btask, long long* dropped) {
  if (batch < 2) fail(MOSES_ERR_INVALID_CONFIG, "batch size must be at least 2");
  if (n < 0 || n_ids < 0) fail(MOSES_ERR_INVALID_ARG, "negative sizes");
  for (int a = 0; a < n_ids; ++a) {
    if (task_ids == nullptr || task_ids[a] == nullptr) fail(MOSES_ERR_INVALID_ARG, "null task id");
    for (int b = 0; b < a; ++b)
      if (std::strcmp(task_ids[a], task_ids[b]) == 0)
        fail(MOSES_ERR_INVALID_ARG, std::string("duplicate task id ") + task_ids[a]);
  }
  std::vector<int> order;  // store_task_ids: first appearance
  std::vector<std::vector<long long>> rows(static_cast<size_t>(n_ids));
  for (long long i = 0; i < n; ++i) {
    const int t = record_task[i];
    if (t < 0 || t >= n_ids) fail(MOSES_ERR_INVALID_TASK, "record " + std::to_string(i) + ": unknown task id");
    if (rows[t].empty()) order.push_back(t);
    rows[t].push_back(i);
  }
  auto shuffle_task = [&](int t) {
    Stream r{Key().add(seed).add("shuffle").add(task_ids[t]).h};
    shuffle_with(rows[t], r);
  };
  if (n >= (1 << 16) && order.size() > 1) {
    std::vector<std::thread> th;
    for (int t : order) th.emplace_back(shuffle_task, t);
    for (auto& x : th) x.join();
  } else {
    for (int t : order) shuffle_task(t);
  }
  struct Chunk {
    int task;
    long long start, len;
  };
  std::vector<Chunk> chunks;
  long long drop = 0;
  for (int t : order) {
    const long long m = (long long)rows[t].size();
    for (long long s = 0; s < m; s += batch) {
      const long long len = std::min<long long>(m, s + batch) - s;
      if (len < 2) {
        ++drop;
        continue;
      }
      chunks.push_back({t, s, len});
    }
  }
  Stream orng{Key().add(seed).add("order").h};
  shuffle_with(chunks, orng);
  long long off = 0;
  for (size_t b = 0; b < chunks.size(); ++b) {
    const Chunk& c = chunks[b];
    if (boff) boff[b] = off;
    if (btask) btask[b] = c.task;
    if (rows_out) std::copy(rows[c.task].begin() + c.start, rows[c.task].begin() + c.start + c.len, rows_out + off);
    off += c.len;
  }
  if (boff) boff[chunks.size()] = off;
  if (dropped) *dropped = drop;
  return (long long)chunks.size();
}

long long replay_rows(long long n_records, long long size, unsigned long long seed, long long* rows_out) {
  if (n_records <= 0) fail(MOSES_ERR_EMPTY_DATASET, "empty record store");
  if (size < 1) fail(MOSES_ERR_INVALID_CONFIG, "replay size must be positive");
  std::vector<long long> rows(static_cast<size_t>(n_records));
  for (long long i = 0; i < n_records; ++i) rows[i] = i;
  Stream r{Key().add(seed).add("replay").h};
  shuffle_with(rows, r);
  const long long k = std::min(n_records, size);
  if (rows_out) std::copy(rows.begin(), rows.begin() + k, rows_out);
  return k;
}

// ---------------------------------------------------------------- line-delimited records
namespace {

// Minimal JSON value reader for one record line. Semantics follow what record_from_json_line
// accepts through nlohmann::json (data.cpp:80-105): any object field order, unknown fields
// ignored, last duplicate wins, numbers convertible between integer and floating kinds and
// booleans usable as numbers (get<double>/get<int64_t> on a boolean yields 0/1), strings only
// from strings, trailing garbage is a parse error.
struct Parser {
  const char* p;
  const char* e;
  [[noreturn]] void bad(const std::string& why) { throw Status(MOSES_ERR_PARSE, why); }
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < e && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) bad(std::string("syntax error: expected '") + c + "'");
  }
  static void utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) out += char(cp);
    else if (cp < 0x800) {
      out += char(0xC0 | (cp >> 6));
      out += char(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += char(0xE0 | (cp >> 12));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    } else {
      out += char(0xF0 | (cp >> 18));
      out += char(0x80 | ((cp >> 12) & 0x3F));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    }
  }
  unsigned hex4() {
    if (e - p < 4) bad("syntax error: truncated \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= unsigned(c - '0');
      else if (c >= 'a' && c <= 'f') v |= unsigned(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= unsigned(c - 'A' + 10);
      else bad("syntax error: bad \\u escape");
    }
    return v;
  }
  std::string str() {
    ws();
    if (p >= e || *p != '"') bad("syntax error: expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= e) bad("syntax error: unterminated string");
      const char c = *p++;
      if (c == '"') break;
      if ((unsigned char)c < 0x20) bad("syntax error: control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p >= e) bad("syntax error: unterminated escape");
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
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (e - p < 6 || p[0] != '\\' || p[1] != 'u') bad("syntax error: unpaired surrogate");
            p += 2;
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) bad("syntax error: unpaired surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            bad("syntax error: unpaired surrogate");
          }
          utf8(out, cp);
          break;
        }
        default: bad("syntax error: bad escape");
      }
    }
    return out;
  }
  // a JSON value; kind: 's' string, 'i' signed int, 'u' unsigned int, 'f' float, 'b' bool, 'n' null,
  // 'a' array of numbers (as doubles + exact ints), 'o' other (object / mixed array)
  struct Val {
    char kind = 'n';
    std::string s;
    long long i = 0;
    unsigned long long u = 0;
    double f = 0;
    std::vector<Val> arr;
  };
  Val num() {
    const char* b = p;
    if (p < e && *p == '-') ++p;
    if (p >= e || !(*p >= '0' && *p <= '9')) bad("syntax error: bad number");
    if (*p == '0') ++p;
    else
      while (p < e && *p >= '0' && *p <= '9') ++p;
    bool is_float = false;
    if (p < e && *p == '.') {
      is_float = true;
      ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) bad("syntax error: bad number");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      is_float = true;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || !(*p >= '0' && *p <= '9')) bad("syntax error: bad number");
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    const std::string tok(b, p);
    Val v;
    if (!is_float) {
      errno = 0;
      if (tok[0] == '-') {
        const long long x = std::strtoll(tok.c_str(), nullptr, 10);
        if (errno == 0) {
          v.kind = 'i';
          v.i = x;
          return v;
        }
      } else {
        const unsigned long long x = std::strtoull(tok.c_str(), nullptr, 10);
        if (errno == 0) {
          v.kind = 'u';
          v.u = x;
          return v;
        }
      }
    }
    v.kind = 'f';
    v.f = std::strtod(tok.c_str(), nullptr);
    if (!std::isfinite(v.f)) bad("number overflow parsing '" + tok + "'");  // nlohmann rejects it too
    return v;
  }
  Val value(int depth = 0) {
    if (depth > 64) bad("syntax error: nesting too deep");
    ws();
    if (p >= e) bad("syntax error: unexpected end of input");
    Val v;
    const char c = *p;
    if (c == '"') {
      v.kind = 's';
      v.s = str();
    } else if (c == '{') {
      ++p;
      v.kind = 'o';
      if (!eat('}')) {
        do {
          str();
          expect(':');
          value(depth + 1);
        } while (eat(','));
        expect('}');
      }
    } else if (c == '[') {
      ++p;
      v.kind = 'a';
      if (!eat(']')) {
        do v.arr.push_back(value(depth + 1));
        while (eat(','));
        expect(']');
      }
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      v = num();
    } else if (e - p >= 4 && std::strncmp(p, "true", 4) == 0) {
      p += 4;
      v.kind = 'b';
      v.u = 1;
    } else if (e - p >= 5 && std::strncmp(p, "false", 5) == 0) {
      p += 5;
      v.kind = 'b';
      v.u = 0;
    } else if (e - p >= 4 && std::strncmp(p, "null", 4) == 0) {
      p += 4;
      v.kind = 'n';
    } else {
      bad("syntax error: invalid literal");
    }
    return v;
  }
};

[[noreturn]] void type_error(const std::string& origin, const char* field, const char* want) {
  fail(MOSES_ERR_PARSE, origin + ": field '" + field + "' must be " + want);
}
double as_double(const Parser::Val& v, const std::string& origin, const char* field) {
  switch (v.kind) {
    case 'f': return v.f;
    case 'i': return double(v.i);
    case 'u': case 'b': return double(v.u);
    default: type_error(origin, field, "a number");
  }
}
long long as_i64(const Parser::Val& v, const std::string& origin, const char* field) {
  switch (v.kind) {
    case 'f': return (long long)v.f;
    case 'i': return v.i;
    case 'u': case 'b': return (long long)v.u;
    default: type_error(origin, field, "a number");
  }
}
unsigned long long as_u64(const Parser::Val& v, const std::string& origin, const char* field) {
  switch (v.kind) {
    case 'f': return (unsigned long long)v.f;
    case 'i': return (unsigned long long)v.i;
    case 'u': case 'b': return v.u;
    default: type_error(origin, field, "a number");
  }
}

int intern(std::vector<std::string>& tab, std::map<std::string, int>& ix, const std::string& s) {
  auto it = ix.find(s);
  if (it != ix.end()) return it->second;
  const int id = int(tab.size());
  tab.push_back(s);
  ix.emplace(s, id);
  return id;
}

// nlohmann::json's number layout (serializer dump_float / to_chars format_buffer) over the shortest
// round-trip digits: k digits d1..dk with the decimal point after position n; fixed notation for
// -4 < n <= 15 (integral values keep ".0"), otherwise d1.d2..dk e+XX with at least two exponent digits.
std::string fmt_double(double x) {
  if (!std::isfinite(x)) return "null";  // nlohmann dumps non-finite numbers as null
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[48];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, x);
    if (std::strtod(buf, nullptr) == x) break;
  }
  std::string s(buf);
  const bool neg = s[0] == '-';
  if (neg) s.erase(0, 1);
  const size_t epos = s.find('e');
  const int e10 = std::atoi(s.c_str() + epos + 1);
  std::string dg = s.substr(0, 1) + (epos > 2 ? s.substr(2, epos - 2) : std::string());
  while (dg.size() > 1 && dg.back() == '0') dg.pop_back();
  const int k = int(dg.size()), n = e10 + 1;
  std::string o;
  if (k <= n && n <= 15) {
    o = dg + std::string(size_t(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    o = dg.substr(0, size_t(n)) + "." + dg.substr(size_t(n));
  } else if (-4 < n && n <= 0) {
    o = "0." + std::string(size_t(-n), '0') + dg;
  } else {
    o = dg.substr(0, 1);
    if (k > 1) o += "." + dg.substr(1);
    const int e = n - 1;
    o += e < 0 ? "e-" : "e+";
    const int ae = e < 0 ? -e : e;
    if (ae < 10) o += '0';
    o += std::to_string(ae);
  }
  return neg ? "-" + o : o;
}
std::string quote(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += char(c);
        }
    }
  }
  return o + "\"";
}

}  // namespace

void Records::parse_line(const std::string& line, const std::string& origin) {
  Parser ps{line.data(), line.data() + line.size()};
  std::map<std::string, Parser::Val> fields;
  try {
    ps.ws();
    if (ps.p >= ps.e || *ps.p != '{') ps.bad("syntax error: expected object");
    ++ps.p;
    if (!ps.eat('}')) {
      do {
        std::string k = ps.str();
        ps.expect(':');
        fields[k] = ps.value(1);
      } while (ps.eat(','));
      ps.expect('}');
    }
    ps.ws();
    if (ps.p != ps.e) ps.bad("syntax error: trailing characters");
  } catch (const Status& s) {
    fail(MOSES_ERR_PARSE, origin + ": " + s.what());
  }
  auto need = [&](const char* f) -> const Parser::Val& {
    auto it = fields.find(f);
    if (it == fields.end()) fail(MOSES_ERR_MISSING_FIELD, origin + ": record missing field '" + f + "'");
    return it->second;
  };
  const Parser::Val& tid = need("task_id");
  if (tid.kind != 's') type_error(origin, "task_id", "a string");
  const Parser::Val& vals = need("values");
  if (vals.kind != 'a') type_error(origin, "values", "an array of integers");
  std::vector<long long> vv;
  vv.reserve(vals.arr.size());
  for (const auto& x : vals.arr) vv.push_back(as_i64(x, origin, "values"));
  const double thr = as_double(need("throughput_gflops"), origin, "throughput_gflops");
  const double lat = as_double(need("latency_ms"), origin, "latency_ms");
  const double wall = as_double(need("wall_cost_ms"), origin, "wall_cost_ms");
  const Parser::Val& did = need("device_id");
  if (did.kind != 's') type_error(origin, "device_id", "a string");
  const unsigned long long sq = as_u64(need("seq"), origin, "seq");
  task.push_back(intern(task_ids, task_ix, tid.s));
  device.push_back(intern(device_ids, device_ix, did.s));
  value_off.push_back(value_off.back() + (long long)vv.size());
  values.insert(values.end(), vv.begin(), vv.end());
  throughput.push_back(thr);
  latency.push_back(lat);
  wall_cost.push_back(wall);
  seq.push_back(sq);
}

Records* Records::read(const char* path) {
  std::ifstream in(path ? path : "", std::ios::binary);
  if (!in) fail(MOSES_ERR_IO, std::string("cannot open record file ") + (path ? path : ""));
  auto* r = new Records();
  try {
    std::string line;
    long long lineno = 0;
    while (std::getline(in, line)) {
      ++lineno;
      if (line.empty()) continue;
      r->parse_line(line, std::string(path) + ":line " + std::to_string(lineno));
    }
  } catch (...) {
    delete r;
    throw;
  }
  return r;
}

std::string Records::line(long long i) const {
  // nlohmann::json objects are key-sorted: device_id, latency_ms, seq, task_id, throughput_gflops,
  // values, wall_cost_ms
  std::string o = "{\"device_id\":" + quote(device_ids[device[i]]) + ",\"latency_ms\":" + fmt_double(latency[i]) +
                  ",\"seq\":" + std::to_string(seq[i]) + ",\"task_id\":" + quote(task_ids[task[i]]) +
                  ",\"throughput_gflops\":" + fmt_double(throughput[i]) + ",\"values\":[";
  for (long long k = value_off[i]; k < value_off[i + 1]; ++k) {
    if (k > value_off[i]) o += ',';
    o += std::to_string(values[k]);
  }
  o += "],\"wall_cost_ms\":" + fmt_double(wall_cost[i]) + "}";
  return o;
}

void Records::write(const char* path) const {
  std::ofstream out(path ? path : "", std::ios::binary | std::ios::trunc);
  if (!out) fail(MOSES_ERR_IO, std::string("cannot open ") + (path ? path : "") + " for writing");
  for (long long i = 0; i < size(); ++i) out << line(i) << '\n';
  if (!out) fail(MOSES_ERR_IO, std::string("short write to ") + path);
}

}  // namespace moses
