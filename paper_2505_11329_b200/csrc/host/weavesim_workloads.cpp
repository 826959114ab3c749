// weavesim_workloads.cpp -- request traces and chunked-prefill batch formation
// (host C++), same semantics and errors as the reference:
//   load_trace / save_trace   proj/src/workloads.cpp:14-54 (JSONL, ParseError)
//   synth_trace               proj/src/workloads.cpp:56-66
//   form_batches              proj/src/workloads.cpp:68-109
// The reference parses with nlohmann::json; this build has a small strict
// JSON reader (full RFC 8259 value grammar, top-level numbers extracted) so
// the library has no third-party dependency.  Parity: tests/test_workloads.py
// against the reference itself (oracle/_ref) and tests/golden/.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <cctype>
#include <string>

#include "weavesim/errors.hpp"
#include "weavesim/workloads.hpp"

namespace weavesim {

namespace {

// One JSON text -> its top-level object's numeric members (other member
// types are parsed and recorded as non-numeric).  Throws std::runtime_error
// on any syntax error.
class JsonLine {
 public:
  explicit JsonLine(const std::string& s) : s_(s) {}

  struct Member {
    bool is_number = false;
    bool is_integer = false;
    double number = 0.0;
    std::int64_t integer = 0;
  };

  // Returns false when the text is valid JSON but not an object.
  bool parse(std::map<std::string, Member>& members) {
    ws();
    bool object = peek() == '{';
    if (object) {
      ++i_;
      ws();
      if (peek() == '}') {
        ++i_;
      } else {
        for (;;) {
          ws();
          std::string key = string();
          ws();
          expect(':');
          ws();
          members[key] = value();  // duplicate keys: last wins, as nlohmann
          ws();
          if (peek() == ',') {
            ++i_;
            continue;
          }
          expect('}');
          break;
        }
      }
    } else {
      (void)value();
    }
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return object;
  }

 private:
  [[noreturn]] void fail(const char* why) const {
    throw std::runtime_error(std::string("syntax error at byte ") + std::to_string(i_ + 1) + ": " + why);
  }
  char peek() const { return i_ < s_.size() ? s_[i_] : '\0'; }
  void expect(char c) {
    if (peek() != c) fail((std::string("expected '") + c + "'").c_str());
    ++i_;
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r')) ++i_;
  }
  void literal(const char* word) {
    const size_t n = std::strlen(word);
    if (s_.compare(i_, n, word) != 0) fail("invalid literal");
    i_ += n;
  }
  std::string string() {
    expect('"');
    std::string out;
    for (;;) {
      if (i_ >= s_.size()) fail("unterminated string");
      const char c = s_[i_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out.push_back(c);
        continue;
      }
      const char e = peek();
      ++i_;
      switch (e) {
        case '"': case '\\': case '/': out.push_back(e); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u':
          for (int k = 0; k < 4; ++k, ++i_)
            if (!std::isxdigit(static_cast<unsigned char>(peek()))) fail("bad \\u escape");
          out.push_back('?');  // key text beyond ASCII is never a trace field
          break;
        default: fail("bad escape");
      }
    }
  }
  Member number() {
    const size_t b = i_;
    bool integral = true;
    if (peek() == '-') ++i_;
    if (peek() == '0') {
      ++i_;
    } else if (peek() >= '1' && peek() <= '9') {
      while (std::isdigit(static_cast<unsigned char>(peek()))) ++i_;
    } else {
      fail("invalid number");
    }
    if (peek() == '.') {
      integral = false;
      ++i_;
      if (!std::isdigit(static_cast<unsigned char>(peek()))) fail("invalid number");
      while (std::isdigit(static_cast<unsigned char>(peek()))) ++i_;
    }
    if (peek() == 'e' || peek() == 'E') {
      integral = false;
      ++i_;
      if (peek() == '+' || peek() == '-') ++i_;
      if (!std::isdigit(static_cast<unsigned char>(peek()))) fail("invalid number");
      while (std::isdigit(static_cast<unsigned char>(peek()))) ++i_;
    }
    Member m;
    m.is_number = true;
    const std::string text = s_.substr(b, i_ - b);
    m.number = std::strtod(text.c_str(), nullptr);
    if (integral) {
      auto r = std::from_chars(text.data(), text.data() + text.size(), m.integer);
      m.is_integer = r.ec == std::errc();  // out of int64 range: stored as a float, like nlohmann
    }
    return m;
  }
  Member value() {
    const char c = peek();
    if (c == '{') {
      ++i_;
      ws();
      if (peek() == '}') {
        ++i_;
        return {};
      }
      for (;;) {
        ws();
        (void)string();
        ws();
        expect(':');
        ws();
        (void)value();
        ws();
        if (peek() == ',') {
          ++i_;
          continue;
        }
        expect('}');
        return {};
      }
    }
    if (c == '[') {
      ++i_;
      ws();
      if (peek() == ']') {
        ++i_;
        return {};
      }
      for (;;) {
        ws();
        (void)value();
        ws();
        if (peek() == ',') {
          ++i_;
          continue;
        }
        expect(']');
        return {};
      }
    }
    if (c == '"') {
      (void)string();
      return {};
    }
    if (c == 't') return literal("true"), Member{};
    if (c == 'f') return literal("false"), Member{};
    if (c == 'n') return literal("null"), Member{};
    return number();
  }

  const std::string& s_;
  size_t i_ = 0;
};

std::string where(const std::string& path, std::int64_t line_no) {
  return "trace " + path + " line " + std::to_string(line_no);
}

std::int64_t as_int(const JsonLine::Member& m, const std::string& ctx, const char* key) {
  if (!m.is_number) throw ParseError(ctx + ": " + key + " must be a number");
  if (m.is_integer) return m.integer;
  if (!std::isfinite(m.number) || std::fabs(m.number) >= 9.2e18) throw ParseError(ctx + ": " + key + " out of range");
  return static_cast<std::int64_t>(m.number);  // nlohmann get<int64_t> truncates a float
}

// Shortest round-trip decimal of a double with a ".0" on integral values --
// the text nlohmann::json::dump writes for a float member.
std::string dump_double(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

}  // namespace

std::vector<Request> load_trace(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open trace: " + path);
  std::vector<Request> requests;
  std::string line;
  std::int64_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::map<std::string, JsonLine::Member> m;
    bool object = false;
    try {
      object = JsonLine(line).parse(m);
    } catch (const std::runtime_error& e) {
      throw ParseError(where(path, line_no) + ": " + e.what());
    }
    const std::string ctx = where(path, line_no);
    if (!object || !m.count("prompt_tokens") || !m.count("output_tokens"))
      throw ParseError(ctx + ": prompt_tokens and output_tokens are required");
    Request r;
    r.id = static_cast<std::int64_t>(requests.size());
    r.prompt_tokens = as_int(m["prompt_tokens"], ctx, "prompt_tokens");
    r.output_tokens = as_int(m["output_tokens"], ctx, "output_tokens");
    if (m.count("arrival_s")) {
      if (!m["arrival_s"].is_number) throw ParseError(ctx + ": arrival_s must be a number");
      r.arrival_s = m["arrival_s"].number;
    }
    if (r.prompt_tokens < 1 || r.output_tokens < 0 || r.arrival_s < 0.0)
      throw ParseError(ctx + ": values out of range");
    requests.push_back(r);
  }
  return requests;
}

void save_trace(const std::vector<Request>& requests, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw ParseError("cannot write trace: " + path);
  for (const Request& r : requests) {
    // Keys in lexicographic order, as nlohmann's std::map-backed object dumps.
    out << '{';
    if (r.arrival_s > 0.0) out << "\"arrival_s\":" << dump_double(r.arrival_s) << ',';
    out << "\"output_tokens\":" << r.output_tokens << ",\"prompt_tokens\":" << r.prompt_tokens << "}\n";
  }
}

std::vector<Request> synth_trace(std::int64_t count, std::int64_t prompt_len, std::int64_t output_len) {
  if (count < 1 || prompt_len < 1 || output_len < 0)
    throw ConfigError("synth_trace: count and prompt_len must be positive");
  std::vector<Request> requests(static_cast<size_t>(count));
  for (std::int64_t i = 0; i < count; ++i) requests[static_cast<size_t>(i)] = {i, prompt_len, output_len, 0.0};
  return requests;
}

std::vector<IterationBatch> form_batches(const std::vector<Request>& requests, std::int64_t chunk_size) {
  if (chunk_size < 1) throw ConfigError("form_batches: chunk_size must be >= 1");
  // FCFS by arrival, stable on ties (workloads.cpp:76-80).
  std::vector<size_t> order(requests.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return requests[a].arrival_s < requests[b].arrival_s; });

  std::vector<std::int64_t> prefilled(requests.size(), 0), decoded(requests.size(), 0);
  // Requests whose prefill is complete and decode is not, in FCFS order; and
  // the FCFS cursor of the first request still prefilling.  Per iteration this
  // touches only live requests instead of rescanning the whole trace.
  std::vector<size_t> decoding;
  size_t next_prefill = 0;
  std::vector<IterationBatch> batches;
  for (;;) {
    IterationBatch batch;
    // Decode-first: one token per request whose prefill has completed.
    // A request enters `decoding` in the iteration its prefill completes, so
    // it decodes from the next iteration on (workloads.cpp:86-95).
    size_t keep = 0;
    for (size_t k = 0; k < decoding.size(); ++k) {
      const size_t i = decoding[k];
      ++decoded[i];
      ++batch.decode_token_count;
      batch.kv_context += requests[i].prompt_tokens + decoded[i] - 1;
      if (decoded[i] < requests[i].output_tokens) decoding[keep++] = i;
    }
    decoding.resize(keep);
    // Then prefill chunks, FCFS, up to the token budget (:96-107).
    std::int64_t budget = chunk_size - batch.decode_token_count;
    std::vector<size_t> completed;
    for (size_t k = next_prefill; k < order.size() && budget > 0; ++k) {
      const size_t i = order[k];
      const Request& r = requests[i];
      if (prefilled[i] == r.prompt_tokens) continue;
      const std::int64_t take = std::min(budget, r.prompt_tokens - prefilled[i]);
      batch.prefill_token_slices.push_back({r.id, prefilled[i], take});
      batch.kv_context += prefilled[i];
      prefilled[i] += take;
      budget -= take;
      if (prefilled[i] == r.prompt_tokens && r.output_tokens > 0) completed.push_back(i);
    }
    while (next_prefill < order.size() && prefilled[order[next_prefill]] == requests[order[next_prefill]].prompt_tokens)
      ++next_prefill;
    batch.total_tokens = batch.decode_token_count;
    for (const PrefillSlice& s : batch.prefill_token_slices) batch.total_tokens += s.len;
    if (batch.total_tokens == 0) break;
    // `decoding` stays in FCFS order: requests complete prefill in FCFS order.
    decoding.insert(decoding.end(), completed.begin(), completed.end());
    batches.push_back(std::move(batch));
  }
  return batches;
}

}  // namespace weavesim

// ---- C-ABI (include/tw/tw_workload.h) ---------------------------------------------

#include "tw/tw_workload.h"

namespace {

thread_local std::string g_workload_error;

template <class F>
tw_status guarded(F&& f) {
  g_workload_error.clear();
  try {
    f();
    return TW_OK;
  } catch (const weavesim::DimensionError& e) {
    g_workload_error = e.what();
    return TW_ERR_DIMENSION;
  } catch (const weavesim::ConfigError& e) {
    g_workload_error = e.what();
    return TW_ERR_CONFIG;
  } catch (const weavesim::ParseError& e) {
    g_workload_error = e.what();
    return TW_ERR_PARSE;
  } catch (const std::exception& e) {
    g_workload_error = e.what();
    return TW_ERR_CONTRACT;
  }
}

std::vector<weavesim::Request> to_requests(const tw_request* r, int64_t n) {
  if (n < 0 || (n > 0 && !r)) throw weavesim::DimensionError("requests: null array or negative count");
  std::vector<weavesim::Request> v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) v[static_cast<size_t>(i)] = {r[i].id, r[i].prompt_tokens, r[i].output_tokens, r[i].arrival_s};
  return v;
}

}  // namespace

extern "C" {

const char* tw_workload_last_error(void) { return g_workload_error.c_str(); }

tw_status tw_synth_trace(int64_t count, int64_t prompt_len, int64_t output_len, tw_request* out) {
  return guarded([&] {
    const std::vector<weavesim::Request> v = weavesim::synth_trace(count, prompt_len, output_len);
    if (!out) throw weavesim::DimensionError("synth_trace: null output");
    for (size_t i = 0; i < v.size(); ++i) out[i] = {v[i].id, v[i].prompt_tokens, v[i].output_tokens, v[i].arrival_s};
  });
}

tw_status tw_load_trace(const char* path, tw_request* out, int64_t capacity, int64_t* count) {
  return guarded([&] {
    if (!path || !count) throw weavesim::DimensionError("load_trace: null argument");
    const std::vector<weavesim::Request> v = weavesim::load_trace(path);
    *count = static_cast<int64_t>(v.size());
    const int64_t n = std::min<int64_t>(capacity, *count);
    for (int64_t i = 0; out && i < n; ++i) {
      const weavesim::Request& r = v[static_cast<size_t>(i)];
      out[i] = {r.id, r.prompt_tokens, r.output_tokens, r.arrival_s};
    }
  });
}

tw_status tw_save_trace(const tw_request* requests, int64_t n, const char* path) {
  return guarded([&] {
    if (!path) throw weavesim::DimensionError("save_trace: null path");
    weavesim::save_trace(to_requests(requests, n), path);
  });
}

tw_status tw_form_batches(const tw_request* requests, int64_t n, int64_t chunk_size, tw_iteration_batch* batches,
                          int64_t max_batches, tw_prefill_slice* slices, int64_t max_slices, int64_t* n_batches,
                          int64_t* n_slices) {
  return guarded([&] {
    if (!n_batches || !n_slices) throw weavesim::DimensionError("form_batches: null count pointer");
    const std::vector<weavesim::IterationBatch> v = weavesim::form_batches(to_requests(requests, n), chunk_size);
    int64_t total_slices = 0;
    for (const auto& b : v) total_slices += static_cast<int64_t>(b.prefill_token_slices.size());
    *n_batches = static_cast<int64_t>(v.size());
    *n_slices = total_slices;
    if (max_batches < *n_batches || max_slices < total_slices || (*n_batches && !batches) || (total_slices && !slices))
      throw weavesim::DimensionError("form_batches: output arrays too small (" + std::to_string(*n_batches) +
                                     " batches, " + std::to_string(total_slices) + " slices needed)");
    int64_t s = 0;
    for (size_t k = 0; k < v.size(); ++k) {
      const auto& b = v[k];
      batches[k] = {b.total_tokens, b.decode_token_count, b.kv_context, s,
                    static_cast<int64_t>(b.prefill_token_slices.size())};
      for (const auto& p : b.prefill_token_slices) slices[s++] = {p.request_id, p.start, p.len};
    }
  });
}

}  // extern "C"
