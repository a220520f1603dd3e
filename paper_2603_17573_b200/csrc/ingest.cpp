// ingest.cpp — DB ingest into HBM: the reference's
// JSONL v1 database file (store.cpp:138-191) parsed natively and
// in parallel into a columnar host image (fp32 keys, fp64 next_actions, payload
// indices, fp32 features), then uploaded to a device collection; plus a binary
// columnar device image (save/load) for fast reload of large shards.
//
// Error behaviour follows load_collection (store.cpp:152-191) line for line:
// the same checks in the same order, hsd::ParseError's line number (exposed as
// hsd_last_error_line), VersionError for version != 1, ConfigError for a
// non-positive dim.  Where the reference lets a nlohmann::json exception escape
// (a non-numeric embedding element, a non-string metric), this loader reports
// a ParseError with the line instead.  Records' features must share one
// length (the device table is [n][d_f]); a mismatch is a SchemaError.
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "hsd/hsd_gpu.h"

// Implemented in api.cu (error plumbing shared with the rest of the ABI).
hsd_status hsd_internal_fail(hsd_status st, const char* msg, long line);

namespace {

// ------------------------------------------------------------------ JSON value
struct JVal {
  enum Type { Null, Bool, Num, Str, Arr, Obj } t = Null;
  bool b = false;
  bool is_int = false;  // number literal without fraction / exponent (nlohmann is_number_integer)
  double num = 0.0;
  std::string str;                                // Str (and the Num literal, for messages)
  std::vector<JVal> arr;                          // Arr
  std::vector<std::pair<std::string, JVal>> obj;  // Obj (duplicate keys: the last one wins on lookup)

  const JVal* get(const char* key) const {
    const JVal* r = nullptr;
    for (const auto& kv : obj)
      if (kv.first == key) r = &kv.second;
    return r;
  }
};

// Strict JSON (RFC 8259) recursive-descent parser over one line.
class Parser {
 public:
  Parser(const char* p, const char* e) : p_(p), e_(e) {}
  bool parse_document(JVal& v) {
    ws();
    if (!value(v, 0)) return false;
    ws();
    return p_ == e_;
  }

 private:
  const char* p_;
  const char* e_;

  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
  }
  bool lit(const char* s) {
    const size_t n = strlen(s);
    if ((size_t)(e_ - p_) < n || memcmp(p_, s, n) != 0) return false;
    p_ += n;
    return true;
  }
  bool value(JVal& v, int depth) {
    if (depth > 64 || p_ >= e_) return false;
    switch (*p_) {
      case '{': return object(v, depth);
      case '[': return array(v, depth);
      case '"': v.t = JVal::Str; return string(v.str);
      case 't': v.t = JVal::Bool; v.b = true; return lit("true");
      case 'f': v.t = JVal::Bool; v.b = false; return lit("false");
      case 'n': v.t = JVal::Null; return lit("null");
      default: return number(v);
    }
  }
  bool number(JVal& v) {
    const char* s = p_;
    if (p_ < e_ && *p_ == '-') ++p_;
    if (p_ >= e_) return false;
    if (*p_ == '0') {
      ++p_;
    } else if (*p_ >= '1' && *p_ <= '9') {
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    } else {
      return false;
    }
    bool is_int = true;
    if (p_ < e_ && *p_ == '.') {
      is_int = false;
      ++p_;
      if (p_ >= e_ || *p_ < '0' || *p_ > '9') return false;
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
      is_int = false;
      ++p_;
      if (p_ < e_ && (*p_ == '+' || *p_ == '-')) ++p_;
      if (p_ >= e_ || *p_ < '0' || *p_ > '9') return false;
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    char buf[64];
    std::string big;
    const size_t n = (size_t)(p_ - s);
    const char* z;
    if (n < sizeof(buf)) {
      memcpy(buf, s, n);
      buf[n] = 0;
      z = buf;
    } else {
      big.assign(s, n);
      z = big.c_str();
    }
    v.t = JVal::Num;
    v.is_int = is_int;
    v.num = strtod(z, nullptr);  // correctly rounded, as nlohmann's number_float parse
    return true;
  }
  static void put_utf8(std::string& out, uint32_t c) {
    if (c < 0x80) {
      out += (char)c;
    } else if (c < 0x800) {
      out += (char)(0xC0 | (c >> 6));
      out += (char)(0x80 | (c & 0x3F));
    } else if (c < 0x10000) {
      out += (char)(0xE0 | (c >> 12));
      out += (char)(0x80 | ((c >> 6) & 0x3F));
      out += (char)(0x80 | (c & 0x3F));
    } else {
      out += (char)(0xF0 | (c >> 18));
      out += (char)(0x80 | ((c >> 12) & 0x3F));
      out += (char)(0x80 | ((c >> 6) & 0x3F));
      out += (char)(0x80 | (c & 0x3F));
    }
  }
  bool hex4(uint32_t& c) {
    if (e_ - p_ < 4) return false;
    c = 0;
    for (int i = 0; i < 4; ++i) {
      const char h = *p_++;
      c <<= 4;
      if (h >= '0' && h <= '9') c |= (uint32_t)(h - '0');
      else if (h >= 'a' && h <= 'f') c |= (uint32_t)(h - 'a' + 10);
      else if (h >= 'A' && h <= 'F') c |= (uint32_t)(h - 'A' + 10);
      else return false;
    }
    return true;
  }
  bool string(std::string& out) {
    ++p_;  // opening quote
    out.clear();
    while (p_ < e_) {
      const unsigned char c = (unsigned char)*p_++;
      if (c == '"') return true;
      if (c < 0x20) return false;  // control characters must be escaped
      if (c != '\\') {
        out += (char)c;
        continue;
      }
      if (p_ >= e_) return false;
      const char x = *p_++;
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
          uint32_t cp;
          if (!hex4(cp)) return false;
          if (cp >= 0xD800 && cp <= 0xDBFF) {  // surrogate pair
            uint32_t lo;
            if (e_ - p_ < 2 || p_[0] != '\\' || p_[1] != 'u') return false;
            p_ += 2;
            if (!hex4(lo) || lo < 0xDC00 || lo > 0xDFFF) return false;
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            return false;
          }
          put_utf8(out, cp);
          break;
        }
        default: return false;
      }
    }
    return false;
  }
  bool array(JVal& v, int depth) {
    ++p_;
    v.t = JVal::Arr;
    ws();
    if (p_ < e_ && *p_ == ']') {
      ++p_;
      return true;
    }
    for (;;) {
      v.arr.emplace_back();
      ws();
      if (!value(v.arr.back(), depth + 1)) return false;
      ws();
      if (p_ >= e_) return false;
      if (*p_ == ',') {
        ++p_;
        continue;
      }
      if (*p_ == ']') {
        ++p_;
        return true;
      }
      return false;
    }
  }
  bool object(JVal& v, int depth) {
    ++p_;
    v.t = JVal::Obj;
    ws();
    if (p_ < e_ && *p_ == '}') {
      ++p_;
      return true;
    }
    for (;;) {
      ws();
      if (p_ >= e_ || *p_ != '"') return false;
      std::string key;
      if (!string(key)) return false;
      ws();
      if (p_ >= e_ || *p_ != ':') return false;
      ++p_;
      ws();
      v.obj.emplace_back(std::move(key), JVal());
      if (!value(v.obj.back().second, depth + 1)) return false;
      ws();
      if (p_ >= e_) return false;
      if (*p_ == ',') {
        ++p_;
        continue;
      }
      if (*p_ == '}') {
        ++p_;
        return true;
      }
      return false;
    }
  }
};

bool parse_line(const std::string& line, JVal& v) {
  Parser ps(line.data(), line.data() + line.size());
  return ps.parse_document(v);
}

// nlohmann get<int>() of a number (floats truncate toward zero).
bool as_int(const JVal* v, int& out) {
  if (!v || v->t != JVal::Num) return false;
  out = (int)v->num;
  return true;
}
bool as_doubles(const JVal* v, std::vector<double>& out) {
  if (!v || v->t != JVal::Arr) return false;
  out.resize(v->arr.size());
  for (size_t i = 0; i < v->arr.size(); ++i) {
    if (v->arr[i].t != JVal::Num) return false;
    out[i] = v->arr[i].num;
  }
  return true;
}

struct Err {
  long line = 0;  // 0 = no error
  hsd_status st = HSD_OK;
  std::string msg;
};

// One parsed record (store.cpp:175-188 + payload_from_json :108-134).
struct Rec {
  std::vector<double> emb;
  double next[21];
  int ep = 0, st = 0;
  bool has_feat = false;
  std::vector<double> feat;
};

bool parse_record(const std::string& line, long line_no, int dim, Rec& r, Err& err) {
  auto perr = [&](const std::string& m) {
    err.line = line_no;
    err.st = HSD_ERR_PARSE;
    err.msg = m;
    return false;
  };
  JVal j;
  if (!parse_line(line, j) || j.t != JVal::Obj) return perr("malformed record");
  const JVal* e = j.get("embedding");
  if (!e || e->t != JVal::Arr) return perr("record lacks an embedding");
  if (!as_doubles(e, r.emb)) return perr("embedding elements must be numbers");
  if ((int)r.emb.size() != dim) return perr("embedding dim mismatch");
  const JVal* p = j.get("payload");
  if (!p) return perr("record lacks a payload");
  // payload_from_json (store.cpp:108-134)
  if (p->t != JVal::Obj) return perr("bad payload: not an object");
  const JVal* dn = p->get("dataset_name");
  if (!dn || dn->t != JVal::Str) return perr("bad payload: dataset_name");
  if (!as_int(p->get("episode_idx"), r.ep)) return perr("bad payload: episode_idx");
  if (!as_int(p->get("step_idx"), r.st)) return perr("bad payload: step_idx");
  const JVal* cur = p->get("current_action");
  if (!cur) return perr("bad payload: current_action");
  if (cur->t != JVal::Arr || cur->arr.size() != 7) return perr("current_action must have 7 entries");
  for (const auto& x : cur->arr)
    if (x.t != JVal::Num) return perr("bad payload: current_action");
  const JVal* nx = p->get("next_actions");
  if (!nx) return perr("bad payload: next_actions");
  if (nx->t != JVal::Arr || nx->arr.size() != 3) return perr("next_actions must have 3 rows");
  for (int s = 0; s < 3; ++s) {
    const JVal& row = nx->arr[(size_t)s];
    if (row.t != JVal::Arr || row.arr.size() != 7) return perr("next_actions rows must have 7 entries");
    for (int i = 0; i < 7; ++i) {
      if (row.arr[(size_t)i].t != JVal::Num) return perr("bad payload: next_actions");
      r.next[s * 7 + i] = row.arr[(size_t)i].num;
    }
  }
  const JVal* li = p->get("language_instruction");
  if (!li || li->t != JVal::Str) return perr("bad payload: language_instruction");
  if (r.ep < 0 || r.st < 0) return perr("negative payload index");
  const JVal* f = j.get("feature");
  r.has_feat = f && f->t != JVal::Null;
  if (r.has_feat && !as_doubles(f, r.feat)) return perr("feature must be an array of numbers");
  return true;
}

}  // namespace

struct hsd_jsonl_db {
  std::string name;
  int dim = 0, d_f = 0;
  int64_t n = 0;
  std::vector<float> emb;       // [n][dim] (fp32 rounding of the parsed doubles)
  std::vector<double> next;     // [n][21]
  std::vector<int32_t> ep, st;  // [n]
  std::vector<float> feat;      // [n][d_f] (zeros where absent)
  std::vector<uint8_t> has_feat;
};

extern "C" {

hsd_status hsd_jsonl_read(const char* path, int threads, hsd_jsonl_db** out) {
  if (!path || !out) return hsd_internal_fail(HSD_ERR_INVALID_INPUT, "null pointer", 0);
  *out = nullptr;
  std::ifstream in(path, std::ios::binary);
  if (!in) return hsd_internal_fail(HSD_ERR_IO, (std::string("cannot open for reading: ") + path).c_str(), 0);
  std::string line;
  long line_no = 0;
  // ---- header (store.cpp:159-171)
  if (!std::getline(in, line)) return hsd_internal_fail(HSD_ERR_PARSE, "missing header line", 1);
  ++line_no;
  JVal h;
  if (!parse_line(line, h) || h.t != JVal::Obj) return hsd_internal_fail(HSD_ERR_PARSE, "malformed header", line_no);
  const JVal* ver = h.get("version");
  if (!ver || ver->t != JVal::Num || !ver->is_int)
    return hsd_internal_fail(HSD_ERR_PARSE, "header lacks a version", line_no);
  if (ver->num != 1.0) {
    char m[96];
    snprintf(m, sizeof m, "unsupported database version %.17g", ver->num);
    return hsd_internal_fail(HSD_ERR_VERSION, m, 0);
  }
  const JVal* met = h.get("metric");
  if (!met || met->t != JVal::Str || met->str != "cosine")
    return hsd_internal_fail(HSD_ERR_PARSE, "unsupported metric", line_no);
  auto* db = new hsd_jsonl_db();
  const JVal* nm = h.get("name");
  if (nm && nm->t == JVal::Str) db->name = nm->str;
  int dim = 0;
  const JVal* dj = h.get("dim");
  if (dj && !as_int(dj, dim)) dim = 0;
  if (dim < 1) {  // Collection(name, dim), store.cpp:36-38
    delete db;
    return hsd_internal_fail(HSD_ERR_CONFIG, "collection dim must be >= 1", 0);
  }
  db->dim = dim;
  // ---- records: parsed in parallel chunks of lines, appended in file order
  const int nt = threads > 0 ? threads : std::max(1u, std::thread::hardware_concurrency());
  constexpr size_t kChunk = 4096;
  std::vector<std::string> lines;
  std::vector<long> nos;
  Err first;
  bool done = false;
  while (!done) {
    lines.clear();
    nos.clear();
    while (lines.size() < kChunk) {
      if (!std::getline(in, line)) {
        done = true;
        break;
      }
      ++line_no;
      if (line.empty()) continue;  // store.cpp:175
      lines.push_back(std::move(line));
      nos.push_back(line_no);
    }
    const size_t m = lines.size();
    if (m == 0) break;
    std::vector<Rec> recs(m);
    std::vector<Err> errs(m);
    auto work = [&](int t) {
      for (size_t i = (size_t)t; i < m; i += (size_t)nt) parse_record(lines[i], nos[i], dim, recs[i], errs[i]);
    };
    if (nt > 1 && m > 64) {
      std::vector<std::thread> pool;
      for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
      for (auto& th : pool) th.join();
    } else {
      for (size_t i = 0; i < m; ++i) parse_record(lines[i], nos[i], dim, recs[i], errs[i]);
    }
    for (size_t i = 0; i < m; ++i) {
      if (errs[i].line) {  // the first failing line in file order (the reference stops there)
        first = errs[i];
        break;
      }
      const Rec& r = recs[i];
      if (r.has_feat) {
        if (db->d_f == 0 && !r.feat.empty()) {
          db->d_f = (int)r.feat.size();
          db->feat.assign((size_t)db->n * db->d_f, 0.f);  // earlier records had none
        }
        if ((int)r.feat.size() != db->d_f) {
          first.line = nos[i];
          first.st = HSD_ERR_SCHEMA;
          first.msg = "feature length differs from the collection's first feature";
          break;
        }
      }
      for (double x : r.emb) db->emb.push_back((float)x);
      db->next.insert(db->next.end(), r.next, r.next + 21);
      db->ep.push_back(r.ep);
      db->st.push_back(r.st);
      db->has_feat.push_back(r.has_feat ? 1 : 0);
      if (db->d_f) {
        if (r.has_feat)
          for (double x : r.feat) db->feat.push_back((float)x);
        else
          db->feat.insert(db->feat.end(), (size_t)db->d_f, 0.f);
      }
      ++db->n;
    }
    if (first.line) break;
  }
  if (first.line) {
    delete db;
    return hsd_internal_fail(first.st, first.msg.c_str(), first.line);
  }
  *out = db;
  return HSD_OK;
}

hsd_status hsd_jsonl_free(hsd_jsonl_db* db) {
  delete db;
  return HSD_OK;
}

hsd_status hsd_jsonl_info(const hsd_jsonl_db* db, int64_t* n, int* dim, int* d_f, const char** name) {
  if (!db) return hsd_internal_fail(HSD_ERR_INVALID_INPUT, "null db", 0);
  if (n) *n = db->n;
  if (dim) *dim = db->dim;
  if (d_f) *d_f = db->d_f;
  if (name) *name = db->name.c_str();
  return HSD_OK;
}

hsd_status hsd_jsonl_data(const hsd_jsonl_db* db, const float** emb, const double** next_actions,
                          const int32_t** episode_idx, const int32_t** step_idx, const float** features,
                          const uint8_t** has_feature) {
  if (!db) return hsd_internal_fail(HSD_ERR_INVALID_INPUT, "null db", 0);
  if (emb) *emb = db->emb.data();
  if (next_actions) *next_actions = db->next.data();
  if (episode_idx) *episode_idx = db->ep.data();
  if (step_idx) *step_idx = db->st.data();
  if (features) *features = db->d_f ? db->feat.data() : nullptr;
  if (has_feature) *has_feature = db->has_feat.data();
  return HSD_OK;
}

hsd_status hsd_collection_from_jsonl(const hsd_jsonl_db* db, int device, int dtype, hsd_collection** out) {
  if (!db || !out) return hsd_internal_fail(HSD_ERR_INVALID_INPUT, "null pointer", 0);
  hsd_status st = hsd_collection_create_ex(device, db->dim, std::max<int64_t>(db->n, 1), dtype, out);
  if (st != HSD_OK) return st;
  if (db->n == 0) return HSD_OK;
  int64_t first = 0;
  st = hsd_collection_insert(*out, db->emb.data(), db->next.data(), db->ep.data(), db->st.data(), db->n, &first);
  if (st == HSD_OK && db->d_f)  // Record::feature rows (store.cpp:184-188) travel to the device too
    st = hsd_collection_set_features(*out, 0, db->n, db->d_f, db->feat.data(), db->has_feat.data());
  if (st != HSD_OK) {
    hsd_collection_destroy(*out);
    *out = nullptr;
  }
  return st;
}

hsd_status hsd_collection_load_jsonl(const char* path, int device, int dtype, hsd_collection** out) {
  hsd_jsonl_db* db = nullptr;
  hsd_status st = hsd_jsonl_read(path, 0, &db);
  if (st != HSD_OK) return st;
  st = hsd_collection_from_jsonl(db, device, dtype, out);
  hsd_jsonl_free(db);
  return st;
}

}  // extern "C"
