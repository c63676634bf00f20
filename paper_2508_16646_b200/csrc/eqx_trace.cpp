// eqx_trace.cpp -- request traces for the ingestion path: the reference's
// CSV trace format (load_trace / write_trace_csv / trace_hash, workload.cpp:312-428) and a binary
// struct-of-arrays format that loads straight into the pinned host arena, so a trace goes
// file -> pinned columns -> eqx_stage_async / eqx_drain without a per-request object.
//
// Host code: parsing and FNV-1a hashing are sequential byte work that belongs on the CPU; the
// columns it produces are exactly the eqx_requests layout the device path consumes.
#include <algorithm>
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/eqx.h"

namespace {

// Column storage: the pinned arena when the driver can register it, plain heap otherwise (a
// trace can be parsed on a machine without a GPU).
struct Col {
  void* p = nullptr;
  bool pinned = false;
  void alloc(size_t bytes) {
    bytes = std::max<size_t>(bytes, 16);
    p = eqx_host_alloc(static_cast<int64_t>(bytes));
    pinned = p != nullptr;
    if (!p) p = std::calloc(1, bytes);
  }
  void release() {
    if (p) {
      if (pinned) eqx_host_free(p);
      else std::free(p);
    }
    p = nullptr;
  }
};

}  // namespace

struct eqx_trace {
  int64_t n = 0;
  double duration_s = 0.0;
  Col client, arrival, in, out, tag;
  std::vector<std::string> clients, tags, warnings;
  std::string client_blob, tag_blob, warning_blob;
  std::string hash;         // trace_hash, computed on demand
  std::string stored_hash;  // the hash a binary trace was saved with
  ~eqx_trace() {
    client.release();
    arrival.release();
    in.release();
    out.release();
    tag.release();
  }
  void alloc(int64_t rows) {
    n = rows;
    const size_t r = static_cast<size_t>(rows);
    client.alloc(4 * r);
    arrival.alloc(8 * r);
    in.alloc(4 * r);
    out.alloc(4 * r);
    tag.alloc(4 * r);
  }
  int32_t* c_client() { return static_cast<int32_t*>(client.p); }
  double* c_arrival() { return static_cast<double*>(arrival.p); }
  int32_t* c_in() { return static_cast<int32_t*>(in.p); }
  int32_t* c_out() { return static_cast<int32_t*>(out.p); }
  int32_t* c_tag() { return static_cast<int32_t*>(tag.p); }
  void blobs() {
    auto join = [](const std::vector<std::string>& v) {
      std::string b;
      for (const auto& s : v) {
        b += s;
        b.push_back('\0');
      }
      return b;
    };
    client_blob = join(clients);
    tag_blob = join(tags);
    warning_blob = join(warnings);
  }
};

namespace {

void set_err(char* err, int32_t len, const std::string& msg) {
  if (err && len > 0) {
    std::strncpy(err, msg.c_str(), static_cast<size_t>(len) - 1);
    err[len - 1] = '\0';
  }
}

constexpr const char* kHeader = "client_id,arrival_time_s,input_tokens,output_tokens,category_tag";

// std::stod (strtod; invalid_argument when nothing converts, out_of_range on ERANGE)
bool parse_double(const std::string& s, double* v) {
  const char* b = s.c_str();
  char* e = nullptr;
  errno = 0;
  const double x = std::strtod(b, &e);
  if (e == b || errno == ERANGE) return false;
  *v = x;
  return true;
}

// std::stoi (strtol, then the int range check)
bool parse_int(const std::string& s, int32_t* v) {
  const char* b = s.c_str();
  char* e = nullptr;
  errno = 0;
  const long x = std::strtol(b, &e, 10);
  if (e == b || errno == ERANGE || x < INT32_MIN || x > INT32_MAX) return false;
  *v = static_cast<int32_t>(x);
  return true;
}

// split_csv_line (workload.cpp:300-307): getline(',') fields, plus one empty field after a
// trailing comma
void split_fields(const char* b, const char* e, std::vector<std::string>& f) {
  f.clear();
  const char* p = b;
  while (p < e) {
    const char* q = static_cast<const char*>(std::memchr(p, ',', static_cast<size_t>(e - p)));
    if (!q) {
      f.emplace_back(p, e);
      p = e;
      break;
    }
    f.emplace_back(p, q);
    p = q + 1;
  }
  if (b < e && e[-1] == ',') f.emplace_back();
}

// FNV-1a (rng.hpp:55-62)
uint64_t fnv1a(uint64_t h, const char* s, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    h ^= static_cast<unsigned char>(s[i]);
    h *= 0x100000001b3ULL;
  }
  return h;
}

// write_trace_csv (workload.cpp:405-414) of rows [lo, hi)
void format_rows(eqx_trace* t, int64_t lo, int64_t hi, std::string& out) {
  char buf[64];
  out.clear();
  out.reserve(static_cast<size_t>(hi - lo) * 40);
  const int32_t* cl = t->c_client();
  const double* ar = t->c_arrival();
  const int32_t* in = t->c_in();
  const int32_t* ot = t->c_out();
  const int32_t* tg = t->c_tag();
  for (int64_t i = lo; i < hi; ++i) {
    out += t->clients[static_cast<size_t>(cl[i])];
    out.push_back(',');
    std::snprintf(buf, sizeof(buf), "%.9f", ar[i]);
    out += buf;
    std::snprintf(buf, sizeof(buf), ",%d,%d,", in[i], ot[i]);
    out += buf;
    if (tg[i] >= 0) out += t->tags[static_cast<size_t>(tg[i])];
    out.push_back('\n');
  }
}

// the canonical CSV in row chunks formatted on all host threads (the chunks concatenate to
// exactly write_trace_csv's output); visit(chunk) in order
template <class Visit>
void canonical_csv(eqx_trace* t, Visit visit) {
  const std::string head = std::string(kHeader) + "\n";
  visit(head);
  const int64_t n = t->n;
  if (n == 0) return;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int64_t chunk = 1 << 16;
  const int64_t n_chunks = (n + chunk - 1) / chunk;
  const int64_t batch = static_cast<int64_t>(hw) * 2;
  std::vector<std::string> bufs(static_cast<size_t>(std::min(n_chunks, batch)));
  for (int64_t c0 = 0; c0 < n_chunks; c0 += batch) {
    const int64_t c1 = std::min(n_chunks, c0 + batch);
    std::vector<std::thread> pool;
    const int64_t per = (c1 - c0 + hw - 1) / hw;
    for (unsigned w = 0; w < hw; ++w) {
      const int64_t a = c0 + w * per, b = std::min(c1, a + per);
      if (a >= b) break;
      pool.emplace_back([&, a, b] {
        for (int64_t c = a; c < b; ++c)
          format_rows(t, c * chunk, std::min(n, (c + 1) * chunk), bufs[static_cast<size_t>(c - c0)]);
      });
    }
    for (auto& th : pool) th.join();
    for (int64_t c = c0; c < c1; ++c) visit(bufs[static_cast<size_t>(c - c0)]);
  }
}

// roster in first-appearance order (workload.cpp:376-383) and dense client / tag indices
struct Interner {
  std::unordered_map<std::string, int32_t> idx;
  std::vector<std::string>* names;
  int32_t operator()(const std::string& s) {
    auto it = idx.find(s);
    if (it != idx.end()) return it->second;
    const int32_t k = static_cast<int32_t>(names->size());
    idx.emplace(s, k);
    names->push_back(s);
    return k;
  }
};

struct BinHeader {
  char magic[8];
  uint32_t version, pad;
  int64_t n;
  int32_t n_clients, n_tags;
  double duration_s;
  uint64_t client_bytes, tag_bytes;
  char hash[16];
};
constexpr char kMagic[8] = {'E', 'Q', 'X', 'T', 'R', 'A', 'C', 'E'};

}  // namespace

extern "C" {

eqx_status eqx_trace_load_csv(const char* path, eqx_trace** out, char* err, int32_t err_len) {
  if (!path || !out) return EQX_ERR_ARG;
  *out = nullptr;
  const std::string p(path);
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    set_err(err, err_len, "cannot open trace file '" + p + "'");
    return EQX_ERR_PARSE;
  }
  std::string text;
  {
    char buf[1 << 16];
    size_t k;
    while ((k = std::fread(buf, 1, sizeof(buf), f)) > 0) text.append(buf, k);
    std::fclose(f);
  }
  const char* s = text.data();
  const char* end = s + text.size();
  auto next_line = [&](const char*& cur, const char*& lb, const char*& le) {  // std::getline
    if (cur >= end) return false;
    lb = cur;
    const char* nl = static_cast<const char*>(std::memchr(cur, '\n', static_cast<size_t>(end - cur)));
    le = nl ? nl : end;
    cur = nl ? nl + 1 : end;
    return true;
  };
  const char* cur = s;
  const char *lb, *le;
  if (!next_line(cur, lb, le)) {
    set_err(err, err_len, "trace file '" + p + "' is empty (missing header)");
    return EQX_ERR_PARSE;
  }
  if (le > lb && le[-1] == '\r') --le;
  if (std::string(lb, le) != kHeader) {
    set_err(err, err_len, "trace file '" + p + "' has unexpected header '" + std::string(lb, le) + "'");
    return EQX_ERR_PARSE;
  }
  auto* t = new eqx_trace();
  std::vector<int32_t> cl, in, ot, tg;
  std::vector<double> ar;
  std::vector<std::string> f5;
  std::vector<std::string> row_client;  // interned after the (stable) sort
  Interner tags{{}, &t->tags};
  int64_t line_no = 1;
  auto fail = [&](const std::string& m) {
    set_err(err, err_len, "trace line " + std::to_string(line_no) + ": " + m);
    delete t;
    return EQX_ERR_PARSE;
  };
  while (next_line(cur, lb, le)) {
    ++line_no;
    if (le > lb && le[-1] == '\r') --le;
    if (le == lb) continue;
    split_fields(lb, le, f5);
    if (f5.size() != 5) return fail("expected 5 fields, got " + std::to_string(f5.size()));
    if (f5[0].empty()) return fail("empty client_id");
    double a;
    int32_t i_in, i_out;
    if (!parse_double(f5[1], &a) || !parse_int(f5[2], &i_in) || !parse_int(f5[3], &i_out))
      return fail("malformed numeric field");
    if (a < 0.0) return fail("negative arrival time");
    if (i_in < 1 || i_out < 1) return fail("token counts must be >= 1");
    row_client.push_back(std::move(f5[0]));
    ar.push_back(a);
    in.push_back(i_in);
    ot.push_back(i_out);
    tg.push_back(f5[4].empty() ? -1 : tags(f5[4]));
  }
  const int64_t n = static_cast<int64_t>(ar.size());
  std::vector<int64_t> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  const bool sorted = std::is_sorted(ar.begin(), ar.end());
  if (!sorted) {
    std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return ar[x] < ar[y]; });
    t->warnings.push_back("arrival times out of order; rows were re-sorted");
  }
  t->alloc(n);
  Interner clients{{}, &t->clients};
  for (int64_t k = 0; k < n; ++k) {
    const int64_t j = order[static_cast<size_t>(k)];
    t->c_client()[k] = clients(row_client[static_cast<size_t>(j)]);
    t->c_arrival()[k] = ar[static_cast<size_t>(j)];
    t->c_in()[k] = in[static_cast<size_t>(j)];
    t->c_out()[k] = ot[static_cast<size_t>(j)];
    t->c_tag()[k] = tg[static_cast<size_t>(j)];
  }
  t->duration_s = n ? t->c_arrival()[n - 1] : 0.0;
  t->blobs();
  *out = t;
  return EQX_OK;
}

eqx_status eqx_trace_create(int64_t n, const int32_t* client, const double* arrival_s, const int32_t* input_tokens,
                            const int32_t* output_tokens, const int32_t* tag, int32_t n_clients,
                            const char* client_names, int32_t n_tags, const char* tag_names, eqx_trace** out) {
  if (!out || n < 0 || n_clients < 0 || n_tags < 0) return EQX_ERR_ARG;
  if (n > 0 && (!client || !arrival_s || !input_tokens || !output_tokens)) return EQX_ERR_ARG;
  if ((n_clients > 0 && !client_names) || (n_tags > 0 && !tag_names)) return EQX_ERR_ARG;
  for (int64_t i = 0; i < n; ++i)
    if (client[i] < 0 || client[i] >= n_clients || (tag && (tag[i] < -1 || tag[i] >= n_tags))) return EQX_ERR_CONFIG;
  auto* t = new eqx_trace();
  const char* p = client_names;
  for (int32_t c = 0; c < n_clients; ++c) {
    t->clients.emplace_back(p);
    p += t->clients.back().size() + 1;
  }
  p = tag_names;
  for (int32_t c = 0; c < n_tags; ++c) {
    t->tags.emplace_back(p);
    p += t->tags.back().size() + 1;
  }
  t->alloc(n);
  const size_t r = static_cast<size_t>(n);
  if (n > 0) {
    std::memcpy(t->c_client(), client, 4 * r);
    std::memcpy(t->c_arrival(), arrival_s, 8 * r);
    std::memcpy(t->c_in(), input_tokens, 4 * r);
    std::memcpy(t->c_out(), output_tokens, 4 * r);
    if (tag) std::memcpy(t->c_tag(), tag, 4 * r);
    else std::fill(t->c_tag(), t->c_tag() + n, -1);
  }
  t->duration_s = n ? arrival_s[n - 1] : 0.0;
  t->blobs();
  *out = t;
  return EQX_OK;
}

void eqx_trace_free(eqx_trace* t) { delete t; }

eqx_status eqx_trace_view_get(eqx_trace* t, eqx_trace_view* v) {
  if (!t || !v) return EQX_ERR_ARG;
  std::memset(v, 0, sizeof(*v));
  v->n = t->n;
  v->n_clients = static_cast<int32_t>(t->clients.size());
  v->n_tags = static_cast<int32_t>(t->tags.size());
  v->n_warnings = static_cast<int32_t>(t->warnings.size());
  v->duration_s = t->duration_s;
  v->client = t->c_client();
  v->arrival_s = t->c_arrival();
  v->input_tokens = t->c_in();
  v->output_tokens = t->c_out();
  v->tag = t->c_tag();
  v->client_names = t->client_blob.c_str();
  v->tag_names = t->tag_blob.c_str();
  v->warnings = t->warning_blob.c_str();
  v->pinned = t->client.pinned ? 1 : 0;
  std::memcpy(v->stored_hash, t->stored_hash.c_str(), t->stored_hash.size() + 1);
  return EQX_OK;
}

eqx_status eqx_trace_hash(eqx_trace* t, char out[17]) {
  if (!t || !out) return EQX_ERR_ARG;
  if (t->hash.empty()) {
    uint64_t h = 0xcbf29ce484222325ULL;
    canonical_csv(t, [&](const std::string& c) { h = fnv1a(h, c.data(), c.size()); });
    char buf[17];
    std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(h));
    t->hash = buf;
  }
  std::memcpy(out, t->hash.c_str(), 17);
  return EQX_OK;
}

eqx_status eqx_trace_save_csv(eqx_trace* t, const char* path) {
  if (!t || !path) return EQX_ERR_ARG;
  FILE* f = std::fopen(path, "wb");
  if (!f) return EQX_ERR_PARSE;
  bool ok = true;
  canonical_csv(t, [&](const std::string& c) { ok = ok && std::fwrite(c.data(), 1, c.size(), f) == c.size(); });
  ok = (std::fclose(f) == 0) && ok;
  return ok ? EQX_OK : EQX_ERR_PARSE;
}

// Binary SoA: header | client names | tag names | client i32 | arrival f64 | input i32 |
// output i32 | tag i32, each section 64-byte aligned; the header carries trace_hash.
eqx_status eqx_trace_save_bin(eqx_trace* t, const char* path) {
  if (!t || !path) return EQX_ERR_ARG;
  char hash[17];
  eqx_trace_hash(t, hash);
  BinHeader h{};
  std::memcpy(h.magic, kMagic, 8);
  h.version = 1;
  h.n = t->n;
  h.n_clients = static_cast<int32_t>(t->clients.size());
  h.n_tags = static_cast<int32_t>(t->tags.size());
  h.duration_s = t->duration_s;
  h.client_bytes = t->client_blob.size();
  h.tag_bytes = t->tag_blob.size();
  std::memcpy(h.hash, hash, 16);
  FILE* f = std::fopen(path, "wb");
  if (!f) return EQX_ERR_PARSE;
  bool ok = true;
  size_t off = 0;
  auto put = [&](const void* p, size_t b) {
    ok = ok && (b == 0 || std::fwrite(p, 1, b, f) == b);
    off += b;
    static const char zeros[64] = {};
    const size_t padn = (64 - off % 64) % 64;
    ok = ok && (padn == 0 || std::fwrite(zeros, 1, padn, f) == padn);
    off += padn;
  };
  const size_t r = static_cast<size_t>(t->n);
  put(&h, sizeof(h));
  put(t->client_blob.data(), t->client_blob.size());
  put(t->tag_blob.data(), t->tag_blob.size());
  put(t->client.p, 4 * r);
  put(t->arrival.p, 8 * r);
  put(t->in.p, 4 * r);
  put(t->out.p, 4 * r);
  put(t->tag.p, 4 * r);
  ok = (std::fclose(f) == 0) && ok;
  return ok ? EQX_OK : EQX_ERR_PARSE;
}

eqx_status eqx_trace_load_bin(const char* path, eqx_trace** out, char* err, int32_t err_len) {
  if (!path || !out) return EQX_ERR_ARG;
  *out = nullptr;
  const std::string p(path);
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    set_err(err, err_len, "cannot open trace file '" + p + "'");
    return EQX_ERR_PARSE;
  }
  BinHeader h{};
  size_t off = 0;
  bool ok = true;
  auto get = [&](void* dst, size_t b) {
    ok = ok && (b == 0 || std::fread(dst, 1, b, f) == b);
    off += b;
    char pad[64];
    const size_t padn = (64 - off % 64) % 64;
    ok = ok && (padn == 0 || std::fread(pad, 1, padn, f) == padn);
    off += padn;
  };
  get(&h, sizeof(h));
  if (!ok || std::memcmp(h.magic, kMagic, 8) != 0 || h.version != 1 || h.n < 0 || h.n_clients < 0 || h.n_tags < 0) {
    std::fclose(f);
    set_err(err, err_len, "trace file '" + p + "' is not a binary eqx trace");
    return EQX_ERR_PARSE;
  }
  auto* t = new eqx_trace();
  std::string cb(h.client_bytes, '\0'), tb(h.tag_bytes, '\0');
  get(cb.data(), cb.size());
  get(tb.data(), tb.size());
  t->alloc(h.n);
  const size_t r = static_cast<size_t>(h.n);
  get(t->client.p, 4 * r);
  get(t->arrival.p, 8 * r);
  get(t->in.p, 4 * r);
  get(t->out.p, 4 * r);
  get(t->tag.p, 4 * r);
  std::fclose(f);
  auto split = [](const std::string& b, int32_t k, std::vector<std::string>& v) {
    size_t q = 0;
    for (int32_t i = 0; i < k; ++i) {
      const size_t z = b.find('\0', q);
      if (z == std::string::npos) return false;
      v.emplace_back(b, q, z - q);
      q = z + 1;
    }
    return true;
  };
  if (!ok || !split(cb, h.n_clients, t->clients) || !split(tb, h.n_tags, t->tags)) {
    delete t;
    set_err(err, err_len, "trace file '" + p + "' is truncated");
    return EQX_ERR_PARSE;
  }
  for (int64_t i = 0; i < h.n; ++i)
    if (t->c_client()[i] < 0 || t->c_client()[i] >= h.n_clients || t->c_tag()[i] < -1 || t->c_tag()[i] >= h.n_tags) {
      delete t;
      set_err(err, err_len, "trace file '" + p + "' has out-of-range client / tag indices");
      return EQX_ERR_PARSE;
    }
  t->duration_s = h.duration_s;
  t->stored_hash.assign(h.hash, 16);
  t->blobs();
  *out = t;
  return EQX_OK;
}

}  // extern "C"
