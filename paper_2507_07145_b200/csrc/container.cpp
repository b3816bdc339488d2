// Host-side .ccq container reader feeding the device upload.
//
// Restates the reference loader (container.cpp:152-319; FORMAT.md §6):
// magic "CCQF", version 1, a length-prefixed JSON header, 8-aligned
// sections.  Validation and FormatError byte offsets follow parse_info
// (container.cpp:171-249) and model_from_bytes (container.cpp:261-319).  The
// sections are kept in the file image and handed to the upload as a borrowed
// ccq_packed_view; only cluster_params is de-interleaved (as the reference
// does, container.cpp:308-316).  CRCs are not checked (readers never do;
// FORMAT.md §6, only `verify` does).
#include <cctype>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ccq_cuda.h"

namespace ccqb {
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
}  // namespace ccqb

namespace {

struct FormatErr {
  std::string what;
  long long offset;
};

// Minimal JSON value + recursive-descent parser (objects, arrays, strings,
// integers, bools, null) - enough for the container header.
struct JVal {
  enum Kind { Null, Bool, Int, Str, Arr, Obj } kind = Null;
  bool b = false;
  long long i = 0;
  bool neg = false;
  bool is_float = false;
  std::string s;
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;
  const JVal* get(const std::string& k) const {
    for (const auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const char* p;
  const char* e;
  void ws() {
    while (p < e && std::isspace(static_cast<unsigned char>(*p))) ++p;
  }
  [[noreturn]] void bad() { throw FormatErr{"header JSON: malformed", 12}; }
  JVal parse() {
    ws();
    if (p >= e) bad();
    JVal v;
    if (*p == '{') {
      v.kind = JVal::Obj;
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return v;
      }
      for (;;) {
        ws();
        JVal k = parse();
        if (k.kind != JVal::Str) bad();
        ws();
        if (p >= e || *p != ':') bad();
        ++p;
        JVal val = parse();
        v.o.emplace_back(k.s, std::move(val));
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          return v;
        }
        bad();
      }
    }
    if (*p == '[') {
      v.kind = JVal::Arr;
      ++p;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return v;
      }
      for (;;) {
        v.a.push_back(parse());
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          return v;
        }
        bad();
      }
    }
    if (*p == '"') {
      v.kind = JVal::Str;
      ++p;
      while (p < e && *p != '"') {
        if (*p == '\\') {
          ++p;
          if (p >= e) bad();
        }
        v.s.push_back(*p++);
      }
      if (p >= e) bad();
      ++p;
      return v;
    }
    if (e - p >= 4 && std::strncmp(p, "true", 4) == 0) {
      v.kind = JVal::Bool;
      v.b = true;
      p += 4;
      return v;
    }
    if (e - p >= 5 && std::strncmp(p, "false", 5) == 0) {
      v.kind = JVal::Bool;
      p += 5;
      return v;
    }
    if (e - p >= 4 && std::strncmp(p, "null", 4) == 0) {
      p += 4;
      return v;
    }
    if (*p == '-' || std::isdigit(static_cast<unsigned char>(*p))) {
      v.kind = JVal::Int;
      if (*p == '-') {
        v.neg = true;
        ++p;
      }
      if (p >= e || !std::isdigit(static_cast<unsigned char>(*p))) bad();
      while (p < e && std::isdigit(static_cast<unsigned char>(*p))) v.i = v.i * 10 + (*p++ - '0');
      if (p < e && (*p == '.' || *p == 'e' || *p == 'E')) {
        v.is_float = true;
        while (p < e && (std::isdigit(static_cast<unsigned char>(*p)) || *p == '.' || *p == 'e' ||
                         *p == 'E' || *p == '+' || *p == '-'))
          ++p;
      }
      if (v.neg) v.i = -v.i;
      return v;
    }
    bad();
  }
};

uint64_t require_u64(const JVal& j, const char* key) {
  const JVal* v = j.get(key);
  if (!v || v->kind != JVal::Int || v->neg || v->is_float)
    throw FormatErr{std::string("header field '") + key + "' missing or not unsigned", 12};
  return uint64_t(v->i);
}

struct Section {
  uint64_t offset = 0, length = 0;
};

struct HostModel {
  std::vector<uint8_t> file;
  std::vector<float> super, cs, czp;
  ccq_packed_view view{};
};

int family_index(const std::string& n) {
  if (n == "2.75") return 0;
  if (n == "2.5" || n == "2.50") return 1;
  if (n == "2.06") return 2;
  return -1;
}

const int kScaleBits[3] = {4, 13, 4};
const int kWordBits[3] = {8, 16, 16};
const std::vector<std::vector<int>> kParts[3] = {
    {{4, 3, 2}}, {{3, 3, 2}, {3, 4, 2}}, {{6, 4, 3}}};

// Group geometry payload bytes / embedded flag (packing.cpp:24-47).
bool geometry(int fam, int gs, int* payload, bool* embedded) {
  const int wpw[3] = {3, 7, 4}, wb[3] = {1, 2, 1};
  if (gs <= 0) return false;
  const int rem = gs % wpw[fam];
  if (rem > 1 || (fam == 1 && rem == 0)) return false;
  *payload = (gs / wpw[fam] + (rem == 1)) * wb[fam];
  *embedded = rem == 1 && fam != 2;
  return true;
}

std::unique_ptr<HostModel> parse(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  auto hm = std::make_unique<HostModel>();
  in.seekg(0, std::ios::end);
  const std::streamoff size = in.tellg();
  in.seekg(0, std::ios::beg);
  hm->file.resize(size_t(size));
  if (size > 0) in.read(reinterpret_cast<char*>(hm->file.data()), size);
  if (!in) throw std::runtime_error("short read from " + path);
  const std::vector<uint8_t>& b = hm->file;

  // parse_info (container.cpp:171-249)
  if (b.size() < 12) throw FormatErr{"file shorter than the fixed prologue", 0};
  if (std::memcmp(b.data(), "CCQF", 4) != 0) throw FormatErr{"bad magic", 0};
  const uint16_t version = uint16_t(b[4] | (b[5] << 8));
  if (version != 1) throw FormatErr{"unsupported version " + std::to_string(version), 4};
  const uint32_t hlen = uint32_t(b[8]) | (uint32_t(b[9]) << 8) | (uint32_t(b[10]) << 16) |
                        (uint32_t(b[11]) << 24);
  if (12 + uint64_t(hlen) > b.size()) throw FormatErr{"header length exceeds file size", 8};
  JParser jp{reinterpret_cast<const char*>(b.data()) + 12,
             reinterpret_cast<const char*>(b.data()) + 12 + hlen};
  JVal j = jp.parse();
  jp.ws();
  if (jp.p != jp.e || j.kind != JVal::Obj) throw FormatErr{"header JSON: malformed", 12};

  const JVal* fam = j.get("family");
  if (!fam || fam->kind != JVal::Str) throw FormatErr{"header field 'family' missing or not a string", 12};
  const int f = family_index(fam->s);
  if (f < 0) throw std::invalid_argument("unknown family '" + fam->s + "'");
  const JVal* shape = j.get("shape");
  if (!shape || shape->kind != JVal::Arr || shape->a.size() != 2 || shape->a[0].kind != JVal::Int ||
      shape->a[1].kind != JVal::Int)
    throw FormatErr{"header field 'shape' must be [rows, cols]", 12};
  const int64_t rows = shape->a[0].i, cols = shape->a[1].i;
  if (rows < 0 || cols < 0) throw FormatErr{"negative shape", 12};
  const int gs = int(require_u64(j, "group_size"));
  const int rounds = int(require_u64(j, "rounds"));
  const int scale_bits = int(require_u64(j, "scale_bits"));
  const JVal* storage = j.get("scale_storage");
  if (!storage || storage->kind != JVal::Str) throw FormatErr{"header field 'scale_storage' missing", 12};
  if (scale_bits != kScaleBits[f]) throw FormatErr{"scale_bits does not match the family", 12};
  const JVal* code = j.get("code");
  if (!code || code->kind != JVal::Obj || !code->get("parts") || !code->get("word_bits"))
    throw FormatErr{"header field 'code' missing or incomplete", 12};
  {
    const JVal* parts = code->get("parts");
    bool ok = parts->kind == JVal::Arr && parts->a.size() == kParts[f].size();
    for (size_t i = 0; ok && i < parts->a.size(); ++i) {
      const JVal& pt = parts->a[i];
      ok = pt.kind == JVal::Arr && pt.a.size() == 3;
      for (size_t k = 0; ok && k < 3; ++k) ok = pt.a[k].kind == JVal::Int && pt.a[k].i == kParts[f][i][k];
    }
    const JVal* wb = code->get("word_bits");
    ok = ok && wb->kind == JVal::Int && wb->i == kWordBits[f];
    if (!ok) throw FormatErr{"code parameters do not match the family", 12};
  }
  const uint64_t header_bytes = 12 + hlen;
  const uint64_t base = (header_bytes + 7) & ~uint64_t(7);
  const JVal* secs = j.get("sections");
  if (!secs || secs->kind != JVal::Obj) throw FormatErr{"header field 'sections' missing", 12};
  std::map<std::string, Section> sec;
  for (const auto& [name, body] : secs->o) {
    Section s;
    s.offset = require_u64(body, "offset");
    s.length = require_u64(body, "length");
    (void)require_u64(body, "crc32");
    if (s.offset % 8 != 0)
      throw FormatErr{"section '" + name + "' offset not 8-aligned", (long long)(base + s.offset)};
    if (base + s.offset + s.length > b.size())
      throw FormatErr{"section '" + name + "' extends past end of file", (long long)(base + s.offset)};
    sec[name] = s;
  }

  // model_from_bytes (container.cpp:261-319)
  if (gs <= 0 || cols % gs != 0) throw FormatErr{"shape is not a whole number of groups", 12};
  int payload = 0;
  bool embedded = false;
  if (!geometry(f, gs, &payload, &embedded)) throw FormatErr{"group_size has no layout for this family", 12};
  auto need = [&](const char* name) -> const Section& {
    auto it = sec.find(name);
    if (it == sec.end()) throw FormatErr{std::string("missing section '") + name + "'", 12};
    return it->second;
  };
  const uint64_t groups = uint64_t(rows) * uint64_t(cols / gs);
  const Section& sc = need("codes");
  if (sc.length != groups * uint64_t(payload))
    throw FormatErr{"codes section length does not match the geometry", (long long)(base + sc.offset)};
  ccq_packed_view& v = hm->view;
  v.rows = rows;
  v.cols = cols;
  v.family = f;
  v.group_size = gs;
  v.rounds = rounds;
  v.code_payload = b.data() + base + sc.offset;
  v.code_bytes = sc.length;
  if (!embedded) {
    const Section& sg = need("group_scales");
    if (sg.length != (groups + 1) / 2)
      throw FormatErr{"group_scales section length does not match the group count",
                      (long long)(base + sg.offset)};
    v.scale_payload = b.data() + base + sg.offset;
    v.scale_bytes = sg.length;
  }
  const Section& ss = need("super_scales");
  if (ss.length != uint64_t(rows) * 4)
    throw FormatErr{"super_scales section length does not match the row count", (long long)(base + ss.offset)};
  hm->super.resize(size_t(rows));
  if (rows) std::memcpy(hm->super.data(), b.data() + base + ss.offset, size_t(rows) * 4);
  v.super_scales = hm->super.data();
  v.n_super_scales = uint64_t(rows);
  if (f == 2) {
    const Section& sp = need("cluster_params");
    if (sp.length != uint64_t(rows) * 8)
      throw FormatErr{"cluster_params section length does not match the row count", (long long)(base + sp.offset)};
    hm->cs.resize(size_t(rows));
    hm->czp.resize(size_t(rows));
    for (int64_t r = 0; r < rows; ++r) {
      std::memcpy(&hm->cs[size_t(r)], b.data() + base + sp.offset + 8 * r, 4);
      std::memcpy(&hm->czp[size_t(r)], b.data() + base + sp.offset + 8 * r + 4, 4);
    }
    v.cluster_scales = hm->cs.data();
    v.cluster_zero_points = hm->czp.data();
    v.n_cluster_scales = v.n_cluster_zero_points = uint64_t(rows);
  }
  return hm;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const FormatErr& e) {
    return ccqb::fail(CCQ_ERR_FORMAT, e.offset >= 0 ? e.what + " (byte offset " +
                                                          std::to_string(e.offset) + ")"
                                                    : e.what);
  } catch (const std::invalid_argument& e) {
    return ccqb::fail(CCQ_ERR_CONFIG, e.what());
  } catch (const std::exception& e) {
    return ccqb::fail(CCQ_ERR_INVALID, e.what());
  }
}

}  // namespace

extern "C" {

int ccq_container_open(const char* path, ccq_packed_view* view, void** owner) {
  if (!path || !view || !owner) return ccqb::fail(CCQ_ERR_INVALID, "null argument");
  return guarded([&] {
    auto hm = parse(path);
    *view = hm->view;
    *owner = hm.release();
    return int(CCQ_OK);
  });
}

void ccq_container_close(void* owner) { delete static_cast<HostModel*>(owner); }

int ccq_cuda_model_load(const char* path, int device, ccq_dev_model** out) {
  if (!path || !out) return ccqb::fail(CCQ_ERR_INVALID, "null argument");
  return guarded([&] {
    auto hm = parse(path);
    return ccq_cuda_model_upload(&hm->view, device, out);
  });
}

}  // extern "C"
