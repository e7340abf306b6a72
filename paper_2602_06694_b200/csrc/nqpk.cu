// nqpk.cu — NQPK packed-model files <-> the device layout.
//
// The on-disk contract is the reference's (io.hpp:27-36, io.cpp:139-193), all
// integers little-endian:
//   "NQPK", version u32 (= 1), layer count u32; per layer: name length u32 +
//   UTF-8 bytes, n u32, m u32, r u32, U words (n * ceil(r/32) u32), V words
//   (m * ceil(r/32) u32), s1 as n binary16, s2 as m binary16.
// Parsing is host work; the binary16 scales go to the device unchanged
// (nqb_layer_upload_f16), so a reference-written model decodes with exactly
// the scales it was saved with, and a device layer written back reproduces
// the reference serialisation byte for byte.
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "common.cuh"

struct nqb_nqpk {
  struct Layer {
    std::string name;
    uint32_t n = 0, m = 0, r = 0;
    std::vector<uint32_t> u, v;
    std::vector<uint16_t> s1h, s2h;
  };
  uint32_t version = 1;
  std::vector<Layer> layers;
};

namespace nqb {
namespace {

constexpr uint32_t kNqpkVersion = 1;  // io.hpp:38

// Little-endian cursor over the file bytes; every read is bounds-checked
// (a short read is a ParseError, io.cpp Reader).
struct Cursor {
  const uint8_t* p;
  size_t n, i = 0;
  void need(size_t k) const {
    NQB_REQUIRE(i + k <= n, NQB_E_PARSE, "truncated NQPK stream");
  }
  uint32_t u32() {
    need(4);
    const uint32_t v = (uint32_t)p[i] | ((uint32_t)p[i + 1] << 8) | ((uint32_t)p[i + 2] << 16) |
                       ((uint32_t)p[i + 3] << 24);
    i += 4;
    return v;
  }
  uint16_t u16() {
    need(2);
    const uint16_t v = (uint16_t)(p[i] | (p[i + 1] << 8));
    i += 2;
    return v;
  }
  std::string str(size_t k) {
    need(k);
    std::string s((const char*)p + i, k);
    i += k;
    return s;
  }
};

void put_u32(std::vector<uint8_t>& o, uint32_t v) {
  for (int b = 0; b < 4; ++b) o.push_back((uint8_t)(v >> (8 * b)));
}
void put_u16(std::vector<uint8_t>& o, uint16_t v) {
  o.push_back((uint8_t)v);
  o.push_back((uint8_t)(v >> 8));
}

// deserialize_packed_model (io.cpp:160-185)
nqb_nqpk* parse(const uint8_t* bytes, size_t len) {
  Cursor c{bytes, len};
  NQB_REQUIRE(c.str(4) == "NQPK", NQB_E_PARSE, "bad NQPK magic");
  auto* f = new nqb_nqpk();
  try {
    f->version = c.u32();
    NQB_REQUIRE(f->version == kNqpkVersion, NQB_E_PARSE, "unsupported NQPK version");
    const uint32_t count = c.u32();
    for (uint32_t k = 0; k < count; ++k) {
      nqb_nqpk::Layer L;
      L.name = c.str(c.u32());
      L.n = c.u32();
      L.m = c.u32();
      L.r = c.u32();
      NQB_REQUIRE(L.n && L.m && L.r, NQB_E_PARSE, "zero layer dimension");
      const size_t wpr = ((size_t)L.r + 31) / 32;
      c.need(4 * wpr * ((size_t)L.n + L.m) + 2 * ((size_t)L.n + L.m));
      L.u.resize((size_t)L.n * wpr);
      for (auto& w : L.u) w = c.u32();
      L.v.resize((size_t)L.m * wpr);
      for (auto& w : L.v) w = c.u32();
      L.s1h.resize(L.n);
      for (auto& h : L.s1h) h = c.u16();
      L.s2h.resize(L.m);
      for (auto& h : L.s2h) h = c.u16();
      f->layers.push_back(std::move(L));
    }
    NQB_REQUIRE(c.i == c.n, NQB_E_PARSE, "trailing bytes in NQPK stream");
  } catch (...) {
    delete f;
    throw;
  }
  return f;
}

// serialize_packed_model (io.cpp:139-158)
void serialize(uint32_t count, const char* const* names, const uint32_t* n, const uint32_t* m,
               const uint32_t* r, const uint32_t* const* u, const uint32_t* const* v,
               const uint16_t* const* s1h, const uint16_t* const* s2h, std::vector<uint8_t>& out) {
  out.insert(out.end(), {'N', 'Q', 'P', 'K'});
  put_u32(out, kNqpkVersion);
  put_u32(out, count);
  for (uint32_t k = 0; k < count; ++k) {
    NQB_REQUIRE(names && names[k], NQB_E_VALIDATION, "null layer name");
    NQB_REQUIRE(n[k] && m[k] && r[k], NQB_E_DIMENSION_MISMATCH, "zero layer dimension");
    const size_t len = std::strlen(names[k]), wpr = ((size_t)r[k] + 31) / 32;
    put_u32(out, (uint32_t)len);
    out.insert(out.end(), names[k], names[k] + len);
    put_u32(out, n[k]);
    put_u32(out, m[k]);
    put_u32(out, r[k]);
    for (size_t i = 0; i < (size_t)n[k] * wpr; ++i) put_u32(out, u[k][i]);
    for (size_t i = 0; i < (size_t)m[k] * wpr; ++i) put_u32(out, v[k][i]);
    for (uint32_t i = 0; i < n[k]; ++i) put_u16(out, s1h[k][i]);
    for (uint32_t i = 0; i < m[k]; ++i) put_u16(out, s2h[k][i]);
  }
}

void write_file(const char* path, const std::vector<uint8_t>& bytes) {
  std::ofstream o(path, std::ios::binary | std::ios::trunc);
  NQB_REQUIRE((bool)o, NQB_E_IO, std::string("cannot open ") + path + " for writing");
  o.write((const char*)bytes.data(), (std::streamsize)bytes.size());
  NQB_REQUIRE((bool)o, NQB_E_IO, std::string("short write to ") + path);
}

}  // namespace

uint16_t host_double_to_half(double x);  // api.cu (half.hpp:83-85 rounding)

}  // namespace nqb

using namespace nqb;

#define NQPK_BEGIN try {
#define NQPK_END                        \
  return NQB_OK;                        \
  }                                     \
  catch (const Failure& e) {            \
    set_error(e.msg);                   \
    return e.code;                      \
  }                                     \
  catch (const std::exception& e) {     \
    set_error(e.what());                \
    return NQB_E_INTERNAL;              \
  }

extern "C" {

int nqb_nqpk_parse(const uint8_t* bytes, uint64_t len, nqb_nqpk** out) {
  NQPK_BEGIN
  NQB_REQUIRE(out != nullptr && (bytes != nullptr || len == 0), NQB_E_VALIDATION, "null argument");
  *out = nullptr;
  *out = parse(bytes, (size_t)len);
  NQPK_END
}

int nqb_nqpk_open(const char* path, nqb_nqpk** out) {
  NQPK_BEGIN
  NQB_REQUIRE(path != nullptr && out != nullptr, NQB_E_VALIDATION, "null argument");
  *out = nullptr;
  std::ifstream in(path, std::ios::binary);  // read_file (io.cpp:89-98)
  NQB_REQUIRE((bool)in, NQB_E_IO, std::string("cannot open ") + path);
  std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  *out = parse(bytes.data(), bytes.size());
  NQPK_END
}

uint32_t nqb_nqpk_count(const nqb_nqpk* f) { return f ? (uint32_t)f->layers.size() : 0u; }

int nqb_nqpk_layer_info(const nqb_nqpk* f, uint32_t i, char* name, uint32_t name_cap,
                        uint32_t* name_len, uint32_t* n, uint32_t* m, uint32_t* r) {
  NQPK_BEGIN
  NQB_REQUIRE(f != nullptr && i < f->layers.size(), NQB_E_VALIDATION, "no such NQPK layer");
  const auto& L = f->layers[i];
  if (name_len) *name_len = (uint32_t)L.name.size();
  if (name && name_cap) {
    const size_t k = std::min<size_t>(L.name.size(), name_cap - 1);
    std::memcpy(name, L.name.data(), k);
    name[k] = 0;
  }
  if (n) *n = L.n;
  if (m) *m = L.m;
  if (r) *r = L.r;
  NQPK_END
}

int nqb_nqpk_layer_data(const nqb_nqpk* f, uint32_t i, const uint32_t** u, const uint32_t** v,
                        const uint16_t** s1_half, const uint16_t** s2_half) {
  NQPK_BEGIN
  NQB_REQUIRE(f != nullptr && i < f->layers.size(), NQB_E_VALIDATION, "no such NQPK layer");
  const auto& L = f->layers[i];
  if (u) *u = L.u.data();
  if (v) *v = L.v.data();
  if (s1_half) *s1_half = L.s1h.data();
  if (s2_half) *s2_half = L.s2h.data();
  NQPK_END
}

int nqb_nqpk_layer_upload(nqb_context* ctx, const nqb_nqpk* f, uint32_t i, nqb_layer** out) {
  if (!f || i >= f->layers.size()) {
    set_error("no such NQPK layer");
    return NQB_E_VALIDATION;
  }
  const auto& L = f->layers[i];
  return nqb_layer_upload_f16(ctx, L.n, L.m, L.r, L.u.data(), L.v.data(), L.s1h.data(),
                              L.s2h.data(), out);
}

void nqb_nqpk_free(nqb_nqpk* f) { delete f; }

int nqb_nqpk_serialize(uint32_t count, const char* const* names, const uint32_t* n,
                       const uint32_t* m, const uint32_t* r, const uint32_t* const* u,
                       const uint32_t* const* v, const uint16_t* const* s1_half,
                       const uint16_t* const* s2_half, uint8_t* buf, uint64_t cap, uint64_t* len) {
  NQPK_BEGIN
  NQB_REQUIRE(len != nullptr, NQB_E_VALIDATION, "null length");
  NQB_REQUIRE(count == 0 || (n && m && r && u && v && s1_half && s2_half), NQB_E_VALIDATION,
              "null layer arrays");
  std::vector<uint8_t> bytes;
  serialize(count, names, n, m, r, u, v, s1_half, s2_half, bytes);
  *len = bytes.size();
  if (buf) {
    NQB_REQUIRE(bytes.size() <= cap, NQB_E_VALIDATION, "NQPK buffer too small");
    std::memcpy(buf, bytes.data(), bytes.size());
  }
  NQPK_END
}

int nqb_nqpk_write_layers(nqb_context* ctx, const char* path, uint32_t count,
                          const char* const* names, const nqb_layer* const* layers) {
  NQPK_BEGIN
  NQB_REQUIRE(path != nullptr && (count == 0 || (names && layers)), NQB_E_VALIDATION,
              "null argument");
  std::vector<uint32_t> n(count), m(count), r(count);
  std::vector<std::vector<uint32_t>> u(count), v(count);
  std::vector<std::vector<uint16_t>> h1(count), h2(count);
  std::vector<const uint32_t*> up(count), vp(count);
  std::vector<const uint16_t*> h1p(count), h2p(count);
  for (uint32_t k = 0; k < count; ++k) {
    NQB_REQUIRE(layers[k] != nullptr, NQB_E_VALIDATION, "null layer");
    const int st = nqb_layer_shape(layers[k], &n[k], &m[k], &r[k]);
    if (st) throw Failure{st, nqb_last_error()};
    const size_t wpr = ((size_t)r[k] + 31) / 32;
    u[k].resize((size_t)n[k] * wpr);
    v[k].resize((size_t)m[k] * wpr);
    std::vector<double> s1(n[k]), s2(m[k]);
    const int sd = nqb_layer_download(ctx, layers[k], u[k].data(), v[k].data(), s1.data(), s2.data());
    if (sd) throw Failure{sd, nqb_last_error()};
    // the device keeps binary16 scales: half -> double -> half is exact
    h1[k].resize(n[k]);
    h2[k].resize(m[k]);
    for (uint32_t i = 0; i < n[k]; ++i) h1[k][i] = host_double_to_half(s1[i]);
    for (uint32_t j = 0; j < m[k]; ++j) h2[k][j] = host_double_to_half(s2[j]);
    up[k] = u[k].data();
    vp[k] = v[k].data();
    h1p[k] = h1[k].data();
    h2p[k] = h2[k].data();
  }
  std::vector<uint8_t> bytes;
  serialize(count, names, n.data(), m.data(), r.data(), up.data(), vp.data(), h1p.data(),
            h2p.data(), bytes);
  write_file(path, bytes);
  NQPK_END
}

}  // extern "C"
