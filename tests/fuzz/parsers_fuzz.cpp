// Mutation fuzzer for the host-side parsers of the two file formats
// (include/maddness.h "File formats": model.mdnm v1, luts.mdnl v1).
//
// Built by tests/test_fuzz_parsers.py with mdn_host.cpp compiled under
// -fsanitize=address,undefined and linked against the library's other
// objects; runs on a machine without a GPU: every mutant must be rejected (or,
// when it is still a valid stream, fail at the first device call) without a
// sanitizer report, a crash or an out-of-range error offset.
//
//   parsers_fuzz <model|luts> <blob file> <mutants> <seed>
//
// Mutations (seeded xorshift): truncation to a random length; 1-8 random bit
// flips; random byte overwrites; a random field-sized (2/4/8 byte) overwrite
// with an extreme value. Half of the non-truncating mutants get their FNV-1a
// trailer recomputed, so the field validation behind the checksum is reached.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "maddness.h"

static uint64_t g_state = 0x9E3779B97F4A7C15ull;
static uint64_t rnd() {
  g_state ^= g_state << 13;
  g_state ^= g_state >> 7;
  g_state ^= g_state << 17;
  return g_state;
}

static uint64_t fnv1a64(const uint8_t* p, size_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001B3ull;
  return h;
}

int main(int argc, char** argv) {
  if (argc != 5) {
    fprintf(stderr, "usage: %s <model|luts> <blob> <mutants> <seed>\n", argv[0]);
    return 2;
  }
  const bool is_model = strcmp(argv[1], "model") == 0;
  FILE* f = fopen(argv[2], "rb");
  if (!f) return 2;
  std::vector<uint8_t> blob;
  for (int c; (c = fgetc(f)) != EOF;) blob.push_back((uint8_t)c);
  fclose(f);
  const long n_mut = atol(argv[3]);
  g_state ^= (uint64_t)atoll(argv[4]) * 0x2545F4914F6CDD1Dull;
  long counts[9] = {0};             // by -status
  if (n_mut == 0) {                 // the unmutated stream: passes every parser check
    size_t off = 0;
    int st;
    if (is_model) {
      mdn_model* h = nullptr;
      st = mdn_model_load(blob.data(), blob.size(), 0, &h, &off);
      if (h) mdn_model_free(h);
    } else {
      mdn_luts* h = nullptr;
      st = mdn_luts_load(blob.data(), blob.size(), 0, &h, &off);
      if (h) mdn_luts_free(h);
    }
    printf("{\"status\": %d}\n", st);
    return 0;
  }
  for (long it = 0; it < n_mut; ++it) {
    std::vector<uint8_t> m = blob;
    const int kind = (int)(rnd() % 4);
    bool truncated = false;
    if (kind == 0) {
      m.resize(rnd() % m.size());
      truncated = true;
    } else if (kind == 1) {
      const int flips = 1 + (int)(rnd() % 8);
      for (int i = 0; i < flips; ++i) m[rnd() % m.size()] ^= (uint8_t)(1u << (rnd() % 8));
    } else if (kind == 2) {
      const int n = 1 + (int)(rnd() % 16);
      for (int i = 0; i < n; ++i) m[rnd() % m.size()] = (uint8_t)rnd();
    } else {
      static const uint64_t extremes[] = {0ull, 1ull, 0xFFull, 0xFFFFull, 0x7FFFFFFFull,
                                          0x80000000ull, 0xFFFFFFFFull, 0x7FC00000ull /*NaN f32*/,
                                          0x7F800000ull /*inf*/, 0xFFFFFFFFFFFFFFFFull};
      const int sz = 2 << (rnd() % 3);
      // bias towards the headers and the per-codebook records
      const size_t lim = m.size() < 512 ? m.size() : 512;
      const size_t at = rnd() % (lim > (size_t)sz ? lim - sz : 1);
      const uint64_t v = extremes[rnd() % (sizeof(extremes) / sizeof(extremes[0]))];
      memcpy(m.data() + at, &v, (size_t)sz <= m.size() - at ? (size_t)sz : m.size() - at);
    }
    if (!truncated && m.size() >= 8 && (rnd() & 1)) {
      const uint64_t h = fnv1a64(m.data(), m.size() - 8);
      memcpy(m.data() + m.size() - 8, &h, 8);
    }
    // the parser gets an exact-size heap copy so any over-read is an ASan report
    uint8_t* buf = (uint8_t*)malloc(m.size() ? m.size() : 1);
    memcpy(buf, m.data(), m.size());
    size_t off = (size_t)-1;
    int st;
    if (is_model) {
      mdn_model* h = nullptr;
      st = mdn_model_load(buf, m.size(), 0, &h, &off);
      if (h) mdn_model_free(h);
    } else {
      mdn_luts* h = nullptr;
      st = mdn_luts_load(buf, m.size(), 0, &h, &off);
      if (h) mdn_luts_free(h);
    }
    free(buf);
    if (st > 0 || st < -8) {
      fprintf(stderr, "mutant %ld: unknown status %d\n", it, st);
      return 1;
    }
    if (st == MDN_OK) {
      fprintf(stderr, "mutant %ld: accepted without a device\n", it);
      return 1;
    }
    if (st == MDN_EFORMAT && off > m.size()) {
      fprintf(stderr, "mutant %ld: err_off %zu beyond the %zu-byte stream\n", it, off, m.size());
      return 1;
    }
    counts[-st]++;
  }
  printf("{\"mutants\": %ld, \"EINVAL\": %ld, \"ESHAPE\": %ld, \"EFORMAT\": %ld, \"EVERSION\": %ld, "
         "\"ESTATE\": %ld, \"ECUDA\": %ld, \"ENOMEM\": %ld}\n",
         n_mut, counts[1], counts[2], counts[3], counts[4], counts[5], counts[6], counts[7]);
  return 0;
}
