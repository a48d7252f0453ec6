// host_rows.cu — first-occurrence de-duplication of encoded candidate rows (host code).
//
// The reference de-duplicates the candidate pool with list(dict.fromkeys(raw)) (acquisition.py:173):
// the first occurrence of each configuration, in draw order.  An encoded row determines its
// configuration and vice versa, so the same pass runs over rows: an open-addressing hash set of row
// indices (64-bit FNV-style hash of the words, full-row comparison on a hash match), one pass in
// draw order.
#include <cstdint>
#include <cstring>
#include <vector>

#include "bx_sm100.h"

extern "C" int64_t bx_unique_rows(const uint32_t* rows, int64_t q, int32_t words, int64_t* first_idx) {
  if (q < 0 || words < 1 || (q > 0 && (!rows || !first_idx))) return -(int64_t)BX_ERR_ARG;
  int64_t cap = 16;
  while (cap < 2 * q) cap <<= 1;
  std::vector<int64_t> slot((size_t)cap, -1);
  const size_t bytes = (size_t)words * 4;
  int64_t n = 0;
  for (int64_t i = 0; i < q; ++i) {
    const uint32_t* r = rows + (size_t)i * words;
    uint64_t h = 0xcbf29ce484222325ull;
    for (int w = 0; w < words; ++w) {
      h ^= r[w];
      h *= 0x100000001b3ull;
      h ^= h >> 29;
    }
    for (int64_t s = (int64_t)(h & (uint64_t)(cap - 1));; s = (s + 1) & (cap - 1)) {
      const int64_t j = slot[(size_t)s];
      if (j < 0) {
        slot[(size_t)s] = i;
        first_idx[n++] = i;
        break;
      }
      if (std::memcmp(rows + (size_t)j * words, r, bytes) == 0) break;  // a repeat: keep the first
    }
  }
  return n;
}
