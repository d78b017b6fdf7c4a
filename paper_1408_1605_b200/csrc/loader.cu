// loader.cu -- edge-list files for real-world graphs (§8(f) NEXT-4; PAPER.md P:774-795, P:843-846:
// "real-world graphs obtained from the Stanford Large Network Dataset Collection").  Host code.
//
// Formats (External Interfaces):
//   snap-text    : lines; a line whose first non-blank character is '#' (or '%') is a comment, a
//                  blank line is skipped; otherwise two whitespace-separated decimal ids (further
//                  fields, e.g. SNAP edge weights / timestamps, are ignored).
//   binary-pairs : consecutive 16-byte records, two little-endian unsigned 64-bit ids each.
// Tuples keep file order, duplicates and self-loops (they count for m_comp).
// nverts = max id + 1 (0 for an empty file); bfs_graph_create pads it.
#include <errno.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "engine.h"

namespace bfs200 {

static constexpr uint64_t kMaxFileId = 1ull << 48;  // id >= 2^48 is unsupported

static int load_text(FILE* f, const char* path, std::vector<uint64_t>& s, std::vector<uint64_t>& d) {
  std::vector<char> buf(1 << 22);
  std::string carry;
  uint64_t lineno = 0;
  auto parse_line = [&](const char* p, const char* e) -> int {
    ++lineno;
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    if (p == e || *p == '#' || *p == '%') return BFS_OK;  // blank line / comment
    uint64_t id[2];
    for (int k = 0; k < 2; ++k) {
      while (p < e && (*p == ' ' || *p == '\t' || *p == ',')) ++p;
      if (p == e || *p < '0' || *p > '9')
        return set_err(BFS_EPARSE, "%s:%llu: expected two decimal vertex ids", path, (unsigned long long)lineno);
      uint64_t v = 0;
      while (p < e && *p >= '0' && *p <= '9') {
        const uint64_t dgt = (uint64_t)(*p - '0');
        if (v > (~0ull - dgt) / 10)
          return set_err(BFS_ERANGE, "%s:%llu: vertex id overflows 64 bits", path, (unsigned long long)lineno);
        v = v * 10 + dgt;
        ++p;
      }
      if (p < e && !(*p == ' ' || *p == '\t' || *p == '\r' || *p == ','))
        return set_err(BFS_EPARSE, "%s:%llu: malformed vertex id", path, (unsigned long long)lineno);
      if (v >= kMaxFileId)
        return set_err(BFS_ERANGE, "%s:%llu: vertex id %llu >= 2^48 (unsupported)", path,
                       (unsigned long long)lineno, (unsigned long long)v);
      id[k] = v;
    }
    s.push_back(id[0]);
    d.push_back(id[1]);
    return BFS_OK;
  };
  for (;;) {
    const size_t got = fread(buf.data(), 1, buf.size(), f);
    if (got == 0) break;
    const char* p = buf.data();
    const char* end = p + got;
    while (p < end) {
      const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(end - p)));
      if (!nl) {  // partial line: keep for the next read
        carry.append(p, (size_t)(end - p));
        break;
      }
      int rc;
      if (!carry.empty()) {
        carry.append(p, (size_t)(nl - p));
        rc = parse_line(carry.data(), carry.data() + carry.size());
        carry.clear();
      } else {
        rc = parse_line(p, nl);
      }
      if (rc) return rc;
      p = nl + 1;
    }
  }
  if (ferror(f)) return set_err(BFS_EPARSE, "%s: read error: %s", path, strerror(errno));
  if (!carry.empty()) return parse_line(carry.data(), carry.data() + carry.size());  // last line without '\n'
  return BFS_OK;
}

static int load_binary(FILE* f, const char* path, std::vector<uint64_t>& s, std::vector<uint64_t>& d) {
  std::vector<unsigned char> buf((size_t)16 << 16);
  uint64_t rec = 0;
  size_t have = 0;
  for (;;) {
    const size_t got = fread(buf.data() + have, 1, buf.size() - have, f);
    have += got;
    const size_t nrec = have / 16;
    for (size_t k = 0; k < nrec; ++k, ++rec) {
      uint64_t id[2] = {0, 0};
      for (int w = 0; w < 2; ++w)
        for (int b = 7; b >= 0; --b) id[w] = (id[w] << 8) | buf[k * 16 + (size_t)w * 8 + (size_t)b];  // little-endian
      for (int w = 0; w < 2; ++w)
        if (id[w] >= kMaxFileId)
          return set_err(BFS_ERANGE, "%s: record %llu: vertex id %llu >= 2^48 (unsupported)", path,
                         (unsigned long long)rec, (unsigned long long)id[w]);
      s.push_back(id[0]);
      d.push_back(id[1]);
    }
    const size_t rest = have - nrec * 16;
    memmove(buf.data(), buf.data() + nrec * 16, rest);
    have = rest;
    if (got == 0) break;
  }
  if (ferror(f)) return set_err(BFS_EPARSE, "%s: read error: %s", path, strerror(errno));
  if (have) return set_err(BFS_EPARSE, "%s: %zu trailing bytes (not a multiple of 16)", path, have);
  return BFS_OK;
}

}  // namespace bfs200

using namespace bfs200;

extern "C" {

int bfs_load_edges(const char* path, int format, uint64_t** src, uint64_t** dst, uint64_t* nedges, uint64_t* nverts) {
  if (!path || !src || !dst || !nedges || !nverts) return set_err(BFS_EINVAL, "null argument");
  *src = *dst = nullptr;
  *nedges = *nverts = 0;
  if (format != BFS_FMT_SNAP_TEXT && format != BFS_FMT_BINARY_PAIRS)
    return set_err(BFS_EINVAL, "format must be BFS_FMT_SNAP_TEXT (0) or BFS_FMT_BINARY_PAIRS (1), got %d", format);
  FILE* f = fopen(path, format == BFS_FMT_SNAP_TEXT ? "r" : "rb");
  if (!f) return set_err(BFS_EINVAL, "%s: cannot open: %s", path, strerror(errno));
  std::vector<uint64_t> s, d;
  int rc;
  try {
    rc = format == BFS_FMT_SNAP_TEXT ? load_text(f, path, s, d) : load_binary(f, path, s, d);
  } catch (std::bad_alloc&) {
    rc = set_err(BFS_ENOMEM, "host allocation failed");
  }
  fclose(f);
  if (rc) return rc;
  const size_t n = s.size();
  uint64_t* a = static_cast<uint64_t*>(malloc((n ? n : 1) * sizeof(uint64_t)));
  uint64_t* b = static_cast<uint64_t*>(malloc((n ? n : 1) * sizeof(uint64_t)));
  if (!a || !b) {
    free(a);
    free(b);
    return set_err(BFS_ENOMEM, "host allocation failed");
  }
  uint64_t mx = 0;
  for (size_t k = 0; k < n; ++k) {
    a[k] = s[k];
    b[k] = d[k];
    mx = s[k] > mx ? s[k] : mx;
    mx = d[k] > mx ? d[k] : mx;
  }
  *src = a;
  *dst = b;
  *nedges = n;
  *nverts = n ? mx + 1 : 0;
  return BFS_OK;
}

void bfs_free_edges(uint64_t* src, uint64_t* dst) {
  free(src);
  free(dst);
}

}  // extern "C"
