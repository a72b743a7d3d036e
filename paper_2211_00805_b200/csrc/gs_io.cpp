// gs_io.cpp -- graph text format (proj/src/sparse.cpp:137-174): header "n nnz" then one
// "i j value" line per stored upper-triangle entry (i <= j), values at precision 17 so the file
// round-trips to the last bit. Loading goes through the device from_triplets (gs_core.cu).
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "geosink_b200.h"

extern "C" int gs_graph_save(gs_ctx* ctx, const gs_graph* g, const char* path) {
  int n = 0;
  int64_t nnz = 0;
  gs_graph_info(g, &n, &nnz);
  std::vector<int> offs(n + 1), cols(nnz);
  std::vector<double> vals(nnz);
  const int rc = gs_graph_download(ctx, g, offs.data(), cols.data(), vals.data(), GS_MEM_HOST);
  if (rc) return rc;
  FILE* fp = std::fopen(path, "w");
  if (!fp) return 16;  // errc::io_error + 1
  int64_t upper = 0;
  for (int i = 0; i < n; ++i)
    for (int p = offs[i]; p < offs[i + 1]; ++p)
      if (cols[p] >= i) ++upper;
  std::fprintf(fp, "%d %lld\n", n, (long long)upper);
  for (int i = 0; i < n; ++i)
    for (int p = offs[i]; p < offs[i + 1]; ++p)
      if (cols[p] >= i) std::fprintf(fp, "%d %d %.17g\n", i, cols[p], vals[p]);
  const bool ok = std::ferror(fp) == 0;
  std::fclose(fp);
  return ok ? 0 : 16;
}

extern "C" int gs_graph_load(gs_ctx* ctx, const char* path, gs_graph** out) {
  *out = nullptr;
  std::ifstream in(path);
  if (!in) return 16;
  int n = 0;
  long long nnz = 0;
  if (!(in >> n >> nnz)) return 16;
  std::vector<int> r(nnz), c(nnz);
  std::vector<double> v(nnz);
  for (long long e = 0; e < nnz; ++e)
    if (!(in >> r[e] >> c[e] >> v[e])) return 16;
  return gs_graph_from_triplets(ctx, n, nnz, r.data(), c.data(), v.data(), GS_MEM_HOST, out);
}
