// hilbert_permute host implementation -- §3.7 "HilbertCurve Permutation"
// and App. A.1: visual tokens of a T x H x W grid are
// flattened along a 3-D Hilbert curve; text-prefix tokens keep their place.
//
// Reading R19: the generalised Hilbert curve for arbitrary extents
// ("gilbert3d", J. Cervený).  A box is described by an origin and three axis
// vectors (a = major, b, c); it is split into 2, 3 or 5 sub-boxes whose
// curves chain end-to-start by unit steps.  This implementation walks the
// decomposition with an explicit work stack (no recursion) and emits cells
// directly into the permutation array.
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "sparge_internal.h"

namespace sparge {

namespace {

struct Box {
  int x, y, z;
  int ax, ay, az, bx, by, bz, cx, cy, cz;
};

inline int sgn(int v) { return (v > 0) - (v < 0); }

struct Emitter {
  int H, W, prefix;
  int32_t* out;
  int64_t pos;
  void cell(int x, int y, int z) {
    out[pos++] = prefix + (z * H + y) * W + x;
  }
};

void walk(Box root, Emitter& em) {
  std::vector<Box> stack;
  stack.push_back(root);
  while (!stack.empty()) {
    const Box q = stack.back();
    stack.pop_back();
    const int w = std::abs(q.ax + q.ay + q.az);
    const int h = std::abs(q.bx + q.by + q.bz);
    const int d = std::abs(q.cx + q.cy + q.cz);
    const int dax = sgn(q.ax), day = sgn(q.ay), daz = sgn(q.az);
    const int dbx = sgn(q.bx), dby = sgn(q.by), dbz = sgn(q.bz);
    const int dcx = sgn(q.cx), dcy = sgn(q.cy), dcz = sgn(q.cz);

    // a box that is one cell thick in two axes is a straight run
    if (h == 1 && d == 1) {
      for (int k = 0; k < w; ++k) em.cell(q.x + k * dax, q.y + k * day, q.z + k * daz);
      continue;
    }
    if (w == 1 && d == 1) {
      for (int k = 0; k < h; ++k) em.cell(q.x + k * dbx, q.y + k * dby, q.z + k * dbz);
      continue;
    }
    if (w == 1 && h == 1) {
      for (int k = 0; k < d; ++k) em.cell(q.x + k * dcx, q.y + k * dcy, q.z + k * dcz);
      continue;
    }

    // half vectors (floor division toward -inf, as for the signed axes)
    auto half = [](int v) { return v >= 0 ? v / 2 : -((-v + 1) / 2); };
    int ax2 = half(q.ax), ay2 = half(q.ay), az2 = half(q.az);
    int bx2 = half(q.bx), by2 = half(q.by), bz2 = half(q.bz);
    int cx2 = half(q.cx), cy2 = half(q.cy), cz2 = half(q.cz);
    const int w2 = std::abs(ax2 + ay2 + az2);
    const int h2 = std::abs(bx2 + by2 + bz2);
    const int d2 = std::abs(cx2 + cy2 + cz2);
    if ((w2 & 1) && w > 2) { ax2 += dax; ay2 += day; az2 += daz; }
    if ((h2 & 1) && h > 2) { bx2 += dbx; by2 += dby; bz2 += dbz; }
    if ((d2 & 1) && d > 2) { cx2 += dcx; cy2 += dcy; cz2 += dcz; }

    Box sub[5];
    int n = 0;
    if (2 * w > 3 * h && 2 * w > 3 * d) {
      sub[n++] = {q.x, q.y, q.z, ax2, ay2, az2, q.bx, q.by, q.bz, q.cx, q.cy, q.cz};
      sub[n++] = {q.x + ax2, q.y + ay2, q.z + az2, q.ax - ax2, q.ay - ay2, q.az - az2,
                  q.bx, q.by, q.bz, q.cx, q.cy, q.cz};
    } else if (3 * h > 4 * d) {
      sub[n++] = {q.x, q.y, q.z, bx2, by2, bz2, q.cx, q.cy, q.cz, ax2, ay2, az2};
      sub[n++] = {q.x + bx2, q.y + by2, q.z + bz2, q.ax, q.ay, q.az,
                  q.bx - bx2, q.by - by2, q.bz - bz2, q.cx, q.cy, q.cz};
      sub[n++] = {q.x + (q.ax - dax) + (bx2 - dbx), q.y + (q.ay - day) + (by2 - dby),
                  q.z + (q.az - daz) + (bz2 - dbz), -bx2, -by2, -bz2, q.cx, q.cy, q.cz,
                  -(q.ax - ax2), -(q.ay - ay2), -(q.az - az2)};
    } else if (3 * d > 4 * h) {
      sub[n++] = {q.x, q.y, q.z, cx2, cy2, cz2, ax2, ay2, az2, q.bx, q.by, q.bz};
      sub[n++] = {q.x + cx2, q.y + cy2, q.z + cz2, q.ax, q.ay, q.az, q.bx, q.by, q.bz,
                  q.cx - cx2, q.cy - cy2, q.cz - cz2};
      sub[n++] = {q.x + (q.ax - dax) + (cx2 - dcx), q.y + (q.ay - day) + (cy2 - dcy),
                  q.z + (q.az - daz) + (cz2 - dcz), -cx2, -cy2, -cz2,
                  -(q.ax - ax2), -(q.ay - ay2), -(q.az - az2), q.bx, q.by, q.bz};
    } else {
      sub[n++] = {q.x, q.y, q.z, bx2, by2, bz2, cx2, cy2, cz2, ax2, ay2, az2};
      sub[n++] = {q.x + bx2, q.y + by2, q.z + bz2, q.cx, q.cy, q.cz, ax2, ay2, az2,
                  q.bx - bx2, q.by - by2, q.bz - bz2};
      sub[n++] = {q.x + (bx2 - dbx) + (q.cx - dcx), q.y + (by2 - dby) + (q.cy - dcy),
                  q.z + (bz2 - dbz) + (q.cz - dcz), q.ax, q.ay, q.az, -bx2, -by2, -bz2,
                  -(q.cx - cx2), -(q.cy - cy2), -(q.cz - cz2)};
      sub[n++] = {q.x + (q.ax - dax) + bx2 + (q.cx - dcx),
                  q.y + (q.ay - day) + by2 + (q.cy - dcy),
                  q.z + (q.az - daz) + bz2 + (q.cz - dcz), -q.cx, -q.cy, -q.cz,
                  -(q.ax - ax2), -(q.ay - ay2), -(q.az - az2),
                  q.bx - bx2, q.by - by2, q.bz - bz2};
      sub[n++] = {q.x + (q.ax - dax) + (bx2 - dbx), q.y + (q.ay - day) + (by2 - dby),
                  q.z + (q.az - daz) + (bz2 - dbz), -bx2, -by2, -bz2, cx2, cy2, cz2,
                  -(q.ax - ax2), -(q.ay - ay2), -(q.az - az2)};
    }
    for (int k = n - 1; k >= 0; --k) stack.push_back(sub[k]);   // LIFO: first sub-box on top
  }
}

}  // namespace

int hilbert_build(int T, int H, int W, int text_prefix, int32_t* perm, int32_t* inv) {
  Emitter em{H, W, text_prefix, perm, 0};
  for (int k = 0; k < text_prefix; ++k) perm[em.pos++] = k;
  Box root;
  if (W >= H && W >= T)
    root = {0, 0, 0, W, 0, 0, 0, H, 0, 0, 0, T};
  else if (H >= W && H >= T)
    root = {0, 0, 0, 0, H, 0, W, 0, 0, 0, 0, T};
  else
    root = {0, 0, 0, 0, 0, T, W, 0, 0, 0, H, 0};
  walk(root, em);
  const int64_t L = em.pos;
  for (int64_t r = 0; r < L; ++r) inv[perm[r]] = static_cast<int32_t>(r);
  return SPARGE_OK;
}

}  // namespace sparge
