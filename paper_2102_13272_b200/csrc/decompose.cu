// decompose.cu -- the decomposition algorithm of section IV.B as a host-side
// planner: F(M, R; S) over one base kernel F(m, r) -> expression tree -> output lengths ->
// reverse Polish token stream.  Host only (no device code); exported as nw_decompose.
//
//  step 1: S > 1 -> stride Winograd, Eq. 2.7: phase t of the filter has
//         ceil((R - t) / S) taps; one term per non-empty phase, in phase order (the
//         (r'+1)-tap phases first, as in Eq. 4.1).  S = 1 and R > r -> nested Winograd
//         (III.A), d = ceil(log_r R) levels of the same kernel.  R <= r -> the kernel.
//  step 2: a kernel outputs m; d levels output O_d distinct contiguous values,
//         O_1 = m, O_j = (m - 1) r^(j-1) + O_(j-1) (m >= r; P:110 gives m^2 for m = r,
//         d = 2); a sum needs equal lengths: each term is repeated n = lcm / length times
//         ("F(n.m, r) = n.F(m, r)", R10a).
//  tokens: K<m>,<r>  NEST<d>  REP<n>  SUM<k>, post-order.
// The CPU oracle (oracle/planner.py) derives the same plan from exact composite matrices;
// tests/test_abi.py compares the two token streams and M over a grid of (R, S, m, r).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "nw_internal.h"

namespace nw {
namespace {

struct PNode {
  enum Kind { kLeaf, kNest, kRepeat, kSum } kind = kLeaf;
  int m = 0, r = 0, levels = 1, n = 1;
  long long M = 0;
  std::vector<PNode> kids;
};

int depth_for(int R, int r) {
  int d = 1;
  long long reach = r;
  while (reach < R) {
    ++d;
    reach *= r;
  }
  return d;
}

long long distinct_outputs(int m, int r, int d) {
  long long O = m, p = 1;
  for (int j = 2; j <= d; ++j) {
    p *= r;
    O = (long long)(m - 1) * p + O;
  }
  return O;
}

long long gcdll(long long a, long long b) {
  while (b) {
    const long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

PNode decompose(int R, int S, int m, int r) {
  PNode p;
  if (S > 1) {
    p.kind = PNode::kSum;
    for (int t = 0; t < S; ++t) {
      const int taps = R - t > 0 ? (R - t + S - 1) / S : 0;
      if (taps > 0) p.kids.push_back(decompose(taps, 1, m, r));
    }
    return p;
  }
  p.m = m;
  p.r = r;
  if (R > r) {
    p.kind = PNode::kNest;
    p.levels = depth_for(R, r);
  }
  return p;
}

void resolve(PNode &p) {
  switch (p.kind) {
    case PNode::kLeaf: p.M = p.m; break;
    case PNode::kNest: p.M = distinct_outputs(p.m, p.r, p.levels); break;
    case PNode::kRepeat:
      resolve(p.kids[0]);
      p.M = p.n * p.kids[0].M;
      break;
    case PNode::kSum: {
      long long L = 1;
      for (auto &k : p.kids) {
        resolve(k);
        L = L / gcdll(L, k.M) * k.M;
      }
      for (auto &k : p.kids) {
        if (k.M != L) {
          PNode rep;
          rep.kind = PNode::kRepeat;
          rep.n = (int)(L / k.M);
          rep.M = L;
          rep.kids.push_back(k);
          k = rep;
        }
      }
      p.M = L;
      break;
    }
  }
}

void emit(const PNode &p, std::string &out) {
  char buf[48];
  auto tok = [&](const char *s) {
    if (!out.empty()) out += ' ';
    out += s;
  };
  switch (p.kind) {
    case PNode::kLeaf:
      snprintf(buf, sizeof buf, "K%d,%d", p.m, p.r);
      tok(buf);
      break;
    case PNode::kNest:
      snprintf(buf, sizeof buf, "K%d,%d", p.m, p.r);
      tok(buf);
      snprintf(buf, sizeof buf, "NEST%d", p.levels);
      tok(buf);
      break;
    case PNode::kRepeat:
      emit(p.kids[0], out);
      snprintf(buf, sizeof buf, "REP%d", p.n);
      tok(buf);
      break;
    case PNode::kSum:
      for (const auto &k : p.kids) emit(k, out);
      snprintf(buf, sizeof buf, "SUM%d", (int)p.kids.size());
      tok(buf);
      break;
  }
}

}  // namespace
}  // namespace nw

extern "C" {

nw_status_t nw_decompose(int R, int S, int m, int r, char *rpn, size_t cap, size_t *len, int *M) {
  if (R < 1 || S < 1 || m < 1 || r < 1 || R > 4096 || S > 64 || m > 64 || r > 64) return NW_ERR_INVALID;
  if (m < r && R > r) return NW_ERR_UNSUPPORTED;  // nesting with m < r leaves holes (R6)
  nw::PNode p = nw::decompose(R, S, m, r);
  nw::resolve(p);
  std::string s;
  nw::emit(p, s);
  if (len) *len = s.size();
  if (M) *M = p.M > 0x7fffffffLL ? -1 : (int)p.M;
  if (rpn) {
    if (cap < s.size() + 1) return NW_ERR_INVALID;
    memcpy(rpn, s.c_str(), s.size() + 1);
  }
  return NW_OK;
}

}  // extern "C"
