// gvo_bytecode.cuh — device evaluation of address-expression bytecode.
//
// Three interpretations of the same postfix program (the host encodes the
// reference's AddressExpr tree, expr.py:47-98, in post-order):
//   * affine_extract : constant + 6 coordinate coefficients with BX/BY/BZ and
//                      the field base bound (reference expr.affine_parts,
//                      expr.py:171-212), or "non-affine";
//   * eval_point     : one address at explicit coordinates (expr._eval_bulk,
//                      expr.py:267-278, floor // and %);
//   * bounds_check   : inclusive interval of every node, exact in 128-bit,
//                      failing when a node leaves int64 (expr.value_bounds,
//                      expr.py:127-168, the AddressOverflowError guard).
#pragma once
// GVO_OUTLINE bit 64 (k_sets.cu): evaluator and guard as one out-of-line copy
#if defined(GVO_OUTLINE) && (GVO_OUTLINE & 64)
#define GVO_BC_ATTR inline __noinline__
#else
#define GVO_BC_ATTR inline
#endif
#include "gvo_common.cuh"

namespace gvo {

struct AffineForm {
  int64_t c[7];  // [0] constant, [1..6] tidx,tidy,tidz,bidx,bidy,bidz
};

// Returns kAffine or kNonAffine.  Coefficients are exact: any intermediate
// that leaves int64 downgrades the access to the per-point evaluator, which
// is exact whenever the bounds check passed (all subexpressions in range).
// *mag (optional) receives the largest |coefficient| of any node, or
// UINT64_MAX when an intermediate left int64 (plan sharing, k_setup.cu).
__device__ inline int affine_extract(const gvo_insn* code, int len, const int32_t bd[3],
                                     const int64_t* field_base, AffineForm* out, uint64_t* mag = nullptr) {
  AffineForm st[kStack];
  int sp = 0;
  uint64_t mx = 0;
  auto amax = [&](int64_t v) {
    const uint64_t a = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
    if (a > mx) mx = a;
  };
  for (int i = 0; i < len; ++i) {
    const gvo_insn in = code[i];
    if (in.op <= GVO_OP_BASE) {
      if (sp >= kStack) return kNonAffine;
      AffineForm f;
#pragma unroll
      for (int k = 0; k < 7; ++k) f.c[k] = 0;
      if (in.op == GVO_OP_CONST) f.c[0] = in.arg;
      else if (in.op == GVO_OP_COORD) f.c[1 + in.arg] = 1;
      else if (in.op == GVO_OP_BDIM) f.c[0] = bd[in.arg];
      else f.c[0] = field_base[in.arg];
      amax(f.c[0]);
      st[sp++] = f;
      continue;
    }
    if (in.op == GVO_OP_FLOORDIV || in.op == GVO_OP_MOD) return kNonAffine;
    if (sp < 2) return kNonAffine;
    AffineForm r = st[--sp];
    AffineForm l = st[--sp];
    AffineForm o;
    if (in.op == GVO_OP_ADD || in.op == GVO_OP_SUB) {
      for (int k = 0; k < 7; ++k) {
        __int128 v = in.op == GVO_OP_ADD ? (__int128)l.c[k] + r.c[k] : (__int128)l.c[k] - r.c[k];
        if (!fits_i64(v)) { if (mag) *mag = ~0ull; return kNonAffine; }
        o.c[k] = (int64_t)v;
        amax(o.c[k]);
      }
    } else {  // MUL: one side must be coordinate-free
      bool lconst = true, rconst = true;
      for (int k = 1; k < 7; ++k) {
        lconst &= l.c[k] == 0;
        rconst &= r.c[k] == 0;
      }
      if (!lconst && !rconst) return kNonAffine;
      const AffineForm& s = lconst ? r : l;
      const int64_t m = lconst ? l.c[0] : r.c[0];
      for (int k = 0; k < 7; ++k) {
        __int128 v = (__int128)s.c[k] * m;
        if (!fits_i64(v)) { if (mag) *mag = ~0ull; return kNonAffine; }
        o.c[k] = (int64_t)v;
        amax(o.c[k]);
      }
    }
    st[sp++] = o;
  }
  if (sp != 1) return kNonAffine;
  *out = st[0];
  if (mag) *mag = mx;
  return kAffine;
}

// Wrapping int64 evaluation; exact whenever bounds_check passed.
__device__ GVO_BC_ATTR int64_t eval_point(const gvo_insn* code, int len, const int64_t coord[6],
                                     const int32_t bd[3], const int64_t* field_base) {
  int64_t st[kStack];
  int sp = 0;
  for (int i = 0; i < len; ++i) {
    const gvo_insn in = code[i];
    switch (in.op) {
      case GVO_OP_CONST: st[sp++] = in.arg; break;
      case GVO_OP_COORD: st[sp++] = coord[in.arg]; break;
      case GVO_OP_BDIM: st[sp++] = bd[in.arg]; break;
      case GVO_OP_BASE: st[sp++] = field_base[in.arg]; break;
      default: {
        const uint64_t r = (uint64_t)st[--sp];
        const uint64_t l = (uint64_t)st[--sp];
        int64_t v;
        if (in.op == GVO_OP_ADD) v = (int64_t)(l + r);
        else if (in.op == GVO_OP_SUB) v = (int64_t)(l - r);
        else if (in.op == GVO_OP_MUL) v = (int64_t)(l * r);
        else if (in.op == GVO_OP_FLOORDIV) v = floordiv((int64_t)l, (int64_t)r);
        else v = floormod((int64_t)l, (int64_t)r);
        st[sp++] = v;
      }
    }
  }
  return st[0];
}

// Interval check of every BinOp node (post-order = the reference's
// recursion order).  Returns -1 when all nodes stay in int64, else the
// instruction index of the first failing node.  lo/hi receive the root
// interval on success.
// *mag (optional) receives the largest |bound| of any BinOp node.
__device__ GVO_BC_ATTR int bounds_check(const gvo_insn* code, int len, const int64_t clo[6],
                                   const int64_t chi[6], const int32_t bd[3],
                                   const int64_t* field_base, int64_t* root_lo,
                                   int64_t* root_hi, uint64_t* mag = nullptr) {
  int64_t slo[kStack], shi[kStack];
  int sp = 0;
  uint64_t mx = 0;
  for (int i = 0; i < len; ++i) {
    const gvo_insn in = code[i];
    if (in.op <= GVO_OP_BASE) {
      int64_t v0, v1;
      if (in.op == GVO_OP_CONST) v0 = v1 = in.arg;
      else if (in.op == GVO_OP_COORD) { v0 = clo[in.arg]; v1 = chi[in.arg]; }
      else if (in.op == GVO_OP_BDIM) v0 = v1 = bd[in.arg];
      else v0 = v1 = field_base[in.arg];
      slo[sp] = v0;
      shi[sp] = v1;
      ++sp;
      continue;
    }
    const int64_t rlo = slo[sp - 1], rhi = shi[sp - 1];
    const int64_t llo = slo[sp - 2], lhi = shi[sp - 2];
    sp -= 2;
    __int128 lo, hi;
    if (in.op == GVO_OP_ADD) { lo = (__int128)llo + rlo; hi = (__int128)lhi + rhi; }
    else if (in.op == GVO_OP_SUB) { lo = (__int128)llo - rhi; hi = (__int128)lhi - rlo; }
    else if (in.op == GVO_OP_MUL) {
      __int128 a = (__int128)llo * rlo, b = (__int128)llo * rhi;
      __int128 c = (__int128)lhi * rlo, d = (__int128)lhi * rhi;
      lo = a; hi = a;
      if (b < lo) lo = b; if (b > hi) hi = b;
      if (c < lo) lo = c; if (c > hi) hi = c;
      if (d < lo) lo = d; if (d > hi) hi = d;
    } else if (in.op == GVO_OP_FLOORDIV) {
      lo = floordiv(llo, rlo);
      hi = floordiv(lhi, rlo);
    } else {
      lo = 0;
      hi = rlo - 1;
    }
    if (!fits_i64(lo) || !fits_i64(hi)) return i;
    slo[sp] = (int64_t)lo;
    shi[sp] = (int64_t)hi;
    ++sp;
    const uint64_t alo = lo < 0 ? (uint64_t)(-lo) : (uint64_t)lo, ahi = hi < 0 ? (uint64_t)(-hi) : (uint64_t)hi;
    if (alo > mx) mx = alo;
    if (ahi > mx) mx = ahi;
  }
  *root_lo = slo[0];
  *root_hi = shi[0];
  if (mag) *mag = mx;
  return -1;
}

}  // namespace gvo
