// Render-row sources (K4 gather, and the rasteriser reading through the
// gather plan): where row r of a view's render set lives — a master row
// (node record / packed master) or a row of a cache block (section-major,
// one touched bit per row after its 23·rows values).
#pragma once
#include "common.cuh"
#include "../../include/glod_b200.h"

namespace glod {

struct Src {
  const double* base;
  long long rows;       // section stride (section-major blocks), or -record stride
  long long idx;
};

// Element (section offset OFF, column col) of a source row: section-major
// blocks/master (rows > 0) or node records (rows = -GLOD_NODE_RECORD).
GLOD_DEV double src_at(const Src& s, int OFF, int COLS, int col) {
  return s.rows > 0 ? s.base[OFF * s.rows + s.idx * COLS + col] : s.base[s.idx * (-s.rows) + OFF + col];
}

// Cache blocks carry one "touched" bit per row after their 23·rows values:
// ADAM sets it instead of writing the updated master row into the block
// (trainer.py:363's refresh made implicit) — a touched row's value IS the
// master row; readers take it from there, and blocks are materialised
// before they are written back.
GLOD_DEV unsigned long long* block_bits(const double* blk, long long rows) {
  return reinterpret_cast<unsigned long long*>(const_cast<double*>(blk) + 23 * rows);
}
GLOD_DEV bool row_touched(const double* blk, long long rows, long long pos) {
  return (block_bits(blk, rows)[pos >> 6] >> (pos & 63)) & 1ull;
}

GLOD_DEV long long master_rows(const glod_gather_plan& p) {
  return p.master_stride ? -p.master_stride : p.capacity;
}

GLOD_DEV Src row_source(const glod_gather_plan& p, long long r, int& node) {
  const long long n_mem = (long long)p.n_upper + p.n_pass;
  Src s;
  if (r < p.n_upper) {
    node = p.upper_ids[r];
    s = {p.master, master_rows(p), node};
  } else if (r < n_mem) {
    node = p.pass_ids[r - p.n_upper];
    s = {p.master, master_rows(p), node};
  } else {
    const long long k = r - n_mem;
    const int j = p.sel_seg[k];
    node = p.sel_node[k];
    const double* blk = reinterpret_cast<const double*>(p.seg_block[j]);
    const long long P = p.seg_rows[j], pos = p.sel_pos[k];
    if (p.spt_from_master || row_touched(blk, P, pos)) s = {p.master, master_rows(p), node};
    else s = {blk, P, pos};
  }
  return s;
}


// The six attribute pointers of one Gaussian (its values at [0, cols)).
struct RowView {
  const double *mean, *scale, *rot, *opac, *base, *sh;
};

GLOD_DEV RowView row_view(const Src& s) {
  RowView v;
  if (s.rows > 0) {                 // section-major block / packed master
    const double* b = s.base;
    v.mean = b + s.idx * 3;
    v.scale = b + 3 * s.rows + s.idx * 3;
    v.rot = b + 6 * s.rows + s.idx * 4;
    v.opac = b + 10 * s.rows + s.idx;
    v.base = b + 11 * s.rows + s.idx * 3;
    v.sh = b + 14 * s.rows + s.idx * 9;
  } else {                          // node record
    const double* r = s.base + s.idx * (-s.rows);
    v.mean = r; v.scale = r + 3; v.rot = r + 6; v.opac = r + 10; v.base = r + 11; v.sh = r + 14;
  }
  return v;
}

}  // namespace glod
