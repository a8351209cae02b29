// Host plan construction (see scc_plan.hpp).
#include "scc_plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <stdexcept>

namespace scc {

namespace {

[[noreturn]] void fail(scc_status_t code, std::string msg) {
  throw Error{code, std::move(msg)};
}

// The cycle walk of compute_channel_cycle (cycle.cpp:9-21): starts 0, +shift
// mod c_in, stop at the first repeat or after c_out windows.
std::vector<int64_t> walk_cycle(int64_t c_in, int64_t c_out, int64_t shift) {
  std::vector<int64_t> starts;
  std::vector<char> seen(static_cast<size_t>(c_in), 0);
  int64_t s = 0;
  while (static_cast<int64_t>(starts.size()) < c_out && !seen[static_cast<size_t>(s)]) {
    seen[static_cast<size_t>(s)] = 1;
    starts.push_back(s);
    s = (s + shift) % c_in;
  }
  return starts;
}

void build_groups(BandSide& side) {
  side.groups.clear();
  const int nb = side.nblk();
  for (int b0 = 0; b0 < nb; b0 += kBlocksPerGroup) {
    const int cnt = std::min(kBlocksPerGroup, nb - b0);
    std::vector<Arc> parts(side.blocks.begin() + b0, side.blocks.begin() + b0 + cnt);
    const Arc a = cover_arcs(parts, side.ring);
    side.groups.insert(side.groups.end(), {b0, cnt, a.start, a.len});
  }
  side.max_block_len = 0;
  for (const Arc& a : side.blocks) side.max_block_len = std::max(side.max_block_len, a.len);
}

}  // namespace

Arc cover_arcs(const std::vector<Arc>& parts, int32_t n) {
  Arc best{0, 0};
  bool any = false;
  int64_t best_len = INT64_MAX;
  for (const Arc& cand : parts) {
    if (cand.len <= 0) continue;
    any = true;
    if (cand.len >= n) return Arc{0, n};
    int64_t need = 0;
    for (const Arc& a : parts) {
      if (a.len <= 0) continue;
      const int64_t off = ((static_cast<int64_t>(a.start) - cand.start) % n + n) % n;
      need = std::max<int64_t>(need, off + a.len);
    }
    if (need < best_len) {
      best_len = need;
      best = Arc{cand.start, static_cast<int32_t>(std::min<int64_t>(need, n))};
    }
  }
  if (!any) return Arc{0, 0};
  if (best.len >= n) best = Arc{0, n};
  return best;
}

int64_t resolve_overlap(int32_t kind, double ratio, int64_t count, int64_t gw) {
  if (kind == SCC_OVERLAP_RATIO) {
    if (!(ratio >= 0.0 && ratio <= 1.0)) {
      fail(SCC_ERR_CONFIG, "overlap fraction " + std::to_string(ratio) + " outside [0, 1]");
    }
    // std::llround: halves round away from zero (config.cpp:45); Python's
    // round() would not (gw=5, co=50% -> 3 here, 2 under banker's rounding).
    return std::llround(ratio * static_cast<double>(gw));
  }
  if (kind != SCC_OVERLAP_CHANNELS) fail(SCC_ERR_ARGUMENT, "unknown overlap kind");
  if (count < 0 || count > gw) {
    fail(SCC_ERR_CONFIG, "overlap of " + std::to_string(count) + " channels outside [0, " +
                             std::to_string(gw) + "] for window width " + std::to_string(gw));
  }
  return count;
}

void parse_overlap(const char* text, int32_t* kind, double* ratio, int64_t* count) {
  if (text == nullptr) fail(SCC_ERR_ARGUMENT, "null overlap text");
  const std::string t(text);
  if (t.empty()) fail(SCC_ERR_ARGUMENT, "empty overlap value");
  try {
    size_t used = 0;
    if (t.back() == '%') {
      const std::string num = t.substr(0, t.size() - 1);
      const double pct = std::stod(num, &used);
      if (used != num.size()) fail(SCC_ERR_ARGUMENT, "bad overlap '" + t + "'");
      *kind = SCC_OVERLAP_RATIO;
      *ratio = pct / 100.0;
      *count = 0;
      return;
    }
    if (t.find_first_of(".eE") != std::string::npos) {
      const double r = std::stod(t, &used);
      if (used != t.size()) fail(SCC_ERR_ARGUMENT, "bad overlap '" + t + "'");
      *kind = SCC_OVERLAP_RATIO;
      *ratio = r;
      *count = 0;
      return;
    }
    const long long c = std::stoll(t, &used);
    if (used != t.size()) fail(SCC_ERR_ARGUMENT, "bad overlap '" + t + "'");
    *kind = SCC_OVERLAP_CHANNELS;
    *ratio = 0.0;
    *count = c;
  } catch (const std::invalid_argument&) {
    fail(SCC_ERR_ARGUMENT, "bad overlap '" + t + "'");
  } catch (const std::out_of_range&) {
    fail(SCC_ERR_ARGUMENT, "overlap '" + t + "' out of numeric range");
  }
}

void build_tc_side(const Plan& p, bool bwd, TcBandPlan& tp) {
  const scc_config_t& c = p.cfg;
  tp = TcBandPlan{};
  const int32_t rows_total = static_cast<int32_t>(bwd ? c.c_in : c.c_out);
  tp.ring = static_cast<int32_t>(bwd ? c.c_out : c.c_in);
  if (tp.ring % 8 != 0) {
    tp.why = "ring length not a multiple of 8";
    return;
  }
  if (bwd) {
    const int32_t D = static_cast<int32_t>(c.cyclic_dist);
    if (c.c_out % D != 0 || (c.c_out / D) % 8 != 0) {
      tp.why = "filters per window class not a multiple of 8";
      return;
    }
    tp.cls = static_cast<int32_t>(c.c_out / D);
    tp.n_class = D;
    tp.rows_per_sample_3d = tp.cls;
    for (int32_t cl = 0; cl < D; ++cl) {
      const int32_t d = p.perm[static_cast<size_t>(cl) * tp.cls];
      if (d >= D) {
        tp.why = "cycle classes are not residues mod cyclic_dist";
        return;
      }
      for (int32_t j = 0; j < tp.cls; ++j) {
        if (p.perm[static_cast<size_t>(cl) * tp.cls + j] != d + D * j) {
          tp.why = "cycle class layout mismatch";
          return;
        }
      }
      tp.class_d.push_back(d);
    }
  } else {
    tp.cls = static_cast<int32_t>(c.c_in);
    tp.n_class = 1;
    tp.rows_per_sample_3d = static_cast<int32_t>(c.c_in);
    tp.class_d = {0};
  }
  // Activation box height: the largest of 32/16/8 rows that divides the ring
  // and the class run, so a box never leaves one contiguous run of rows.
  tp.rb = 8;
  for (int32_t rb : {32, 16}) {
    if (tp.ring % rb == 0 && tp.cls % rb == 0) {
      tp.rb = rb;
      break;
    }
  }
  // Output view for TMA stores (32-row groups of the tile's rows).
  if (bwd) {
    tp.out_cls = static_cast<int32_t>(c.c_in);
    tp.out_n_class = 1;
    tp.out_class_d = {0};
    tp.store_ok = c.c_in % 32 == 0;
  } else {
    const int32_t D = static_cast<int32_t>(c.cyclic_dist);
    tp.store_ok = c.c_out % D == 0 && (c.c_out / D) % 32 == 0;
    if (tp.store_ok) {
      tp.out_cls = static_cast<int32_t>(c.c_out / D);
      tp.out_n_class = D;
      for (int32_t cl = 0; cl < D && tp.store_ok; ++cl) {
        const int32_t d = p.perm[static_cast<size_t>(cl) * tp.out_cls];
        for (int32_t j = 0; j < tp.out_cls; ++j) {
          if (d >= D || p.perm[static_cast<size_t>(cl) * tp.out_cls + j] != d + D * j) tp.store_ok = false;
        }
        tp.out_class_d.push_back(d);
      }
    }
    if (!tp.store_ok) tp.out_class_d.assign(1, 0);
  }
  // Row-tile width: fewest padded rows, ties to the wider tile.
  int32_t best = 0;
  int64_t best_pad = INT64_MAX;
  for (int32_t nt : {128, 64}) {
    const int64_t tiles = (rows_total + nt - 1) / nt;
    const int64_t pad = tiles * nt;
    if (pad < best_pad) {
      best_pad = pad;
      best = nt;
    }
  }
  // gw = 64 with tight 64-row arcs (<= 96 ring rows, i.e. co = 50 %): 64-row
  // tiles measured 2-10 % faster at 14x14 and 56x56 (scripts/band_ab.py: each
  // CTA keeps one row tile's panel resident, the band padding halves).  With
  // wider arcs (co = 25 / 75 %: more, shorter class runs) every extra
  // activation row re-read costs more than that (measured 5-15 % slower), and
  // for gw >= 256 they lose up to 40 %, so those keep the widest tile.
  if (c.group_width == 64 && rows_total % 64 == 0) {
    int32_t max_arc = 0;
    for (int32_t t0 = 0; t0 < rows_total; t0 += 64) {
      std::vector<Arc> arcs;
      for (int32_t i = t0; i < std::min(t0 + 64, rows_total); ++i) {
        arcs.push_back(bwd ? p.ic_arcs[static_cast<size_t>(i)]
                           : Arc{static_cast<int32_t>(p.start_of(p.perm[static_cast<size_t>(i)])),
                                 static_cast<int32_t>(c.group_width)});
      }
      max_arc = std::max(max_arc, cover_arcs(arcs, tp.ring).len);
    }
    if (max_arc <= 96) best = 64;
  }
  tp.nt = best;
  tp.n_rt = (rows_total + tp.nt - 1) / tp.nt;
  tp.rows.assign(static_cast<size_t>(tp.n_rt) * tp.nt, -1);
  tp.chunk_base.assign(1, 0);
  const int32_t gw = static_cast<int32_t>(c.group_width);
  for (int32_t rt = 0; rt < tp.n_rt; ++rt) {
    std::vector<Arc> arcs;
    for (int32_t r = 0; r < tp.nt; ++r) {
      const int32_t i = rt * tp.nt + r;
      if (i >= rows_total) break;
      if (bwd) {
        tp.rows[static_cast<size_t>(i)] = i;
        arcs.push_back(p.ic_arcs[static_cast<size_t>(i)]);
      } else {
        const int32_t oc = p.perm[static_cast<size_t>(i)];
        tp.rows[static_cast<size_t>(i)] = oc;
        arcs.push_back(Arc{static_cast<int32_t>(p.start_of(oc)), gw});
      }
    }
    const Arc cov = cover_arcs(arcs, tp.ring);
    // Align the arc to the TMA box height so every box stays inside one ring
    // class and never wraps.
    int32_t start8 = (cov.start / tp.rb) * tp.rb;
    int32_t nk8 = (cov.start + cov.len - start8 + tp.rb - 1) / tp.rb * (tp.rb / 8);
    if (nk8 < tp.rb / 8) nk8 = tp.rb / 8;  // uncovered rows still get written (as zeros)
    if (nk8 * 8 >= tp.ring) {
      start8 = 0;
      nk8 = tp.ring / 8;
    }
    const int32_t chunks = (nk8 + 3) / 4;
    tp.rt_info.insert(tp.rt_info.end(),
                      {start8, nk8, tp.chunk_base.back() * 2 * tp.nt * 32, chunks});
    tp.chunk_base.push_back(tp.chunk_base.back() + chunks);
  }
  tp.total_chunks = tp.chunk_base.back();
  tp.ok = true;
}

void build_tc_weight(const Plan& p, TcWeightPlan& tw) {
  const scc_config_t& c = p.cfg;
  tw = TcWeightPlan{};
  if (!p.tc_bwd.ok || c.c_in % 8 != 0) {
    tw.why = "needs the backward-data class layout and c_in % 8 == 0";
    return;
  }
  tw.cls = p.tc_bwd.cls;
  tw.n_class = p.tc_bwd.n_class;
  tw.class_d = p.tc_bwd.class_d;
  const int32_t ring = static_cast<int32_t>(c.c_in);
  const int32_t gw = static_cast<int32_t>(c.group_width);
  tw.n_rt = static_cast<int32_t>((c.c_out + 127) / 128);
  int32_t max_cols = 0;
  for (int32_t rt = 0; rt < tw.n_rt; ++rt) {
    std::vector<Arc> arcs;
    for (int32_t r = 0; r < 128; ++r) {
      const int64_t i = static_cast<int64_t>(rt) * 128 + r;
      if (i >= c.c_out) break;
      arcs.push_back(Arc{static_cast<int32_t>(p.start_of(p.perm[static_cast<size_t>(i)])), gw});
    }
    const Arc cov = cover_arcs(arcs, ring);
    int32_t start8 = (cov.start / 8) * 8;
    int32_t ncols = ((cov.start + cov.len - start8 + 7) / 8) * 8;
    if (ncols >= ring) {
      start8 = 0;
      ncols = ring;
    }
    tw.rt_info.insert(tw.rt_info.end(), {start8, ncols});
    max_cols = std::max(max_cols, ncols);
  }
  // Column chunk: multiple of 32 (four 8-row quarters, M=128 MMA).  Up to 384
  // columns stay one chunk (the kernel splits the MMA's N at 256, TMEM holds
  // 384 accumulator columns next to its A stages): a second chunk would be a
  // second CTA re-reading the tile's dy -- co = 25 / 75 % at gw = 256 gives
  // 320-384-column arcs (measured 1.7x the backward-weight time of co = 50 %).
  const int32_t w32 = (max_cols + 31) / 32 * 32;
  tw.n_nc = w32 <= 384 ? 1 : (w32 + 255) / 256;
  tw.nw = ((w32 + tw.n_nc - 1) / tw.n_nc + 31) / 32 * 32;
  // dy boxes: each converter warp loads its 32 filter rows; one box when the
  // 32 rows are one contiguous class run.
  tw.rba = (tw.cls % 32 == 0) ? 32 : (tw.cls % 16 == 0 ? 16 : 8);
  // x boxes: a warp loads nw/4 consecutive arc rows; a box must not wrap the
  // ring, so its height divides the ring, every arc start and the quarter.
  tw.rbb = 8;
  for (int32_t rb : {64, 32, 16}) {
    bool ok = (tw.nw / 4) % rb == 0 && ring % rb == 0;
    for (int32_t rt = 0; rt < tw.n_rt && ok; ++rt) ok = tw.rt_info[2 * rt] % rb == 0;
    if (ok) {
      tw.rbb = rb;
      break;
    }
  }
  // Generation-1 kernel: the producer tiles each chunk's arc rows with boxes
  // of rbb1 rows; the tallest box (multiple of 8: 1 KB swizzle atoms) that
  // divides the chunk width and never straddles the ring end.  Fewer, larger
  // boxes keep more bytes in flight per TMA issue.
  tw.rbb1 = 8;
  for (int32_t rb = std::min(tw.nw, 256); rb > 8; rb -= 8) {
    bool ok = tw.nw % rb == 0;
    for (int32_t rt = 0; rt < tw.n_rt && ok; ++rt) {
      for (int32_t r = 0; r < tw.n_nc * tw.nw && ok; r += rb) {
        if (r >= tw.rt_info[2 * rt + 1]) break;
        const int32_t pos = (tw.rt_info[2 * rt] + r) % ring;
        ok = pos + rb <= ring;
      }
    }
    if (ok) {
      tw.rbb1 = rb;
      break;
    }
  }
  tw.c_in = static_cast<int32_t>(p.cfg.c_in);
  tw.c_out = static_cast<int32_t>(p.cfg.c_out);
  tw.ok = true;
}

void build_plan(Plan& p, int64_t c_in, int64_t c_out, int64_t cg, int32_t kind,
                double ratio, int64_t count, int32_t has_bias) {
  // scc_config_new (config.cpp:62-83).
  if (c_in < 1) fail(SCC_ERR_CONFIG, "c_in must be >= 1, got " + std::to_string(c_in));
  if (c_out < 1) fail(SCC_ERR_CONFIG, "c_out must be >= 1, got " + std::to_string(c_out));
  if (cg < 1 || cg > c_in) {
    fail(SCC_ERR_CONFIG, "cg must be in [1, c_in=" + std::to_string(c_in) + "], got " +
                             std::to_string(cg));
  }
  if (c_in % cg != 0) {
    fail(SCC_ERR_CONFIG,
         "cg=" + std::to_string(cg) + " does not divide c_in=" + std::to_string(c_in));
  }
  if (c_in > (1 << 24) || c_out > (1 << 24)) {
    fail(SCC_ERR_CONFIG, "channel counts above 2^24 are not supported by the device tables");
  }
  scc_config_t& c = p.cfg;
  c.c_in = c_in;
  c.c_out = c_out;
  c.cg = cg;
  c.group_width = c_in / cg;
  c.overlap_channels = resolve_overlap(kind, ratio, count, c.group_width);
  c.shift = c.group_width - c.overlap_channels;
  c.has_bias = has_bias ? 1 : 0;
  c.fully_overlapped = (c.shift == 0 && cg > 1) ? 1 : 0;
  p.cycle_starts = walk_cycle(c_in, c_out, c.shift);
  c.cyclic_dist = static_cast<int64_t>(p.cycle_starts.size());

  // The closed form the device uses must agree with the cycle lookup.
  for (int64_t oc = 0; oc < c_out; ++oc) {
    if (p.cycle_starts[static_cast<size_t>(oc % c.cyclic_dist)] != p.start_of(oc)) {
      fail(SCC_ERR_INTERNAL, "window-start closed form disagrees with the cycle walk");
    }
  }

  p.starts.resize(static_cast<size_t>(c_out));
  for (int64_t oc = 0; oc < c_out; ++oc) p.starts[static_cast<size_t>(oc)] = static_cast<int32_t>(p.start_of(oc));

  // Cycle-sorted order of the filters: by window start, then oc.
  p.perm.resize(static_cast<size_t>(c_out));
  std::iota(p.perm.begin(), p.perm.end(), 0);
  std::stable_sort(p.perm.begin(), p.perm.end(), [&](int32_t a, int32_t b) {
    return p.start_of(a) < p.start_of(b);
  });
  p.inv_perm.resize(static_cast<size_t>(c_out));
  for (int64_t i = 0; i < c_out; ++i) p.inv_perm[static_cast<size_t>(p.perm[i])] = static_cast<int32_t>(i);

  const int32_t gw = static_cast<int32_t>(c.group_width);

  // Forward: rows = filters in sorted order, ring = input channels.
  {
    BandSide& f = p.fwd;
    f.ring = static_cast<int32_t>(c_in);
    f.ring_map.clear();
    const int nb = static_cast<int>((c_out + kRowsPerBlock - 1) / kRowsPerBlock);
    f.rows.assign(static_cast<size_t>(nb) * kRowsPerBlock, -1);
    f.blocks.resize(static_cast<size_t>(nb));
    for (int b = 0; b < nb; ++b) {
      std::vector<Arc> parts;
      for (int j = 0; j < kRowsPerBlock; ++j) {
        const int64_t i = static_cast<int64_t>(b) * kRowsPerBlock + j;
        if (i >= c_out) break;
        const int32_t oc = p.perm[static_cast<size_t>(i)];
        f.rows[static_cast<size_t>(i)] = oc;
        parts.push_back(Arc{static_cast<int32_t>(p.start_of(oc)), gw});
      }
      f.blocks[static_cast<size_t>(b)] = cover_arcs(parts, f.ring);
    }
    build_groups(f);
  }

  // Backward-data: rows = input channels, ring = filters in sorted order.
  // The filters covering ic are those with start in (ic-gw, ic] (cyclic), a
  // contiguous run of the sorted order (verified below against the direct
  // membership test of ChannelWindow::contains, cycle.hpp:18-20).
  {
    BandSide& d = p.bwd;
    d.ring = static_cast<int32_t>(c_out);
    d.ring_map = p.perm;
    const int nb = static_cast<int>((c_in + kRowsPerBlock - 1) / kRowsPerBlock);
    d.rows.assign(static_cast<size_t>(nb) * kRowsPerBlock, -1);
    d.blocks.resize(static_cast<size_t>(nb));
    std::vector<int32_t> covered;
    p.ic_arcs.assign(static_cast<size_t>(c_in), Arc{0, 0});
    for (int b = 0; b < nb; ++b) {
      std::vector<Arc> parts;
      for (int j = 0; j < kRowsPerBlock; ++j) {
        const int64_t ic = static_cast<int64_t>(b) * kRowsPerBlock + j;
        if (ic >= c_in) break;
        d.rows[static_cast<size_t>(ic)] = static_cast<int32_t>(ic);
        covered.clear();
        for (int64_t i = 0; i < c_out; ++i) {
          if (p.slot_of(p.perm[static_cast<size_t>(i)], ic) >= 0) covered.push_back(static_cast<int32_t>(i));
        }
        if (covered.empty()) continue;
        // Find the arc: the covered positions are contiguous modulo c_out.
        const int32_t n = static_cast<int32_t>(c_out);
        int32_t first = covered.front();
        if (static_cast<int64_t>(covered.size()) < n && covered.front() == 0 &&
            covered.back() == n - 1) {
          // Wrapping run: starts after the first gap.
          for (size_t k = 1; k < covered.size(); ++k) {
            if (covered[k] != covered[k - 1] + 1) {
              first = covered[k];
              break;
            }
          }
        }
        const Arc a{first, static_cast<int32_t>(covered.size())};
        p.ic_arcs[static_cast<size_t>(ic)] = a;
        for (int32_t k = 0; k < a.len; ++k) {
          const int32_t pos = (a.start + k) % n;
          if (p.slot_of(p.perm[static_cast<size_t>(pos)], ic) < 0) {
            fail(SCC_ERR_INTERNAL, "covering filters are not contiguous in cycle order");
          }
        }
        parts.push_back(a);
      }
      d.blocks[static_cast<size_t>(b)] = cover_arcs(parts, d.ring);
    }
    build_groups(d);
  }
  build_tc_side(p, false, p.tc_fwd);
  build_tc_side(p, true, p.tc_bwd);
  build_tc_weight(p, p.tc_wgt);
}

}  // namespace scc
