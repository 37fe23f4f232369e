// Host builder of the K5 "colored_smem" format (C++17/OpenMP).
//
// K5 executes the RACE distance-2 colouring (§4.2: rows
// of one colour have disjoint write sets, so they run "in parallel without
// write conflicts") inside a shared-memory window of one
// GPU tile:
//   * a K5 tile is a run of consecutive schedule tiles of ONE level group
//     (level groups of >= k levels; tiles never straddle
//     a group), merged while its window |own rows ∪ targets| <= wcap and its
//     stored entries <= nnzcap;
//   * inside the tile the rows are greedily coloured so that the write sets
//     W(r) = {r} ∪ {c : a_rc stored in row r} of one colour are disjoint
//     (the distance-2 condition of PAPER.md:787-789 for upper storage); a
//     colour whose entries would not fit the kernel's shared-memory ring is
//     split into several (a subset of a colour is still a colour);
//   * within a colour the rows are sorted by their number of off-diagonal
//     entries (descending) and cut into slices of 32 (one lane per row);
//   * the off-diagonal entries of a slice are stored jagged-diagonal (JDS) in
//     pieces of <= 16 steps: step j holds one entry of every lane whose row is
//     longer than j, so a warp reads a step as one contiguous run, and no
//     padding is stored.  WHICH entry of a row goes to step j is chosen so
//     that the 16 lanes of each half warp address 16 different shared-memory
//     bank pairs (window id mod 16): the x gather and the y read-modify-write
//     of a step are then conflict-free (measured 3.1x the throughput of
//     random addresses on B200, tools/micro3.cu).  Summation order is free
//     (reading R5).
//
// Global layout of one tile: a HEAD (one bulk copy into shared memory)
// followed by CHUNKS (<= chunk bytes, one bulk copy each into a ring stage)
// holding whole pieces:
//   head:  CsHeadHdr | cslc u16[nc+1] | srec CsSliceRec[ns] | ploc u32[np] |
//          pw u16[np] | tgt i32[S] | clen u32[nch]      (16-B aligned sections)
//   piece: eo u16[16] | (first piece of a slice: rowid u16[32] | len u16[32] |
//          diag f64[32]) | val f64[nnz_p] | lcol u16[nnz_p] | pad to 16 B
// cslc[c] = first slice of colour c; srec[s] = slice record (first piece, its
// location, pieces, steps, rows); ploc[p] = (chunk index in tile << 20) | byte
// offset of piece p in its chunk; pw[p] = release weight of piece p (the
// weights of the pieces of one chunk sum to kCsReleaseUnits, so the warps
// that finish the pieces of a chunk release its ring stage together);
// eo[u] = end of step u's run inside the piece (eo[15] = nnz_p).
#include <algorithm>
#include <cstring>
#include <functional>
#include <vector>

#include "internal.h"

namespace symm {

namespace {
inline int64_t al16(int64_t v) { return (v + 15) & ~int64_t(15); }
constexpr int kPieceSteps = 16;
constexpr int kSliceMeta = 32 + 64 + 64 + 256;  // eo + rowid + len + diag of a first piece
using Ent = std::pair<uint16_t, double>;        // (window id, value)
}  // namespace

// Greedy write-set colouring of rows [r0, r1) of the permuted upper CRS.
// Local target ids: own rows 0..T-1, targets >= r1 at T + position in tgt.
// Rows take, in ascending order, the smallest colour whose write set is
// disjoint from theirs.  Returns the number of colours.
int32_t color_rows_writeset(const int32_t* rp, const int32_t* pc, int32_t r0, int32_t r1,
                            const std::vector<int32_t>& tgt, std::vector<int32_t>& color) {
  const int32_t T = r1 - r0;
  const size_t W = (size_t)T + tgt.size();
  auto local = [&](int32_t c) -> size_t {
    if (c < r1) return (size_t)(c - r0);
    return (size_t)T + (size_t)(std::lower_bound(tgt.begin(), tgt.end(), c) - tgt.begin());
  };
  size_t nw = 1;
  std::vector<uint64_t> m(W, 0);
  color.assign((size_t)T, 0);
  int32_t ncolors = 0;
  std::vector<size_t> tg;
  for (int32_t r = r0; r < r1; ++r) {
    tg.clear();
    tg.push_back((size_t)(r - r0));
    for (int32_t i = rp[r]; i < rp[r + 1]; ++i)
      if (pc[i] != r) tg.push_back(local(pc[i]));
    int32_t col = -1;
    for (size_t word = 0; col < 0; ++word) {
      if (word == nw) {  // grow every mask by one word
        std::vector<uint64_t> m2(W * (nw + 1), 0);
        for (size_t l = 0; l < W; ++l)
          for (size_t w = 0; w < nw; ++w) m2[l * (nw + 1) + w] = m[l * nw + w];
        m.swap(m2);
        ++nw;
      }
      uint64_t forbid = 0;
      for (size_t l : tg) forbid |= m[l * nw + word];
      if (~forbid) {
        const int bit = __builtin_ctzll(~forbid);
        col = (int32_t)(word * 64) + bit;
        for (size_t l : tg) m[l * nw + word] |= (uint64_t(1) << bit);
      }
    }
    color[(size_t)(r - r0)] = col;
    ncolors = std::max(ncolors, col + 1);
  }
  return ncolors;
}

namespace {

// Bank-aware step order of one slice with V lanes per row (lane = i * V +
// sub; entry t * V + sub of row i is handled by lane (i, sub) at step t): the
// rows' entry lists are reordered in place so that at every step the active
// lanes of each half warp use distinct banks (window id mod 16) where
// possible: per (step, half) a bipartite matching lane -> bank over the
// entries the lane's row has left (augmenting paths).  Returns the number of
// (step, half) pairs that still conflict.
int64_t bank_order(std::vector<std::vector<Ent>>& ent, int V) {
  const int m = (int)ent.size();
  int maxlen = 0;
  for (auto& e : ent) maxlen = std::max(maxlen, (int)e.size());
  const int nsteps = (maxlen + V - 1) / V;
  int64_t conflicts = 0;
  std::vector<char> seen(16);
  std::vector<Ent> rest;
  for (int t = 0; t < nsteps; ++t) {
    for (int h = 0; h < 2; ++h) {
      int lrow[16], lsub[16], nl = 0;  // active lanes of this half
      for (int ln = 16 * h; ln < 16 * h + 16; ++ln) {
        const int i = ln / V, sub = ln % V;
        if (i < m && (int)ent[(size_t)i].size() > t * V + sub) {
          lrow[nl] = i;
          lsub[nl] = sub;
          ++nl;
        }
      }
      if (!nl) continue;
      int owner[16];
      std::fill(owner, owner + 16, -1);
      std::function<bool(int)> aug = [&](int li) -> bool {
        auto& e = ent[(size_t)lrow[li]];
        for (size_t q = (size_t)t * V; q < e.size(); ++q) {
          const int bk = e[q].first & 15;
          if (seen[(size_t)bk]) continue;
          seen[(size_t)bk] = 1;
          if (owner[bk] < 0 || aug(owner[bk])) {
            owner[bk] = li;
            return true;
          }
        }
        return false;
      };
      int matched = 0;
      for (int li = 0; li < nl; ++li) {
        std::fill(seen.begin(), seen.end(), 0);
        matched += aug(li) ? 1 : 0;
      }
      conflicts += (matched < nl);
      int bank_of[16];
      std::fill(bank_of, bank_of + 16, -1);
      for (int bk = 0; bk < 16; ++bk)
        if (owner[bk] >= 0) bank_of[owner[bk]] = bk;
      // place row by row: matched lanes take an entry of their bank, the
      // others any remaining entry; the rest keeps its order after them
      for (int li = 0; li < nl;) {
        const int i = lrow[li];
        int lj = li;
        while (lj < nl && lrow[lj] == i) ++lj;
        auto& e = ent[(size_t)i];
        rest.assign(e.begin() + (size_t)t * V, e.end());
        Ent placed[16];
        bool got[16] = {false};
        for (int k = li; k < lj; ++k)
          if (bank_of[k] >= 0)
            for (size_t q = 0; q < rest.size(); ++q)
              if ((rest[q].first & 15) == bank_of[k]) {
                placed[lsub[k]] = rest[q];
                got[lsub[k]] = true;
                rest.erase(rest.begin() + (long)q);
                break;
              }
        for (int k = li; k < lj; ++k)
          if (!got[lsub[k]]) {
            placed[lsub[k]] = rest.front();
            got[lsub[k]] = true;
            rest.erase(rest.begin());
          }
        size_t w = (size_t)t * V;
        for (int k = li; k < lj; ++k) e[w + (size_t)lsub[k]] = placed[lsub[k]];
        w += (size_t)(lj - li);
        for (auto& r : rest) e[w++] = r;
        li = lj;
      }
    }
  }
  return conflicts;
}

}  // namespace

int64_t bank_order_rows(std::vector<std::vector<std::pair<uint16_t, double>>>& ent, int V) { return bank_order(ent, V); }

int build_cs_format(const Schedule& S, int32_t t_begin, int32_t t_end, int32_t wcap, int32_t nnzcap,
                    int32_t chunk_bytes, int32_t stages, int32_t V, CsHost* out) {
  if (V != 1 && V != 2 && V != 4) return set_error(SYMM_ERR_ARG, "lanes per row %d (1, 2 or 4)", V);
  const int32_t R = 32 / V;  // rows per slice
  const int32_t* rp = S.prow_ptr.data();
  const int32_t* pc = S.pcol.data();
  const double* pv = S.pval.data();
  if (chunk_bytes < 8192 || (chunk_bytes & 15) || chunk_bytes >= (1 << 20))
    return set_error(SYMM_ERR_ARG, "chunk bytes %d", chunk_bytes);
  if (stages < 3) return set_error(SYMM_ERR_ARG, "ring stages %d", stages);
  // a colour's pieces must fit the ring at once: <= stages - 2 chunks of data
  // (so it spans at most stages - 1 chunks)
  const int64_t colour_cap = (int64_t)(stages - 2) * chunk_bytes;
  // ---- merge schedule tiles of one level group -----------------------------
  std::vector<int32_t> cut{S.tile_ptr[(size_t)t_begin]};
  {
    std::vector<int32_t> tg, nt, merged;
    int32_t r0 = S.tile_ptr[(size_t)t_begin], r1 = r0, grp = -1;
    auto extend = [&](int32_t e) {  // targets of [r0, e) from the targets of [r0, r1)
      nt.clear();
      for (int32_t r = r1; r < e; ++r)
        for (int32_t i = rp[r]; i < rp[r + 1]; ++i)
          if (pc[i] >= e) nt.push_back(pc[i]);
      std::sort(nt.begin(), nt.end());
      nt.erase(std::unique(nt.begin(), nt.end()), nt.end());
      merged.clear();
      auto it = std::lower_bound(tg.begin(), tg.end(), e);
      std::set_union(it, tg.end(), nt.begin(), nt.end(), std::back_inserter(merged));
    };
    for (int32_t t = t_begin; t < t_end; ++t) {
      const int32_t e = S.tile_ptr[(size_t)t + 1];
      const int32_t g = S.tile_group[(size_t)t];
      if (r1 > r0 && g == grp) {
        extend(e);
        const int64_t W = (int64_t)(e - r0) + (int64_t)merged.size();
        const int64_t nnz = rp[e] - rp[r0];
        if (W <= wcap && nnz <= nnzcap) {
          tg.swap(merged);
          r1 = e;
          continue;
        }
      }
      if (r1 > r0) cut.push_back(r1);  // close [r0, r1), start a new tile at r1
      r0 = r1;
      grp = g;
      tg.clear();
      extend(e);
      tg.swap(merged);
      r1 = e;
    }
    if (r1 > r0) cut.push_back(r1);
  }
  const int32_t nt = (int32_t)cut.size() - 1;
  // ---- per tile: targets, colours, slices, pieces, chunks -----------------
  struct TileTmp {
    std::vector<int32_t> tgt, cslc;
    std::vector<CsSliceRec> srec;
    std::vector<uint32_t> ploc;
    std::vector<int64_t> chunk_bytes, chunk_start;
    std::vector<unsigned char> data;  // the tile's chunks, concatenated
    int64_t nnz = 0, conflicts = 0, steps = 0;
    int32_t maxspan = 1;
  };
  std::vector<TileTmp> tmp((size_t)nt);
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 2) reduction(| : bad)
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t r0 = cut[(size_t)t], r1 = cut[(size_t)t + 1], T = r1 - r0;
    TileTmp& X = tmp[(size_t)t];
    for (int32_t r = r0; r < r1; ++r)
      for (int32_t i = rp[r]; i < rp[r + 1]; ++i)
        if (pc[i] >= r1) X.tgt.push_back(pc[i]);
    std::sort(X.tgt.begin(), X.tgt.end());
    X.tgt.erase(std::unique(X.tgt.begin(), X.tgt.end()), X.tgt.end());
    if ((int64_t)T + (int64_t)X.tgt.size() > 65535) {  // u16 window ids
      bad |= 1;
      continue;
    }
    auto local = [&](int32_t c) -> int32_t {
      if (c < r1) return c - r0;
      return T + (int32_t)(std::lower_bound(X.tgt.begin(), X.tgt.end(), c) - X.tgt.begin());
    };
    auto has_diag = [&](int32_t r) { return rp[r] < rp[r + 1] && pc[rp[r]] == r; };
    auto offd = [&](int32_t r) { return rp[r + 1] - rp[r] - (has_diag(r) ? 1 : 0); };
    std::vector<int32_t> color;
    const int32_t nc0 = color_rows_writeset(rp, pc, r0, r1, X.tgt, color);
    // slot order: colour, then off-diagonal length descending, then row
    std::vector<int32_t> rows((size_t)T);
    for (int32_t i = 0; i < T; ++i) rows[(size_t)i] = r0 + i;
    std::stable_sort(rows.begin(), rows.end(), [&](int32_t a, int32_t b) {
      const int32_t ca = color[(size_t)(a - r0)], cb = color[(size_t)(b - r0)];
      if (ca != cb) return ca < cb;
      return offd(a) > offd(b);
    });
    // slices of <= R slots inside a colour; a colour is split before a slice
    // that would push its bytes past colour_cap
    std::vector<int32_t> sl_begin, sl_end;
    X.cslc.push_back(0);
    {
      int32_t p = 0;
      for (int32_t c = 0; c < nc0; ++c) {
        int32_t q = p;
        while (q < T && color[(size_t)(rows[(size_t)q] - r0)] == c) ++q;
        int64_t acc = 0;
        for (int32_t s0 = p; s0 < q; s0 += R) {
          const int32_t s1 = std::min(s0 + R, q);
          int64_t b = kSliceMeta;
          for (int32_t u = s0; u < s1; ++u) b += 10 * (int64_t)offd(rows[(size_t)u]);
          b += 48 * (1 + offd(rows[(size_t)s0]) / (V * kPieceSteps));
          if (acc > 0 && acc + b > colour_cap) {
            X.cslc.push_back((int32_t)sl_begin.size());  // split the colour here
            acc = 0;
          }
          acc += b;
          sl_begin.push_back(s0);
          sl_end.push_back(s1);
        }
        if ((int32_t)sl_begin.size() > X.cslc.back()) X.cslc.push_back((int32_t)sl_begin.size());
        p = q;
      }
    }
    const int32_t ns = (int32_t)sl_begin.size();
    // pieces and chunks
    X.chunk_start.push_back(0);
    int64_t cur = 0;
    auto open_piece = [&](int64_t bytes) -> uint32_t {
      if (cur + bytes > chunk_bytes) {
        X.chunk_bytes.push_back(cur);
        X.chunk_start.push_back((int64_t)X.data.size());
        cur = 0;
      }
      const uint32_t loc = ((uint32_t)(X.chunk_start.size() - 1) << 20) | (uint32_t)cur;
      cur += bytes;
      return loc;
    };
    std::vector<std::vector<Ent>> ent;
    for (int32_t s = 0; s < ns; ++s) {
      const int32_t p = sl_begin[(size_t)s], q = sl_end[(size_t)s], m = q - p;
      ent.assign((size_t)m, {});
      int32_t maxlen = 0;
      for (int32_t u = p; u < q; ++u) {
        const int32_t r = rows[(size_t)u];
        auto& e = ent[(size_t)(u - p)];
        for (int32_t i = rp[r] + (has_diag(r) ? 1 : 0); i < rp[r + 1]; ++i) e.push_back({(uint16_t)local(pc[i]), pv[i]});
        maxlen = std::max(maxlen, (int32_t)e.size());
      }
      X.conflicts += bank_order(ent, V);
      const int32_t nsteps = (maxlen + V - 1) / V;
      X.steps += 2 * nsteps;
      // lane (i, sub) holds entry t * V + sub of row i at step t
      auto valid = [&](int32_t ln, int32_t t) {
        const int32_t i = ln / V, sub = ln % V;
        return i < m && (int32_t)ent[(size_t)i].size() > t * V + sub;
      };
      const int32_t npc = std::max(1, (nsteps + kPieceSteps - 1) / kPieceSteps);
      if (npc > 255 || nsteps >= 65536) bad |= 4;
      CsSliceRec Rc{};
      Rc.p0 = (uint16_t)X.ploc.size();
      Rc.npieces = (uint8_t)npc;
      Rc.nsteps = (uint16_t)nsteps;
      Rc.m = (uint8_t)m;
      for (int32_t k = 0; k < npc; ++k) {
        const int32_t j0 = k * kPieceSteps, j1 = std::min(nsteps, j0 + kPieceSteps);
        int64_t nnzp = 0;
        for (int32_t t = j0; t < j1; ++t)
          for (int32_t ln = 0; ln < 32; ++ln) nnzp += valid(ln, t) ? 1 : 0;
        const int64_t bytes = al16((k == 0 ? kSliceMeta : 32) + 10 * nnzp);
        const uint32_t loc = open_piece(bytes);
        if (k == 0) Rc.ploc0 = loc;
        X.ploc.push_back(loc);
        const size_t at = X.data.size();
        X.data.resize(at + (size_t)bytes, 0);
        unsigned char* b = X.data.data() + at;
        uint16_t* eo = reinterpret_cast<uint16_t*>(b);
        int64_t acc = 0;
        for (int32_t u = 0; u < kPieceSteps; ++u) {
          if (j0 + u < j1)
            for (int32_t ln = 0; ln < 32; ++ln) acc += valid(ln, j0 + u) ? 1 : 0;
          eo[u] = (uint16_t)acc;
        }
        b += 32;
        if (k == 0) {  // per lane: its row's window id, length, diagonal
          uint16_t* rid = reinterpret_cast<uint16_t*>(b);
          uint16_t* len = reinterpret_cast<uint16_t*>(b + 64);
          double* dg = reinterpret_cast<double*>(b + 128);
          for (int32_t ln = 0; ln < 32; ++ln) {
            const int32_t i = ln / V;
            if (i >= m) continue;
            const int32_t r = rows[(size_t)(p + i)];
            rid[ln] = (uint16_t)(r - r0);
            len[ln] = (uint16_t)std::min<int64_t>(offd(r), 65535);
            dg[ln] = has_diag(r) ? pv[rp[r]] : 0.0;
          }
          b += kSliceMeta - 32;
        }
        double* val = reinterpret_cast<double*>(b);
        uint16_t* lcol = reinterpret_cast<uint16_t*>(b + 8 * nnzp);
        int64_t e = 0;
        for (int32_t t = j0; t < j1; ++t)
          for (int32_t ln = 0; ln < 32; ++ln)
            if (valid(ln, t)) {
              const Ent& en = ent[(size_t)(ln / V)][(size_t)(t * V + ln % V)];
              val[e] = en.second;
              lcol[e] = en.first;
              ++e;
            }
        X.nnz += nnzp;
      }
      X.srec.push_back(Rc);
    }
    X.chunk_bytes.push_back(cur);
    if (X.ploc.size() >= 65535) bad |= 2;
    // ring requirement: chunks spanned by one colour
    for (int32_t c = 0; c + 1 < (int32_t)X.cslc.size(); ++c) {
      const int32_t s0 = X.cslc[(size_t)c], s1 = X.cslc[(size_t)c + 1] - 1;
      if (s1 < s0) continue;
      const uint32_t pl = X.ploc[(size_t)X.srec[(size_t)s1].p0 + X.srec[(size_t)s1].npieces - 1];
      X.maxspan = std::max<int32_t>(X.maxspan, (int32_t)(pl >> 20) - (int32_t)(X.srec[(size_t)s0].ploc0 >> 20) + 1);
    }
  }
  if (bad & 1) return set_error(SYMM_ERR_UNSUPPORTED, "colored_smem: a tile window exceeds 65535 entries");
  if (bad & 4) return set_error(SYMM_ERR_UNSUPPORTED, "colored_smem: a row has more than %d entries", 255 * kPieceSteps);
  if (bad) return set_error(SYMM_ERR_UNSUPPORTED, "colored_smem: a tile has too many pieces");
  // ---- offsets: head then chunks per tile ----------------------------------
  out->desc.assign((size_t)nt, CsDesc{});
  out->chunk_off.clear();
  out->chunk_len.clear();
  out->tile_chunk0.clear();
  int64_t off = 0;
  out->Wcap = out->Hcap = 16;
  out->nnz_offdiag = out->sum_colors = out->sum_spill = out->conflicts = out->steps = out->sum_slices = 0;
  out->max_colour_chunks = 1;
  for (int32_t t = 0; t < nt; ++t) {
    const TileTmp& X = tmp[(size_t)t];
    CsDesc& D = out->desc[(size_t)t];
    const int32_t T = cut[(size_t)t + 1] - cut[(size_t)t], S_ = (int32_t)X.tgt.size();
    D.row0 = cut[(size_t)t];
    D.T = T;
    D.S = S_;
    D.ncolors = (int32_t)X.cslc.size() - 1;
    D.nslices = (int32_t)X.srec.size();
    D.npieces = (int32_t)X.ploc.size();
    D.nchunks = (int32_t)X.chunk_bytes.size();
    int64_t o = al16((int64_t)sizeof(CsHeadHdr));
    D.o_cslc = (uint16_t)o; o = al16(o + 2 * (int64_t)(D.ncolors + 1));
    D.o_srec = (uint16_t)o; o = al16(o + (int64_t)sizeof(CsSliceRec) * D.nslices);
    D.o_ploc = (uint16_t)o; o = al16(o + 4 * (int64_t)D.npieces);
    D.o_pw = (uint16_t)o; o = al16(o + 2 * (int64_t)D.npieces);
    D.o_tgt = (uint16_t)o; o = al16(o + 4 * (int64_t)S_);
    D.o_clen = (uint16_t)o; o = al16(o + 4 * (int64_t)D.nchunks);
    if (o >= 65536) return set_error(SYMM_ERR_UNSUPPORTED, "colored_smem: tile %d head is %lld B (> 64 KB)", t, (long long)o);
    D.head_bytes = (int32_t)o;
    D.head_off = off;
    off += o;
    out->tile_chunk0.push_back((int32_t)out->chunk_off.size());
    for (size_t c = 0; c < X.chunk_bytes.size(); ++c) {
      out->chunk_off.push_back(off);
      out->chunk_len.push_back((int32_t)X.chunk_bytes[c]);
      off += X.chunk_bytes[c];
    }
    if (off - D.head_off >= ((int64_t)1 << 31)) return set_error(SYMM_ERR_UNSUPPORTED, "colored_smem: tile %d >= 2 GB", t);
    D.block_bytes = (int32_t)(off - D.head_off);
    out->Wcap = std::max(out->Wcap, T + S_);
    out->Hcap = std::max<int32_t>(out->Hcap, (int32_t)o);
    out->nnz_offdiag += X.nnz;
    out->sum_colors += D.ncolors;
    out->sum_slices += D.nslices;
    out->sum_spill += S_;
    out->conflicts += X.conflicts;
    out->steps += X.steps;
    out->max_colour_chunks = std::max(out->max_colour_chunks, X.maxspan);
  }
  out->blocks.assign((size_t)off, 0);
  // ---- fill ------------------------------------------------------------------
#pragma omp parallel for schedule(dynamic, 4)
  for (int32_t t = 0; t < nt; ++t) {
    const TileTmp& X = tmp[(size_t)t];
    const CsDesc& D = out->desc[(size_t)t];
    unsigned char* b = out->blocks.data() + D.head_off;
    CsHeadHdr H{};
    H.chunk_base = D.head_off + D.head_bytes;
    H.row0 = D.row0;
    H.T = D.T;
    H.S = D.S;
    H.ncolors = D.ncolors;
    H.nslices = D.nslices;
    H.npieces = D.npieces;
    H.nchunks = D.nchunks;
    H.o_cslc = D.o_cslc;
    H.o_srec = D.o_srec;
    H.o_ploc = D.o_ploc;
    H.o_pw = D.o_pw;
    H.o_tgt = D.o_tgt;
    H.o_clen = D.o_clen;
    std::memcpy(b, &H, sizeof H);
    uint16_t* cslc = reinterpret_cast<uint16_t*>(b + D.o_cslc);
    for (int32_t c = 0; c <= D.ncolors; ++c) cslc[c] = (uint16_t)X.cslc[(size_t)c];
    std::memcpy(b + D.o_srec, X.srec.data(), sizeof(CsSliceRec) * X.srec.size());
    uint32_t* ploc = reinterpret_cast<uint32_t*>(b + D.o_ploc);
    for (int32_t p = 0; p < D.npieces; ++p) ploc[p] = X.ploc[(size_t)p];
    uint16_t* pw = reinterpret_cast<uint16_t*>(b + D.o_pw);
    for (int32_t p = 0; p < D.npieces;) {  // pieces of one chunk are consecutive
      int32_t q = p;
      while (q < D.npieces && (X.ploc[(size_t)q] >> 20) == (X.ploc[(size_t)p] >> 20)) ++q;
      for (int32_t i = p; i < q; ++i) pw[i] = 1;
      pw[p] = (uint16_t)(kCsReleaseUnits - (q - p - 1));
      p = q;
    }
    int32_t* tgt = reinterpret_cast<int32_t*>(b + D.o_tgt);
    for (int32_t i = 0; i < D.S; ++i) tgt[i] = X.tgt[(size_t)i];
    uint32_t* clen = reinterpret_cast<uint32_t*>(b + D.o_clen);
    for (int32_t c = 0; c < D.nchunks; ++c) clen[c] = (uint32_t)X.chunk_bytes[(size_t)c];
    for (int32_t c = 0; c < D.nchunks; ++c)
      std::memcpy(out->blocks.data() + out->chunk_off[(size_t)out->tile_chunk0[(size_t)t] + c],
                  X.data.data() + X.chunk_start[(size_t)c], (size_t)X.chunk_bytes[(size_t)c]);
  }
  // ---- stamping validator: inside a colour every window id is written once --
  if (S.cfg.validate) {
    int bad_t = -1;
#pragma omp parallel for schedule(dynamic, 8) reduction(max : bad_t)
    for (int32_t t = 0; t < nt; ++t) {
      const CsDesc& D = out->desc[(size_t)t];
      const unsigned char* hb = out->blocks.data() + D.head_off;
      const uint16_t* cslc = reinterpret_cast<const uint16_t*>(hb + D.o_cslc);
      const CsSliceRec* srec = reinterpret_cast<const CsSliceRec*>(hb + D.o_srec);
      const uint32_t* ploc = reinterpret_cast<const uint32_t*>(hb + D.o_ploc);
      std::vector<int32_t> stamp((size_t)(D.T + D.S), -1);
      auto piece = [&](uint32_t loc) {
        return out->blocks.data() + out->chunk_off[(size_t)out->tile_chunk0[(size_t)t] + (loc >> 20)] + (loc & 0xfffff);
      };
      for (int32_t c = 0; c < D.ncolors; ++c)
        for (int32_t s = cslc[c]; s < cslc[c + 1]; ++s) {
          const CsSliceRec& R = srec[s];
          auto hit = [&](int32_t l) {
            if (l < 0 || l >= D.T + D.S || stamp[(size_t)l] == c) bad_t = std::max(bad_t, t);
            else stamp[(size_t)l] = c;
          };
          const unsigned char* b0 = piece(R.ploc0);
          const uint16_t* rid = reinterpret_cast<const uint16_t*>(b0 + 32);
          for (int32_t i = 0; i < R.m; ++i) hit(rid[i * V]);
          for (int32_t k = 0; k < R.npieces; ++k) {
            const unsigned char* b = piece(ploc[R.p0 + k]);
            const int32_t nnzp = reinterpret_cast<const uint16_t*>(b)[15];
            b += k == 0 ? kSliceMeta : 32;
            const uint16_t* lcol = reinterpret_cast<const uint16_t*>(b + 8 * nnzp);
            for (int32_t e = 0; e < nnzp; ++e) hit(lcol[e]);
          }
        }
    }
    if (bad_t >= 0) return set_error(SYMM_ERR_SCHEDULE, "validator: colored_smem tile %d colour not write-disjoint", bad_t);
  }
  return SYMM_OK;
}

}  // namespace symm
