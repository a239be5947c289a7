// psa_plan.cpp — deterministic work-item planner. Restated in oracle/plan.py;
// tests/test_plan.py checks the two produce byte-identical int32 tables.
#include "psa_plan.h"

#include <algorithm>
#include <array>
#include <numeric>
#include <utility>

#include "../../include/psa.h"

namespace psa {

namespace {

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

struct Chunking {
  int64_t chunk;
  // Split [0, L) into near-equal chunks of <= chunk keys, boundaries on kChunkAlign.
  int64_t per(int64_t L) const {
    int64_t n = ceil_div(L, chunk);
    return round_up(ceil_div(L, n), kChunkAlign);
  }
};

}  // namespace

int32_t dtype_bytes(int32_t dtype) {
  switch (dtype) {
    case PSA_DTYPE_F32: return 4;
    case PSA_DTYPE_BF16: return 2;
    case PSA_DTYPE_F16: return 2;
    case PSA_DTYPE_F64: return 8;
    default: return 0;
  }
}

std::string validate_offsets(const PlanInput& in) {
  if (in.G < 1) return "num_groups must be >= 1";
  if (in.R < 1) return "num_requests must be >= 1";
  if (in.Hkv < 1 || in.Hq < in.Hkv || in.Hq % in.Hkv != 0)
    return "num_q_heads must be a positive multiple of num_kv_heads";
  if (in.d < 1 || in.dv < 1) return "head dims must be positive";
  if (!in.cu_req || !in.cu_q || !in.cu_prefix || !in.cu_distinct)
    return "offset tables must not be NULL";
  if (in.cu_req[0] != 0 || in.cu_req[in.G] != in.R)
    return "cu_req must start at 0 and end at num_requests";
  if (in.cu_q[0] != 0 || in.cu_prefix[0] != 0 || in.cu_distinct[0] != 0)
    return "offset tables must start at 0";
  const int64_t kMax = (int64_t(1) << 31) - 1;
  const int64_t gqa = in.Hq / in.Hkv;
  for (int32_t g = 0; g < in.G; ++g) {
    if (in.cu_req[g + 1] <= in.cu_req[g]) return "group " + std::to_string(g) + " has no requests";
    int64_t P = in.cu_prefix[g + 1] - in.cu_prefix[g];
    if (P < 0) return "cu_prefix must be non-decreasing";
    if (P > kMax) return "prefix too long";
    int64_t t0 = in.cu_q[in.cu_req[g]], t1 = in.cu_q[in.cu_req[g + 1]];
    if ((t1 - t0) * gqa > kMax) return "too many stacked rows in one group";
    for (int64_t r = in.cu_req[g]; r < in.cu_req[g + 1]; ++r) {
      if (in.cu_q[r + 1] <= in.cu_q[r])
        return "queries[" + std::to_string(r) + "] must be a 2-D matrix with positive dimensions";
      int64_t D = in.cu_distinct[r + 1] - in.cu_distinct[r];
      if (D < 0) return "cu_distinct must be non-decreasing";
      if (D > kMax) return "distinct segment too long";
      if (P == 0 && D == 0) return "request has neither prefix nor distinct keys";
    }
  }
  if (in.cu_q[in.R] * in.Hq > kMax * 64) return "batch too large";
  return "";
}

bool tiles_supported(const PlanInput& in, const PlanOptions& opt) {
  if (opt.disable_tiles) return false;
  if (in.dtype != PSA_DTYPE_BF16 && in.dtype != PSA_DTYPE_F16) return false;
  if (!(in.d == 64 || in.d == 128) || in.dv != in.d) return false;
  return (in.Hq / in.Hkv) <= kTileM;
}

// Row segments of one group (identical for every kv head). A segment is a run of
// group rows evaluated against one key space: the prefix alone, or — with
// fuse_own, for a request whose own rows go to TILE items — [prefix ++ that
// request's distinct KV] in one online softmax (no merge between the two).
struct Segment {
  int64_t row0, rows;
  int64_t req;  // -1: prefix-only run; else the request whose distinct KV is appended
  int64_t P, D; // keys: P prefix keys, then D distinct keys of `req`
};

std::string build_plan(const PlanInput& in, const PlanOptions& opt, Plan* out) {
  std::string err = validate_offsets(in);
  if (!err.empty()) return err;
  const int64_t gqa = in.Hq / in.Hkv;
  const bool tiles = tiles_supported(in, opt);
  const int64_t tile_rows = tiles ? gqa * (kTileM / gqa) : 0;
  const int64_t item_rows = opt.tile_pair ? 2 * tile_rows : tile_rows;
  const int64_t elt = dtype_bytes(in.dtype);
  const int64_t width = int64_t(in.d) + in.dv;

  auto kind_for = [&](int64_t rows) -> int32_t {
    return (tiles && rows >= opt.tile_min_rows) ? kItemTile : kItemVec;
  };
  auto step_for = [&](int32_t kind) -> int64_t { return kind == kItemTile ? item_rows : kVecRows; };

  // 0. Segments per group, and the requests whose distinct KV runs as separate items.
  std::vector<std::vector<Segment>> segs(in.G);
  std::vector<std::vector<int64_t>> sep(in.G);  // requests with separate distinct items
  for (int32_t g = 0; g < in.G; ++g) {
    const int64_t tok0 = in.cu_q[in.cu_req[g]];
    const int64_t Ng = gqa * (in.cu_q[in.cu_req[g + 1]] - tok0);
    const int64_t P = in.cu_prefix[g + 1] - in.cu_prefix[g];
    if (!opt.fuse_own) {
      if (P > 0) segs[g].push_back({0, Ng, -1, P, 0});
      for (int64_t r = in.cu_req[g]; r < in.cu_req[g + 1]; ++r)
        if (in.cu_distinct[r + 1] > in.cu_distinct[r]) sep[g].push_back(r);
      continue;
    }
    int64_t run0 = -1;  // first row of the open prefix-only run
    for (int64_t r = in.cu_req[g]; r < in.cu_req[g + 1]; ++r) {
      const int64_t rb = gqa * (in.cu_q[r] - tok0), nr = gqa * (in.cu_q[r + 1] - in.cu_q[r]);
      const int64_t D = in.cu_distinct[r + 1] - in.cu_distinct[r];
      if (D > 0 && kind_for(nr) == kItemTile) {
        if (run0 >= 0 && P > 0) segs[g].push_back({run0, rb - run0, -1, P, 0});
        run0 = -1;
        segs[g].push_back({rb, nr, r, P, D});
      } else {
        if (run0 < 0) run0 = rb;
        if (D > 0) sep[g].push_back(r);
      }
    }
    if (run0 >= 0 && P > 0) segs[g].push_back({run0, Ng - run0, -1, P, 0});
  }

  // 1. Chunk sizes from the (row block x key) volume of each item kind.
  //    TILE items (CTA-level) aim at target_waves waves over all CTAs: every tile
  //    item writes a 128-row fp32 partial, so fewer, longer tiles are cheaper.
  //    VEC items (warp-level) aim at kVecWaves waves over all warps, capped at
  //    kVecMaxKeys keys so a long segment spreads over many warps.
  int64_t total_vec = 0;
  std::vector<std::pair<int64_t, int64_t>> tile_segs;  // (row blocks x Hkv, keys)
  for (int32_t g = 0; g < in.G; ++g) {
    for (const Segment& sg : segs[g]) {
      const int32_t k = kind_for(sg.rows);
      const int64_t blocks = ceil_div(sg.rows, step_for(k));
      if (k == kItemTile) tile_segs.emplace_back(blocks * in.Hkv, sg.P + sg.D);
      else total_vec += blocks * (sg.P + sg.D);
    }
    for (int64_t r : sep[g]) {
      const int64_t D = in.cu_distinct[r + 1] - in.cu_distinct[r];
      const int64_t nr = gqa * (in.cu_q[r + 1] - in.cu_q[r]);
      const int32_t k = kind_for(nr);
      const int64_t blocks = ceil_div(nr, step_for(k));
      if (k == kItemTile) tile_segs.emplace_back(blocks * in.Hkv, D);
      else total_vec += blocks * D;
    }
  }
  total_vec *= in.Hkv;
  const int64_t ctas = int64_t(std::max(1, opt.num_sms)) * std::max(1, opt.ctas_per_sm);
  // VEC queue consumers: warps of the legacy kernel, or the decode pipelines of the
  // v2 kernel (two per CTA) — sized so both see the same chunking.
  const int64_t vec_ctas = opt.tile_pair ? int64_t(std::max(1, opt.num_sms)) * 2 : ctas;
  // Tile chunk: the smallest multiple of kChunkAlign in [min, max] whose item count
  // fits target_waves waves of CTAs (binary search; item count is monotone).
  const int64_t tile_target = ctas * std::max(1, opt.target_waves);
  auto tile_items = [&](int64_t ck) {
    int64_t n = 0;
    for (const auto& sg : tile_segs) n += sg.first * ceil_div(sg.second, ck);
    return n;
  };
  int64_t lo = round_up(std::max<int64_t>(opt.min_chunk_keys, 1), kChunkAlign);
  int64_t hi = std::max(lo, round_up(std::max<int64_t>(opt.max_chunk_keys, 1), kChunkAlign));
  if (tile_items(lo) > tile_target) {
    while (lo < hi) {
      const int64_t mid = round_up((lo + hi) / 2, kChunkAlign);
      if (mid >= hi) break;
      if (tile_items(mid) <= tile_target) hi = mid; else lo = mid + kChunkAlign;
    }
    lo = tile_items(lo) <= tile_target ? lo : hi;
  }
  const int64_t chunk = lo;
  // consumers: every warp of the legacy kernel; the v2 kernel's decode pipelines
  // (two per CTA) each take whole items
  const int64_t vec_consumers = opt.tile_pair ? vec_ctas * kVecWaves : vec_ctas * kVecWarps * kVecWaves;
  int64_t vchunk = ceil_div(total_vec, vec_consumers);
  vchunk = std::min<int64_t>(std::max<int64_t>(vchunk, kChunkAlign), kVecMaxKeys);
  vchunk = round_up(vchunk, kChunkAlign);
  const Chunking ck{chunk};
  const Chunking ckv{vchunk};
  out->chunk_keys = int32_t(chunk);

  // 2. Canonical items and merge units.
  using Rec = std::array<int32_t, kItemWords>;
  std::vector<Rec> items;
  std::vector<std::array<int32_t, kUnitWords>> units;
  std::vector<std::vector<int32_t>> unit_items;

  for (int32_t g = 0; g < in.G; ++g) {
    const int64_t tok0 = in.cu_q[in.cu_req[g]];
    const int64_t Ng = gqa * (in.cu_q[in.cu_req[g + 1]] - tok0);
    for (int32_t h = 0; h < in.Hkv; ++h) {
      const size_t first = items.size();
      auto push = [&](int32_t kind, int64_t row0, int64_t rows, int64_t req, int64_t pk0,
                      int64_t pk1, int64_t dk0, int64_t dk1) {
        Rec it{};
        it[kItKind] = kind; it[kItGroup] = g; it[kItHead] = h;
        it[kItRow0] = int32_t(row0); it[kItRows] = int32_t(rows);
        it[kItRequest] = int32_t(req);
        it[kItPk0] = int32_t(pk0); it[kItPk1] = int32_t(pk1);
        it[kItDk0] = int32_t(dk0); it[kItDk1] = int32_t(dk1);
        it[kItWsRow] = -1;
        it[kItCanon] = int32_t(items.size());
        items.push_back(it);
      };
      for (const Segment& sg : segs[g]) {
        const int32_t kind = kind_for(sg.rows);
        const int64_t L = sg.P + sg.D;
        const int64_t step = step_for(kind), per = (kind == kItemTile ? ck : ckv).per(L);
        for (int64_t o = 0; o < sg.rows; o += step)
          for (int64_t k0 = 0; k0 < L; k0 += per) {
            const int64_t k1 = std::min(L, k0 + per);
            push(kind, sg.row0 + o, std::min(step, sg.rows - o), sg.req, std::min(k0, sg.P),
                 std::min(k1, sg.P), std::max<int64_t>(k0 - sg.P, 0),
                 std::max<int64_t>(k1 - sg.P, 0));
          }
      }
      for (int64_t r : sep[g]) {
        const int64_t D = in.cu_distinct[r + 1] - in.cu_distinct[r];
        const int64_t rb = gqa * (in.cu_q[r] - tok0), nr = gqa * (in.cu_q[r + 1] - in.cu_q[r]);
        const int32_t kind = kind_for(nr);
        const int64_t step = step_for(kind), per = (kind == kItemTile ? ck : ckv).per(D);
        for (int64_t o = 0; o < nr; o += step)
          for (int64_t k0 = 0; k0 < D; k0 += per)
            push(kind, rb + o, std::min(step, nr - o), r, 0, 0, k0, std::min(D, k0 + per));
      }
      // Merge units: intervals between item boundaries and request boundaries.
      std::vector<int64_t> cuts{0, Ng};
      for (size_t i = first; i < items.size(); ++i) {
        cuts.push_back(items[i][kItRow0]);
        cuts.push_back(int64_t(items[i][kItRow0]) + items[i][kItRows]);
        // paired tiles: each 128-row slot arrives at its own units
        if (items[i][kItKind] == kItemTile && items[i][kItRows] > tile_rows)
          cuts.push_back(int64_t(items[i][kItRow0]) + tile_rows);
      }
      for (int64_t r = in.cu_req[g]; r < in.cu_req[g + 1]; ++r) cuts.push_back(gqa * (in.cu_q[r] - tok0));
      std::sort(cuts.begin(), cuts.end());
      cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
      const int32_t ubase = int32_t(units.size());
      for (size_t u = 0; u + 1 < cuts.size(); ++u) {
        std::array<int32_t, kUnitWords> rec{};
        rec[kUnGroup] = g; rec[kUnHead] = h;
        rec[kUnRow0] = int32_t(cuts[u]); rec[kUnRows] = int32_t(cuts[u + 1] - cuts[u]);
        units.push_back(rec);
        unit_items.emplace_back();
      }
      for (size_t i = first; i < items.size(); ++i) {
        const int64_t a = items[i][kItRow0], b = a + items[i][kItRows];
        const int32_t u0 = int32_t(std::lower_bound(cuts.begin(), cuts.end(), a) - cuts.begin());
        const int32_t u1 = int32_t(std::lower_bound(cuts.begin(), cuts.end(), b) - cuts.begin());
        items[i][kItUnit0] = ubase + u0;
        items[i][kItUnit1] = ubase + u1;
        for (int32_t u = u0; u < u1; ++u) unit_items[ubase + u].push_back(int32_t(i));
      }
      for (size_t u = ubase; u < units.size(); ++u)
        if (unit_items[u].empty()) return "internal: merge unit without contributions";
    }
  }

  // 3. Direct items (sole contributor of every unit they cover) skip the workspace.
  int64_t ws = 0;
  for (auto& it : items) {
    bool direct = true;
    for (int32_t u = it[kItUnit0]; u < it[kItUnit1]; ++u)
      if (unit_items[u].size() != 1) { direct = false; break; }
    if (!direct) { it[kItWsRow] = int32_t(ws); ws += it[kItRows]; }
  }
  if (ws > (int64_t(1) << 31) - 1) return "workspace rows overflow";
  std::vector<int32_t> contribs;
  for (size_t u = 0; u < units.size(); ++u) {
    units[u][kUnContribBegin] = int32_t(contribs.size());
    units[u][kUnContribCount] = int32_t(unit_items[u].size());
    for (int32_t i : unit_items[u]) {
      const auto& it = items[i];
      contribs.push_back(it[kItWsRow] < 0 ? -1 : it[kItWsRow] + (units[u][kUnRow0] - it[kItRow0]));
    }
  }

  // Pair merges: an item that shares its single unit (spanning exactly its rows) with
  // one other item can merge that item's partial itself when it arrives last — the
  // decode pipeline's in-register merge; precomputed so the kernel needs one load.
  for (auto& it : items) {
    int64_t pair = -1;
    if (it[kItWsRow] >= 0 && it[kItUnit1] - it[kItUnit0] == 1) {
      const auto& u = units[it[kItUnit0]];
      if (u[kUnRow0] == it[kItRow0] && u[kUnRows] == it[kItRows] && u[kUnContribCount] == 2) {
        const int32_t c0 = contribs[u[kUnContribBegin]], c1 = contribs[u[kUnContribBegin] + 1];
        const bool first = c0 != it[kItWsRow];
        pair = int64_t(first ? c0 : c1) * 2 + (first ? 1 : 0);
        if (pair > INT32_MAX) pair = -1;
      }
    }
    it[kItPair] = int32_t(pair);
  }

  // 4. LPT queue order: cost descending; ties: tiles by canonical index, VEC items
  //    heads-fastest (below).
  std::vector<int64_t> cost(items.size());
  for (size_t i = 0; i < items.size(); ++i) {
    const auto& it = items[i];
    const int64_t keys = int64_t(it[kItPk1] - it[kItPk0]) + (it[kItDk1] - it[kItDk0]);
    const int64_t bytes = (keys + it[kItRows]) * width * elt;
    if (it[kItKind] == kItemTile) {
      const int64_t slots = ceil_div(it[kItRows], std::max<int64_t>(tile_rows, 1));
      cost[i] = std::max(bytes * kByteWeight, 2 * int64_t(kTileM) * slots * keys * width);
    } else {
      cost[i] = std::max(bytes * kByteWeight, 2 * round_up(it[kItRows], 4) * keys * width * kVecFlopWeight);
    }
  }
  // Queue order: TILE items first (CTA-level queue), then VEC items (warp-level
  // queue). TILE items go by (group, kv head) bundle — all tiles that read one
  // group's prefix for one head, in bundle-cost order (LPT over bundles), each
  // bundle's items by cost — so a group's prefix is streamed by tiles running at the
  // same time and re-read from L2, not DRAM (c3: a group's decode-row prefix tile no
  // longer waits behind every prefill tile of the batch). VEC items by cost.
  std::vector<int64_t> bundle(int64_t(in.G) * in.Hkv, 0);
  for (size_t i = 0; i < items.size(); ++i)
    if (items[i][kItKind] == kItemTile)
      bundle[int64_t(items[i][kItGroup]) * in.Hkv + items[i][kItHead]] += cost[i];
  std::vector<int32_t> order(items.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    const bool ta = items[a][kItKind] == kItemTile, tb = items[b][kItKind] == kItemTile;
    if (ta != tb) return ta;
    if (ta) {
      const int64_t ka = int64_t(items[a][kItGroup]) * in.Hkv + items[a][kItHead];
      const int64_t kb = int64_t(items[b][kItGroup]) * in.Hkv + items[b][kItHead];
      if (bundle[ka] != bundle[kb]) return bundle[ka] > bundle[kb];
      if (ka != kb) return ka < kb;
      return cost[a] > cost[b];
    }
    if (cost[a] != cost[b]) return cost[a] > cost[b];
    // equal-cost VEC items: the kv heads of one (request, key chunk) side by side, so
    // the pipelines running at the same time read whole token rows of the cache
    const auto& x = items[a];
    const auto& y = items[b];
    const std::array<int32_t, 6> kx{x[kItGroup], x[kItRequest], x[kItRow0], x[kItPk0], x[kItDk0], x[kItHead]};
    const std::array<int32_t, 6> ky{y[kItGroup], y[kItRequest], y[kItRow0], y[kItPk0], y[kItDk0], y[kItHead]};
    return kx < ky;
  });
  out->tile_cost = out->total_cost = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    out->total_cost += cost[i];
    if (items[i][kItKind] == kItemTile) out->tile_cost += cost[i];
  }

  out->items.clear();
  out->items.reserve(items.size() * kItemWords);
  out->num_tile_items = 0;
  for (int32_t i : order) {
    out->items.insert(out->items.end(), items[i].begin(), items[i].end());
    out->num_tile_items += items[i][kItKind] == kItemTile;
  }
  out->units.clear();
  for (auto& u : units) out->units.insert(out->units.end(), u.begin(), u.end());
  out->contribs = std::move(contribs);
  out->num_items = int32_t(items.size());
  out->num_units = int32_t(units.size());
  out->workspace_rows = ws;
  out->tile_ctas = out->num_tile_items > 0 ? int32_t(ctas) : 0;
  out->max_vec_rows = 0;
  out->vec_fan_in = 0;
  for (const auto& it : items) {
    if (it[kItKind] != kItemVec) continue;
    out->max_vec_rows = std::max(out->max_vec_rows, it[kItRows]);
    for (int32_t u = it[kItUnit0]; u < it[kItUnit1]; ++u)
      out->vec_fan_in = std::max(out->vec_fan_in, int32_t(unit_items[u].size()));
  }
  return "";
}

void group_costs(const PlanInput& in, int64_t* cost) {
  const int64_t elt = dtype_bytes(in.dtype), width = int64_t(in.d) + in.dv;
  for (int32_t g = 0; g < in.G; ++g) {
    const int64_t P = in.cu_prefix[g + 1] - in.cu_prefix[g];
    int64_t keys = P, tokens = 0, pairs = 0;
    for (int64_t r = in.cu_req[g]; r < in.cu_req[g + 1]; ++r) {
      const int64_t n = in.cu_q[r + 1] - in.cu_q[r];
      const int64_t D = in.cu_distinct[r + 1] - in.cu_distinct[r];
      keys += D;
      tokens += n;
      pairs += n * (P + D);
    }
    const int64_t bytes = in.Hkv * keys * width * elt + tokens * in.Hq * width * elt;
    const int64_t flops = 2 * int64_t(in.Hq) * pairs * width;
    cost[g] = std::max(bytes * kRidge, flops);
  }
}

void shard_groups(int32_t G, const int64_t* cost, int32_t world, int32_t* owner) {
  std::vector<int32_t> order(G);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return cost[a] > cost[b]; });
  std::vector<int64_t> load(world, 0);
  for (int32_t g : order) {
    int32_t best = 0;
    for (int32_t w = 1; w < world; ++w)
      if (load[w] < load[best]) best = w;
    owner[g] = best;
    load[best] += cost[g];
  }
}

}  // namespace psa
