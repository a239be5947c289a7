// psa_plan.h — deterministic work-item planner (host, pure C++).
//
// Turns the packed batch's offset tables into the int32 tables the persistent
// kernel consumes. Restated bit-exactly in oracle/plan.py; see DESIGN.md §3.
//
// Row space: for group g and kv head h the "group rows" are the stacked query
// rows of the reference's prefix call (attention.py:174): row i of group g is
// token tok0(g) + i / gqa, query head h*gqa + i % gqa. Request r owns the row
// range [gqa*(cu_q[r]-tok0(g)), gqa*(cu_q[r+1]-tok0(g))) — the implicit row
// cursor of attention.py:182-200.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace psa {

enum ItemKind : int32_t { kItemVec = 0, kItemTile = 1 };

// Item record layout (int32 words).
enum ItemField : int {
  kItKind = 0, kItGroup, kItHead, kItRow0, kItRows, kItRequest,
  kItPk0, kItPk1, kItDk0, kItDk1, kItUnit0, kItUnit1, kItWsRow, kItCanon,
  kItPair,  // one of exactly two contributors of one unit spanning its rows: the other
            // contribution's workspace row * 2 + (it comes first); else -1
  kItReserved1, kItemWords
};
// Merge-unit record layout (int32 words).
enum UnitField : int {
  kUnGroup = 0, kUnHead, kUnRow0, kUnRows, kUnContribBegin, kUnContribCount,
  kUnReserved0, kUnReserved1, kUnitWords
};

constexpr int32_t kTileM = 128;        // tcgen05 M (rows per tile)
constexpr int32_t kVecRows = 8;        // rows per CUDA-core item
constexpr int32_t kChunkAlign = 64;    // KV chunk boundaries align to 64 keys
constexpr int64_t kVecMaxKeys = 512;   // warp-level VEC items: at most 512 keys each
constexpr int64_t kVecWarps = 8;       // warps per CTA that pull VEC items
constexpr int64_t kVecWaves = 2;       // VEC items per warp the chunking aims at
constexpr int64_t kByteWeight = 356;   // ~ (tensor FLOP/clk/SM) / (HBM B/clk/SM)
constexpr int64_t kVecFlopWeight = 32; // tensor / CUDA-core FLOP rate per SM
constexpr int64_t kRidge = 257;        // measured B200 ridge (FLOP/B) for group costs

struct PlanInput {
  int32_t G = 0, R = 0, Hq = 0, Hkv = 0, d = 0, dv = 0, dtype = 0;
  const int64_t* cu_req = nullptr;
  const int64_t* cu_q = nullptr;
  const int64_t* cu_prefix = nullptr;
  const int64_t* cu_distinct = nullptr;
};

struct PlanOptions {
  int32_t num_sms = 148;
  int32_t ctas_per_sm = 2;
  int32_t tile_min_rows = 32;
  int32_t disable_tiles = 0;
  int32_t min_chunk_keys = 512;
  int32_t max_chunk_keys = 16384;
  int32_t target_waves = 1;
  // v2 kernel (1 CTA/SM, two 128-row softmax slots sharing each K/V block):
  int32_t tile_pair = 0;  // TILE items cover up to 2 x tile_rows rows (slot 0 + slot 1)
  int32_t fuse_own = 0;   // a multi-token request's tiles run [prefix ++ own distinct] in one item
};

struct Plan {
  std::vector<int32_t> items;     // queue order (cost desc, canonical asc)
  std::vector<int32_t> units;
  std::vector<int32_t> contribs;
  int32_t num_items = 0, num_units = 0, num_tile_items = 0;
  int64_t workspace_rows = 0;
  int32_t chunk_keys = 0;
  int64_t tile_cost = 0, total_cost = 0;  // LPT cost model totals (host heuristics only)
  int32_t tile_ctas = 0;  // v2: CTAs that start on the TILE queue (the rest on decode)
  int32_t max_vec_rows = 0;  // rows of the largest VEC item
  int32_t vec_fan_in = 0;    // most contributions of a merge unit a VEC item shares
};

// Returns "" on success, else the validation message (maps to PSA_INVALID_ARGUMENT).
std::string validate_offsets(const PlanInput& in);
bool tiles_supported(const PlanInput& in, const PlanOptions& opt);
std::string build_plan(const PlanInput& in, const PlanOptions& opt, Plan* out);
void group_costs(const PlanInput& in, int64_t* cost);
void shard_groups(int32_t G, const int64_t* cost, int32_t world, int32_t* owner);
int32_t dtype_bytes(int32_t dtype);

}  // namespace psa
