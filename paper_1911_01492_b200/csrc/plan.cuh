// Symbolic plans for SPAI(1) assembly.
//
// The local least-squares problem of column k depends on the pattern only
// through the *relative* row offsets of the gathered CSC lists (rows - k).
// Columns with identical relative structure (every interior column of a
// structured FEM matrix, and each of the boundary classes) therefore share
// all index work: I_k, local ranks, the sparse overlap structure of
// G = (A^T A)[J,J] and the position of e_k.  A plan stores that once:
//   - jrel[a] = J_a - k, jcls[a] = class of column J_a  (exact match key)
//   - loff[nj+1], listid[e] (list of entry e; byte listid_pos(e): each group
//     of 128 entries is stored lane-interleaved, so lane L's 32-bit word holds
//     entries L, L+32, L+64, L+96 of the group)
//   - rhsidx[a]                          (entry holding A[k, J_a], or -1)
//   - product program in "rounds": the G entries with a nonzero overlap are
//     sorted by overlap length and dealt 32 per round (one per lane); round r
//     runs rlen[r] steps (rounded up to even), step t of lane l is ops[t*32 + l] = the byte
//     offsets of its two factors in the value list (lo | hi << 16), shorter
//     entries padded with 0 * 0 from the zero slot, and ends with one store
//     G[rdst[r][l]] -- no per-step bookkeeping.
// The numeric kernel then only gathers values, replays the product program
// and factors G -- no hashing, sorting or searching per column.  Exact
// A column's structure is fixed exactly by J_k's relative offsets and the
// *class* of every J member, where the class of a CSC column is its exact
// relative row pattern (de-duplicated with full comparison, class_kernel).
// The replay verifies (jrel, jcls) exactly, so a column can only use a plan
// built from a column with identical relative structure; a mismatch sends it
// to the direct path.
#pragma once
#include "common.cuh"

namespace spai {

constexpr int kPlanNJ = 32;          // max |J_k| on the plan path
constexpr int kPlanCap = 1024;       // max gathered entries per column
constexpr int kPlanSteps = 192;      // max product-program length per lane
constexpr int kPlanTable = 8192;     // signature hash-table slots (power of 2)
constexpr int kMaxPlans = 2048;
constexpr int kPadIdx = 1023;        // max entries+1 on the plan path (pad ops read slot `total`)

// plan layout in 32-bit words
constexpr int kPH_nj = 0, kPH_total = 1, kPH_nsteps = 2, kPH_nrounds = 3;
constexpr int kMaxRounds = (kPlanNJ * (kPlanNJ + 1) / 2 + 31) / 32;   // 17
constexpr int kPO_loff = 4;
constexpr int kPO_rhs = kPO_loff + kPlanNJ + 1;
constexpr int kPO_listid = kPO_rhs + kPlanNJ;                 // uint8, packed
constexpr int kPO_jrel = kPO_listid + kPlanCap / 4;
constexpr int kPO_jcls = kPO_jrel + kPlanNJ;
constexpr int kPO_rlen = kPO_jcls + kPlanNJ;                  // [kMaxRounds]
constexpr int kPO_rdst = kPO_rlen + kMaxRounds + 1;           // uint16 [kMaxRounds][32]
constexpr int kPO_ops = (kPO_rdst + kMaxRounds * 16 + 31) & ~31;   // 128-B aligned (8-byte op pairs)
constexpr int kClassTable = 8192;    // column-class hash table (exact de-dup)
// the op program is padded to whole groups of kOpGroupSteps steps (0 * 0 from
// the zero slot) and followed by one more group of slack, so the replay reads
// whole groups and prefetches one group ahead without bounds checks
#ifndef SPAI_OP_GROUP_STEPS
#define SPAI_OP_GROUP_STEPS 8
#endif
constexpr int kOpGroupSteps = SPAI_OP_GROUP_STEPS;
constexpr int kPlanWords = ((kPO_ops + 32 * (kPlanSteps + kOpGroupSteps)) + 31) & ~31;

// steps t and t + 1 of a lane are adjacent words (one 8-byte load per pair)
__host__ __device__ __forceinline__ int op_index(int t, int lane) {
  return (t >> 1) * 64 + lane * 2 + (t & 1);
}

__host__ __device__ __forceinline__ int listid_pos(int e) {
  return (e & ~127) | ((e & 31) << 2) | ((e >> 5) & 3);
}

__device__ __forceinline__ uint32_t op_pack(int ea, int eb) {   // byte offsets of two doubles
  return (uint32_t)(ea * 8) | ((uint32_t)(eb * 8) << 16);
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct PlanWs {
  unsigned long long* keys;   // [kPlanTable]  0 = empty
  int32_t* rep;               // [kPlanTable]  representative column
  int32_t* slot_plan;         // [kPlanTable]  plan index of a slot (-1 invalid)
  int32_t* plan_slot;         // [n]           table slot of each column (-1 = direct)
  unsigned long long* ckeys;  // [kClassTable] column-class hashes
  int32_t* crep;              // [kClassTable] representative column (-1 until published)
  int32_t* col_class;         // [n]           class of every column (-1 = none)
  int* nclass;                // distinct classes
  int64_t ntot;               // columns of the matrix (class kernel range)
  int* nplans;                // distinct signatures
  int* nbuilt;                // plans built
  uint32_t* plans;            // [kMaxPlans * kPlanWords]
};

}  // namespace spai
