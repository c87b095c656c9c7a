// canon.h — host-side decode, validation and canonicalisation of predicate programs
// (SURVEY §8a row a2). Independent of the CPU oracle (oracle/oracle.c): shares no code.
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace sel {

struct Instr {
  uint8_t op, col;
  uint16_t a, b;
};

struct Program {
  std::vector<Instr> ins;
  std::vector<uint64_t> consts;
};

struct Interval {
  uint64_t lo, hi;  // inclusive, in the column's key space
};

struct PlanLeaf {
  int col;
  std::vector<Interval> iv;  // sorted, disjoint, non-adjacent, non-empty, not the full space
  int bitmap = -1;           // >= 0: an IN_BITMAP leaf on key set `bitmap` (iv unused)
  bool negate = false;       // IN_BITMAP leaf: NOT(v in set)
};

struct Plan {
  int path = 0;                 // Path (sel_internal.h)
  bool const_value = false;     // PATH_CONST: the predicate folded to TRUE or FALSE
  bool conj = false;            // PATH_CONJ: AND of leaves on distinct columns
  std::vector<PlanLeaf> leaves;
  std::vector<uint8_t> op;      // postfix DevOpcode
  std::vector<uint8_t> arg;     // leaf index for DOP_LEAF
  int max_depth = 0;
  size_t n_intervals = 0;
};

// Returns a sel_status (0 = OK); fills *out on success. `types` are sel_type codes.
int decode_program(const void* bytes, size_t len, const int* types, uint32_t ncols, Program* out,
                   std::string* msg);

// Canonicalises a decoded, validated program (see sel_internal.h). Always succeeds.
void plan_program(const Program& prog, const int* types, Plan* out);

// Key-space helpers, exported for the device-parameter packing in plan.cpp (host.h).
int key_bits(int type);
uint64_t key_sign_bias(int type);   // XOR applied to a key to get the raw lower bound

}  // namespace sel
