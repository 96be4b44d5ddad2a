// L-BFGS / Armijo on articulated trees (LbfgsSolver, reference
// src/optim.cpp:141-232): the k_tree_lbfgs kernel of pbad_tree.cu, built as
// a separate translation unit.  Sharing one TU with k_tree_step changed
// ptxas's register allocation for the LM kernel (252 -> 168 registers with
// spills, C4 +14 %), so each kernel gets its own.
#define PBAD_TREE_LBFGS_TU 1
#include "pbad_tree.cu"
