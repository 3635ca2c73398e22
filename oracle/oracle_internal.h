/* oracle_internal.h -- oracle-private structures (TEST INFRASTRUCTURE ONLY, see oracle.h) */
#ifndef FC_ORACLE_INTERNAL_H
#define FC_ORACLE_INTERNAL_H
#include <stdint.h>

struct orc_forest {
  int64_t P;
  int T, m, lmax;
  int8_t* level;
  int32_t* tree;
  int64_t *x, *y;        /* leaf origin in units of level-Lmax leaves */
  uint64_t* start;       /* Morton start of the leaf in the 4^Lmax index space of its tree */
  int64_t* tree_first;   /* [T+1] */
  int32_t* t2t;
  int8_t *t2f, *bc;
  int32_t* table;        /* lazily built [P][G][8] ghost records */
};

const int32_t* orc_cached_table(const orc_forest* f, int* rc);
/* first solver error since the last call (physical-state guard of orc_step_patch), then clear */
int orc_take_step_error(void);

/* padded index of 1-based cell (i, j), i, j in [-1, m+2], in an n x n array (x fastest) */
#define ORC_N(m) ((m) + 4)
#define ORC_IDX(m, i, j) (((j) + 1) * ORC_N(m) + ((i) + 1))

#endif
