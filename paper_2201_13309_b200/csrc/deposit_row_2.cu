// deposit_row_2.cu -- instance set 2 of the row kernel (deposit_row.cu, end of file): compiled
// as its own translation unit so that the four instance sets build in parallel.
#define DAXM_ROW_TU 2
#include "deposit_row.cu"
