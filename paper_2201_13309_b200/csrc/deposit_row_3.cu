// deposit_row_3.cu -- instance set 3 of the row kernel (deposit_row.cu, end of file): compiled
// as its own translation unit so that the four instance sets build in parallel.
#define DAXM_ROW_TU 3
#include "deposit_row.cu"
