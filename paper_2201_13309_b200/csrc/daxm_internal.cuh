// daxm_internal.cuh -- internal data layout shared by the plan (pre-pass) and
// the deposit kernels.  Not part of the ABI.  See DESIGN.md "Data layout".
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "daxm.h"

namespace daxm {

// Deposit tile: TILE_R detector rows x TILE_C detector columns.  Tiles are
// aligned to GLOBAL detector rows/cols, so a row-band plan reproduces the
// full-detector plan bit for bit (every per-tile reference is a function of
// the global tile only).
constexpr int TILE_R = 32;
constexpr int TILE_C = 32;
constexpr int TILE_E = TILE_C + 1;  // pixel edge columns per tile (finite pixels)
constexpr int NCOEF = 4;            // cubic depth model per edge point

// Geometry constants for the fp64 pre-pass (by value into kernels).
struct GeomConst {
    double rho[9];          // detector rotation (Rodrigues)
    double trans[3];        // det_trans
    double pitch_col, pitch_row;
    double axis[3];         // unit wire axis
    double beam[3];         // unit beam direction
    double origin[3];       // depth origin
    double w0[3];           // first wire centre
    double d[3];            // unit scan direction, perpendicular to the axis
    double r;               // wire radius
    double lo0;             // lower edge of bin 0 (um)
    double dz;              // bin width (um)
    int R, C, S, M;
    int edge;               // 0 leading, 1 trailing
    int point_mode;         // 1: POINT pixel model
    int m_ref;              // integer bin offset of the fp32 depth coordinate
};

// Per deposit tile (global tile index).
struct TileInfo {
    double t_ref;   // wire-travel reference (um) the cubic is expanded about
    int k_lo;       // first wire step (point) any pixel of the tile reads
    int k_hi;       // last wire step (point) any pixel of the tile reads (inclusive); k_hi < k_lo: empty
    int dir;        // +1: depth increases with the step index, -1: decreases
    int pad;
};

// Pre-pass failure flags (device word, read back by the host).
enum : unsigned {
    FLAG_NONMONOTONE = 1u,
    FLAG_NAN_IN_WINDOW = 2u,
    FLAG_MIXED_DIR = 4u,
    FLAG_FIT_NAN = 8u,
};

// Device-side plan view passed to the deposit kernels by value.
struct DepositArgs {
    const double* t;          // [S] wire travel t_k (um)
    const TileInfo* tiles;    // [n_tr][n_tc]
    const int2* win;          // [pre_rows][C] pair window [kb, ke) per pixel (global pixel indexing)
    const float* coef;        // [n_tiles][NCOEF][TILE_E][TILE_R]
    int R, C, S, M;
    int row_begin, row_end;   // band (global rows)
    int pre_row0;             // first global row of win[]
    int tr0, n_tr, n_tc;      // tile rows covered (global tile-row index tr0 ..)
    int m_ref;
    int point_mode;
    float sign;               // s: +1 leading, -1 trailing (reading R2)
};

// Launchers (deposit.cu).
cudaError_t launch_deposit(const DepositArgs& a, const void* stack, int dtype, float* out, cudaStream_t st);

}  // namespace daxm
