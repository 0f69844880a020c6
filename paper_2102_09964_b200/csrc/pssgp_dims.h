// pssgp_dims.h — state dimensions compiled for the warp-per-chain path (posterior: d >= 4; the
// general-model NLL gradient: every d, including d <= 3 models other than one Matern component).  One object per
// entry is built from pssgp_wide_inst.cu (-DPSSGP_WD=d; _native.build() reads this list).
#pragma once
#define PSSGP_WIDE_DIMS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) X(18) X(19) X(20)
