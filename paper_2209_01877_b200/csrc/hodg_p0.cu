// Order-0 instantiation of the tetrahedral DG kernels (generated layout; see hodg_kernels.cuh)
#include "tables_p0.cuh"
#define ORDER 0
#define NB NB_P0
#define NQV NQV_P0
#define NQF NQF_P0
#define VB_D VB_P0_d
#define VB_F VB_P0_f
#define VB_FX VB_P0_fx
#define VD_D VD_P0_d
#define VD_F VD_P0_f
#define VD_FX VD_P0_fx
#define FB_D FB_P0_d
#define FB_F FB_P0_f
#define FG_D FG_P0_d
#define FG_F FG_P0_f
#define FG_FX FG_P0_fx
#define WV_D WV_P0_d
#define WV_F WV_P0_f
#define WV_FX WV_P0_fx
#define FBG_D FBG_P0_d
#define FBG_F FBG_P0_f
#define MINV_T MINV_P0
#define MEAN_T MEAN_P0
#include "hodg_kernels.cuh"
