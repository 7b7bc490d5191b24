// Order-2 instantiation of the tetrahedral DG kernels (generated layout; see hodg_kernels.cuh)
#include "tables_p2.cuh"
#define ORDER 2
#define NB NB_P2
#define NQV NQV_P2
#define NQF NQF_P2
#define VB_D VB_P2_d
#define VB_F VB_P2_f
#define VB_FX VB_P2_fx
#define VD_D VD_P2_d
#define VD_F VD_P2_f
#define VD_FX VD_P2_fx
#define FB_D FB_P2_d
#define FB_F FB_P2_f
#define FG_D FG_P2_d
#define FG_F FG_P2_f
#define FG_FX FG_P2_fx
#define WV_D WV_P2_d
#define WV_F WV_P2_f
#define WV_FX WV_P2_fx
#define FBG_D FBG_P2_d
#define FBG_F FBG_P2_f
#define MINV_T MINV_P2
#define MEAN_T MEAN_P2
#include "hodg_kernels.cuh"
