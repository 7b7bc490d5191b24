// Order-1 instantiation of the tetrahedral DG kernels (generated layout; see hodg_kernels.cuh)
#include "tables_p1.cuh"
#define ORDER 1
#define NB NB_P1
#define NQV NQV_P1
#define NQF NQF_P1
#define VB_D VB_P1_d
#define VB_F VB_P1_f
#define VB_FX VB_P1_fx
#define VD_D VD_P1_d
#define VD_F VD_P1_f
#define VD_FX VD_P1_fx
#define FB_D FB_P1_d
#define FB_F FB_P1_f
#define FG_D FG_P1_d
#define FG_F FG_P1_f
#define FG_FX FG_P1_fx
#define WV_D WV_P1_d
#define WV_F WV_P1_f
#define WV_FX WV_P1_fx
#define FBG_D FBG_P1_d
#define FBG_F FBG_P1_f
#define MINV_T MINV_P1
#define MEAN_T MEAN_P1
#include "hodg_kernels.cuh"
