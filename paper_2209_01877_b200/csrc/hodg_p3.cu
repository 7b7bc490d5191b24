// Order-3 instantiation of the tetrahedral DG kernels (generated layout; see hodg_kernels.cuh)
#include "tables_p3.cuh"
#define ORDER 3
#define NB NB_P3
#define NQV NQV_P3
#define NQF NQF_P3
#define VB_D VB_P3_d
#define VB_F VB_P3_f
#define VB_FX VB_P3_fx
#define VD_D VD_P3_d
#define VD_F VD_P3_f
#define VD_FX VD_P3_fx
#define FB_D FB_P3_d
#define FB_F FB_P3_f
#define FG_D FG_P3_d
#define FG_F FG_P3_f
#define FG_FX FG_P3_fx
#define WV_D WV_P3_d
#define WV_F WV_P3_f
#define WV_FX WV_P3_fx
#define FBG_D FBG_P3_d
#define FBG_F FBG_P3_f
#define MINV_T MINV_P3
#define MEAN_T MEAN_P3
#include "hodg_kernels.cuh"
