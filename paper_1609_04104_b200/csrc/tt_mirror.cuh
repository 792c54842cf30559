// Shared-memory plan of the mirrored rows kernel (tt_rows2.cu) and its entry points for tt_rows.cu's
// dispatcher (tt_track_rows).
#pragma once

#include "tt_common.cuh"

struct MirrorPlan {
  int CL, nJm, Rp, ysr, sblk, eblk, rs64, rs32;
  int o_ahf, o_bhl, o_bh64, o_u, o_ahs, o_wacc, o_zrecv, o_hrecv, o_ynrecv, o_gbrecv, o_gbfull, o_G, o_gaf, o_gbf,
      o_aown, o_vec, o_tab, o_colb, o_flags, o_rows, o_forced, o_usm, o_red, o_zown, o_eown;
  int smem;
};

// true (and the plan) when the mirrored kernel runs this launch at cluster size CL
bool tt_rows_mirror_plan(const tt_rows_args* a, int CL, MirrorPlan* pl);
int tt_rows_mirror_launch(void* stream, const tt_rows_args* a, const MirrorPlan& pl);
