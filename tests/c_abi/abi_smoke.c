/* Plain-C client of include/spa.h (no Python, no torch): creates host-only rank groups and plans, checks
 * validation errors and the stage split / workspace / message descriptions of a PipeSP plan, and the
 * padding helper.  Built and run by tests/test_abi.py::test_plain_c_client (CPU only, no GPU calls). */
#include <stdio.h>
#include <stdint.h>
#include <string.h>

#include "spa.h"

#define CHECK(cond, msg)                                        \
    do {                                                        \
        if (!(cond)) {                                          \
            fprintf(stderr, "FAIL %s: %s\n", msg, spa_last_error()); \
            return 1;                                           \
        }                                                       \
    } while (0)

int main(void) {
    int pad = -1;
    CHECK(spa_pad_heads(24, 7, &pad) == 28 && pad == 4, "pad_heads 24/7");
    CHECK(strcmp(spa_status_string(SPA_ERR_BUSY), "SPA_ERR_BUSY") == 0, "status string");

    spa_comm *comm = NULL;
    CHECK(spa_comm_init_host(&comm, 8, 3) == SPA_OK, "host comm");
    int n = 0, r = 0, kind = -1;
    CHECK(spa_comm_info(comm, &n, &r, &kind) == SPA_OK && n == 8 && r == 3 && kind == 2, "comm info");

    spa_shape bad;
    memset(&bad, 0, sizeof bad);
    bad.B = 1; bad.S = 256; bad.H = 12; bad.D = 80; bad.stages = 1;
    spa_plan *plan = NULL;
    CHECK(spa_plan_create(&plan, comm, &bad) == SPA_ERR_UNSUPPORTED, "D=80 rejected");

    spa_shape s;
    memset(&s, 0, sizeof s);
    s.B = 1; s.S = 118800; s.H = 24; s.D = 128; s.stages = 24;   /* configs[3]: 720p, P=8, N_st=24 */
    CHECK(spa_plan_create(&plan, comm, &s) == SPA_OK, "plan");
    int G_h = 0, C = 0, g = 0;
    CHECK(spa_plan_stage_split(plan, &G_h, &C, &g) == SPA_OK && G_h == 3 && C == 8 && g == 1, "stage split");
    size_t ws = 0;
    CHECK(spa_plan_workspace_bytes(plan, &ws) == SPA_OK && ws >= (size_t)8 * 14850 * 24 * 128 * 2, "workspace");
    spa_msg msgs[64];
    int nm = 0;
    CHECK(spa_plan_describe_messages(plan, 0, 0, 3, msgs, 64, &nm) == SPA_OK && nm > 0, "messages");
    long long sent = 0, recvd = 0;
    for (int i = 0; i < nm; ++i) {
        if (msgs[i].is_recv) recvd += msgs[i].bytes; else sent += msgs[i].bytes;
    }
    CHECK(sent > 0 && sent == recvd, "stage 0 sends == receives for a uniform plan");
    spa_attn_desc a;
    CHECK(spa_plan_describe_attention(plan, 0, 3, &a) == SPA_OK && a.Skv == 118800 && a.n_heads == 1, "attn desc");
    /* the fused QKV projection's packed weight: 3 head groups of 3*8*1*128 rows of C, + fp32 bias */
    size_t wb = 0;
    CHECK(spa_plan_qkv_weight_bytes(plan, 3072, &wb) == SPA_OK && wb >= (size_t)9216 * 3072 * 2 + 9216 * 4, "qkv w");
    CHECK(spa_plan_qkv_weight_bytes(plan, 3071, &wb) == SPA_ERR_SHAPE, "C % 8 rejected");
    /* host-buffer SP workspace = the plan's + device copies of this rank's Q, K, V, O */
    size_t hb = 0;
    CHECK(spa_plan_host_sp_workspace_bytes(plan, &hb) == SPA_OK && hb >= ws + (size_t)4 * 14850 * 24 * 128 * 2, "hostbuf ws");
    /* NCCL symmetric windows are for NCCL plans only (refused here before any device call); free(NULL) is a no-op */
    CHECK(spa_plan_window_register(plan, (void *)(uintptr_t)4096) == SPA_ERR_INVALID, "window: not an NCCL plan");
    CHECK(spa_mem_free(NULL) == SPA_OK, "mem_free(NULL)");
    CHECK(spa_plan_destroy(plan) == SPA_OK, "destroy plan");
    /* a ring plan: step 0 of rank 3 sends K, V to rank 4 and receives from rank 2 */
    spa_shape rs;
    memset(&rs, 0, sizeof rs);
    rs.B = 1; rs.S = 8 * 64; rs.H = 5; rs.D = 64; rs.stages = 1; rs.ring = 1;
    CHECK(spa_plan_create(&plan, comm, &rs) == SPA_OK, "ring plan");
    CHECK(spa_plan_describe_ring(plan, 0, 3, msgs, 64, &nm) == SPA_OK && nm == 4 && msgs[0].peer == 4 &&
              msgs[2].peer == 2 && msgs[2].is_recv, "ring step");
    CHECK(spa_plan_destroy(plan) == SPA_OK && spa_comm_destroy(comm) == SPA_OK, "destroy");
    printf("c abi ok: %s\n", spa_version());
    return 0;
}
