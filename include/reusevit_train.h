/*
 * reusevit_train.h — C-ABI of libreusevit's gate trainer: offline
 * training of the decision and restoration layers of a frozen ViT (§4).
 *
 *   Eq. 11  M_soft = GumbelSoftmax(MLP_decision(v)) — two logits, reuse = d and
 *                   recompute = 0; the Gumbel draws are INPUTS of every call
 *   Eq. 12  T_soft = M_soft * reused + (1 - M_soft) * recomputed, applied (reading T2,
 *                   DESIGN.md §3) to the layer output and to the key / value a token
 *                   contributes to attention; both branches are evaluated for every token
 *   Eq. 13-15  L = mean_f(1 - cos(Z_f, Z_hat_f)) + alpha max(0, R_target - L_reuse)
 *                   per frame group, averaged over the groups of a batch
 *   §4.3 frames come in groups (default pattern 1-5-9-13-11-12 = I, P, P, P, B2,
 *                   B1 with its references inside the group); the plan of one group is given
 *                   at creation and shared by every group of a batch
 *   P:401          backward runs for the gate parameters only: the ViT is frozen
 * Decision features (s, provider, t, r, c) carry no gradient (reading T3).
 *
 * Arithmetic: fp32 on the CUDA cores (toy-scale training; the inference hot path is
 * rv_embed).  Layouts: frames of a batch are [B][G] (group-major; frame b*G + k is local frame
 * k of group b, local frames in ascending display order); patches [B][G][N][pp], codec
 * [B][G][N], gumbel [B][G][L][N][2] (index 0: the reuse logit's draw, 1: recompute's),
 * Z [B][G][D], M and d [B][G][L][N].  All array arguments are DEVICE pointers on `stream`.
 * Gate parameters are the RVG1 blob (include/reusevit.h rv_load_gates order).
 * Errors: negative rv_status + rv_trainer_last_error(); RV_ECONTRACT for B > groups capacity
 * or non-positive temperature.  A trainer is bound to one device, thread-compatible.
 */
#ifndef REUSEVIT_TRAIN_H
#define REUSEVIT_TRAIN_H

#include "reusevit.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rv_trainer rv_trainer;

typedef struct {
  int32_t groups;          /* B: capacity in frame groups per call                          */
  int32_t group_size;      /* G: frames per group                                           */
  const int8_t* type;      /* [G] frame types (RV_I..RV_B1) of the group plan (host, copied) */
  const int32_t* past;     /* [G] local reference index or -1                                */
  const int32_t* future;   /* [G]                                                            */
  const int32_t* order;    /* [G] computation order (references first)                      */
  float alpha;             /* Eq. 15 weight                                                 */
  float r_target;          /* Eq. 15 target reuse rate                                      */
  float lr, beta1, beta2, eps;   /* Adam                                            */
} rv_train_config;

typedef struct {
  double l_sim, l_reuse, l_total;   /* batch means of Eq. 13, 14, 15                       */
  double cos_mean;                  /* mean cos(Z, Z_hat) over the batch's frames          */
  int32_t step;                     /* Adam steps taken so far                             */
} rv_train_log;

/* Create a trainer: the frozen ViT (RVW1 blob) and the initial gates (RVG1 blob) are copied
 * to the device as fp32.  The group plan is validated like rv_plan_check (RV_EPLAN). */
rv_status rv_trainer_create(const rv_config* cfg, int device, const float* vit_blob, size_t vit_floats,
                            const float* gate_blob, size_t gate_floats, const rv_train_config* tc,
                            rv_trainer** out);

/* flags for rv_trainer_forward */
#define RV_TRAIN_DENSE 1u  /* M = 0 everywhere: the frozen ViT's embedding (Z of Eq. 13)         */
#define RV_TRAIN_FORCE 2u  /* M read from `force` [B][G][L][N] (soft-to-hard limit diagnostic)   */

/* Soft-gated forward (Eq. 1-12) of B groups at temperature tau.  Z, M, d may be NULL. */
rv_status rv_trainer_forward(rv_trainer* tr, const float* patches, const float* codec, const float* gumbel,
                             int32_t B, float tau, uint32_t flags, const float* force, float* Z, float* M,
                             float* d, void* stream);

/* Forward at tau, the frozen ViT's Z, Eq. 15 and the backward pass: the gradient of the batch
 * loss w.r.t. every gate parameter is left in the trainer (and copied to grad_blob, a device
 * array of rv_gate_blob_floats floats, when non-NULL).  log may be NULL.  Synchronises. */
rv_status rv_trainer_loss_grad(rv_trainer* tr, const float* patches, const float* codec, const float* gumbel,
                               int32_t B, float tau, float* grad_blob, rv_train_log* log, void* stream);

/* rv_trainer_loss_grad followed by one Adam update of the gate parameters. */
rv_status rv_trainer_step(rv_trainer* tr, const float* patches, const float* codec, const float* gumbel, int32_t B,
                          float tau, rv_train_log* log, void* stream);

/* Current gate parameters as an RVG1 blob (HOST array of rv_gate_blob_floats floats), ready
 * for rv_load_gates.  Synchronises the trainer's device. */
rv_status rv_trainer_gates(rv_trainer* tr, float* gate_blob_host);

const char* rv_trainer_last_error(const rv_trainer* tr);
void rv_trainer_destroy(rv_trainer* tr);

#ifdef __cplusplus
}
#endif
#endif
