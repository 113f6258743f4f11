/*
 * kr_host.h — C ABI of the product's host side (libkrhost.so): the
 * reference's instance loader, betting skeleton, Kronecker payoff assembly,
 * Technique A/B sparsifier, postprocessing and factor bundles, restated in
 * C++ for the B200 build (everything upstream of the gradient oracle).
 *
 * Reference interfaces replaced (paths under /root/reference/proj):
 *   readInstance / instanceFromJson     include/kronriver/instance_io.hpp:103-247
 *   buildSkeleton / payoffComponents    include/kronriver/skeleton.hpp:316-349
 *   makeRiverInstance / assemble        include/kronriver/kron.hpp:39-166
 *   densePayoffNonzeros                 include/kronriver/kron.hpp:198-207
 *   sparsifyW / techniqueA / techniqueB include/kronriver/sparsify.hpp:68-312
 *   postprocess / size / validate       include/kronriver/sparsify.hpp:123-406
 *   writeSparsification / read...       include/kronriver/bundle_io.hpp:27-94
 *   built-in instances                  include/kronriver/instances.hpp:19-194
 * Status codes are those of kr_engine.h.
 */
#ifndef KR_HOST_H
#define KR_HOST_H

#include <stdint.h>

#include "kr_engine.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct krh_instance krh_instance; /* RiverInstance + KronPayoff */
typedef struct krh_factors krh_factors;   /* Sparsification            */

/* Instance JSON schema v1 (instance_io.hpp:103-229). */
int krh_instance_from_json(const char* path, krh_instance** out);

/* Built-in games.  name: golden | twenty_card | bluffing | all_tie |
 * random_small (seed, hands; `skip` earlier draws of the same stream) |
 * bench (seed, hands, shared) | river_full (board code, deck 52 or 26,
 * tree 1 = reference menus, 3 = three-bet tree; beliefs from seed). */
int krh_instance_builtin(const char* name, uint64_t seed, int hands, int shared, const char* board, int deck,
                         int tree, krh_instance** out);

void krh_instance_free(krh_instance* h);

/* A river instance with explicit pieces (makeRiverInstance + assemble,
 * kron.hpp:39-166): board = 5 card ids, deck 52 or 26, hands as card-id pairs
 * with belief weights per player, and a betting configuration with one
 * menu (pot fractions) for every context and both players (skeleton.hpp:44-78;
 * stack per player, pot = each player's contribution, all-in flag, raise cap,
 * raise_cap < 0 = none).  Used to build the river continuations of a turn
 * endgame. */
int krh_instance_custom(const int32_t board[5], int deck, const uint8_t* cards1, const double* w1, int m1,
                        const uint8_t* cards2, const double* w2, int m2, double stack, double pot,
                        const double* menu, int nmenu, int all_in, int raise_cap, krh_instance** out);

/* m1 m2 n1 n2 rows cols nodes decisions1 decisions2 terminals folds
 * showdowns nnzF nnzS actions1 actions2 */
int krh_instance_dims(const krh_instance* h, int64_t out[16]);
double krh_instance_beta(const krh_instance* h);
double krh_instance_pot(const krh_instance* h); /* 2 * potContribution */
/* 4 characters per hand, strength-sorted (kron.hpp:74-83) */
int krh_instance_hands(const krh_instance* h, int player, char* out);
/* mu1 mu2 lambda1 lambda2 (sorted-hand order) */
int krh_instance_vectors(const krh_instance* h, double* mu1, double* mu2, double* lam1, double* lam2);
/* Treeplex of `player` for the solver: parent[nodes], action_ptr[nodes+1],
 * action_seq[actions] (skeleton.hpp:89-126). */
int krh_instance_treeplex(const krh_instance* h, int player, int32_t* parent, int32_t* action_ptr,
                          int32_t* action_seq);
int64_t krh_dense_nnz(const krh_instance* h);
/* Kronecker view for kr_engine_create_kron (pointers valid while h lives). */
int krh_instance_kron_view(const krh_instance* h, kr_kron_board* out);

/* technique 0 = A (rectangle peel, peel_iters), 1 = B.  post != 0 applies
 * postprocess (Technique B post is built in closed form, bit-identical to
 * postprocess(techniqueB(kp))). */
int krh_sparsify(const krh_instance* h, int technique, int post, int peel_iters, krh_factors** out);
int krh_postprocess(const krh_factors* f, krh_factors** out);
int krh_factors_from_arrays(const kr_factors* f, int technique, int postprocessed, krh_factors** out);
void krh_factors_free(krh_factors* f);
/* rows cols k nnzAhat nnzU nnzM nnzV technique postprocessed */
int krh_factors_dims(const krh_factors* f, int64_t out[9]);
/* Zero-copy view for kr_engine_create (valid while f lives). */
int krh_factors_view(const krh_factors* f, kr_factors* out);
/* validateSparsification (sparsify.hpp:133-145) */
int krh_factors_validate(const krh_factors* f);

/* Bundle directory: header.json + ahat/u/m/v.mtx (bundle_io.hpp:27-94). */
int krh_bundle_write(const krh_factors* f, const char* dir);
int krh_bundle_read(const char* dir, krh_factors** out);

const char* krh_last_error(int* code);

#ifdef __cplusplus
}
#endif

#endif /* KR_HOST_H */
