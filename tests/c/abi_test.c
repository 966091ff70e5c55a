/* abi_test.c -- a plain C99 program compiled against include/sigattn.h and linked against
 * libsigattn.so (no Python, no torch): the header is self-contained C, every declared host-side
 * entry point links, and the calls that need no GPU behave as documented.
 *   - sigattn_valid_flops: the App. B.1 pins.
 *   - sigattn_worklist_host: padded-tile skipping: items = sum_b ceil(n_b / 128) per head.
 *   - argument errors return SIGATTN_EINVAL / SIGATTN_EWORKSPACE before any CUDA call.
 * Exit status 0 on success; prints the first failing check otherwise.                          */
#include <stdio.h>
#include <string.h>

#include "sigattn.h"

static int failures = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (!(cond)) {                                                           \
      fprintf(stderr, "abi_test: check failed at line %d: %s\n", __LINE__, #cond); \
      ++failures;                                                            \
    }                                                                        \
  } while (0)

int main(void) {
  /* FLOP credit: (b, h, n, d) = (1, 1, 2, 1) -> 16 forward / 40 backward; (1, 16, 16384, 128) */
  int32_t two[1] = {2};
  CHECK(sigattn_valid_flops(1, 1, 1, two, two, 1) == 16);
  CHECK(sigattn_valid_flops(1, 1, 1, two, two, 0) == 40);
  int32_t n16k[1] = {16384};
  CHECK(sigattn_valid_flops(1, 16, 128, n16k, n16k, 1) == 2199023255552LL);
  CHECK(sigattn_valid_flops(0, 1, 1, two, two, 1) == -1);

  /* work list: lengths {300, 0, 129} at N = 384 -> 3 + 0 + 2 forward items per head */
  int32_t lens[3] = {300, 0, 129};
  int32_t items[4 * 16];
  CHECK(sigattn_worklist_host(0, 3, 2, 384, 384, lens, lens, NULL, 0) == 10);
  CHECK(sigattn_worklist_host(0, 3, 2, 384, 384, lens, lens, items, 16) == 10);
  CHECK(items[0] == 0 && items[3] == 3);            /* longest sequence first, cost = key tiles */
  CHECK(sigattn_worklist_host(3, 3, 2, 384, 384, lens, lens, NULL, 0) == -1);

  /* parameter validation happens before any launch (works without a GPU) */
  sigattn_params p;
  memset(&p, 0, sizeof(p));
  p.B = 1; p.H = 1; p.Nq = 128; p.Nk = 128; p.d = 64; p.dtype = SIGATTN_BF16; p.scale = 0.125f;
  size_t fws = sigattn_fwd_workspace_bytes(&p), bws = sigattn_bwd_workspace_bytes(&p);
  CHECK(fws >= 32 && fws % 256 == 0);
  CHECK(bws >= (size_t)128 * 64 * 4);
  void* fake = (void*)(uintptr_t)(1u << 20);
  CHECK(sigattn_fwd(&p, fake, fake, fake, fake, fake, fws - 1, NULL) == SIGATTN_EWORKSPACE);
  CHECK(sigattn_fwd(&p, NULL, fake, fake, fake, fake, fws, NULL) == SIGATTN_EINVAL);
  CHECK(strlen(sigattn_last_error()) > 0);
  CHECK(sigattn_bwd(&p, fake, fake, fake, fake, fake, fake, fake, fake, bws - 1, NULL) == SIGATTN_EWORKSPACE);
  p.d = 96;
  CHECK(sigattn_fwd(&p, fake, fake, fake, fake, fake, fws, NULL) == SIGATTN_EINVAL);
  CHECK(sigattn_fwd_workspace_bytes(&p) == 0 && sigattn_bwd_workspace_bytes(&p) == 0);
  p.d = 64;
  p.flags = SIGATTN_F_DQ_F32_PARTIAL | SIGATTN_F_LAYOUT_BSHD;
  CHECK(sigattn_bwd(&p, fake, fake, fake, fake, fake, fake, fake, fake, bws, NULL) == SIGATTN_EUNSUPPORTED);
  CHECK(strstr(sigattn_version(), "sm_100a") != NULL);
  if (failures == 0) printf("abi_test: OK (%s)\n", sigattn_version());
  return failures == 0 ? 0 : 1;
}
