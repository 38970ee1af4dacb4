/* Plain-C consumer of the C-ABI (include/gridnlp_b200.h): what a cgo / FFI / C host
 * binding sees.  Runs without a GPU: version, device count, argument validation, the
 * CPU-side load profile.  Built and run by tests/test_abi.py. */
#include <stdio.h>
#include <string.h>

#include "gridnlp_b200.h"

int main(void) {
  int32_t ndev = -1;
  int rc;
  gn_error err;
  double scale[2 * 3];
  memset(&err, 0, sizeof err);
  if (gn_abi_version() != GN_ABI_VERSION) return 1;
  rc = gn_device_count(&ndev); /* GN_ERR_CUDA without a device */
  if ((rc != GN_OK && rc != GN_ERR_CUDA) || ndev < 0) return 2;
  /* null handles are rejected, never dereferenced */
  if (gn_eval_f(NULL, NULL, NULL, GN_MEM_HOST, &err) != GN_ERR_INVALID) return 3;
  if (gn_kkt_values(NULL, NULL, NULL, GN_MEM_HOST) != GN_ERR_INVALID) return 4;
  if (gn_ipm_destroy(NULL) != GN_OK) return 5;
  /* generate_load_profile on the host (network.hpp:104-140) */
  if (gn_load_profile(3, 2, 60.0, 1, 0.2, 0.02, scale, &err) != GN_OK) return 6;
  printf("abi %d devices %d scale0 %.17g\n", gn_abi_version(), (int)ndev, scale[0]);
  return 0;
}
