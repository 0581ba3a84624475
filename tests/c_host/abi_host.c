/* A plain C host linking libtetris_b200.so through include/tetris_b200.h (no Python, no torch): what a non-Python
 * serving process (or a cgo / JNI shim) compiles against.  CPU-only calls: version, workspace sizing, argument
 * validation with the thread-local error string, and the NCCL binding's null-communicator check. */
#include <stdio.h>
#include <string.h>

#include "tetris_b200.h"

int main(void) {
  if (tetris_abi_version() != 1) return 1;
  const size_t ws = tetris_workspace_bytes(TETRIS_OP_ALL, 1024, 16, 128256);
  if (ws == 0) return 2;
  /* capacity < 0 is the reference's ValueError (selector.py:145-146): rejected before any device work */
  int rc = tetris_select_f64(NULL, NULL, 4, 2, -1, 0, NULL, NULL, NULL, NULL, NULL, NULL, 0, NULL);
  if (rc != TETRIS_INVALID_ARGUMENT || strstr(tetris_last_error(), "capacity") == NULL) return 3;
  int32_t rank = -1, world = -1;
  rc = tetris_nccl_comm_info(NULL, &rank, &world);
  if (rc != TETRIS_INVALID_ARGUMENT && rc != TETRIS_NCCL_ERROR) return 4;
  printf("ok %zu\n", ws);
  return 0;
}
