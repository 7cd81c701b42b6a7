/* sparsesync_peer.h — NVLink peer-memory plumbing for the bucket transfer (row a6).
 *
 * The paper ships buckets Trainer -> Rollout over the framework's process groups
 * (Alg. 2 l.10 SendToRollout / Alg. 3 l.2 RecvFromUpdater). On one
 * NVSwitch node this library instead lets a Rollout process map a Trainer
 * process's bucket buffer (CUDA IPC) and pull the bytes with the copy engines
 * (no SMs, no NCCL kernels competing with the extract / decode kernels), or let
 * the decode kernel read them in place. Cross-process ordering uses IPC events:
 * the Trainer records "ready" after the encode, the Rollout records "consumed"
 * after its decode; the host control plane (gloo) orders the record/wait calls.
 *
 * All calls are thin wrappers over the CUDA runtime/driver; they return
 * SYNC_OK (0) or SYNC_ERR_CUDA (-5) / SYNC_ERR_ARG (-1) and never throw.
 * Handles are opaque 64-byte blobs (cudaIpcMemHandle_t / cudaIpcEventHandle_t)
 * that the caller ships between processes of the same node.                   */
#ifndef SPARSESYNC_PEER_H
#define SPARSESYNC_PEER_H
#include <stddef.h>
#include <stdint.h>

#include "sparsesync.h"

#ifdef __cplusplus
extern "C" {
#endif

#define SYNC_PEER_HANDLE_BYTES 64

/* Export the device allocation containing d_ptr: out_handle (64 B) names the
 * whole allocation, *offset = d_ptr - allocation base, *alloc_bytes its size. */
int sync_peer_mem_export(const void* d_ptr, uint8_t* out_handle, uint64_t* offset, uint64_t* alloc_bytes);
/* Map a peer process's exported allocation into the calling thread's current
 * device (lazy peer access); *d_base = the mapped allocation base. Must not be
 * called on a handle exported by the same process. */
int sync_peer_mem_open(const uint8_t* handle, void** d_base);
int sync_peer_mem_close(void* d_base);

/* Interprocess event (timing disabled): create + export, open a peer's, record, wait, destroy. */
int sync_peer_event_create(void** ev, uint8_t* out_handle);
int sync_peer_event_open(const uint8_t* handle, void** ev);
int sync_peer_event_record(void* ev, sync_stream_t stream);
int sync_peer_stream_wait(sync_stream_t stream, void* ev);
int sync_peer_event_destroy(void* ev);

/* Asynchronous device-to-device copy on `stream` (copy engine; src or dst may be a mapped peer pointer). */
int sync_peer_copy(void* d_dst, const void* d_src, uint64_t bytes, sync_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSESYNC_PEER_H */
