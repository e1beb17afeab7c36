// The streaming bucket kernel with 512 consumer threads (16 warps) per CTA:
// more warps to hide latency on levels made of many small items (config 3
// default), at 96 registers per thread.  Selected per level by the batch.
#define QTN_STREAM_COMPUTE 512
#define QTN_STREAM_NS s512
#include "qtn_stream_tile.cuh"
