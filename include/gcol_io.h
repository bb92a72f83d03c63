/*
 * gcol_io.h -- C ABI of the host-side text loaders (libgcol_io.so; host only,
 * no CUDA).  What a binding of the reference's ingestion would call:
 *
 *   reference                                                   replaced by
 *   load_edge_list      /root/reference/proj/include/gcol/graph_io.hpp:83-106   gcol_io_parse / gcol_io_load (GCOL_IO_EDGELIST)
 *   load_matrix_market  graph_io.hpp:124-221                    gcol_io_parse / gcol_io_load (GCOL_IO_MM)
 *   load_graph          /root/reference/proj/tools/gcol_main.cpp:25-35  gcol_io_load (GCOL_IO_AUTO: by extension)
 *   save_edge_list      graph_io.hpp:110-117                    gcol_io_format_edge_list
 *   read_coloring_file  gcol_main.cpp:72-108                    gcol_io_parse_coloring
 *   build_graph         graph.hpp:98-138                        gcol_io_build_graph
 *
 * Every loader returns the canonical CSR the colouring ABI takes
 * (include/gcol_cuda.h: int64 offsets[n+1], int32 cols[m], rows ascending,
 * symmetric, no loops).  Arrays are owned by the returned handle.
 * Status: 0 ok, else a gcol_io_status; the message (the reference's wording,
 * "line N: ..." for parse errors) is in gcol_io_last_error() (thread-local).
 */
#ifndef GCOL_IO_H
#define GCOL_IO_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GCOL_IO_OK = 0,
  GCOL_IO_ERR_INPUT = 1,       /* gcol::input_error (errors.hpp:11-14)            -> CLI exit 2 */
  GCOL_IO_ERR_PARSE = 2,       /* gcol::parse_error (errors.hpp:17-28), has a line -> CLI exit 2 */
  GCOL_IO_ERR_UNSUPPORTED = 3, /* gcol::unsupported_format_error (errors.hpp:32-35)  -> CLI exit 2 */
  GCOL_IO_ERR_CAPACITY = 4,    /* gcol::capacity_error (errors.hpp:38-41)           -> CLI exit 2 */
  GCOL_IO_ERR_IO = 5           /* gcol::io_error (errors.hpp:50-53)                 -> CLI exit 4 */
} gcol_io_status;

typedef enum { GCOL_IO_AUTO = 0, GCOL_IO_EDGELIST = 1, GCOL_IO_MM = 2 } gcol_io_format;

typedef struct gcol_io_graph gcol_io_graph;

const char* gcol_io_last_error(void);
/* 1-based line of the last parse error on this thread, 0 if it had none. */
uint64_t gcol_io_last_error_line(void);

/* Parses `len` bytes of text.  format: EDGELIST or MM (AUTO = EDGELIST).
 * num_vertices < 0: 1 + the largest id seen (edge lists only; ignored for MM). */
int gcol_io_parse(const char* text, uint64_t len, int32_t format, int64_t num_vertices,
                  gcol_io_graph** out);
/* Reads and parses a file; AUTO picks MM for .mtx / .mm, else an edge list. */
int gcol_io_load(const char* path, int32_t format, gcol_io_graph** out);
/* build_graph over raw pairs (u0, v0, u1, v1, ...), any order/orientation. */
int gcol_io_build_graph(const uint32_t* pairs, uint64_t num_pairs, uint64_t num_vertices,
                        gcol_io_graph** out);
void gcol_io_graph_free(gcol_io_graph* g);
int64_t gcol_io_num_vertices(const gcol_io_graph* g);
int64_t gcol_io_num_adjacency(const gcol_io_graph* g); /* m = 2 * edges */
int32_t gcol_io_max_degree(const gcol_io_graph* g);
const int64_t* gcol_io_offsets(const gcol_io_graph* g);
const int32_t* gcol_io_cols(const gcol_io_graph* g);

/* Edge-list text of the graph (save_edge_list).  Returns its length; the
 * buffer lives until the next call on this handle or its release. */
uint64_t gcol_io_format_edge_list(gcol_io_graph* g, const char** text);
int gcol_io_save_edge_list(gcol_io_graph* g, const char* path);

/* One colour per line.  *colors is malloc'ed (release with gcol_io_free). */
int gcol_io_parse_coloring(const char* text, uint64_t len, int32_t** colors, uint64_t* count);
void gcol_io_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
