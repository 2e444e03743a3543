/*
 * route.c — generator-side routing helper (NOT part of the simulated method).
 *
 * The paper takes routes as inputs "from the input demand data after the
 * routing"; this helper produces them for the synthetic workloads:
 * free-flow shortest paths (integer millisecond costs) with a
 * heap-order-independent tie-break — the parent of node v is the lowest-id
 * tight in-edge — so the routes are a pure function of (graph, OD pairs).
 *
 * One Dijkstra per origin group, groups spread over pthreads.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t n_nodes, n_edges;
  const int64_t *row_ptr;
  const int32_t *dst;
  const int64_t *cost;
  const int32_t *src;
  const int64_t *in_ptr;   /* in-edges of v: in_edge[in_ptr[v] .. in_ptr[v+1]) ascending */
  const int32_t *in_edge;
  int64_t n_groups;
  const int32_t *group_origin;
  const int64_t *group_ptr;
  const int64_t *trip_idx;
  const int32_t *dest;
  int64_t *route_len;      /* [n_trips] */
  int32_t **group_buf;     /* per group: concatenated routes of its trips (in trip_idx order) */
  int64_t next_group;
  pthread_mutex_t mu;
} job_t;

typedef struct { int64_t d; int32_t v; } hitem;

static void heap_push(hitem *h, int64_t *n, hitem x) {
  int64_t i = (*n)++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (h[p].d < x.d || (h[p].d == x.d && h[p].v <= x.v)) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = x;
}

static hitem heap_pop(hitem *h, int64_t *n) {
  hitem top = h[0];
  hitem x = h[--(*n)];
  int64_t i = 0;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= *n) break;
    if (c + 1 < *n && (h[c + 1].d < h[c].d || (h[c + 1].d == h[c].d && h[c + 1].v < h[c].v))) ++c;
    if (x.d < h[c].d || (x.d == h[c].d && x.v <= h[c].v)) break;
    h[i] = h[c];
    i = c;
  }
  h[i] = x;
  return top;
}

static void *worker(void *arg) {
  job_t *J = (job_t *)arg;
  int64_t *dist = (int64_t *)malloc(sizeof(int64_t) * (size_t)J->n_nodes);
  hitem *heap = (hitem *)malloc(sizeof(hitem) * (size_t)(J->n_edges + J->n_nodes + 1));
  int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(J->n_nodes + 1));
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int64_t g = J->next_group++;
    pthread_mutex_unlock(&J->mu);
    if (g >= J->n_groups) break;
    int32_t o = J->group_origin[g];
    for (int32_t v = 0; v < J->n_nodes; ++v) dist[v] = INT64_MAX;
    int64_t hn = 0;
    dist[o] = 0;
    heap_push(heap, &hn, (hitem){0, o});
    while (hn > 0) {
      hitem it = heap_pop(heap, &hn);
      if (it.d != dist[it.v]) continue;
      for (int64_t e = J->row_ptr[it.v]; e < J->row_ptr[it.v + 1]; ++e) {
        int32_t w = J->dst[e];
        int64_t nd = it.d + J->cost[e];
        if (nd < dist[w]) {
          dist[w] = nd;
          heap_push(heap, &hn, (hitem){nd, w});
        }
      }
    }
    /* walk back from every destination of the group */
    int64_t total = 0;
    int64_t t0 = J->group_ptr[g], t1 = J->group_ptr[g + 1];
    int64_t cap = 1024;
    int32_t *buf = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
    for (int64_t ti = t0; ti < t1; ++ti) {
      int64_t trip = J->trip_idx[ti];
      int32_t d = J->dest[trip];
      if (dist[d] == INT64_MAX || d == o) { J->route_len[trip] = -1; continue; }
      int32_t len = 0, v = d;
      while (v != o) {
        int32_t pe = -1;
        for (int64_t q = J->in_ptr[v]; q < J->in_ptr[v + 1]; ++q) {
          int32_t e = J->in_edge[q];
          int32_t u = J->src[e];
          if (dist[u] != INT64_MAX && dist[u] + J->cost[e] == dist[v]) { pe = e; break; }
        }
        tmp[len++] = pe;
        v = J->src[pe];
      }
      if (total + len > cap) {
        while (total + len > cap) cap *= 2;
        buf = (int32_t *)realloc(buf, sizeof(int32_t) * (size_t)cap);
      }
      for (int32_t i = 0; i < len; ++i) buf[total + i] = tmp[len - 1 - i];
      total += len;
      J->route_len[trip] = len;
    }
    J->group_buf[g] = buf;
  }
  free(dist);
  free(heap);
  free(tmp);
  return NULL;
}

typedef struct {
  job_t J;
  int32_t *src;
  int64_t *in_ptr;
  int32_t *in_edge;
} handle_t;

/* Computes all routes; returns a handle (route_len filled, −1 = unreachable). */
void *route_batch_begin(int32_t n_nodes, int32_t n_edges, const int64_t *row_ptr, const int32_t *dst,
                        const int64_t *cost, int64_t n_groups, const int32_t *group_origin,
                        const int64_t *group_ptr, const int64_t *trip_idx, const int32_t *dest,
                        int64_t *route_len, int32_t n_threads) {
  handle_t *H = (handle_t *)calloc(1, sizeof(handle_t));
  H->src = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_edges + 1));
  H->in_ptr = (int64_t *)calloc((size_t)n_nodes + 1, sizeof(int64_t));
  H->in_edge = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_edges + 1));
  for (int32_t u = 0; u < n_nodes; ++u)
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) H->src[e] = u;
  for (int32_t e = 0; e < n_edges; ++e) H->in_ptr[dst[e] + 1]++;
  for (int32_t v = 0; v < n_nodes; ++v) H->in_ptr[v + 1] += H->in_ptr[v];
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_nodes + 1));
  memcpy(fill, H->in_ptr, sizeof(int64_t) * (size_t)(n_nodes + 1));
  for (int32_t e = 0; e < n_edges; ++e) H->in_edge[fill[dst[e]]++] = e; /* ascending e */
  free(fill);
  job_t *J = &H->J;
  J->n_nodes = n_nodes; J->n_edges = n_edges; J->row_ptr = row_ptr; J->dst = dst; J->cost = cost;
  J->src = H->src; J->in_ptr = H->in_ptr; J->in_edge = H->in_edge;
  J->n_groups = n_groups; J->group_origin = group_origin; J->group_ptr = group_ptr;
  J->trip_idx = trip_idx; J->dest = dest; J->route_len = route_len;
  J->group_buf = (int32_t **)calloc((size_t)(n_groups > 0 ? n_groups : 1), sizeof(int32_t *));
  J->next_group = 0;
  pthread_mutex_init(&J->mu, NULL);
  if (n_threads < 1) n_threads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int32_t i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, worker, J);
  for (int32_t i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
  free(th);
  return H;
}

/* Scatters the routes into out (laid out by trip id via route_ptr) and frees the handle. */
void route_batch_finish(void *h, const int64_t *route_ptr, int32_t *out) {
  handle_t *H = (handle_t *)h;
  job_t *J = &H->J;
  for (int64_t g = 0; g < J->n_groups; ++g) {
    int64_t off = 0;
    for (int64_t ti = J->group_ptr[g]; ti < J->group_ptr[g + 1]; ++ti) {
      int64_t trip = J->trip_idx[ti];
      int64_t len = J->route_len[trip];
      if (len <= 0) continue;
      memcpy(out + route_ptr[trip], J->group_buf[g] + off, sizeof(int32_t) * (size_t)len);
      off += len;
    }
    free(J->group_buf[g]);
  }
  free(J->group_buf);
  pthread_mutex_destroy(&J->mu);
  free(H->src); free(H->in_ptr); free(H->in_edge);
  free(H);
}
