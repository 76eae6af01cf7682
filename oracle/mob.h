/* mob.h — tiny tagged-blob container used to move test/bench data between the
 * Python harness, the compiled reference driver (oracle/_ref) and the C
 * restatement (oracle/mo_oracle.c).
 *
 * TEST INFRASTRUCTURE ONLY: this file is part of the oracle (checker) and is
 * never linked into the product library.
 *
 * Layout (little endian):
 *   "MOB1" u32 n_records
 *   repeat n_records: u16 name_len, name bytes, u8 dtype, u64 n_elems, payload
 * dtype: 0=f32 1=f64 2=u8 3=i32 4=i64 5=u64
 */
#ifndef MOB_H_
#define MOB_H_

#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { MOB_F32 = 0, MOB_F64 = 1, MOB_U8 = 2, MOB_I32 = 3, MOB_I64 = 4, MOB_U64 = 5 };

static inline size_t mob_dsize(int dt) {
  static const size_t s[6] = {4, 8, 1, 4, 8, 8};
  return (dt >= 0 && dt < 6) ? s[dt] : 0;
}

typedef struct {
  char name[128];
  int dtype;
  uint64_t n;
  void* data;
} mob_rec;

typedef struct {
  int count;
  mob_rec* recs;
} mob_file;

static inline int mob_read(const char* path, mob_file* out) {
  FILE* f = fopen(path, "rb");
  char magic[4];
  uint32_t n;
  out->count = 0;
  out->recs = NULL;
  if (!f) return -1;
  if (fread(magic, 1, 4, f) != 4 || memcmp(magic, "MOB1", 4) != 0 || fread(&n, 4, 1, f) != 1) {
    fclose(f);
    return -2;
  }
  out->recs = (mob_rec*)calloc(n ? n : 1, sizeof(mob_rec));
  for (uint32_t i = 0; i < n; ++i) {
    uint16_t len;
    uint8_t dt;
    mob_rec* r = &out->recs[i];
    if (fread(&len, 2, 1, f) != 1 || len >= sizeof(r->name)) { fclose(f); return -3; }
    if (fread(r->name, 1, len, f) != len) { fclose(f); return -3; }
    r->name[len] = 0;
    if (fread(&dt, 1, 1, f) != 1 || fread(&r->n, 8, 1, f) != 1) { fclose(f); return -3; }
    r->dtype = dt;
    size_t bytes = (size_t)r->n * mob_dsize(dt);
    r->data = malloc(bytes ? bytes : 1);
    if (bytes && fread(r->data, 1, bytes, f) != bytes) { fclose(f); return -4; }
    out->count = (int)(i + 1);
  }
  fclose(f);
  return 0;
}

static inline const mob_rec* mob_find(const mob_file* m, const char* name) {
  for (int i = 0; i < m->count; ++i)
    if (strcmp(m->recs[i].name, name) == 0) return &m->recs[i];
  return NULL;
}

static inline void mob_free(mob_file* m) {
  for (int i = 0; i < m->count; ++i) free(m->recs[i].data);
  free(m->recs);
  m->recs = NULL;
  m->count = 0;
}

/* Streaming writer: header count is patched on close. */
typedef struct {
  FILE* f;
  uint32_t count;
} mob_writer;

static inline int mob_open_w(mob_writer* w, const char* path) {
  w->f = fopen(path, "wb");
  w->count = 0;
  if (!w->f) return -1;
  fwrite("MOB1", 1, 4, w->f);
  fwrite(&w->count, 4, 1, w->f);
  return 0;
}

static inline void mob_put(mob_writer* w, const char* name, int dtype, const void* data,
                           uint64_t n) {
  uint16_t len = (uint16_t)strlen(name);
  uint8_t dt = (uint8_t)dtype;
  fwrite(&len, 2, 1, w->f);
  fwrite(name, 1, len, w->f);
  fwrite(&dt, 1, 1, w->f);
  fwrite(&n, 8, 1, w->f);
  if (n) fwrite(data, mob_dsize(dtype), (size_t)n, w->f);
  w->count++;
}

static inline void mob_close_w(mob_writer* w) {
  fseek(w->f, 4, SEEK_SET);
  fwrite(&w->count, 4, 1, w->f);
  fclose(w->f);
  w->f = NULL;
}

#endif /* MOB_H_ */
