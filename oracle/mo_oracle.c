/* mo_oracle.c — C restatement of the reference solver path (see mo_oracle.h).
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline arm, never by the product. */
#include "mo_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MOO_MAXF 32
#define MOO_MAXOUT 512
#define MOO_MAXT 256

typedef struct {
  uint8_t op, sub;
  uint16_t dst, a, b, c;
  uint32_t gid;
  int32_t field, channel;
  int graph;
  int16_t off[3];
  int16_t slot;
  double imm;
  long long pnum, pden;
} Ins;
typedef struct {
  uint32_t gid, begin, end;
} Blk;
typedef struct {
  uint32_t nregs;
  int ni, nb, ng, no;
  Ins* ins;
  Blk* blk;
  uint16_t* greg;
  int* ooff;
  uint32_t* rgid;
  uint16_t* rreg;
} Prog;
typedef struct {
  int nd;
  int dims[3];
} Dom;
typedef struct {
  char name[64];
  int ch, mode;
  Dom dom;
} Fld;
typedef struct {
  int graph;
  Dom dom;
  int graph_idx;
} Res;
/* One template's Jacobian lanes (plan.hpp:47-72): grid lanes carry stencil
 * offsets, graph lanes edge slots. */
typedef struct {
  int tmpl, guard, nl;
  int *out, *f, *c, *slot;
  int (*off)[3];
} JTmpl;
typedef struct {
  Dom dom;
  int nt;
  int tmpl[MOO_MAXT];
  Prog cost, evalf;
  int njt;
  JTmpl* jt;
  Prog evalj;
} GridSetO;
typedef struct {
  Dom dom;
  int nc;
  int cf[MOO_MAXOUT], cc[MOO_MAXOUT];
  Prog bm, jtj;
} GatherSetO;
typedef struct {
  int graph, nt, ns;
  int tmpl[MOO_MAXT];
  int sslot[MOO_MAXOUT], sfield[MOO_MAXOUT], sch[MOO_MAXOUT];
  Prog cost, evalf, bm, jtj;
  int njt;
  JTmpl* jt;
  Prog evalj;
} GraphSetO;
typedef struct {
  int index;
  Dom dom;
  Prog prog;
} CompK;
typedef struct {
  Dom dom;
  Prog prog;
} ExclK;
typedef struct {
  int arity, bound;
  int64_t E;
  uint64_t* verts;
} Graph;

struct moo {
  int f64;
  moo_config cfg;
  int ndims;
  char dimname[16][64];
  int64_t dimext[16];
  int np, nu, na, nc, ng, nres, ngs, nqs, nhs, nck, nek;
  Fld unk[MOO_MAXF], arr[MOO_MAXF], cmp[MOO_MAXF];
  int garity[MOO_MAXF];
  Res res[MOO_MAXT];
  int64_t ubase[MOO_MAXF];
  int64_t num_cols;
  GridSetO* gs;
  GatherSetO* qs;
  GraphSetO* hs;
  CompK* ck;
  ExclK* ek;
  uint32_t max_regs;
  /* bound data */
  double* params;
  int x_bound, params_bound;
  int64_t arr_bound[MOO_MAXF];
  Graph graphs[MOO_MAXF];
  uint8_t* excluded;
  int64_t rowbase[MOO_MAXT];
  int64_t rows, unconstrained;
  int nonfinite_seen;
  void* st;
  /* materialized J (solver.hpp:278-376): 0 kNone, 1 kJ, 2 kJtJ */
  int materialize, jvalid;
  int64_t rows_seen;
  int64_t* joffs; /* CSR of J: rows + 1 */
  int64_t* jcol;
  void* jval;
  int64_t jnnz, jcap;
  int64_t* hoffs; /* kJtJ: CSR of H = 2 J^T J */
  int64_t* hcol;
  void* hval;
  int64_t hnnz;
};

static char g_err[512];
const char* moo_error(void) { return g_err; }
static int err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1 + code;
}
enum { E_SHAPE = 9, E_INDEX = 10, E_FORMAT = 11, E_TRUNC = 12, E_BIND = 14, E_INTERNAL = 17 };

static int dom_eq(const Dom* a, const Dom* b) {
  if (a->nd != b->nd) return 0;
  for (int i = 0; i < a->nd; ++i)
    if (a->dims[i] != b->dims[i]) return 0;
  return 1;
}
static void dom_shape(const moo* o, const Dom* d, int64_t* s) {
  s[0] = s[1] = s[2] = 1;
  for (int i = 0; i < d->nd; ++i) s[i] = o->dimext[d->dims[i]];
}
static int64_t dom_extent(const moo* o, const Dom* d) {
  int64_t n = 1;
  for (int i = 0; i < d->nd; ++i) n *= o->dimext[d->dims[i]];
  return n;
}

/* ------------------------------------------------------------ plan parsing */
typedef struct {
  const char* p;
  const char* end;
  int bad;
} Lex;
static int tok(Lex* L, char* out, size_t cap) {
  while (L->p < L->end && (*L->p == ' ' || *L->p == '\n' || *L->p == '\t' || *L->p == '\r')) ++L->p;
  size_t n = 0;
  while (L->p < L->end && !(*L->p == ' ' || *L->p == '\n' || *L->p == '\t' || *L->p == '\r')) {
    if (n + 1 < cap) out[n++] = *L->p;
    ++L->p;
  }
  out[n] = 0;
  if (n == 0) L->bad = 1;
  return (int)n;
}
static long long geti(Lex* L) {
  char b[64];
  tok(L, b, sizeof b);
  return strtoll(b, NULL, 10);
}
static double getd(Lex* L) {
  char b[64];
  tok(L, b, sizeof b);
  return strtod(b, NULL);
}
static void expect(Lex* L, const char* kw) {
  char b[64];
  tok(L, b, sizeof b);
  if (strcmp(b, kw) != 0) L->bad = 1;
}
static Dom getdom(Lex* L) {
  Dom d = {0, {0, 0, 0}};
  d.nd = (int)geti(L);
  if (d.nd < 0 || d.nd > 3) {
    L->bad = 1;
    d.nd = 0;
  }
  for (int i = 0; i < d.nd; ++i) d.dims[i] = (int)geti(L);
  return d;
}
static Prog getprog(Lex* L, const char* name, uint32_t* maxr) {
  Prog p;
  memset(&p, 0, sizeof p);
  expect(L, "program");
  expect(L, name);
  p.nregs = (uint32_t)geti(L);
  p.ni = (int)geti(L);
  p.nb = (int)geti(L);
  p.ng = (int)geti(L);
  p.no = (int)geti(L);
  if (L->bad || p.ni < 0 || p.nb < 0 || p.no < 0 || p.no > MOO_MAXOUT ||
      (p.ng < 1 && (p.ni || p.nb || p.no))) { /* empty = not compiled by the plan */
    L->bad = 1;
    return p;
  }
  if (p.nregs > *maxr) *maxr = p.nregs;
  p.ins = (Ins*)calloc((size_t)p.ni + 1, sizeof(Ins));
  for (int i = 0; i < p.ni; ++i) {
    Ins* in = &p.ins[i];
    expect(L, "i");
    in->op = (uint8_t)geti(L);
    in->sub = (uint8_t)geti(L);
    in->dst = (uint16_t)geti(L);
    in->a = (uint16_t)geti(L);
    in->b = (uint16_t)geti(L);
    in->c = (uint16_t)geti(L);
    in->gid = (uint32_t)geti(L);
    in->field = (int32_t)geti(L);
    in->channel = (int32_t)geti(L);
    in->graph = (int)geti(L);
    for (int k = 0; k < 3; ++k) in->off[k] = (int16_t)geti(L);
    in->slot = (int16_t)geti(L);
    in->imm = getd(L);
    in->pnum = geti(L);
    in->pden = geti(L);
  }
  p.blk = (Blk*)calloc((size_t)p.nb + 1, sizeof(Blk));
  for (int i = 0; i < p.nb; ++i) {
    expect(L, "b");
    p.blk[i].gid = (uint32_t)geti(L);
    p.blk[i].begin = (uint32_t)geti(L);
    p.blk[i].end = (uint32_t)geti(L);
  }
  p.greg = (uint16_t*)calloc((size_t)(p.ng > 0 ? p.ng : 1), sizeof(uint16_t));
  for (int i = 0; i < p.ng; ++i) {
    expect(L, "g");
    p.greg[i] = (uint16_t)geti(L);
  }
  p.ooff = (int*)calloc((size_t)p.no + 1, sizeof(int));
  int cap = 16, nr = 0;
  p.rgid = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)cap);
  p.rreg = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)cap);
  for (int o = 0; o < p.no; ++o) {
    expect(L, "o");
    int n = (int)geti(L);
    p.ooff[o] = nr;
    for (int k = 0; k < n; ++k) {
      if (nr == cap) {
        cap *= 2;
        p.rgid = (uint32_t*)realloc(p.rgid, sizeof(uint32_t) * (size_t)cap);
        p.rreg = (uint16_t*)realloc(p.rreg, sizeof(uint16_t) * (size_t)cap);
      }
      p.rgid[nr] = (uint32_t)geti(L);
      p.rreg[nr] = (uint16_t)geti(L);
      ++nr;
    }
  }
  p.ooff[p.no] = nr;
  return p;
}
static void freeprog(Prog* p) {
  free(p->ins);
  free(p->blk);
  free(p->greg);
  free(p->ooff);
  free(p->rgid);
  free(p->rreg);
}

static void relayout(moo* o) {
  int64_t col = 0;
  for (int f = 0; f < o->nu; ++f) {
    o->ubase[f] = col;
    col += dom_extent(o, &o->unk[f].dom) * o->unk[f].ch;
  }
  o->num_cols = col;
}

/* ------------------------------------------------------------ typed bodies */
#define REAL float
#define F(x) x##_f
#define POWF powf
#define SQRTF sqrtf
#define SINF sinf
#define COSF cosf
#define EXPF expf
#define LOGF logf
#define FABSF fabsf
#define ATANF atanf
#include "mo_oracle_impl.h"
#undef REAL
#undef F
#undef POWF
#undef SQRTF
#undef SINF
#undef COSF
#undef EXPF
#undef LOGF
#undef FABSF
#undef ATANF
#undef PUSH_ROW
#define REAL double
#define F(x) x##_d
#define POWF pow
#define SQRTF sqrt
#define SINF sin
#define COSF cos
#define EXPF exp
#define LOGF log
#define FABSF fabs
#define ATANF atan
#include "mo_oracle_impl.h"

static void jt_alloc(JTmpl* t) {
  size_t n = (size_t)t->nl + 1;
  t->out = (int*)calloc(n, sizeof(int));
  t->f = (int*)calloc(n, sizeof(int));
  t->c = (int*)calloc(n, sizeof(int));
  t->slot = (int*)calloc(n, sizeof(int));
  t->off = (int(*)[3])calloc(n, sizeof(int[3]));
}
static void jt_free(JTmpl* t, int n) {
  for (int k = 0; t && k < n; ++k) {
    free(t[k].out);
    free(t[k].f);
    free(t[k].c);
    free(t[k].slot);
    free(t[k].off);
  }
  free(t);
}

/* ------------------------------------------------------------ API */
int moo_create(const char* text, size_t len, int f64, moo** out) {
  moo* o = (moo*)calloc(1, sizeof(moo));
  Lex L = {text, text + len, 0};
  char w[64];
  o->f64 = f64;
  expect(&L, "moplan");
  if (geti(&L) != 1) L.bad = 1;
  expect(&L, "cfg");
  o->cfg.method = (int)geti(&L);
  (void)geti(&L); /* precision: chosen by the caller */
  o->cfg.nonlinear_iters = (int)geti(&L);
  o->cfg.linear_iters = (int)geti(&L);
  o->cfg.pcg_rel_tol = getd(&L);
  o->cfg.pcg_abs_tol = getd(&L);
  o->cfg.use_preconditioner = (int)geti(&L);
  o->cfg.lm_radius0 = getd(&L);
  o->cfg.lm_radius_min = getd(&L);
  o->cfg.lm_radius_max = getd(&L);
  o->cfg.lm_diag_min = getd(&L);
  o->cfg.lm_diag_max = getd(&L);
  o->cfg.lm_min_decrease = getd(&L);
  o->cfg.cost_stop_tol = getd(&L);
  {
    const char* save = L.p;
    tok(&L, w, sizeof w);
    if (strcmp(w, "materialize") == 0) o->materialize = (int)geti(&L);
    else L.p = save;
  }
  expect(&L, "dims");
  o->ndims = (int)geti(&L);
  for (int i = 0; i < o->ndims && i < 16; ++i) {
    expect(&L, "dim");
    tok(&L, o->dimname[i], 64);
    o->dimext[i] = geti(&L);
  }
  expect(&L, "params");
  o->np = (int)geti(&L);
  for (int i = 0; i < o->np; ++i) {
    expect(&L, "param");
    tok(&L, w, sizeof w);
  }
  expect(&L, "unknowns");
  o->nu = (int)geti(&L);
  for (int i = 0; i < o->nu && i < MOO_MAXF; ++i) {
    expect(&L, "unknown");
    tok(&L, o->unk[i].name, 64);
    o->unk[i].ch = (int)geti(&L);
    o->unk[i].dom = getdom(&L);
  }
  expect(&L, "arrays");
  o->na = (int)geti(&L);
  for (int i = 0; i < o->na && i < MOO_MAXF; ++i) {
    expect(&L, "array");
    tok(&L, o->arr[i].name, 64);
    o->arr[i].ch = (int)geti(&L);
    o->arr[i].dom = getdom(&L);
  }
  expect(&L, "computed");
  o->nc = (int)geti(&L);
  for (int i = 0; i < o->nc && i < MOO_MAXF; ++i) {
    expect(&L, "computed");
    tok(&L, o->cmp[i].name, 64);
    o->cmp[i].mode = (int)geti(&L);
    o->cmp[i].ch = (int)geti(&L);
    o->cmp[i].dom = getdom(&L);
  }
  expect(&L, "graphs");
  o->ng = (int)geti(&L);
  for (int i = 0; i < o->ng && i < MOO_MAXF; ++i) {
    expect(&L, "graph");
    tok(&L, w, sizeof w);
    o->garity[i] = (int)geti(&L);
  }
  expect(&L, "residuals");
  o->nres = (int)geti(&L);
  for (int i = 0; i < o->nres && i < MOO_MAXT; ++i) {
    expect(&L, "residual");
    tok(&L, w, sizeof w);
    if (strcmp(w, "grid") == 0) {
      o->res[i].graph = 0;
      o->res[i].dom = getdom(&L);
    } else {
      o->res[i].graph = 1;
      o->res[i].graph_idx = (int)geti(&L);
    }
  }
  expect(&L, "ubase");
  int nub = (int)geti(&L);
  for (int i = 0; i < nub; ++i) (void)geti(&L);
  expect(&L, "num_cols");
  (void)geti(&L);
  expect(&L, "grid_sets");
  o->ngs = (int)geti(&L);
  o->gs = (GridSetO*)calloc((size_t)o->ngs + 1, sizeof(GridSetO));
  for (int i = 0; i < o->ngs; ++i) {
    expect(&L, "grid_set");
    o->gs[i].dom = getdom(&L);
    o->gs[i].nt = (int)geti(&L);
    for (int t = 0; t < o->gs[i].nt; ++t) o->gs[i].tmpl[t] = (int)geti(&L);
    o->gs[i].cost = getprog(&L, "cost", &o->max_regs);
    o->gs[i].evalf = getprog(&L, "evalf", &o->max_regs);
    /* optional Jacobian-lane section (force_evalj / materialized plans) */
    const char* save = L.p;
    tok(&L, w, sizeof w);
    if (strcmp(w, "evalj") == 0) {
      GridSetO* g = &o->gs[i];
      g->njt = (int)geti(&L);
      g->jt = (JTmpl*)calloc((size_t)g->njt + 1, sizeof(JTmpl));
      for (int k = 0; k < g->njt; ++k) {
        expect(&L, "jtemplate");
        JTmpl* t = &g->jt[k];
        t->tmpl = (int)geti(&L);
        t->guard = (int)geti(&L);
        (void)geti(&L); /* origin flag: device-side only */
        t->nl = (int)geti(&L);
        jt_alloc(t);
        for (int q = 0; q < t->nl; ++q) {
          t->out[q] = (int)geti(&L);
          t->f[q] = (int)geti(&L);
          t->c[q] = (int)geti(&L);
          for (int a = 0; a < 3; ++a) t->off[q][a] = (int)geti(&L);
          t->slot[q] = -1;
        }
      }
      g->evalj = getprog(&L, "evalj", &o->max_regs);
    } else {
      L.p = save;
    }
  }
  expect(&L, "gather_sets");
  o->nqs = (int)geti(&L);
  o->qs = (GatherSetO*)calloc((size_t)o->nqs + 1, sizeof(GatherSetO));
  for (int i = 0; i < o->nqs; ++i) {
    expect(&L, "gather_set");
    o->qs[i].dom = getdom(&L);
    o->qs[i].nc = (int)geti(&L);
    for (int t = 0; t < o->qs[i].nc; ++t) {
      o->qs[i].cf[t] = (int)geti(&L);
      o->qs[i].cc[t] = (int)geti(&L);
    }
    o->qs[i].bm = getprog(&L, "bm", &o->max_regs);
    o->qs[i].jtj = getprog(&L, "jtj", &o->max_regs);
  }
  expect(&L, "graph_sets");
  o->nhs = (int)geti(&L);
  o->hs = (GraphSetO*)calloc((size_t)o->nhs + 1, sizeof(GraphSetO));
  for (int i = 0; i < o->nhs; ++i) {
    expect(&L, "graph_set");
    o->hs[i].graph = (int)geti(&L);
    o->hs[i].nt = (int)geti(&L);
    for (int t = 0; t < o->hs[i].nt; ++t) o->hs[i].tmpl[t] = (int)geti(&L);
    o->hs[i].ns = (int)geti(&L);
    for (int t = 0; t < o->hs[i].ns; ++t) {
      o->hs[i].sslot[t] = (int)geti(&L);
      o->hs[i].sfield[t] = (int)geti(&L);
      o->hs[i].sch[t] = (int)geti(&L);
    }
    o->hs[i].cost = getprog(&L, "cost", &o->max_regs);
    o->hs[i].evalf = getprog(&L, "evalf", &o->max_regs);
    o->hs[i].bm = getprog(&L, "bm", &o->max_regs);
    o->hs[i].jtj = getprog(&L, "jtj", &o->max_regs);
    const char* save = L.p;
    tok(&L, w, sizeof w);
    if (strcmp(w, "gevalj") == 0) {
      GraphSetO* g = &o->hs[i];
      g->njt = (int)geti(&L);
      g->jt = (JTmpl*)calloc((size_t)g->njt + 1, sizeof(JTmpl));
      for (int k = 0; k < g->njt; ++k) {
        expect(&L, "gjtemplate");
        JTmpl* t = &g->jt[k];
        t->tmpl = (int)geti(&L);
        t->guard = -1;
        t->nl = (int)geti(&L);
        jt_alloc(t);
        for (int q = 0; q < t->nl; ++q) {
          t->out[q] = (int)geti(&L);
          t->f[q] = (int)geti(&L);
          t->c[q] = (int)geti(&L);
          t->slot[q] = (int)geti(&L);
        }
      }
      g->evalj = getprog(&L, "evalj", &o->max_regs);
    } else {
      L.p = save;
    }
  }
  expect(&L, "computed_kernels");
  o->nck = (int)geti(&L);
  o->ck = (CompK*)calloc((size_t)o->nck + 1, sizeof(CompK));
  for (int i = 0; i < o->nck; ++i) {
    expect(&L, "computed_kernel");
    o->ck[i].index = (int)geti(&L);
    o->ck[i].dom = getdom(&L);
    o->ck[i].prog = getprog(&L, "prog", &o->max_regs);
  }
  expect(&L, "exclude_kernels");
  o->nek = (int)geti(&L);
  o->ek = (ExclK*)calloc((size_t)o->nek + 1, sizeof(ExclK));
  for (int i = 0; i < o->nek; ++i) {
    expect(&L, "exclude_kernel");
    o->ek[i].dom = getdom(&L);
    o->ek[i].prog = getprog(&L, "prog", &o->max_regs);
  }
  expect(&L, "end");
  if (L.bad || o->nu > MOO_MAXF || o->na > MOO_MAXF || o->nc > MOO_MAXF || o->nres > MOO_MAXT) {
    moo_destroy(o);
    return err(E_FORMAT, "moplan: malformed plan");
  }
  for (int a = 0; a < MOO_MAXF; ++a) o->arr_bound[a] = -1;
  relayout(o);
  *out = o;
  return 0;
}

static void free_data(moo* o) {
  if (o->st) {
    if (o->f64) free_state_d(o);
    else free_state_f(o);
  }
  free(o->excluded);
  o->excluded = NULL;
}

void moo_destroy(moo* o) {
  if (!o) return;
  free_data(o);
  for (int i = 0; i < o->ngs; ++i) {
    freeprog(&o->gs[i].cost);
    freeprog(&o->gs[i].evalf);
  }
  for (int i = 0; i < o->nqs; ++i) {
    freeprog(&o->qs[i].bm);
    freeprog(&o->qs[i].jtj);
  }
  for (int i = 0; i < o->nhs; ++i) {
    freeprog(&o->hs[i].cost);
    freeprog(&o->hs[i].evalf);
    freeprog(&o->hs[i].bm);
    freeprog(&o->hs[i].jtj);
  }
  for (int i = 0; i < o->ngs; ++i) {
    jt_free(o->gs[i].jt, o->gs[i].njt);
    if (o->gs[i].njt) freeprog(&o->gs[i].evalj);
  }
  for (int i = 0; i < o->nhs; ++i) {
    jt_free(o->hs[i].jt, o->hs[i].njt);
    if (o->hs[i].njt) freeprog(&o->hs[i].evalj);
  }
  free(o->joffs);
  free(o->jcol);
  free(o->jval);
  free(o->hoffs);
  free(o->hcol);
  free(o->hval);
  for (int i = 0; i < o->nck; ++i) freeprog(&o->ck[i].prog);
  for (int i = 0; i < o->nek; ++i) freeprog(&o->ek[i].prog);
  free(o->gs);
  free(o->qs);
  free(o->hs);
  free(o->ck);
  free(o->ek);
  free(o->params);
  for (int g = 0; g < MOO_MAXF; ++g) free(o->graphs[g].verts);
  free(o);
}

static void ensure_state(moo* o) {
  if (o->st) return;
  o->excluded = (uint8_t*)calloc((size_t)o->num_cols + 1, 1);
  if (o->f64) alloc_d(o);
  else alloc_f(o);
}

int moo_set_dim(moo* o, const char* name, int64_t extent) {
  if (o->st) return err(E_BIND, "set dims before binding data");
  for (int i = 0; i < o->ndims; ++i)
    if (strcmp(o->dimname[i], name) == 0) {
      o->dimext[i] = extent;
      relayout(o);
      return 0;
    }
  return err(1, "no such dim");
}

int moo_set_config(moo* o, const moo_config* c) {
  o->cfg = *c;
  if (o->cfg.pcg_rel_tol < 0) o->cfg.pcg_rel_tol = o->f64 ? 1e-8 : 1e-4;
  return 0;
}

int64_t moo_num_cols(moo* o) { return o->num_cols; }

#define RSZ(o) ((o)->f64 ? sizeof(double) : sizeof(float))

int moo_bind_x(moo* o, const void* x, int64_t n) {
  if (n != o->num_cols) return err(E_BIND, "unknown vector size does not match the plan layout");
  ensure_state(o);
  void* dst = o->f64 ? (void*)((State_d*)o->st)->x : (void*)((State_f*)o->st)->x;
  memcpy(dst, x, (size_t)n * RSZ(o));
  o->x_bound = 1;
  return 0;
}

int moo_bind_array(moo* o, int i, const void* a, int64_t n) {
  if (i < 0 || i >= o->na) return err(E_BIND, "array count does not match the declaration");
  if (n != dom_extent(o, &o->arr[i].dom) * o->arr[i].ch) return err(E_BIND, "array has the wrong size");
  ensure_state(o);
  void* dst = o->f64 ? (void*)((State_d*)o->st)->arrays[i] : (void*)((State_f*)o->st)->arrays[i];
  memcpy(dst, a, (size_t)n * RSZ(o));
  o->arr_bound[i] = n;
  return 0;
}

int moo_bind_params(moo* o, const double* p, int64_t n) {
  if (n != o->np) return err(E_BIND, "parameter count does not match the declaration");
  free(o->params);
  o->params = (double*)calloc((size_t)n + 1, sizeof(double));
  if (n) memcpy(o->params, p, (size_t)n * sizeof(double));
  o->params_bound = 1;
  return 0;
}

int moo_bind_graph(moo* o, int i, const uint64_t* v, int64_t n, int arity) {
  if (i < 0 || i >= o->ng) return err(E_BIND, "graph count does not match the declaration");
  Graph* g = &o->graphs[i];
  free(g->verts);
  g->verts = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n + 1));
  if (n) memcpy(g->verts, v, sizeof(uint64_t) * (size_t)n);
  g->arity = arity;
  g->E = arity ? n / arity : 0;
  g->bound = 1;
  return 0;
}

/* validate (solver.hpp:529-546) + vertex bounds (exec.hpp:238-259) */
static int validate(moo* o) {
  if (!o->x_bound) return err(E_BIND, "unknown vector size does not match the plan layout");
  if (!o->params_bound && o->np) return err(E_BIND, "parameter count does not match the declaration");
  for (int a = 0; a < o->na; ++a)
    if (o->arr_bound[a] < 0) return err(E_BIND, "array has the wrong size");
  for (int g = 0; g < o->ng; ++g) {
    if (!o->graphs[g].bound) return err(E_BIND, "graph count does not match the declaration");
    if (o->graphs[g].arity != o->garity[g]) return err(E_BIND, "graph arity does not match the declaration");
  }
  for (int s = 0; s < o->nhs; ++s) {
    const GraphSetO* h = &o->hs[s];
    const Graph* G = &o->graphs[h->graph];
    int64_t bound[64];
    for (int k = 0; k < 64; ++k) bound[k] = INT64_MAX;
    const Prog* ps[4] = {&h->cost, &h->evalf, &h->bm, &h->jtj};
    for (int q = 0; q < 4; ++q)
      for (int k = 0; k < ps[q]->ni; ++k) {
        const Ins* in = &ps[q]->ins[k];
        if (in->op < 3 || in->op > 6 || !in->graph) continue;
        const Fld* f = in->op == 4 ? &o->arr[in->field] : in->op == 5 ? &o->cmp[in->field] : &o->unk[in->field];
        int64_t ext = dom_extent(o, &f->dom);
        if (in->slot >= 0 && in->slot < 64 && ext < bound[in->slot]) bound[in->slot] = ext;
      }
    for (int k = 0; k < h->ns; ++k) {
      int64_t ext = dom_extent(o, &o->unk[h->sfield[k]].dom);
      if (ext < bound[h->sslot[k]]) bound[h->sslot[k]] = ext;
    }
    for (int64_t e = 0; e < G->E; ++e)
      for (int sl = 0; sl < G->arity && sl < 64; ++sl)
        if (G->verts[e * G->arity + sl] >= (uint64_t)bound[sl])
          return err(E_INDEX, "edge references a vertex beyond the bound extent");
  }
  return 0;
}

int moo_refresh(moo* o) {
  int rc = validate(o);
  if (rc) return rc;
  ensure_state(o);
  if (o->f64) {
    ensure_elemcost_d(o);
    refresh_d(o);
  } else {
    ensure_elemcost_f(o);
    refresh_f(o);
  }
  return 0;
}

int64_t moo_num_rows(moo* o) { return o->rows; }
int moo_excluded(moo* o, uint8_t* out) {
  memcpy(out, o->excluded, (size_t)o->num_cols);
  return 0;
}
int moo_cost(moo* o, double* out) {
  *out = o->f64 ? cost_at_d(o, ((State_d*)o->st)->x) : cost_at_f(o, ((State_f*)o->st)->x);
  return 0;
}
int moo_residuals(moo* o, void* out) {
  if (o->f64) residuals_d(o, (double*)out);
  else residuals_f(o, (float*)out);
  return 0;
}
int moo_build_normal(moo* o, void* b, void* m) {
  if (o->f64) {
    build_normal_d(o);
    memcpy(b, ((State_d*)o->st)->b, (size_t)o->num_cols * 8);
    memcpy(m, ((State_d*)o->st)->m, (size_t)o->num_cols * 8);
  } else {
    build_normal_f(o);
    memcpy(b, ((State_f*)o->st)->b, (size_t)o->num_cols * 4);
    memcpy(m, ((State_f*)o->st)->m, (size_t)o->num_cols * 4);
  }
  return 0;
}
int moo_apply_jtj(moo* o, const void* v, void* out) {
  return o->f64 ? apply_jtj_d(o, (const double*)v, (double*)out) : apply_jtj_f(o, (const float*)v, (float*)out);
}
int moo_solve(moo* o, moo_result* r, int* ti, double* tc, int* ta, double* tr, int* tp) {
  int rc = validate(o);
  if (rc) return rc;
  if (o->f64) {
    ensure_elemcost_d(o);
    rc = solve_d(o, r, ti, tc, ta, tr, tp);
  } else {
    ensure_elemcost_f(o);
    rc = solve_f(o, r, ti, tc, ta, tr, tp);
  }
  return rc;
}
int moo_linearize(moo* o) {
  int rc = validate(o);
  if (rc) return rc;
  return o->f64 ? linearize_d(o) : linearize_f(o);
}
int moo_normal_matrix(moo* o, int64_t* nnz, int64_t* offs, int64_t* col, void* val) {
  if (!o->jvalid || o->materialize != 2) return err(E_BIND, "no normal matrix has been assembled");
  *nnz = o->hnnz;
  if (offs) memcpy(offs, o->hoffs, (size_t)(o->num_cols + 1) * sizeof(int64_t));
  if (col) memcpy(col, o->hcol, (size_t)o->hnnz * sizeof(int64_t));
  if (val) memcpy(val, o->hval, (size_t)o->hnnz * RSZ(o));
  return 0;
}
int moo_jacobian(moo* o, int64_t* rows, int64_t* nnz, int64_t* offs, int64_t* col, void* val) {
  if (!o->jvalid) return err(E_BIND, "no Jacobian has been materialized");
  *rows = o->rows;
  *nnz = o->jnnz;
  if (offs) memcpy(offs, o->joffs, (size_t)(o->rows + 1) * sizeof(int64_t));
  if (col) memcpy(col, o->jcol, (size_t)o->jnnz * sizeof(int64_t));
  if (val) memcpy(val, o->jval, (size_t)o->jnnz * RSZ(o));
  return 0;
}
int moo_get_x(moo* o, void* out) {
  memcpy(out, o->f64 ? (void*)((State_d*)o->st)->x : (void*)((State_f*)o->st)->x, (size_t)o->num_cols * RSZ(o));
  return 0;
}
