/* mo_oracle_impl.h — Real-typed body of the C restatement; included twice by
 * mo_oracle.c with REAL = float / double and F(x) = x##_f / x##_d.
 * TEST INFRASTRUCTURE ONLY. */

typedef struct {
  const REAL* data;
  int ch, nd;
  int64_t shape[3];
} F(View);

typedef struct {
  const double* params;
  F(View) unk[MOO_MAXF], arr[MOO_MAXF], cmp[MOO_MAXF], pf[MOO_MAXF];
  int64_t dshape[3];
  int dnd;
  int64_t pix[3];
  const uint64_t* edge;
} F(Env);

typedef struct {
  REAL* data;
  int64_t offset, stride, extent;
  int slot;
} F(Out);

/* ipow / pow_eval: common.hpp:102-124 */
static REAL F(ipow)(REAL x, long long n) {
  if (n < 0) return (REAL)1 / F(ipow)(x, -n);
  REAL r = (REAL)1;
  while (n > 0) {
    if (n & 1) r *= x;
    x *= x;
    n >>= 1;
  }
  return r;
}
static REAL F(pow_eval)(REAL x, long long num, long long den) {
  if (den == 1) {
    if (num >= -32 && num <= 32) return F(ipow)(x, num);
    return (REAL)POWF(x, (REAL)num);
  }
  if (den == 2) return F(ipow)((REAL)SQRTF(x), num);
  return (REAL)POWF(x, (REAL)num / (REAL)den);
}

/* EvalEnv::read (eval.hpp:41-55): OOB against the field's own shape -> 0 */
static REAL F(read)(const F(Env) * e, const F(View) * f, const Ins* in) {
  int64_t elem;
  if (in->graph) {
    elem = (int64_t)e->edge[in->slot];
  } else {
    int64_t c[3] = {0, 0, 0};
    for (int a = 0; a < f->nd; ++a) {
      c[a] = e->pix[a] + in->off[a];
      if (c[a] < 0 || c[a] >= f->shape[a]) return (REAL)0;
    }
    elem = 0;
    for (int a = 0; a < f->nd; ++a) elem = elem * f->shape[a] + c[a];
  }
  return f->data[elem * f->ch + in->channel];
}

/* EvalEnv::inbounds (eval.hpp:57-61): against the iteration domain */
static int F(inbounds)(const F(Env) * e, const Ins* in) {
  for (int a = 0; a < e->dnd; ++a) {
    int64_t c = e->pix[a] + in->off[a];
    if (c < 0 || c >= e->dshape[a]) return 0;
  }
  return 1;
}

/* run_program (program.hpp:89-167) */
static void F(run_program)(const Prog* p, const F(Env) * e, REAL* r, REAL* out) {
  for (uint32_t i = 0; i < p->nregs; ++i) r[i] = (REAL)0;
  for (int b = 0; b < p->nb; ++b) {
    const Blk* blk = &p->blk[b];
    if (blk->gid != 0 && r[p->greg[blk->gid]] == (REAL)0) continue;
    for (uint32_t i = blk->begin; i < blk->end; ++i) {
      const Ins* in = &p->ins[i];
      REAL v = 0, x, y;
      switch (in->op) {
        case 0: v = (REAL)in->imm; break;
        case 1: v = (REAL)e->params[in->field]; break;
        case 2: v = (REAL)e->pix[in->field]; break;
        case 3: v = F(read)(e, &e->unk[in->field], in); break;
        case 4: v = F(read)(e, &e->arr[in->field], in); break;
        case 5: v = F(read)(e, &e->cmp[in->field], in); break;
        case 6: v = F(read)(e, &e->pf[in->field], in); break;
        case 7: v = (REAL)(F(inbounds)(e, in) ? 1 : 0); break;
        case 8: v = r[in->a] + r[in->b]; break;
        case 9: v = r[in->a] * r[in->b]; break;
        case 10: v = F(pow_eval)(r[in->a], in->pnum, in->pden); break;
        case 11:
          x = r[in->a];
          switch (in->sub) {
            case 0: v = (REAL)SQRTF(x); break;
            case 1: v = (REAL)SINF(x); break;
            case 2: v = (REAL)COSF(x); break;
            case 3: v = (REAL)EXPF(x); break;
            case 4: v = (REAL)LOGF(x); break;
            case 5: v = (REAL)FABSF(x); break;
            case 6: v = (REAL)ATANF(x); break;
            default: v = 0;
          }
          break;
        case 12: {
          int t = 0;
          x = r[in->a];
          y = r[in->b];
          switch (in->sub) {
            case 0: t = x == y; break;
            case 1: t = x != y; break;
            case 2: t = x < y; break;
            case 3: t = x <= y; break;
            case 4: t = x > y; break;
            case 5: t = x >= y; break;
          }
          v = (REAL)(t ? 1 : 0);
          break;
        }
        case 13: v = (REAL)((r[in->a] != (REAL)0 && r[in->b] != (REAL)0) ? 1 : 0); break;
        case 14: v = (REAL)((r[in->a] != (REAL)0 || r[in->b] != (REAL)0) ? 1 : 0); break;
        case 15: v = (REAL)(r[in->a] == (REAL)0 ? 1 : 0); break;
        case 16: v = r[in->a] != (REAL)0 ? r[in->b] : r[in->c]; break;
      }
      r[in->dst] = v;
    }
  }
  for (int o = 0; o < p->no; ++o) {
    REAL acc = (REAL)0;
    for (int k = p->ooff[o]; k < p->ooff[o + 1]; ++k) {
      uint32_t gid = p->rgid[k];
      if (gid != 0 && r[p->greg[gid]] == (REAL)0) continue;
      acc += r[p->rreg[k]];
    }
    out[o] = acc;
  }
}

typedef struct {
  REAL *x, *b, *m, *md, *damp, *delta, *xt, *aptmp, *r, *z, *p, *ap;
  double* base_diag;
  REAL* arrays[MOO_MAXF];
  REAL* comp[MOO_MAXF];
  REAL* maskval[MOO_MAXF];
  uint8_t* masks[MOO_MAXF];
  REAL* regs;
  REAL* outs;
  REAL* elemcost;
  REAL* jtmp; /* materialized apply: J v (solver.hpp:280) */
  int64_t jtmp_cap;
} F(State);

static void F(coord_of)(const int64_t* shape, int nd, int64_t e, int64_t* c) {
  c[0] = c[1] = c[2] = 0;
  for (int a = nd - 1; a >= 0; --a) {
    c[a] = e % shape[a];
    e /= shape[a];
  }
}

static void F(env)(moo* o, const REAL* x, const REAL* pv, const Dom* d, F(Env) * e) {
  F(State)* S = (F(State)*)o->st;
  memset(e, 0, sizeof *e);
  e->params = o->params;
  for (int f = 0; f < o->nu; ++f) {
    const Fld* u = &o->unk[f];
    F(View) v = {x + o->ubase[f], u->ch, u->dom.nd, {1, 1, 1}};
    dom_shape(o, &u->dom, v.shape);
    e->unk[f] = v;
    v.data = pv ? pv + o->ubase[f] : NULL;
    e->pf[f] = v;
  }
  for (int a = 0; a < o->na; ++a) {
    F(View) v = {S->arrays[a], o->arr[a].ch, o->arr[a].dom.nd, {1, 1, 1}};
    dom_shape(o, &o->arr[a].dom, v.shape);
    e->arr[a] = v;
  }
  for (int c = 0; c < o->nc; ++c) {
    F(View) v = {S->comp[c], o->cmp[c].ch, o->cmp[c].dom.nd, {1, 1, 1}};
    dom_shape(o, &o->cmp[c].dom, v.shape);
    e->cmp[c] = v;
  }
  e->dshape[0] = e->dshape[1] = e->dshape[2] = 1;
  e->dnd = 1;
  if (d) {
    dom_shape(o, d, e->dshape);
    e->dnd = d->nd ? d->nd : 1;
  }
}

/* exec_grid (exec.hpp:151-214), sequential: write outputs, excluded -> 0 */
static void F(exec_grid)(moo* o, const Prog* p, F(Env) * e, const F(Out) * outs, const uint8_t* excl) {
  F(State)* S = (F(State)*)o->st;
  const int64_t ext = e->dshape[0] * e->dshape[1] * e->dshape[2];
  for (int64_t el = 0; el < ext; ++el) {
    if (excl && excl[el]) {
      for (int k = 0; k < p->no; ++k) outs[k].data[outs[k].offset + el * outs[k].stride] = (REAL)0;
      continue;
    }
    F(coord_of)(e->dshape, e->dnd, el, e->pix);
    F(run_program)(p, e, S->regs, S->outs);
    for (int k = 0; k < p->no; ++k) {
      REAL v = S->outs[k];
      if (!isfinite((double)v)) o->nonfinite_seen = 1;
      outs[k].data[outs[k].offset + el * outs[k].stride] = v;
    }
  }
}

/* exec_graph (exec.hpp:223-309), sequential edge order */
static void F(exec_graph)(moo* o, const Prog* p, F(Env) * e, int g, const F(Out) * outs) {
  F(State)* S = (F(State)*)o->st;
  const Graph* G = &o->graphs[g];
  for (int64_t ed = 0; ed < G->E; ++ed) {
    e->edge = G->verts + ed * G->arity;
    e->pix[0] = e->pix[1] = e->pix[2] = 0;
    F(run_program)(p, e, S->regs, S->outs);
    for (int k = 0; k < p->no; ++k) {
      REAL v = S->outs[k];
      if (!isfinite((double)v)) o->nonfinite_seen = 1;
      if (outs[k].slot < 0) {
        outs[k].data[outs[k].offset + ed * outs[k].stride] = v;
      } else {
        int64_t vert = (int64_t)e->edge[outs[k].slot];
        outs[k].data[outs[k].offset + vert * outs[k].stride] += v;
      }
    }
  }
}

static const uint8_t* F(mask_for)(moo* o, const Dom* d) {
  F(State)* S = (F(State)*)o->st;
  for (int i = 0; i < o->nek; ++i)
    if (dom_eq(&o->ek[i].dom, d)) return S->masks[i];
  return NULL;
}

/* refresh (solver.hpp:125-168): computed arrays, masks, excluded columns */
static void F(refresh)(moo* o) {
  F(State)* S = (F(State)*)o->st;
  F(Env) e;
  F(Out) outs[MOO_MAXOUT];
  o->jvalid = 0; /* solver.hpp:167 */
  for (int i = 0; i < o->nck; ++i) {
    const CompK* ck = &o->ck[i];
    int tc = o->cmp[ck->index].ch;
    F(env)(o, S->x, NULL, &ck->dom, &e);
    for (int c = 0; c < tc; ++c) outs[c] = (F(Out)){S->comp[ck->index], c, tc, 0, -1};
    F(exec_grid)(o, &ck->prog, &e, outs, NULL);
  }
  for (int i = 0; i < o->nek; ++i) {
    const ExclK* ek = &o->ek[i];
    int64_t ext = dom_extent(o, &ek->dom);
    F(env)(o, S->x, NULL, &ek->dom, &e);
    outs[0] = (F(Out)){S->maskval[i], 0, 1, ext, -1};
    F(exec_grid)(o, &ek->prog, &e, outs, NULL);
    for (int64_t k = 0; k < ext; ++k) S->masks[i][k] = S->maskval[i][k] != (REAL)0 ? 1 : 0;
  }
  memset(o->excluded, 0, (size_t)o->num_cols);
  for (int i = 0; i < o->nek; ++i)
    for (int f = 0; f < o->nu; ++f) {
      if (!dom_eq(&o->unk[f].dom, &o->ek[i].dom)) continue;
      int64_t ext = dom_extent(o, &o->ek[i].dom);
      for (int64_t k = 0; k < ext; ++k)
        if (S->masks[i][k])
          for (int c = 0; c < o->unk[f].ch; ++c) o->excluded[o->ubase[f] + k * o->unk[f].ch + c] = 1;
    }
  int64_t row = 0;
  for (int t = 0; t < o->nres; ++t) {
    o->rowbase[t] = row;
    row += o->res[t].graph ? o->graphs[o->res[t].graph_idx].E : dom_extent(o, &o->res[t].dom);
  }
  o->rows = row;
}

/* cost_at (solver.hpp:176-193): per-element buffer, sequential Real sum */
static double F(cost_at)(moo* o, const REAL* x) {
  F(State)* S = (F(State)*)o->st;
  F(Env) e;
  REAL total = (REAL)0;
  for (int i = 0; i < o->ngs; ++i) {
    const GridSetO* g = &o->gs[i];
    int64_t ext = dom_extent(o, &g->dom);
    F(env)(o, x, NULL, &g->dom, &e);
    F(Out) out = {S->elemcost, 0, 1, ext, -1};
    F(exec_grid)(o, &g->cost, &e, &out, NULL);
    for (int64_t k = 0; k < ext; ++k) total += S->elemcost[k];
  }
  for (int i = 0; i < o->nhs; ++i) {
    const GraphSetO* g = &o->hs[i];
    int64_t E = o->graphs[g->graph].E;
    F(env)(o, x, NULL, NULL, &e);
    F(Out) out = {S->elemcost, 0, 1, E, -1};
    F(exec_graph)(o, &g->cost, &e, g->graph, &out);
    for (int64_t k = 0; k < E; ++k) total += S->elemcost[k];
  }
  return (double)total;
}

static void F(residuals)(moo* o, REAL* f) {
  F(State)* S = (F(State)*)o->st;
  F(Env) e;
  F(Out) outs[MOO_MAXOUT];
  for (int i = 0; i < o->ngs; ++i) {
    const GridSetO* g = &o->gs[i];
    F(env)(o, S->x, NULL, &g->dom, &e);
    for (int k = 0; k < g->nt; ++k) outs[k] = (F(Out)){f, o->rowbase[g->tmpl[k]], 1, 0, -1};
    F(exec_grid)(o, &g->evalf, &e, outs, NULL);
  }
  for (int i = 0; i < o->nhs; ++i) {
    const GraphSetO* g = &o->hs[i];
    F(env)(o, S->x, NULL, NULL, &e);
    for (int k = 0; k < g->nt; ++k) outs[k] = (F(Out)){f, o->rowbase[g->tmpl[k]], 1, 0, -1};
    F(exec_graph)(o, &g->evalf, &e, g->graph, outs);
  }
}

/* build_normal (solver.hpp:220-251) */
static void F(build_normal)(moo* o) {
  F(State)* S = (F(State)*)o->st;
  F(Env) e;
  F(Out) outs[MOO_MAXOUT];
  for (int i = 0; i < o->nqs; ++i) {
    const GatherSetO* g = &o->qs[i];
    F(env)(o, S->x, NULL, &g->dom, &e);
    for (int k = 0; k < g->nc; ++k) {
      const Fld* u = &o->unk[g->cf[k]];
      outs[2 * k] = (F(Out)){S->b, o->ubase[g->cf[k]] + g->cc[k], u->ch, 0, -1};
      outs[2 * k + 1] = (F(Out)){S->m, o->ubase[g->cf[k]] + g->cc[k], u->ch, 0, -1};
    }
    F(exec_grid)(o, &g->bm, &e, outs, F(mask_for)(o, &g->dom));
  }
  for (int i = 0; i < o->nhs; ++i) {
    const GraphSetO* g = &o->hs[i];
    F(env)(o, S->x, NULL, NULL, &e);
    for (int k = 0; k < g->ns; ++k) {
      const Fld* u = &o->unk[g->sfield[k]];
      outs[2 * k] = (F(Out)){S->b, o->ubase[g->sfield[k]] + g->sch[k], u->ch, 0, g->sslot[k]};
      outs[2 * k + 1] = (F(Out)){S->m, o->ubase[g->sfield[k]] + g->sch[k], u->ch, 0, g->sslot[k]};
    }
    F(exec_graph)(o, &g->bm, &e, g->graph, outs);
  }
  o->unconstrained = 0;
  for (int64_t i = 0; i < o->num_cols; ++i) {
    if (o->excluded[i]) {
      S->b[i] = (REAL)0;
      S->m[i] = (REAL)1;
    } else if (S->m[i] == (REAL)0) {
      ++o->unconstrained;
      S->m[i] = (REAL)1;
    }
  }
}

/* H = 2 J^T J (solver.hpp:370-374): transpose by counting sort, Gustavson
 * spgemm with a dense accumulator (rows of J^T in order, touched columns
 * sorted), scale_inplace (sparse.hpp). */
static int F(cmp_i64)(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : x > y;
}
static void F(assemble_h)(moo* o) {
  const int64_t n = o->num_cols, nnz = o->jnnz;
  const REAL* jv = (const REAL*)o->jval;
  int64_t* toffs = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* tcol = (int64_t*)malloc((size_t)nnz * sizeof(int64_t) + 8);
  REAL* tval = (REAL*)malloc((size_t)nnz * sizeof(REAL) + 8);
  for (int64_t k = 0; k < nnz; ++k) ++toffs[o->jcol[k] + 1];
  for (int64_t i = 0; i < n; ++i) toffs[i + 1] += toffs[i];
  int64_t* cur = (int64_t*)malloc((size_t)n * sizeof(int64_t) + 8);
  memcpy(cur, toffs, (size_t)n * sizeof(int64_t));
  for (int64_t r = 0; r < o->rows; ++r)
    for (int64_t k = o->joffs[r]; k < o->joffs[r + 1]; ++k) {
      int64_t d = cur[o->jcol[k]]++;
      tcol[d] = r;
      tval[d] = jv[k];
    }
  REAL* acc = (REAL*)calloc((size_t)n + 1, sizeof(REAL));
  char* used = (char*)calloc((size_t)n + 1, 1);
  int64_t* touched = (int64_t*)malloc((size_t)n * sizeof(int64_t) + 8);
  free(o->hoffs);
  free(o->hcol);
  free(o->hval);
  o->hoffs = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t cap = 1024, hn = 0;
  o->hcol = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
  o->hval = malloc((size_t)cap * sizeof(REAL));
  for (int64_t i = 0; i < n; ++i) {
    int64_t nt = 0;
    for (int64_t ka = toffs[i]; ka < toffs[i + 1]; ++ka) {
      int64_t mid = tcol[ka];
      REAL av = tval[ka];
      for (int64_t kb = o->joffs[mid]; kb < o->joffs[mid + 1]; ++kb) {
        int64_t cc = o->jcol[kb];
        if (!used[cc]) {
          used[cc] = 1;
          acc[cc] = (REAL)0;
          touched[nt++] = cc;
        }
        acc[cc] += av * jv[kb];
      }
    }
    qsort(touched, (size_t)nt, sizeof(int64_t), F(cmp_i64));
    for (int64_t k = 0; k < nt; ++k) {
      if (hn == cap) {
        cap *= 2;
        o->hcol = (int64_t*)realloc(o->hcol, (size_t)cap * sizeof(int64_t));
        o->hval = realloc(o->hval, (size_t)cap * sizeof(REAL));
      }
      o->hcol[hn] = touched[k];
      ((REAL*)o->hval)[hn] = acc[touched[k]] * (REAL)2;
      ++hn;
      used[touched[k]] = 0;
    }
    o->hoffs[i + 1] = hn;
  }
  o->hnnz = hn;
  free(toffs);
  free(tcol);
  free(tval);
  free(cur);
  free(acc);
  free(used);
  free(touched);
}

/* linearize (solver.hpp:291-376): evalj lanes per template set, then the
 * CSR of J with the SparseCSR push checks (sparse.hpp:30-37). */
static int F(jpush)(moo* o, int64_t c, REAL v) {
  if (c < 0 || c >= o->num_cols) return err(E_INDEX, "CSR column out of range");
  int64_t r = o->rows_seen;
  if (!(o->jnnz == o->joffs[r - 1] || o->jcol[o->jnnz - 1] < c))
    return err(E_INTERNAL, "CSR row entries must arrive in increasing column order");
  if (o->jnnz == o->jcap) {
    o->jcap = o->jcap ? 2 * o->jcap : 1024;
    o->jcol = (int64_t*)realloc(o->jcol, (size_t)o->jcap * sizeof(int64_t));
    o->jval = realloc(o->jval, (size_t)o->jcap * sizeof(REAL));
  }
  o->jcol[o->jnnz] = c;
  ((REAL*)o->jval)[o->jnnz] = v;
  ++o->jnnz;
  o->joffs[r] = o->jnnz;
  return 0;
}
static int F(linearize)(moo* o) {
  F(State)* S = (F(State)*)o->st;
  F(Env) e;
  F(Out) outs[MOO_MAXOUT];
  REAL* lg[MOO_MAXT] = {0};
  REAL* lh[MOO_MAXT] = {0};
  int rc = 0;
  for (int i = 0; i < o->ngs; ++i) {
    const GridSetO* g = &o->gs[i];
    if (!g->njt) continue;
    int64_t ext = dom_extent(o, &g->dom);
    lg[i] = (REAL*)calloc((size_t)(g->evalj.no * ext) + 1, sizeof(REAL));
    for (int l = 0; l < g->evalj.no; ++l) outs[l] = (F(Out)){lg[i], (int64_t)l * ext, 1, ext, -1};
    F(env)(o, S->x, NULL, &g->dom, &e);
    F(exec_grid)(o, &g->evalj, &e, outs, NULL);
  }
  for (int i = 0; i < o->nhs; ++i) {
    const GraphSetO* g = &o->hs[i];
    if (!g->njt) continue;
    int64_t E = o->graphs[g->graph].E;
    lh[i] = (REAL*)calloc((size_t)(g->evalj.no * E) + 1, sizeof(REAL));
    for (int l = 0; l < g->evalj.no; ++l) outs[l] = (F(Out)){lh[i], (int64_t)l * E, 1, E, -1};
    F(env)(o, S->x, NULL, NULL, &e);
    F(exec_graph)(o, &g->evalj, &e, g->graph, outs);
  }
  free(o->joffs);
  o->joffs = (int64_t*)calloc((size_t)o->rows + 1, sizeof(int64_t));
  o->jnnz = 0;
  o->rows_seen = 0;
  for (int t = 0; t < o->nres && !rc; ++t) {
    int found = 0;
    for (int i = 0; i < o->ngs && !found; ++i) {
      const GridSetO* g = &o->gs[i];
      for (int k = 0; k < g->njt && !found; ++k) {
        const JTmpl* jt = &g->jt[k];
        if (jt->tmpl != t) continue;
        found = 1;
        int64_t sh[3], ext = dom_extent(o, &g->dom);
        dom_shape(o, &g->dom, sh);
        for (int64_t el = 0; el < ext && !rc; ++el) {
          o->joffs[++o->rows_seen] = o->jnnz; /* begin_row */
          if (lg[i][(int64_t)jt->guard * ext + el] == (REAL)0) continue;
          for (int q = 0; q < jt->nl && !rc; ++q) {
            int64_t lin = ((int64_t)jt->off[q][0] * sh[1] + jt->off[q][1]) * sh[2] + jt->off[q][2];
            rc = F(jpush)(o, o->ubase[jt->f[q]] + (el + lin) * o->unk[jt->f[q]].ch + jt->c[q],
                          lg[i][(int64_t)jt->out[q] * ext + el]);
          }
        }
      }
    }
    for (int i = 0; i < o->nhs && !found; ++i) {
      const GraphSetO* g = &o->hs[i];
      for (int k = 0; k < g->njt && !found; ++k) {
        const JTmpl* jt = &g->jt[k];
        if (jt->tmpl != t) continue;
        found = 1;
        const Graph* G = &o->graphs[g->graph];
        int64_t cols[MOO_MAXOUT];
        REAL vals[MOO_MAXOUT];
        for (int64_t ed = 0; ed < G->E && !rc; ++ed) {
          o->joffs[++o->rows_seen] = o->jnnz;
          int n = 0;
          for (int q = 0; q < jt->nl; ++q) { /* stable insertion sort by column */
            int64_t c = o->ubase[jt->f[q]] + (int64_t)G->verts[ed * G->arity + jt->slot[q]] * o->unk[jt->f[q]].ch +
                        jt->c[q];
            REAL v = lh[i][(int64_t)jt->out[q] * G->E + ed];
            int j = n++;
            while (j > 0 && cols[j - 1] > c) {
              cols[j] = cols[j - 1];
              vals[j] = vals[j - 1];
              --j;
            }
            cols[j] = c;
            vals[j] = v;
          }
          for (int q = 0; q < n && !rc;) { /* degenerate edges: merge columns */
            int64_t c = cols[q];
            REAL v = vals[q];
            for (++q; q < n && cols[q] == c; ++q) v += vals[q];
            rc = F(jpush)(o, c, v);
          }
        }
      }
    }
    if (!found) rc = err(E_BIND, "plan was compiled without Jacobian kernels");
  }
  for (int i = 0; i < MOO_MAXT; ++i) {
    free(lg[i]);
    free(lh[i]);
  }
  if (!rc && o->materialize == 2) F(assemble_h)(o);
  o->jvalid = rc == 0;
  return rc;
}

/* spmv / spmv_t (sparse.hpp): y = J v row by row; y = J^T x by row-ordered scatter */
static void F(apply_materialized)(moo* o, const REAL* v, REAL* out) {
  F(State)* S = (F(State)*)o->st;
  const REAL* val = (const REAL*)o->jval;
  for (int64_t r = 0; r < o->rows; ++r) {
    REAL acc = (REAL)0;
    for (int64_t k = o->joffs[r]; k < o->joffs[r + 1]; ++k) acc += val[k] * v[o->jcol[k]];
    S->jtmp[r] = acc;
  }
  for (int64_t i = 0; i < o->num_cols; ++i) out[i] = (REAL)0;
  for (int64_t r = 0; r < o->rows; ++r) {
    REAL xr = S->jtmp[r];
    for (int64_t k = o->joffs[r]; k < o->joffs[r + 1]; ++k) out[o->jcol[k]] += val[k] * xr;
  }
  for (int64_t i = 0; i < o->num_cols; ++i) out[i] *= (REAL)2;
}

/* apply_jtj (solver.hpp:255-285): matrix-free, or the materialized J */
static int F(apply_jtj)(moo* o, const REAL* v, REAL* out) {
  F(State)* S = (F(State)*)o->st;
  F(Env) e;
  F(Out) outs[MOO_MAXOUT];
  if (o->materialize) {
    if (!o->jvalid) return err(E_INTERNAL, "normal-matrix apply before linearize()");
    if (o->rows > S->jtmp_cap) {
      free(S->jtmp);
      S->jtmp = (REAL*)calloc((size_t)o->rows, sizeof(REAL));
      S->jtmp_cap = o->rows;
    }
    if (o->materialize == 2) { /* spmv(H, v) */
      const REAL* hv = (const REAL*)o->hval;
      for (int64_t i = 0; i < o->num_cols; ++i) {
        REAL acc = (REAL)0;
        for (int64_t k = o->hoffs[i]; k < o->hoffs[i + 1]; ++k) acc += hv[k] * v[o->hcol[k]];
        out[i] = acc;
      }
      return 0;
    }
    F(apply_materialized)(o, v, out);
    return 0;
  }
  for (int i = 0; i < o->nqs; ++i) {
    const GatherSetO* g = &o->qs[i];
    F(env)(o, S->x, v, &g->dom, &e);
    for (int k = 0; k < g->nc; ++k)
      outs[k] = (F(Out)){out, o->ubase[g->cf[k]] + g->cc[k], o->unk[g->cf[k]].ch, 0, -1};
    F(exec_grid)(o, &g->jtj, &e, outs, F(mask_for)(o, &g->dom));
  }
  for (int i = 0; i < o->nhs; ++i) {
    const GraphSetO* g = &o->hs[i];
    F(env)(o, S->x, v, NULL, &e);
    for (int k = 0; k < g->ns; ++k)
      outs[k] = (F(Out)){out, o->ubase[g->sfield[k]] + g->sch[k], o->unk[g->sfield[k]].ch, 0, g->sslot[k]};
    F(exec_graph)(o, &g->jtj, &e, g->graph, outs);
  }
  return 0;
}

static REAL F(dot)(const REAL* a, const REAL* b, int64_t n) {
  REAL acc = (REAL)0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}
static void F(zero_excl)(moo* o, REAL* v) {
  for (int64_t i = 0; i < o->num_cols; ++i)
    if (o->excluded[i]) v[i] = (REAL)0;
}
static void F(apply_damped)(moo* o, const REAL* v, REAL* out, int lm) {
  F(State)* S = (F(State)*)o->st;
  F(apply_jtj)(o, v, out);
  if (lm)
    for (int64_t i = 0; i < o->num_cols; ++i) out[i] += S->damp[i] * v[i];
}

/* pcg (pcg.hpp:63-130) */
static void F(pcg)(moo* o, int lm, int* iters, int* indefinite, int* nonfinite) {
  F(State)* S = (F(State)*)o->st;
  const int64_t n = o->num_cols;
  const REAL* m = S->md;
  *iters = 0;
  *indefinite = 0;
  *nonfinite = 0;
  for (int64_t i = 0; i < n; ++i) {
    S->delta[i] = (REAL)0;
    S->r[i] = S->b[i];
  }
  F(zero_excl)(o, S->r);
  for (int64_t i = 0; i < n; ++i) S->z[i] = o->cfg.use_preconditioner ? S->r[i] / m[i] : S->r[i];
  F(zero_excl)(o, S->z);
  REAL rz = F(dot)(S->r, S->z, n);
  if (!isfinite((double)rz)) {
    *nonfinite = 1;
    return;
  }
  REAL stop = (REAL)o->cfg.pcg_rel_tol * (REAL)o->cfg.pcg_rel_tol * rz;
  if ((REAL)o->cfg.pcg_abs_tol > stop) stop = (REAL)o->cfg.pcg_abs_tol;
  if (rz <= stop) return;
  for (int64_t i = 0; i < n; ++i) S->p[i] = S->z[i];
  for (int k = 0; k < o->cfg.linear_iters; ++k) {
    F(apply_damped)(o, S->p, S->ap, lm);
    F(zero_excl)(o, S->ap);
    REAL pap = F(dot)(S->p, S->ap, n);
    if (!isfinite((double)pap)) {
      *nonfinite = 1;
      return;
    }
    if (pap <= (REAL)0) {
      *indefinite = 1;
      return;
    }
    REAL alpha = rz / pap;
    for (int64_t i = 0; i < n; ++i) S->delta[i] += alpha * S->p[i];
    F(zero_excl)(o, S->delta);
    for (int64_t i = 0; i < n; ++i) S->r[i] -= alpha * S->ap[i];
    F(zero_excl)(o, S->r);
    for (int64_t i = 0; i < n; ++i) S->z[i] = o->cfg.use_preconditioner ? S->r[i] / m[i] : S->r[i];
    F(zero_excl)(o, S->z);
    REAL rzn = F(dot)(S->r, S->z, n);
    if (!isfinite((double)rzn)) {
      *nonfinite = 1;
      return;
    }
    ++*iters;
    if (rzn <= stop) return;
    REAL beta = rzn / rz;
    for (int64_t i = 0; i < n; ++i) S->p[i] = S->z[i] + beta * S->p[i];
    F(zero_excl)(o, S->p);
    rz = rzn;
  }
}

#define PUSH_ROW(IT, C, A, R, P)                                 \
  do {                                                           \
    if (nt < 4096) {                                             \
      t_iter[nt] = (IT);                                         \
      t_cost[nt] = (C);                                          \
      t_acc[nt] = (A);                                           \
      t_radius[nt] = (R);                                        \
      t_pcg[nt] = (P);                                           \
    }                                                            \
    ++nt;                                                        \
  } while (0)

/* solve (solver.hpp:389-515), no callbacks */
static int F(solve)(moo* o, moo_result* res, int* t_iter, double* t_cost, int* t_acc, double* t_radius,
                    int* t_pcg) {
  F(State)* S = (F(State)*)o->st;
  const moo_config* c = &o->cfg;
  const int lm = c->method == 1;
  const int64_t n = o->num_cols;
  double mu = c->lm_radius0, nu = 2.0;
  int nt = 0;
  memset(res, 0, sizeof *res);
  res->reason = 0;
  for (int it = 0; it < c->nonlinear_iters; ++it) {
    F(refresh)(o);
    double cost_old = F(cost_at)(o, S->x);
    if (!isfinite(cost_old)) {
      PUSH_ROW(it, cost_old, 0, lm ? mu : 0.0, 0);
      res->reason = 3;
      res->final_cost = cost_old;
      goto done;
    }
    F(build_normal)(o);
    if (o->materialize) { /* solver.hpp:426 */
      int rc = F(linearize)(o);
      if (rc) return rc;
    }
    if (lm)
      for (int64_t i = 0; i < n; ++i) {
        double v = (double)S->m[i] / 2.0;
        S->base_diag[i] = v < c->lm_diag_min ? c->lm_diag_min : (c->lm_diag_max < v ? c->lm_diag_max : v);
      }
    double cost_after = cost_old;
    int stepped = 0;
    while (!stepped) {
      if (lm)
        for (int64_t i = 0; i < n; ++i) S->damp[i] = o->excluded[i] ? (REAL)0 : (REAL)(2.0 / mu * S->base_diag[i]);
      for (int64_t i = 0; i < n; ++i) S->md[i] = S->m[i] + S->damp[i];
      int iters, indef, nonf;
      F(pcg)(o, lm, &iters, &indef, &nonf);
      res->indefinite |= indef;
      if (nonf && !lm) {
        res->reason = 3;
        res->final_cost = cost_old;
        PUSH_ROW(it, cost_old, 0, 0.0, iters);
        goto done;
      }
      for (int64_t i = 0; i < n; ++i) S->xt[i] = o->excluded[i] ? S->x[i] : S->x[i] + S->delta[i];
      double cost_new = nonf ? INFINITY : F(cost_at)(o, S->xt);
      if (!lm) {
        memcpy(S->x, S->xt, (size_t)n * sizeof(REAL));
        PUSH_ROW(it, cost_new, 1, 0.0, iters);
        if (!isfinite(cost_new)) {
          res->reason = 3;
          res->final_cost = cost_new;
          goto done;
        }
        cost_after = cost_new;
        stepped = 1;
        break;
      }
      F(apply_jtj)(o, S->delta, S->aptmp);
      double predicted = 0, dot_b = 0;
      for (int64_t i = 0; i < n; ++i) {
        dot_b += (double)S->b[i] * (double)S->delta[i];
        predicted -= 0.5 * (double)S->delta[i] * (double)S->aptmp[i];
      }
      predicted += dot_b;
      double rho = predicted > 0 ? (cost_old - cost_new) / predicted : -1.0;
      if (isfinite(cost_new) && predicted > 0 && rho > c->lm_min_decrease) {
        memcpy(S->x, S->xt, (size_t)n * sizeof(REAL));
        double t = 2.0 * rho - 1.0;
        double shrink = 1.0 - t * t * t;
        if (shrink < 1.0 / 3.0) shrink = 1.0 / 3.0;
        PUSH_ROW(it, cost_new, 1, mu, iters);
        mu = mu / shrink;
        if (mu < c->lm_radius_min) mu = c->lm_radius_min;
        if (mu > c->lm_radius_max) mu = c->lm_radius_max;
        nu = 2.0;
        cost_after = cost_new;
        stepped = 1;
      } else {
        PUSH_ROW(it, cost_new, 0, mu, iters);
        int zero_step = 1;
        for (int64_t i = 0; i < n; ++i)
          if (S->delta[i] != (REAL)0) {
            zero_step = 0;
            break;
          }
        mu /= nu;
        nu *= 2.0;
        if (zero_step || mu < c->lm_radius_min) {
          res->reason = 2;
          res->final_cost = cost_old;
          goto done;
        }
      }
    }
    {
      double denom = cost_old > 1e-300 ? cost_old : 1e-300;
      double rel = (cost_old - cost_after) / denom;
      if (rel >= 0 && rel < c->cost_stop_tol) {
        res->reason = 1;
        break;
      }
    }
  }
  F(refresh)(o);
  res->final_cost = F(cost_at)(o, S->x);
  if (!isfinite(res->final_cost)) res->reason = 3;
done:
  res->n_trace = nt;
  res->nonfinite_kernels = o->nonfinite_seen;
  res->unconstrained = o->unconstrained;
  return 0;
}

static void F(alloc)(moo* o) {
  F(State)* S = (F(State)*)calloc(1, sizeof(F(State)));
  const size_t n = (size_t)o->num_cols + 1;
  o->st = S;
  REAL** vecs[] = {&S->x, &S->b, &S->m, &S->md, &S->damp, &S->delta, &S->xt, &S->aptmp, &S->r, &S->z, &S->p, &S->ap};
  for (size_t k = 0; k < sizeof vecs / sizeof vecs[0]; ++k) *vecs[k] = (REAL*)calloc(n, sizeof(REAL));
  S->base_diag = (double*)calloc(n, sizeof(double));
  for (int a = 0; a < o->na; ++a) S->arrays[a] = (REAL*)calloc((size_t)(dom_extent(o, &o->arr[a].dom) * o->arr[a].ch + 1), sizeof(REAL));
  for (int c = 0; c < o->nc; ++c) S->comp[c] = (REAL*)calloc((size_t)(dom_extent(o, &o->cmp[c].dom) * o->cmp[c].ch + 1), sizeof(REAL));
  for (int i = 0; i < o->nek; ++i) {
    size_t ext = (size_t)dom_extent(o, &o->ek[i].dom) + 1;
    S->maskval[i] = (REAL*)calloc(ext, sizeof(REAL));
    S->masks[i] = (uint8_t*)calloc(ext, 1);
  }
  S->regs = (REAL*)calloc((size_t)o->max_regs + 1, sizeof(REAL));
  S->outs = (REAL*)calloc(MOO_MAXOUT, sizeof(REAL));
  S->elemcost = NULL;
}

static void F(free_state)(moo* o) {
  F(State)* S = (F(State)*)o->st;
  if (!S) return;
  REAL* vecs[] = {S->x, S->b, S->m, S->md, S->damp, S->delta, S->xt, S->aptmp, S->r, S->z, S->p, S->ap, S->regs, S->outs, S->elemcost};
  for (size_t k = 0; k < sizeof vecs / sizeof vecs[0]; ++k) free(vecs[k]);
  free(S->base_diag);
  free(S->jtmp);
  for (int a = 0; a < MOO_MAXF; ++a) {
    free(S->arrays[a]);
    free(S->comp[a]);
    free(S->maskval[a]);
    free(S->masks[a]);
  }
  free(S);
  o->st = NULL;
}

static void F(ensure_elemcost)(moo* o) {
  F(State)* S = (F(State)*)o->st;
  int64_t need = 1;
  for (int i = 0; i < o->ngs; ++i) {
    int64_t e = dom_extent(o, &o->gs[i].dom);
    if (e > need) need = e;
  }
  for (int g = 0; g < o->ng; ++g)
    if (o->graphs[g].E > need) need = o->graphs[g].E;
  free(S->elemcost);
  S->elemcost = (REAL*)calloc((size_t)need, sizeof(REAL));
}
