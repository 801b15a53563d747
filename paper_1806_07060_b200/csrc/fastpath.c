/* fastpath.c -- CPython extension: the reference's numpy-in / numpy-out call
 * convention straight into the C-ABI, without per-call ctypes marshalling.
 *
 * gemm_execute(shape, config, A, B, C, caps, out) (kernels.py:328-349) with
 * numpy operands is: legality (ConfigError) -> operand checks (ShapeError,
 * kernels.py:271-283, same order and messages as kernels._check_operands)
 * -> ag_gemm_host_ex (H2D, family path, D2H in one blocking call; pageable
 * operands staged through the library's pinned rings, AG_HOST_STAGE; the
 * library's own device scratch) with the GIL released -> (out, device
 * seconds of the family path).  A fresh result (out=None) of 64 KB or more is
 * a numpy array over a block of the library's caching pinned allocator.
 *
 * Operands that are not plain row-major float32/float64 numpy arrays make
 * `execute` return NotImplemented; the Python path then handles them.
 * Built by build.py against libadaptgemm_b200.so (rpath $ORIGIN/_lib).
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <string.h>

#include "adaptgemm_b200.h"

static PyObject* ConfigError = NULL;
static PyObject* ShapeError = NULL;
static PyObject* np_empty = NULL;
static PyObject* np_frombuffer = NULL;
static PyObject* np_f32 = NULL;
static PyObject* np_f64 = NULL;

static PyObject *s_M, *s_N, *s_K, *s_alpha, *s_beta, *s_transA, *s_transB;
static PyObject *s_family_code, *s_block_m, *s_block_n, *s_block_k, *s_tile_m, *s_tile_n, *s_unroll_k;
static PyObject *s_tmc, *s_rtd, *s_rti, *s_es, *s_mt;

static int get_i64(PyObject* o, PyObject* name, int64_t* v) {
    PyObject* x = PyObject_GetAttr(o, name);
    if (!x) return -1;
    *v = PyLong_AsLongLong(x);
    Py_DECREF(x);
    return (*v == -1 && PyErr_Occurred()) ? -1 : 0;
}
static int get_f64(PyObject* o, PyObject* name, double* v) {
    PyObject* x = PyObject_GetAttr(o, name);
    if (!x) return -1;
    *v = PyFloat_AsDouble(x);
    Py_DECREF(x);
    return (*v == -1.0 && PyErr_Occurred()) ? -1 : 0;
}
static int get_bool(PyObject* o, PyObject* name, int32_t* v) {
    PyObject* x = PyObject_GetAttr(o, name);
    if (!x) return -1;
    const int t = PyObject_IsTrue(x);
    Py_DECREF(x);
    if (t < 0) return -1;
    *v = t;
    return 0;
}

static int read_shape(PyObject* o, ag_shape* s) {
    if (get_i64(o, s_M, &s->m) || get_i64(o, s_N, &s->n) || get_i64(o, s_K, &s->k)) return -1;
    if (get_f64(o, s_alpha, &s->alpha) || get_f64(o, s_beta, &s->beta)) return -1;
    return (get_bool(o, s_transA, &s->trans_a) || get_bool(o, s_transB, &s->trans_b)) ? -1 : 0;
}

static int read_config(PyObject* o, ag_config* c) {
    int64_t v[7];
    PyObject* names[7] = {s_family_code, s_block_m, s_block_n, s_block_k, s_tile_m, s_tile_n, s_unroll_k};
    for (int i = 0; i < 7; ++i)
        if (get_i64(o, names[i], &v[i])) return -1;
    c->family = (int32_t)v[0];
    c->bm = (int32_t)v[1]; c->bn = (int32_t)v[2]; c->bk = (int32_t)v[3];
    c->tm = (int32_t)v[4]; c->tn = (int32_t)v[5]; c->uk = (int32_t)v[6];
    return 0;
}

static int read_caps(PyObject* o, ag_caps* k) {
    if (get_i64(o, s_tmc, &k->tile_memory_cap) || get_i64(o, s_rtd, &k->register_tile_cap_direct) ||
        get_i64(o, s_rti, &k->register_tile_cap_indirect) || get_i64(o, s_es, &k->element_size))
        return -1;
    k->max_threads = 1024;
    PyObject* x = PyObject_GetAttr(o, s_mt);
    if (!x) {
        PyErr_Clear();
        return 0;
    }
    k->max_threads = PyLong_AsLongLong(x);
    Py_DECREF(x);
    return (k->max_threads == -1 && PyErr_Occurred()) ? -1 : 0;
}

/* A page-locked block from the library's caching host allocator
 * (ag_host_alloc), exported through the buffer protocol: the numpy result of
 * an out=None call lives in one, so the D2H lands by DMA with no staging
 * copy and no page faults; freeing the array returns the block to the cache. */
typedef struct {
    PyObject_HEAD
    void* p;
    Py_ssize_t n;
} PinnedBlock;

static int pb_getbuffer(PyObject* self, Py_buffer* view, int flags) {
    PinnedBlock* b = (PinnedBlock*)self;
    return PyBuffer_FillInfo(view, self, b->p, b->n, 0, flags);
}
static void pb_dealloc(PyObject* self) {
    ag_host_free(((PinnedBlock*)self)->p);
    Py_TYPE(self)->tp_free(self);
}
static PyBufferProcs pb_buffer = {pb_getbuffer, NULL};
static PyTypeObject PinnedBlockType = {
    PyVarObject_HEAD_INIT(NULL, 0)
    .tp_name = "_fastpath.PinnedBlock",
    .tp_basicsize = sizeof(PinnedBlock),
    .tp_dealloc = pb_dealloc,
    .tp_as_buffer = &pb_buffer,
    .tp_flags = Py_TPFLAGS_DEFAULT,
    .tp_doc = "page-locked result block (ag_host_alloc)",
};

#define PINNED_OUT_MIN (64 << 10) /* smaller results: np.empty (the small-call path stages them anyway) */

/* a fresh m x n result: pinned when large enough and the cache can pin it,
 * else np.empty */
static PyObject* new_result(int64_t m, int64_t n, int code) {
    const size_t nbytes = (size_t)(m * n) * (code == 0 ? 4 : 8);
    PyObject* dtype = code == 0 ? np_f32 : np_f64;
    if (nbytes >= PINNED_OUT_MIN) {
        void* p = ag_host_alloc(nbytes);
        if (p) {
            PinnedBlock* blk = PyObject_New(PinnedBlock, &PinnedBlockType);
            if (!blk) {
                ag_host_free(p);
                return NULL;
            }
            blk->p = p;
            blk->n = (Py_ssize_t)nbytes;
            PyObject* flat = PyObject_CallFunctionObjArgs(np_frombuffer, (PyObject*)blk, dtype, NULL);
            Py_DECREF(blk);
            if (!flat) return NULL;
            PyObject* arr = PyObject_CallMethod(flat, "reshape", "(LL)", (long long)m, (long long)n);
            Py_DECREF(flat);
            return arr;
        }
    }
    PyObject* dims = Py_BuildValue("(LL)", (long long)m, (long long)n);
    if (!dims) return NULL;
    PyObject* arr = PyObject_CallFunctionObjArgs(np_empty, dims, dtype, NULL);
    Py_DECREF(dims);
    return arr;
}

/* cache_bytes() -> bytes the pinned result cache holds free (ag_host_cache_bytes) */
static PyObject* fp_cache_bytes(PyObject* self, PyObject* unused) {
    (void)self;
    (void)unused;
    return PyLong_FromSize_t(ag_host_cache_bytes());
}

/* a 2-D float32 / float64 buffer; dtype code 0 / 1, -1 other, -2 not a buffer */
typedef struct {
    Py_buffer view;
    int held, code;
} Buf;

static void release(Buf* b) {
    if (b->held) PyBuffer_Release(&b->view);
    b->held = 0;
}

static int acquire(PyObject* o, Buf* b, int writable) {
    b->held = 0;
    b->code = -2;
    if (!PyObject_CheckBuffer(o)) return 0;
    if (PyObject_GetBuffer(o, &b->view, PyBUF_RECORDS_RO | (writable ? PyBUF_WRITABLE : 0)) < 0) {
        PyErr_Clear();
        return 0;
    }
    b->held = 1;
    const char* f = b->view.format ? b->view.format : "B";
    if (*f == '<' || *f == '=' || *f == '@') ++f;
    b->code = (!strcmp(f, "f") && b->view.itemsize == 4) ? 0 : (!strcmp(f, "d") && b->view.itemsize == 8) ? 1 : -1;
    return 0;
}

/* row-major: unit column stride, row stride a whole number of elements >= cols */
static int row_major(const Buf* b, int64_t* ld) {
    const Py_ssize_t it = b->view.itemsize, r = b->view.shape[0], c = b->view.shape[1];
    const Py_ssize_t s0 = b->view.strides[0], s1 = b->view.strides[1];
    if (c > 1 && s1 != it) return 0;
    if (r > 1 && (s0 % it != 0 || s0 < c * it)) return 0;
    *ld = r > 1 ? s0 / it : c;
    if (*ld < c) *ld = c;
    if (*ld < 1) *ld = 1;
    return 1;
}

static PyObject* shape_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    PyObject* msg = PyUnicode_FromFormatV(fmt, ap);
    va_end(ap);
    if (msg) {
        PyErr_SetObject(ShapeError, msg);
        Py_DECREF(msg);
    }
    return NULL;
}

static PyObject* raise_rc(int rc) {
    const char* msg = ag_last_error();
    PyObject* exc = rc == 1 ? ConfigError : rc == 2 ? ShapeError : PyExc_RuntimeError;
    if (rc == 3)
        PyErr_Format(exc, "CUDA failure in adaptgemm-b200: %s", msg ? msg : "");
    else
        PyErr_SetString(exc, msg ? msg : "adaptgemm-b200 error");
    return NULL;
}

/* execute(shape, config, A, B, C, caps, out) -> (out, seconds) | NotImplemented */
static PyObject* fp_execute(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
    (void)self;
    if (nargs != 7) {
        PyErr_SetString(PyExc_TypeError, "execute(shape, config, A, B, C, caps, out)");
        return NULL;
    }
    PyObject *shape = args[0], *config = args[1], *caps = args[5], *out = args[6];
    ag_shape s;
    ag_config c;
    ag_caps k;
    if (read_shape(shape, &s) || read_config(config, &c) || read_caps(caps, &k)) return NULL;
    if (!ag_is_legal(&c, &k)) {  /* ConfigError before any operand check (kernels.py:336-338) */
        PyObject* canon = PyObject_CallMethod(config, "canonical", NULL);
        if (canon) {
            PyErr_Format(ConfigError, "illegal config %U for caps %R", canon, caps);
            Py_DECREF(canon);
        }
        return NULL;
    }
    Buf a, b, cc, o;
    o.held = 0;
    acquire(args[2], &a, 0);
    acquire(args[3], &b, 0);
    acquire(args[4], &cc, 0);
    PyObject* result = NULL;
    int64_t lda = 0, ldb = 0, ldc = 0, ldo = 0;
    if (a.code == -2 || b.code == -2 || cc.code == -2 || a.view.ndim != 2 || b.view.ndim != 2 || cc.view.ndim != 2) {
        result = Py_NewRef(Py_NotImplemented);
        goto done;
    }
    {
        const int64_t ar = s.trans_a ? s.k : s.m, ac = s.trans_a ? s.m : s.k;
        const int64_t br = s.trans_b ? s.n : s.k, bc = s.trans_b ? s.k : s.n;
        if (a.view.shape[0] != ar || a.view.shape[1] != ac) {
            shape_error("A has shape (%zd, %zd), expected (%lld, %lld)", a.view.shape[0], a.view.shape[1],
                        (long long)ar, (long long)ac);
            goto done;
        }
        if (b.view.shape[0] != br || b.view.shape[1] != bc) {
            shape_error("B has shape (%zd, %zd), expected (%lld, %lld)", b.view.shape[0], b.view.shape[1],
                        (long long)br, (long long)bc);
            goto done;
        }
        if (cc.view.shape[0] != s.m || cc.view.shape[1] != s.n) {
            shape_error("C has shape (%zd, %zd), expected (%lld, %lld)", cc.view.shape[0], cc.view.shape[1],
                        (long long)s.m, (long long)s.n);
            goto done;
        }
    }
    if (!(a.code == b.code && b.code == cc.code)) {
        result = Py_NewRef(Py_NotImplemented);  /* mixed dtypes: the Python path words the error */
        goto done;
    }
    if (a.code < 0) {
        result = Py_NewRef(Py_NotImplemented);
        goto done;
    }
    if (!row_major(&a, &lda) || !row_major(&b, &ldb) || !row_major(&cc, &ldc)) {
        result = Py_NewRef(Py_NotImplemented);
        goto done;
    }
    PyObject* dst;
    if (out == Py_None) {
        dst = new_result(s.m, s.n, a.code);
        if (!dst) goto done;
    } else {
        dst = Py_NewRef(out);
    }
    acquire(dst, &o, 1);
    if (o.code == -2 || o.view.ndim != 2 || !row_major(&o, &ldo)) {
        Py_DECREF(dst);
        result = Py_NewRef(Py_NotImplemented);
        goto done;
    }
    if (o.view.shape[0] != s.m || o.view.shape[1] != s.n || o.code != a.code) {
        Py_DECREF(dst);
        shape_error("out buffer has wrong shape or dtype");
        goto done;
    }
    {
        double secs = 0.0;
        int rc;
        Py_BEGIN_ALLOW_THREADS
        rc = ag_gemm_host_ex(&s, &c, &k, a.code, a.view.buf, lda, b.view.buf, ldb, cc.view.buf, ldc, o.view.buf,
                             ldo, NULL, 0, 0, AG_HOST_STAGE, NULL, &secs);
        Py_END_ALLOW_THREADS
        if (rc) {
            Py_DECREF(dst);
            raise_rc(rc);
            goto done;
        }
        result = Py_BuildValue("(Nd)", dst, secs > 1e-9 ? secs : 1e-9);
    }
done:
    release(&a);
    release(&b);
    release(&cc);
    release(&o);
    return result;
}

/* legal(config, caps) -> bool: ag_is_legal (the C mirror of spaces.is_legal_tuple) */
static PyObject* fp_legal(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
    (void)self;
    if (nargs != 2) {
        PyErr_SetString(PyExc_TypeError, "legal(config, caps)");
        return NULL;
    }
    ag_config c;
    ag_caps k;
    if (read_config(args[0], &c) || read_caps(args[1], &k)) return NULL;
    return PyBool_FromLong(ag_is_legal(&c, &k));
}

/* set_errors(ConfigError, ShapeError) */
static PyObject* fp_set_errors(PyObject* self, PyObject* const* args, Py_ssize_t nargs) {
    (void)self;
    if (nargs != 2) {
        PyErr_SetString(PyExc_TypeError, "set_errors(ConfigError, ShapeError)");
        return NULL;
    }
    Py_XSETREF(ConfigError, Py_NewRef(args[0]));
    Py_XSETREF(ShapeError, Py_NewRef(args[1]));
    Py_RETURN_NONE;
}

static PyMethodDef methods[] = {
    {"execute", (PyCFunction)(void (*)(void))fp_execute, METH_FASTCALL, "gemm_execute over numpy operands"},
    {"legal", (PyCFunction)(void (*)(void))fp_legal, METH_FASTCALL, "ag_is_legal(config, caps)"},
    {"set_errors", (PyCFunction)(void (*)(void))fp_set_errors, METH_FASTCALL, "bind the exception classes"},
    {"cache_bytes", fp_cache_bytes, METH_NOARGS, "bytes held free by the pinned result cache"},
    {NULL, NULL, 0, NULL},
};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_fastpath", NULL, -1, methods, NULL, NULL, NULL, NULL};

PyMODINIT_FUNC PyInit__fastpath(void) {
#define INTERN(var, str) \
    if (!(var = PyUnicode_InternFromString(str))) return NULL;
    INTERN(s_M, "M") INTERN(s_N, "N") INTERN(s_K, "K") INTERN(s_alpha, "alpha") INTERN(s_beta, "beta")
    INTERN(s_transA, "transA") INTERN(s_transB, "transB") INTERN(s_family_code, "family_code")
    INTERN(s_block_m, "block_m") INTERN(s_block_n, "block_n") INTERN(s_block_k, "block_k")
    INTERN(s_tile_m, "tile_m") INTERN(s_tile_n, "tile_n") INTERN(s_unroll_k, "unroll_k")
    INTERN(s_tmc, "tile_memory_cap") INTERN(s_rtd, "register_tile_cap_direct")
    INTERN(s_rti, "register_tile_cap_indirect") INTERN(s_es, "element_size") INTERN(s_mt, "max_threads")
#undef INTERN
    PyObject* np = PyImport_ImportModule("numpy");
    if (!np) return NULL;
    np_empty = PyObject_GetAttrString(np, "empty");
    np_frombuffer = PyObject_GetAttrString(np, "frombuffer");
    np_f32 = PyObject_GetAttrString(np, "float32");
    np_f64 = PyObject_GetAttrString(np, "float64");
    Py_DECREF(np);
    if (!np_empty || !np_frombuffer || !np_f32 || !np_f64) return NULL;
    if (PyType_Ready(&PinnedBlockType) < 0) return NULL;
    ConfigError = Py_NewRef(PyExc_ValueError);
    ShapeError = Py_NewRef(PyExc_ValueError);
    return PyModule_Create(&module);
}
