/* _sites: host-side helper of the public API -- builds the list[Site] that
 * centroidal_update() and lrcvt() return (tessellation.py:245-247 builds it
 * with a Python loop) from the float64[S, 3] positions and int32[S]
 * components the device wrote, at C speed.
 *
 * Site is the slotted dataclass of seeding.py (fields position, component_id,
 * no __post_init__): its instances are filled through the slots' member
 * offsets exactly as the generated __init__ would assign them -- position a
 * tuple of three Python floats, component_id a Python int. */
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#include <structmember.h>

static Py_ssize_t member_offset(PyTypeObject* t, const char* name) {
  for (PyTypeObject* b = t; b; b = b->tp_base) {
    PyMemberDef* m = b->tp_members;
    if (!m) continue;
    for (; m->name; m++)
      if (strcmp(m->name, name) == 0 && m->type == T_OBJECT_EX) return m->offset;
  }
  return -1;
}

/* make_sites(cls, pos_bytes, comp_bytes) -> list[cls] */
static PyObject* make_sites(PyObject* self, PyObject* args) {
  PyObject* cls_obj;
  Py_buffer pos, comp;
  if (!PyArg_ParseTuple(args, "Oy*y*", &cls_obj, &pos, &comp)) return NULL;
  PyObject* out = NULL;
  if (!PyType_Check(cls_obj)) {
    PyErr_SetString(PyExc_TypeError, "make_sites: cls must be a type");
    goto done;
  }
  PyTypeObject* cls = (PyTypeObject*)cls_obj;
  const Py_ssize_t n = comp.len / (Py_ssize_t)sizeof(int);
  if (pos.len != n * 3 * (Py_ssize_t)sizeof(double) || comp.len != n * (Py_ssize_t)sizeof(int)) {
    PyErr_SetString(PyExc_ValueError, "make_sites: need float64[S, 3] positions and int32[S] components");
    goto done;
  }
  const Py_ssize_t off_pos = member_offset(cls, "position"), off_comp = member_offset(cls, "component_id");
  if (off_pos < 0 || off_comp < 0) {
    PyErr_SetString(PyExc_TypeError, "make_sites: cls needs the slots position and component_id");
    goto done;
  }
  const double* p = (const double*)pos.buf;
  const int* c = (const int*)comp.buf;
  out = PyList_New(n);
  if (!out) goto done;
  for (Py_ssize_t i = 0; i < n; i++) {
    PyObject* t = PyTuple_New(3);
    PyObject* id = PyLong_FromLong(c[i]);
    PyObject* o = cls->tp_alloc(cls, 0);
    if (!t || !id || !o) {
      Py_XDECREF(t);
      Py_XDECREF(id);
      Py_XDECREF(o);
      Py_CLEAR(out);
      goto done;
    }
    for (int k = 0; k < 3; k++) {
      PyObject* f = PyFloat_FromDouble(p[3 * i + k]);
      if (!f) {
        Py_DECREF(t);
        Py_DECREF(id);
        Py_DECREF(o);
        Py_CLEAR(out);
        goto done;
      }
      PyTuple_SET_ITEM(t, k, f);
    }
    *(PyObject**)((char*)o + off_pos) = t;
    *(PyObject**)((char*)o + off_comp) = id;
    // a tuple of floats cannot be part of a reference cycle: off the cyclic
    // collector's lists, as CPython's own collector leaves such tuples
    if (PyObject_GC_IsTracked(t)) PyObject_GC_UnTrack(t);
    PyList_SET_ITEM(out, i, o);
  }
done:
  PyBuffer_Release(&pos);
  PyBuffer_Release(&comp);
  return out;
}

static PyMethodDef methods[] = {
    {"make_sites", make_sites, METH_VARARGS, "list of Site objects from position / component buffers"},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_sites", NULL, -1, methods};

PyMODINIT_FUNC PyInit__sites(void) { return PyModule_Create(&module); }
