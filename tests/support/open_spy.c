/* open_spy.c — LD_PRELOAD shim for tests/test_isolation.py:
 * while the environment variable JM_OPEN_SPY_LOG names a file, every path
 * passed to open/open64/openat/openat64/fopen/fopen64 is appended to it.
 * Test infrastructure only; shares nothing with the library. */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <fcntl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static __thread int in_spy = 0;

static void spy(const char *path) {
  const char *log = getenv("JM_OPEN_SPY_LOG");
  if (!log || !path || in_spy) return;
  in_spy = 1;
  static int (*real_open)(const char *, int, ...) = 0;
  if (!real_open) real_open = (int (*)(const char *, int, ...))dlsym(RTLD_NEXT, "open");
  int fd = real_open(log, O_WRONLY | O_APPEND | O_CREAT, 0644);
  if (fd >= 0) {
    size_t n = strlen(path);
    ssize_t w = write(fd, path, n);
    w += write(fd, "\n", 1);
    (void)w;
    close(fd);
  }
  in_spy = 0;
}

#define FWD_OPEN(name)                                                   \
  int name(const char *path, int flags, ...) {                           \
    static int (*real)(const char *, int, ...) = 0;                      \
    if (!real) real = (int (*)(const char *, int, ...))dlsym(RTLD_NEXT, #name); \
    mode_t mode = 0;                                                     \
    if (flags & (O_CREAT | O_TMPFILE)) {                                 \
      va_list ap;                                                        \
      va_start(ap, flags);                                               \
      mode = (mode_t)va_arg(ap, int);                                    \
      va_end(ap);                                                        \
    }                                                                    \
    spy(path);                                                           \
    return real(path, flags, mode);                                      \
  }
FWD_OPEN(open)
FWD_OPEN(open64)

#define FWD_OPENAT(name)                                                 \
  int name(int dirfd, const char *path, int flags, ...) {                \
    static int (*real)(int, const char *, int, ...) = 0;                 \
    if (!real) real = (int (*)(int, const char *, int, ...))dlsym(RTLD_NEXT, #name); \
    mode_t mode = 0;                                                     \
    if (flags & (O_CREAT | O_TMPFILE)) {                                 \
      va_list ap;                                                        \
      va_start(ap, flags);                                               \
      mode = (mode_t)va_arg(ap, int);                                    \
      va_end(ap);                                                        \
    }                                                                    \
    spy(path);                                                           \
    return real(dirfd, path, flags, mode);                               \
  }
FWD_OPENAT(openat)
FWD_OPENAT(openat64)

#define FWD_FOPEN(name)                                                  \
  FILE *name(const char *path, const char *mode) {                       \
    static FILE *(*real)(const char *, const char *) = 0;                \
    if (!real) real = (FILE * (*)(const char *, const char *)) dlsym(RTLD_NEXT, #name); \
    spy(path);                                                           \
    return real(path, mode);                                             \
  }
FWD_FOPEN(fopen)
FWD_FOPEN(fopen64)
