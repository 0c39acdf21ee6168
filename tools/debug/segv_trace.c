/* LD_PRELOAD helper: on SIGSEGV / SIGABRT print the native backtrace
 * (module + offset, resolvable with addr2line -e <module> <offset>) to stderr,
 * then re-raise.  Debug aid for crashes on the GPU box (no gdb in the image).
 *   gcc -shared -fPIC -O1 -o tools/debug/segv_trace.so tools/debug/segv_trace.c */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <stdio.h>
#include <string.h>
#include <unistd.h>

static void on_fault(int sig, siginfo_t* si, void* uc) {
  (void)uc;
  void* pcs[64];
  int n = backtrace(pcs, 64);
  char line[512];
  int len = snprintf(line, sizeof line, "\n[segv_trace] signal %d at address %p\n", sig, si->si_addr);
  write(2, line, len);
  for (int i = 0; i < n; ++i) {
    Dl_info info;
    if (dladdr(pcs[i], &info) && info.dli_fname) {
      len = snprintf(line, sizeof line, "[segv_trace] #%d %s +0x%lx (%s)\n", i, info.dli_fname,
                     (unsigned long)((char*)pcs[i] - (char*)info.dli_fbase),
                     info.dli_sname ? info.dli_sname : "?");
    } else {
      len = snprintf(line, sizeof line, "[segv_trace] #%d %p\n", i, pcs[i]);
    }
    write(2, line, len);
  }
  signal(sig, SIG_DFL);
  raise(sig);
}

__attribute__((constructor)) static void install(void) {
  struct sigaction sa;
  memset(&sa, 0, sizeof sa);
  sa.sa_sigaction = on_fault;
  sa.sa_flags = SA_SIGINFO;
  sigaction(SIGSEGV, &sa, NULL);
  sigaction(SIGBUS, &sa, NULL);
}
