#ifndef SELECT_TF32_NN_H
#define SELECT_TF32_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_nn_config;

static inline select_tf32_nn_config select_tf32_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(35480)) {
        if (m < INT64_C(4435)) {
            if (n < INT64_C(2897)) {
                if (k < INT64_C(176)) {
                    if (k < INT64_C(79)) {
                        if (m < INT64_C(278)) {
                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(1109)) {
                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(2218)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (n < INT64_C(544)) {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(555)) {
                                    if (m < INT64_C(278)) {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(124)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(111)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(136)) {
                                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(136)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(555)) {
                        if (n < INT64_C(1145)) {
                            if (m < INT64_C(70)) {
                                if (k < INT64_C(1145)) {
                                    if (k < INT64_C(744)) {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(992)) {
                                            if (n < INT64_C(227)) {
                                                select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(4345)) {
                                        if (k < INT64_C(1620)) {
                                            if (m < INT64_C(12)) {
                                                if (m < INT64_C(3)) {
                                                    if (m < INT64_C(2)) {
                                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(2)) {
                                                if (k < INT64_C(2897)) {
                                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(2897)) {
                                                    if (m < INT64_C(4)) {
                                                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(12)) {
                                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (m < INT64_C(29)) {
                                                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        }
                                                    }
                                                } else {
                                                    if (m < INT64_C(3)) {
                                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(6)) {
                                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (m < INT64_C(12)) {
                                                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        }
                                                    }
                                                }
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(444)) {
                                    if (k < INT64_C(314)) {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(79)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(2173)) {
                                        if (k < INT64_C(744)) {
                                            if (m < INT64_C(139)) {
                                                select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (n < INT64_C(124)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(544)) {
                                                        if (m < INT64_C(278)) {
                                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (n < INT64_C(512)) {
                                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        }
                                                    } else {
                                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(1449)) {
                                                if (m < INT64_C(139)) {
                                                    if (k < INT64_C(992)) {
                                                        if (n < INT64_C(227)) {
                                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(278)) {
                                                        select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(3259)) {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(139)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(278)) {
                                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(196)) {
                                if (k < INT64_C(725)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(725)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(351)) {
                            if (n < INT64_C(725)) {
                                if (n < INT64_C(91)) {
                                    if (m < INT64_C(2218)) {
                                        if (m < INT64_C(1109)) {
                                            if (n < INT64_C(46)) {
                                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (n < INT64_C(46)) {
                                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(222)) {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(257)) {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(2218)) {
                                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(405)) {
                                if (k < INT64_C(744)) {
                                    if (k < INT64_C(544)) {
                                        if (n < INT64_C(182)) {
                                            if (m < INT64_C(2218)) {
                                                if (k < INT64_C(444)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(1109)) {
                                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (k < INT64_C(444)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(79)) {
                                                select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(1109)) {
                                        if (k < INT64_C(1630)) {
                                            if (k < INT64_C(992)) {
                                                if (n < INT64_C(227)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(1087)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(1087)) {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(2218)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(1630)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(2218)) {
                                    if (k < INT64_C(1449)) {
                                        if (k < INT64_C(725)) {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(1024)) {
                                                select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(6)) {
                    if (k < INT64_C(10138)) {
                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(12)) {
                        if (k < INT64_C(10138)) {
                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (n < INT64_C(222)) {
                if (n < INT64_C(111)) {
                    if (k < INT64_C(30)) {
                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(79)) {
                            if (m < INT64_C(8870)) {
                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(17740)) {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(17740)) {
                                if (k < INT64_C(168)) {
                                    if (k < INT64_C(146)) {
                                        if (m < INT64_C(8870)) {
                                            if (k < INT64_C(118)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(118)) {
                                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(8870)) {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(333)) {
                                            select_tf32_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(146)) {
                                    if (k < INT64_C(118)) {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(194)) {
                                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(385)) {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(17740)) {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(91)) {
                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(544)) {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(544)) {
                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(815)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(118)) {
                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (k < INT64_C(1630)) {
                    if (k < INT64_C(544)) {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(8870)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(17740)) {
                                select_tf32_nn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(363)) {
                        if (m < INT64_C(12544)) {
                            select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {4u, 1u, 8u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_config out = {4u, 1u, 8u, 8u, 8u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(79)) {
            if (n < INT64_C(40)) {
                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                return out;
            } else {
                if (m < INT64_C(567677)) {
                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(125)) {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(70960)) {
                if (k < INT64_C(815)) {
                    if (k < INT64_C(20)) {
                        select_tf32_nn_config out = {1u, 1u, 4u, 8u, 8u};
                        return out;
                    } else {
                        if (n < INT64_C(193)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 4u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    select_tf32_nn_config out = {4u, 1u, 8u, 8u, 8u};
                    return out;
                }
            } else {
                select_tf32_nn_config out = {1u, 1u, 4u, 8u, 8u};
                return out;
            }
        }
    }
}

#endif /* SELECT_TF32_NN_H */
