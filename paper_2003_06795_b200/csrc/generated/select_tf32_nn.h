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
    if (m < INT64_C(3584)) {
        if (n < INT64_C(2897)) {
            if (m < INT64_C(448)) {
                if (m < INT64_C(12)) {
                    if (m < INT64_C(6)) {
                        if (k < INT64_C(2897)) {
                            if (m < INT64_C(3)) {
                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(1620)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(2)) {
                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(3)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(444)) {
                        if (m < INT64_C(57)) {
                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(317)) {
                                if (n < INT64_C(203)) {
                                    if (n < INT64_C(111)) {
                                        if (n < INT64_C(79)) {
                                            if (m < INT64_C(112)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(272)) {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(992)) {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(1536)) {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(992)) {
                                    if (k < INT64_C(471)) {
                                        if (k < INT64_C(157)) {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(79)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(405)) {
                            if (m < INT64_C(278)) {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(287)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(725)) {
                                if (m < INT64_C(70)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (n < INT64_C(1449)) {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(29)) {
                                    if (k < INT64_C(2897)) {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(139)) {
                                        if (n < INT64_C(1024)) {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(70)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (n < INT64_C(1024)) {
                                            if (m < INT64_C(278)) {
                                                if (k < INT64_C(3072)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(2173)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(222)) {
                    if (n < INT64_C(46)) {
                        if (m < INT64_C(1109)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(167)) {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(167)) {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(111)) {
                            if (n < INT64_C(167)) {
                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(1109)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(744)) {
                                if (k < INT64_C(444)) {
                                    if (m < INT64_C(2218)) {
                                        if (m < INT64_C(1109)) {
                                            if (k < INT64_C(222)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(272)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (n < INT64_C(79)) {
                                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(1109)) {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(544)) {
                        if (m < INT64_C(1109)) {
                            if (m < INT64_C(634)) {
                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(992)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(3259)) {
                                        if (k < INT64_C(1449)) {
                                            if (n < INT64_C(363)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (n < INT64_C(363)) {
                                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(444)) {
                                if (k < INT64_C(1630)) {
                                    if (k < INT64_C(725)) {
                                        if (k < INT64_C(182)) {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(768)) {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
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
                        }
                    } else {
                        if (m < INT64_C(2218)) {
                            if (n < INT64_C(1620)) {
                                if (k < INT64_C(203)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(725)) {
                                        if (n < INT64_C(1145)) {
                                            if (m < INT64_C(1109)) {
                                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(363)) {
                                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(6)) {
                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                return out;
            } else {
                if (m < INT64_C(12)) {
                    if (k < INT64_C(10138)) {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(146)) {
            if (n < INT64_C(46)) {
                if (m < INT64_C(17740)) {
                    if (k < INT64_C(118)) {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(8870)) {
                            select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(28)) {
                                select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (k < INT64_C(63)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(141920)) {
                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(30)) {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(8870)) {
                    if (k < INT64_C(91)) {
                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(118)) {
                            if (m < INT64_C(17740)) {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(32)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(363)) {
                    if (m < INT64_C(8870)) {
                        if (k < INT64_C(815)) {
                            if (k < INT64_C(363)) {
                                if (n < INT64_C(91)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(182)) {
                            if (n < INT64_C(46)) {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(17740)) {
                                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(91)) {
                                        select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (m < INT64_C(567677)) {
                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    select_tf32_nn_config out = {2u, 1u, 2u, 8u, 8u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_TF32_NN_H */
