#ifndef SELECT_F32_TN_H
#define SELECT_F32_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_tn_config;

static inline select_f32_tn_config select_f32_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(7168)) {
        if (m < INT64_C(57)) {
            if (k < INT64_C(227)) {
                select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                return out;
            } else {
                if (n < INT64_C(2290)) {
                    if (m < INT64_C(29)) {
                        if (m < INT64_C(12)) {
                            if (k < INT64_C(1620)) {
                                if (m < INT64_C(2)) {
                                    select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(6)) {
                                        select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(1620)) {
                                select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(3)) {
                        select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(6)) {
                            select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(12)) {
                                select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(10138)) {
                                    select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(444)) {
                if (m < INT64_C(2218)) {
                    if (m < INT64_C(225)) {
                        if (m < INT64_C(159)) {
                            if (m < INT64_C(80)) {
                                select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(203)) {
                                if (k < INT64_C(471)) {
                                    if (n < INT64_C(79)) {
                                        select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(256)) {
                                    select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(1536)) {
                                        select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(111)) {
                            if (m < INT64_C(555)) {
                                select_f32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(1109)) {
                                    if (k < INT64_C(471)) {
                                        select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(46)) {
                                        select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(176)) {
                                    if (k < INT64_C(363)) {
                                        select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(725)) {
                                        if (m < INT64_C(1109)) {
                                            if (k < INT64_C(128)) {
                                                select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(128)) {
                                                select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(28)) {
                        if (m < INT64_C(4435)) {
                            if (k < INT64_C(118)) {
                                select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(46)) {
                            if (m < INT64_C(4435)) {
                                if (k < INT64_C(28)) {
                                    select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(28)) {
                                    select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(4435)) {
                                if (n < INT64_C(46)) {
                                    select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(111)) {
                                        select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(182)) {
                                            select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (n < INT64_C(182)) {
                                    if (n < INT64_C(91)) {
                                        if (k < INT64_C(222)) {
                                            select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(4435)) {
                    if (m < INT64_C(139)) {
                        if (n < INT64_C(1109)) {
                            select_f32_tn_config out = {8u, 2u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(1145)) {
                            if (m < INT64_C(634)) {
                                if (k < INT64_C(725)) {
                                    if (m < INT64_C(278)) {
                                        select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(744)) {
                                            select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(1449)) {
                                        if (m < INT64_C(278)) {
                                            select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_tn_config out = {2u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(544)) {
                                    if (m < INT64_C(1109)) {
                                        select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            if (k < INT64_C(182)) {
                                                select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                                return out;
                                            } else {
                                                select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(896)) {
                                        select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(157)) {
                                            if (m < INT64_C(2218)) {
                                                select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(1268)) {
                                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(2218)) {
                                                    select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                                    return out;
                                                } else {
                                                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(1268)) {
                                if (m < INT64_C(555)) {
                                    if (m < INT64_C(278)) {
                                        if (k < INT64_C(405)) {
                                            select_f32_tn_config out = {8u, 4u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(405)) {
                                            select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                            return out;
                                        } else {
                                            select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(146)) {
            if (n < INT64_C(118)) {
                if (m < INT64_C(283839)) {
                    if (k < INT64_C(46)) {
                        select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(35480)) {
                            if (n < INT64_C(28)) {
                                select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(96)) {
                                        select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                } else {
                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                    return out;
                }
            } else {
                if (m < INT64_C(17740)) {
                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(35480)) {
                        select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                        return out;
                    } else {
                        select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(182)) {
                    if (k < INT64_C(363)) {
                        if (m < INT64_C(17740)) {
                            if (k < INT64_C(168)) {
                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_tn_config out = {1u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_tn_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(17740)) {
                            select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(91)) {
                                select_f32_tn_config out = {8u, 8u, 4u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                    return out;
                }
            } else {
                select_f32_tn_config out = {4u, 8u, 8u, 16u, 8u};
                return out;
            }
        }
    }
}

#endif /* SELECT_F32_TN_H */
